/* gf2_mul_sharded from plain C with NCCL (world size 1 here; with N ranks
 * each process passes its own row shard and the same communicator):
 *
 *   gcc examples/sharded_demo.c -Iinclude -I/usr/local/cuda/include \
 *       -Lpaper_0811_1714_b200 -lgf2b200 -lnccl \
 *       -Wl,-rpath,$PWD/paper_0811_1714_b200 -o sharded_demo
 *
 * Checks the K-panel broadcast + multiply against gf2_strassen, C += A.B,
 * and the error for a missing communicator. */
#include <nccl.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "gf2b200.h"

#define CHECK(x)                                                                   \
    do {                                                                           \
        int rc_ = (x);                                                             \
        if (rc_ != GF2_OK) {                                                       \
            fprintf(stderr, "%s -> %d: %s\n", #x, rc_, gf2_last_error());          \
            return 1;                                                              \
        }                                                                          \
    } while (0)

int main(void) {
    ncclUniqueId id;
    ncclComm_t comm;
    if (ncclGetUniqueId(&id) != ncclSuccess || ncclCommInitRank(&comm, 1, id, 0) != ncclSuccess) {
        fprintf(stderr, "NCCL init failed\n");
        return 1;
    }
    const int64_t m = 3000, l = 5000, n = 4100, wn = (n + 63) / 64;
    gf2_view a, b, c, ref;
    CHECK(gf2_alloc(m, l, &a, NULL));
    CHECK(gf2_alloc(l, n, &b, NULL));
    CHECK(gf2_alloc(m, n, &c, NULL));
    CHECK(gf2_alloc(m, n, &ref, NULL));
    CHECK(gf2_random(&a, 11, 0, NULL));
    CHECK(gf2_random(&b, 12, 0, NULL));
    CHECK(gf2_strassen(&ref, &a, &b, 2048, 8, 0, NULL));
    CHECK(gf2_mul_sharded(&c, &a, &b, comm, 0, 3, 2048, 0, NULL));
    uint64_t *h1 = malloc((size_t)(m * wn) * 8), *h2 = malloc((size_t)(m * wn) * 8);
    CHECK(gf2_download(&c, h1, wn, NULL));
    CHECK(gf2_download(&ref, h2, wn, NULL));
    CHECK(gf2_stream_sync(NULL));
    if (memcmp(h1, h2, (size_t)(m * wn) * 8)) {
        fprintf(stderr, "sharded product differs from gf2_strassen\n");
        return 1;
    }
    /* src = -1: rank r supplies block r of B's rows (all of B on rank 0 here) */
    CHECK(gf2_mul_sharded(&c, &a, &b, comm, -1, 2, 2048, 1, NULL)); /* C += A.B -> 0 */
    CHECK(gf2_download(&c, h1, wn, NULL));
    CHECK(gf2_stream_sync(NULL));
    for (int64_t i = 0; i < m * wn; ++i)
        if (h1[i]) {
            fprintf(stderr, "C + A.B + A.B != 0\n");
            return 1;
        }
    if (gf2_mul_sharded(&c, &a, &b, NULL, 0, 2, 2048, 0, NULL) != GF2_ERR_PARAMETER) {
        fprintf(stderr, "null communicator accepted\n");
        return 1;
    }
    free(h1);
    free(h2);
    CHECK(gf2_free(&a, NULL));
    CHECK(gf2_free(&b, NULL));
    CHECK(gf2_free(&c, NULL));
    CHECK(gf2_free(&ref, NULL));
    ncclCommDestroy(comm);
    printf("sharded demo OK\n");
    return 0;
}
