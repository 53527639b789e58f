/* Plain-C use of the drop-in boundary (include/gf2b200.h): no CUDA headers,
 * no torch -- device matrices are gf2_views from gf2_alloc, host data moves
 * through gf2_upload/gf2_download, and gf2_stream_sync waits for results.
 *
 *   gcc examples/abi_demo.c -Iinclude -Lpaper_0811_1714_b200 -lgf2b200 \
 *       -Wl,-rpath,$PWD/paper_0811_1714_b200 -o abi_demo && ./abi_demo
 *
 * Checks: the reference's random() known answer, a Strassen
 * product with tensor-core leaves against the M4RM entry, C += A.B
 * (accumulating the same product cancels it over GF(2)), and that a shape
 * error comes back as GF2_ERR_DIMENSION with a message. */
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

static int64_t words(int64_t ncols) { return (ncols + 63) / 64; }

int main(void) {
    printf("%s\n", gf2_version());

    /* core.random(1, 128, seed=0) */
    gf2_view k;
    uint64_t kw[2];
    CHECK(gf2_alloc(1, 128, &k, NULL));
    CHECK(gf2_random(&k, 0, 0, NULL));
    CHECK(gf2_download(&k, kw, 2, NULL));
    CHECK(gf2_stream_sync(NULL));
    if (kw[0] != 0xe220a8397b1dcdafULL || kw[1] != 0x6e789e6aa1b965f4ULL) {
        fprintf(stderr, "random() KAT mismatch: %016llx %016llx\n", (unsigned long long)kw[0],
                (unsigned long long)kw[1]);
        return 1;
    }

    const int64_t m = 3000, l = 2500, n = 3500;
    gf2_view a, b, c1, c2;
    CHECK(gf2_alloc(m, l, &a, NULL));
    CHECK(gf2_alloc(l, n, &b, NULL));
    CHECK(gf2_alloc(m, n, &c1, NULL));
    CHECK(gf2_alloc(m, n, &c2, NULL));
    CHECK(gf2_random(&a, 1, 0, NULL));
    CHECK(gf2_random(&b, 2, 0, NULL));
    CHECK(gf2_strassen(&c1, &a, &b, 1024, 8, 0, NULL)); /* depth 1, tensor-core leaves */
    CHECK(gf2_m4rm(&c2, &a, &b, 8, 0, NULL));

    const int64_t wn = words(n);
    uint64_t *h1 = malloc((size_t)(m * wn) * 8), *h2 = malloc((size_t)(m * wn) * 8);
    CHECK(gf2_download(&c1, h1, wn, NULL));
    CHECK(gf2_download(&c2, h2, wn, NULL));
    CHECK(gf2_stream_sync(NULL));
    if (memcmp(h1, h2, (size_t)(m * wn) * 8) != 0) {
        fprintf(stderr, "strassen and m4rm products differ\n");
        return 1;
    }
    uint64_t fold = 0;
    for (int64_t i = 0; i < m * wn; ++i) fold ^= h1[i] * (uint64_t)(i + 1);

    CHECK(gf2_strassen(&c1, &a, &b, 1024, 8, 1, NULL)); /* C += A.B -> 0 */
    CHECK(gf2_download(&c1, h1, wn, NULL));
    CHECK(gf2_stream_sync(NULL));
    for (int64_t i = 0; i < m * wn; ++i)
        if (h1[i]) {
            fprintf(stderr, "C + A.B + A.B != 0 at word %lld\n", (long long)i);
            return 1;
        }

    int rc = gf2_strassen(&c1, &b, &a, 1024, 8, 0, NULL); /* 2500x3500 . 3000x2500 */
    if (rc != GF2_ERR_DIMENSION) {
        fprintf(stderr, "expected GF2_ERR_DIMENSION, got %d\n", rc);
        return 1;
    }
    printf("dimension error reported: %s\n", gf2_last_error());

    free(h1);
    free(h2);
    CHECK(gf2_free(&a, NULL));
    CHECK(gf2_free(&b, NULL));
    CHECK(gf2_free(&c1, NULL));
    CHECK(gf2_free(&c2, NULL));
    CHECK(gf2_free(&k, NULL));
    CHECK(gf2_stream_sync(NULL));
    printf("product fold %016llx\nabi demo OK\n", (unsigned long long)fold);
    return 0;
}
