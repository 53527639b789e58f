// Row-sharded multi-GPU multiply for hosts that drive NCCL themselves
// (the Python layer does the same over torch.distributed,
// paper_0811_1714_b200/sharded.py). Each rank holds its row shard of A and C
// and a device buffer for all of B; B's contents matter on the root (or, with
// src < 0, rank r's block of rows on rank r), which broadcasts it on a
// communication stream while this rank multiplies the K-panels that have
// landed: C_p (^)= A_p[:, panel] . B[panel, :].
// XOR accumulation is shard-local, so the broadcast is the only collective.
//
// NCCL is resolved at run time (dlopen of libnccl.so.2 -- the copy already
// loaded in the process when there is one), so the library itself has no
// link-time NCCL dependency; only nccl.h's types are used at compile time.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <string>
#include <vector>

#include "gf2_internal.cuh"

namespace gf2 {
int strassen_mul(const gf2_view &C, const gf2_view &A, const gf2_view &B, int64_t cutoff, int accumulate,
                 cudaStream_t s);

namespace {

typedef ncclResult_t (*BroadcastFn)(const void *, void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
typedef const char *(*ErrStrFn)(ncclResult_t);
typedef ncclResult_t (*CountFn)(const ncclComm_t, int *);
BroadcastFn g_bcast = nullptr;
ErrStrFn g_errstr = nullptr;
CountFn g_count = nullptr;

int load_nccl() {
    if (g_bcast) return GF2_OK;
    void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return set_error(GF2_ERR_NCCL, std::string("libnccl.so.2 not loadable: ") + dlerror());
    g_bcast = (BroadcastFn)dlsym(h, "ncclBroadcast");
    g_errstr = (ErrStrFn)dlsym(h, "ncclGetErrorString");
    g_count = (CountFn)dlsym(h, "ncclCommCount");
    if (!g_bcast || !g_count)
        return set_error(GF2_ERR_NCCL, "ncclBroadcast / ncclCommCount not found in libnccl.so.2");
    return GF2_OK;
}

int check_nccl(ncclResult_t r, const char *what) {
    if (r == ncclSuccess) return GF2_OK;
    return set_error(GF2_ERR_NCCL, std::string(what) + ": " + (g_errstr ? g_errstr(r) : std::to_string((int)r)));
}

struct CommStream {
    cudaStream_t s = nullptr;
    std::vector<cudaEvent_t> landed;
};

int comm_stream(CommStream **out, size_t npanels) {
    static CommStream cs[64];
    int dev = 0;
    GF2_TRY(check_cuda(cudaGetDevice(&dev), "cudaGetDevice"));
    if (dev < 0 || dev >= 64) return set_error(GF2_ERR_CUDA, "device index out of range");
    CommStream &c = cs[dev];
    if (!c.s) GF2_TRY(check_cuda(cudaStreamCreateWithFlags(&c.s, cudaStreamNonBlocking), "comm stream"));
    while (c.landed.size() < npanels) {
        cudaEvent_t e;
        GF2_TRY(check_cuda(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "panel event"));
        c.landed.push_back(e);
    }
    *out = &c;
    return GF2_OK;
}

}  // namespace

// Word-aligned K-panels [k0, k1) covering l (sharded.py k_panels).
std::vector<std::pair<int64_t, int64_t>> k_panels(int64_t l, int npanels) {
    std::vector<std::pair<int64_t, int64_t>> out;
    if (l <= 0) return out;
    const int64_t words = words_per_row(l);
    const int64_t np = std::max<int64_t>(1, std::min<int64_t>(npanels, words));
    const int64_t per = (words + np - 1) / np;
    for (int64_t p = 0; p < np; ++p) {
        const int64_t k0 = p * per * kWordBits, k1 = std::min(l, (p + 1) * per * kWordBits);
        if (k0 < k1) out.push_back({k0, k1});
    }
    return out;
}

int mul_sharded(const gf2_view &c, const gf2_view &a, const gf2_view &b, ncclComm_t comm, int src, int npanels,
                int64_t cutoff, int accumulate, cudaStream_t s) {
    GF2_TRY(load_nccl());
    const auto panels = k_panels(a.ncols, npanels);
    if (!accumulate) GF2_TRY(launch_zero(c, s));
    if (panels.empty()) return GF2_OK;
    // src >= 0: one broadcast per compute panel, from rank src. src < 0: B's
    // rows split into nranks word-aligned blocks, block r broadcast from rank
    // r (sharded.py owned_rows); a panel waits for every block it overlaps.
    std::vector<std::pair<int64_t, int64_t>> pieces = panels;
    if (src < 0) {
        int nranks = 1;
        GF2_TRY(check_nccl(g_count(comm, &nranks), "ncclCommCount"));
        pieces = k_panels(a.ncols, nranks);
    }
    CommStream *cs = nullptr;
    GF2_TRY(comm_stream(&cs, pieces.size()));
    // B goes over the wire as whole rows of `width` words. A B whose pitch is
    // its width (an owned matrix without padding words, or whole rows of
    // one) is broadcast in place. Any other B -- a window at a word offset,
    // a ragged window, or a padded pitch -- is staged through a contiguous
    // buffer: packed here, broadcast, and unpacked with the edge-preserving
    // copy, so no word outside B's window is written and the byte counts do
    // not depend on each rank's pitch.
    const int64_t W = words_per_row(b.ncols);
    const bool staged = b.pitch != W;
    u64 *stage = nullptr;
    if (staged) {
        cudaError_t e = cudaMallocAsync((void **)&stage, (size_t)(b.nrows * W) * 8, s);
        if (e != cudaSuccess) {
            cudaGetLastError();
            return set_error(GF2_ERR_OOM, std::string("sharded B staging: ") + cudaGetErrorString(e));
        }
        const gf2_view sv{stage, W, b.nrows, b.ncols};
        GF2_TRY(launch_ewise(sv, &b, nullptr, 1, s));
    }
    u64 *wire = staged ? stage : b.data;
    const int64_t wp = staged ? W : b.pitch;
    // the broadcast may overwrite B only after earlier work on `s` is done
    cudaEvent_t ready = cs->landed[0];
    GF2_TRY(check_cuda(cudaEventRecord(ready, s), "ready"));
    GF2_TRY(check_cuda(cudaStreamWaitEvent(cs->s, ready, 0), "ready wait"));
    for (size_t i = 0; i < pieces.size(); ++i) {
        const int64_t k0 = pieces[i].first, k1 = pieces[i].second;
        // rows k0..k1 of B: one contiguous byte range
        GF2_TRY(check_nccl(g_bcast(wire + k0 * wp, wire + k0 * wp, (size_t)((k1 - k0) * wp) * 8,
                                   ncclUint8, src >= 0 ? src : (int)i, comm, cs->s),
                           "ncclBroadcast"));
        GF2_TRY(check_cuda(cudaEventRecord(cs->landed[i], cs->s), "panel landed"));
    }
    size_t next = 0;
    for (size_t i = 0; i < panels.size(); ++i) {
        const int64_t k0 = panels[i].first, k1 = panels[i].second;
        for (; next < pieces.size() && pieces[next].first < k1; ++next) {
            GF2_TRY(check_cuda(cudaStreamWaitEvent(s, cs->landed[next], 0), "panel wait"));
            if (staged) {
                const int64_t p0 = pieces[next].first, p1 = pieces[next].second;
                const gf2_view sv{stage + p0 * W, W, p1 - p0, b.ncols};
                GF2_TRY(launch_ewise(sub_view(b, p0, 0, p1 - p0, b.ncols), &sv, nullptr, 1, s));
            }
        }
        GF2_TRY(strassen_mul(c, sub_view(a, 0, k0, a.nrows, k1 - k0), sub_view(b, k0, 0, k1 - k0, b.ncols), cutoff,
                             1, s));
    }
    if (staged) GF2_TRY(check_cuda(cudaFreeAsync(stage, s), "free staging"));
    return GF2_OK;
}

}  // namespace gf2
