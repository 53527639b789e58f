// Strassen-Winograd over GF(2) on device windows, breadth first.
//
// Same mathematics as strassen.py:141-204 (7 products, 15 additions per
// level, Winograd's schedule) and the same peeling (strassen.py:66-84,
// 219-249), re-scheduled for a GPU: instead of walking the recursion tree
// depth first with two scratch quadrants per level (a CPU cache design),
// every level is one batched launch.
//
//   level s -> s+1 (pre):  for every level-s problem p and product i,
//       A_{s+1}[7p+i] = XOR of A_s[p]'s quadrants in SA[i]   (one launch)
//       B_{s+1}[7p+i] = XOR of B_s[p]'s quadrants in SB[i]   (one launch)
//   leaves: all 7^d products in ONE batched M4RM launch
//   level s+1 -> s (post): C_s[p] quadrant Q = XOR of C_{s+1}[7p+i], i in SC[Q]
//
// Over GF(2) every S/T/U step of the schedule is an XOR, so Winograd's
// operand sums and output combination reduce to these subset tables
// (derived from the 22-step schedule, strassen.py:183-204):
//   P1 = A11.B11                     -> C11 C12 C21 C22
//   P2 = A12.B21                     -> C11
//   P3 = (A11+A12+A21+A22).B22       -> C12
//   P4 = A22.(B11+B12+B21+B22)       -> C21
//   P5 = (A21+A22).(B11+B12)         -> C12 C22
//   P6 = (A11+A21+A22).(B11+B12+B22) -> C12 C21 C22
//   P7 = (A11+A21).(B12+B22)         -> C21 C22
// HBM is plentiful (180 GB), so every level's operands get their own
// buffers (stream-ordered pool) and the 7^d leaf products run concurrently.
#include <stdlib.h>

#include "gf2_internal.cuh"

namespace gf2 {

namespace {
// quadrant bits: 1 = X11, 2 = X12, 4 = X21, 8 = X22
constexpr unsigned kSA[7] = {1, 2, 15, 8, 12, 13, 5};
constexpr unsigned kSB[7] = {1, 4, 8, 15, 3, 11, 10};
// product bits: 1 << (i-1) for P_i
constexpr unsigned kSC[4] = {0x03, 0x35, 0x69, 0x71};


int m4rm_view(const gf2_view &c, const gf2_view &a, const gf2_view &b, int accumulate, cudaStream_t s) {
    M4rmBatch mb{a.data, a.pitch, 0, b.data, b.pitch, 0, c.data, c.pitch, 0,
                 a.nrows,  a.ncols, b.ncols, 1, accumulate};
    return launch_product(mb, s);
}

// the same quadrant mask on a transposed operand (X12 <-> X21)
constexpr unsigned swap12(unsigned m) { return (m & 9u) | ((m & 2u) << 1) | ((m & 4u) >> 1); }

// product q = 7p + i lands in these quadrants of C_p (transpose of kSC)
constexpr unsigned kSCT[7] = {0xF, 0x1, 0x2, 0x4, 0xA, 0xE, 0xC};

// Tensor-core leaves when the batch is big enough to amortize the expansion
// and each leaf is at least tensor_min_leaf() (640) on every side; smaller
// leaves run faster on M4RM.
bool tc_leaves(int64_t m, int64_t l, int64_t n, int depth) {
    if (g_engine == 0) return false;
    const int64_t lm = m >> depth, ll = l >> depth, ln = n >> depth;
    double leaf = (double)lm * (double)ll * (double)ln;
    for (int i = 0; i < depth; ++i) leaf *= 7.0;
    const int64_t ml = tensor_min_leaf();
    return leaf >= tensor_min_work() && lm >= ml && ln >= ml && ll >= ml;
}

// Workspace layout of strassen_core_tc at `depth`: which levels are
// materialized and where (64-bit words from the workspace base).
struct TcLayout {
    bool fpost, bt;
    int last, fp, lastA;
    int64_t offA[24], offB[24], offC[24], offBt0, total;
};
TcLayout tc_layout(const int64_t *M, const int64_t *L, const int64_t *N, const int64_t *Lw, const int64_t *Nw,
                   const int64_t *P, int depth) {
    TcLayout y{};
    // Post-additions of the last level fused into the GEMM epilogue (red.xor
    // into C_{d-1}) unless the leaves are shallow in K: below
    // GF2_POST_FUSE_MIN_K the leaf products are stored plainly into C_d and
    // one more combine pass folds them up (red.xor traffic, not MMA time,
    // bounds short-K tiles).
    // Default: 1024-deep leaves (cfg2 at the reference's cutoff 1024) store
    // plainly -- cfg2 63.7 -> 60.6 us, 8192^3 at cutoff 1024 310 -> 285 us --
    // while deeper leaves (2048: even; 4096+: fused faster) and the shallow
    // 512-cutoff leaves (736 deep: fused 1.3 us faster) keep the fused form.
    static const int64_t post_min_k = getenv("GF2_POST_FUSE_MIN_K") ? atoll(getenv("GF2_POST_FUSE_MIN_K")) : -1;
    y.fpost = post_min_k >= 0 ? L[depth] >= post_min_k : !(L[depth] >= 1024 && L[depth] < 2048);
    y.last = y.fpost ? depth - 1 : depth;  // deepest materialized C level
    // pre-addition levels fused into the expansion (GF2_FUSE_LEVELS=2 folds
    // two levels into it; one is faster on B200)
    static const int fuse_env = getenv("GF2_FUSE_LEVELS") ? atoi(getenv("GF2_FUSE_LEVELS")) : 1;
    y.fp = (depth >= 2 && fuse_env >= 2) ? 2 : 1;
    y.lastA = depth - y.fp;             // deepest materialized A/B level
    // FP4 engine: its MMA wants B K-major, so B0 is transposed once here and
    // the B side of the recursion runs on B^T (quadrants 12 and 21 swap)
    y.bt = g_engine == 3;
    int64_t total = 0;
    for (int i = 1; i <= y.last; ++i) {
        if (i <= y.lastA) {
            y.offA[i] = total;
            total += P[i] * M[i] * Lw[i];
            y.offB[i] = total;
            total += P[i] * L[i] * Nw[i];
        }
        y.offC[i] = total;
        total += P[i] * M[i] * Nw[i];
    }
    // B^T of the whole operand is materialized only when no pre-addition level
    // is (lastA == 0); otherwise level 0's B pre-addition writes transposed
    y.offBt0 = total;
    if (y.bt && y.lastA == 0) total += N[0] * Lw[0];
    y.total = total;
    return y;
}

// Tensor-core engine: levels 0..d-2 as below, and the LAST level fused into
// the product launch -- its pre-additions into the byte expansion, its
// post-additions into the UMMA epilogue (red.global.xor into C_{d-1}).
int strassen_core_tc(const gf2_view &C0, const gf2_view &A0, const gf2_view &B0, int depth, int accumulate,
                     cudaStream_t s) {
    int64_t M[24], L[24], N[24], Lw[24], Nw[24], P[24];
    for (int i = 0; i <= depth; ++i) {
        M[i] = A0.nrows >> i;
        L[i] = A0.ncols >> i;
        N[i] = B0.ncols >> i;
        Lw[i] = L[i] / kWordBits;
        Nw[i] = N[i] / kWordBits;
        P[i] = i == 0 ? 1 : P[i - 1] * 7;
    }
    const TcLayout ly = tc_layout(M, L, N, Lw, Nw, P, depth);
    const bool fpost = ly.fpost, bt = ly.bt;
    const int last = ly.last, fp = ly.fp, lastA = ly.lastA;
    const int64_t *offA = ly.offA, *offB = ly.offB, *offC = ly.offC;
    const int64_t offBt0 = ly.offBt0, total = ly.total;
    GF2_TRY(pool_setup());
    u64 *ws = nullptr;
    if (total) {
        cudaError_t e = cudaMallocAsync((void **)&ws, (size_t)total * 8, s);
        if (e != cudaSuccess) {
            cudaGetLastError();
            return set_error(GF2_ERR_OOM, std::string("strassen workspace: ") + cudaGetErrorString(e));
        }
    }
    int rc = GF2_OK;
    gf2_view Bt0{ws + offBt0, Lw[0], N[0], L[0]};
    // depth 1: transpose B0 on a side stream, overlapping the A-side
    // expansion; only the B-side expansion waits for it (UmmaJob::b_ready)
    cudaEvent_t bt_ready = nullptr;
    if (bt && lastA == 0) {
        SideStream *sd = nullptr;
        rc = side_stream(&sd);
        if (rc == GF2_OK) rc = check_cuda(cudaEventRecord(sd->fork, s), "fork");
        if (rc == GF2_OK) rc = check_cuda(cudaStreamWaitEvent(sd->s, sd->fork, 0), "fork wait");
        if (rc == GF2_OK) rc = launch_transpose(Bt0, B0, sd->s);
        if (rc == GF2_OK) rc = check_cuda(cudaEventRecord(sd->join, sd->s), "join");
        if (sd) bt_ready = sd->join;  // null when the side stream could not be created
    }
    for (int lv = 0; lv < lastA && rc == GF2_OK; ++lv) {
        for (int side = 0; side < 2 && rc == GF2_OK; ++side) {
            CombineArgs c{};
            const bool isA = side == 0;
            if (bt && !isA && lv == 0) {  // (quadrant combinations of B0)^T
                c.src = B0.data;
                c.src_pitch = B0.pitch;
                c.R = L[1];
                c.W = Nw[1];
                c.src_off[1] = c.W;
                c.src_off[2] = c.R * c.src_pitch;
                c.src_off[3] = c.src_off[2] + c.W;
                c.dst = ws + offB[1];
                c.dst_pitch = Lw[1];
                c.dst_stride = N[1] * Lw[1];
                for (int q = 0; q < 7; ++q) c.mask[q] = kSB[q];
                c.nq = 7;
                c.nprob = 1;
                rc = launch_combine_t(c, s);
                continue;
            }
            const int64_t R = isA ? M[lv + 1] : (bt ? N[lv + 1] : L[lv + 1]);
            const int64_t W = isA ? Lw[lv + 1] : (bt ? Lw[lv + 1] : Nw[lv + 1]);
            if (lv == 0) {
                c.src = isA ? A0.data : (bt ? Bt0.data : B0.data);
                c.src_pitch = isA ? A0.pitch : (bt ? Bt0.pitch : B0.pitch);
            } else {
                c.src = ws + (isA ? offA[lv] : offB[lv]);
                c.src_pitch = isA ? Lw[lv] : (bt ? Lw[lv] : Nw[lv]);
                c.src_stride = (isA ? M[lv] : (bt ? N[lv] : L[lv])) * c.src_pitch;
            }
            c.src_off[1] = W;
            c.src_off[2] = R * c.src_pitch;
            c.src_off[3] = R * c.src_pitch + W;
            c.dst = ws + (isA ? offA[lv + 1] : offB[lv + 1]);
            c.dst_pitch = W;
            c.dst_stride = 7 * R * W;
            for (int q = 0; q < 7; ++q) {
                c.dst_off[q] = q * R * W;
                c.mask[q] = isA ? kSA[q] : (bt ? swap12(kSB[q]) : kSB[q]);
            }
            c.nq = 7;
            c.R = R;
            c.W = W;
            c.nprob = P[lv];
            rc = launch_combine(c, s);
        }
    }
    if (rc == GF2_OK) {
        UmmaJob jb{};
        if (lastA == 0) {
            jb.A = A0.data; jb.pa = A0.pitch;
            jb.B = bt ? Bt0.data : B0.data; jb.pb = bt ? Bt0.pitch : B0.pitch;
        } else {
            jb.A = ws + offA[lastA]; jb.pa = Lw[lastA]; jb.sa = M[lastA] * Lw[lastA];
            jb.B = ws + offB[lastA];
            jb.pb = bt ? Lw[lastA] : Nw[lastA];
            jb.sb = bt ? N[lastA] * Lw[lastA] : L[lastA] * Nw[lastA];
        }
        jb.b_trans = bt ? 1 : 0;
        jb.b_ready = bt_ready;
        if (last == 0) {
            jb.C = C0.data; jb.pc = C0.pitch;
            if (!accumulate) rc = launch_zero(C0, s);
        } else {
            jb.C = ws + offC[last]; jb.pc = Nw[last]; jb.sc = M[last] * Nw[last];
            if (fpost)  // red.xor targets start from zero; plain stores overwrite
                rc = check_cuda(cudaMemsetAsync(ws + offC[last], 0, (size_t)(P[last] * M[last] * Nw[last]) * 8, s),
                                "zero C_{d-1}");
        }
        jb.m = M[depth]; jb.l = L[depth]; jb.n = N[depth];
        jb.nsrc = P[lastA];
        jb.fuse_pre = fp;
        jb.fuse_post = fpost ? 1 : 0;
        for (int i = 0; i < 7; ++i) {
            jb.maskA[i] = kSA[i];
            jb.maskB[i] = bt ? swap12(kSB[i]) : kSB[i];
            jb.maskC[i] = kSCT[i];
        }
        if (rc == GF2_OK) rc = launch_umma_job(jb, g_engine - 1, s);
    }
    for (int lv = last - 1; lv >= 0 && rc == GF2_OK; --lv) {
        CombineArgs c{};
        const int64_t R = M[lv + 1], W = Nw[lv + 1];
        c.src = ws + offC[lv + 1];
        c.src_pitch = W;
        c.src_stride = 7 * R * W;
        for (int i = 0; i < 7; ++i) c.src_off[i] = i * R * W;
        if (lv == 0) {
            c.dst = C0.data;
            c.dst_pitch = C0.pitch;
        } else {
            c.dst = ws + offC[lv];
            c.dst_pitch = Nw[lv];
            c.dst_stride = M[lv] * Nw[lv];
        }
        c.dst_off[1] = W;
        c.dst_off[2] = R * c.dst_pitch;
        c.dst_off[3] = R * c.dst_pitch + W;
        for (int q = 0; q < 4; ++q) c.mask[q] = kSC[q];
        c.nq = 4;
        c.R = R;
        c.W = W;
        c.nprob = P[lv];
        c.accumulate = lv == 0 ? accumulate : 0;
        rc = launch_combine(c, s);
    }
    if (bt_ready) cudaStreamWaitEvent(s, bt_ready, 0);  // side work done before ws is released
    if (ws) cudaFreeAsync(ws, s);
    return rc;
}

int strassen_core(const gf2_view &C0, const gf2_view &A0, const gf2_view &B0, int depth, int accumulate,
                  cudaStream_t s) {
    if (tc_leaves(A0.nrows, A0.ncols, B0.ncols, depth)) return strassen_core_tc(C0, A0, B0, depth, accumulate, s);
    int64_t M[24], L[24], N[24], Lw[24], Nw[24], P[24];
    for (int i = 0; i <= depth; ++i) {
        M[i] = A0.nrows >> i;
        L[i] = A0.ncols >> i;
        N[i] = B0.ncols >> i;
        Lw[i] = L[i] / kWordBits;
        Nw[i] = N[i] / kWordBits;
        P[i] = i == 0 ? 1 : P[i - 1] * 7;
    }
    // workspace: per level s >= 1, A_s, B_s and C_s for all 7^s problems
    int64_t offA[24], offB[24], offC[24], total = 0;
    for (int i = 1; i <= depth; ++i) {
        offA[i] = total;
        total += P[i] * M[i] * Lw[i];
        offB[i] = total;
        total += P[i] * L[i] * Nw[i];
        offC[i] = total;
        total += P[i] * M[i] * Nw[i];
    }
    GF2_TRY(pool_setup());
    u64 *ws = nullptr;
    cudaError_t e = cudaMallocAsync((void **)&ws, (size_t)total * 8, s);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return set_error(GF2_ERR_OOM, std::string("strassen workspace: ") + cudaGetErrorString(e));
    }
    int rc = GF2_OK;
    // ---- pre-additions, level by level
    for (int lv = 0; lv < depth && rc == GF2_OK; ++lv) {
        for (int side = 0; side < 2 && rc == GF2_OK; ++side) {
            CombineArgs c{};
            const bool isA = side == 0;
            const int64_t R = isA ? M[lv + 1] : L[lv + 1];
            const int64_t W = isA ? Lw[lv + 1] : Nw[lv + 1];
            if (lv == 0) {
                c.src = isA ? A0.data : B0.data;
                c.src_pitch = isA ? A0.pitch : B0.pitch;
                c.src_stride = 0;
            } else {
                c.src = ws + (isA ? offA[lv] : offB[lv]);
                c.src_pitch = isA ? Lw[lv] : Nw[lv];
                c.src_stride = (isA ? M[lv] : L[lv]) * c.src_pitch;
            }
            c.src_off[0] = 0;
            c.src_off[1] = W;
            c.src_off[2] = R * c.src_pitch;
            c.src_off[3] = R * c.src_pitch + W;
            c.dst = ws + (isA ? offA[lv + 1] : offB[lv + 1]);
            c.dst_pitch = W;
            c.dst_stride = 7 * R * W;
            for (int q = 0; q < 7; ++q) {
                c.dst_off[q] = q * R * W;
                c.mask[q] = isA ? kSA[q] : kSB[q];
            }
            c.nq = 7;
            c.R = R;
            c.W = W;
            c.nprob = P[lv];
            c.accumulate = 0;
            rc = launch_combine(c, s);
        }
    }
    // ---- all 7^d leaf products in one batched M4RM launch
    if (rc == GF2_OK) {
        M4rmBatch mb{ws + offA[depth], Lw[depth], M[depth] * Lw[depth],
                     ws + offB[depth], Nw[depth], L[depth] * Nw[depth],
                     ws + offC[depth], Nw[depth], M[depth] * Nw[depth],
                     M[depth], L[depth], N[depth], P[depth], 0};
        rc = launch_product(mb, s);
    }
    // ---- post-combination, deepest level first
    for (int lv = depth - 1; lv >= 0 && rc == GF2_OK; --lv) {
        CombineArgs c{};
        const int64_t R = M[lv + 1], W = Nw[lv + 1];
        c.src = ws + offC[lv + 1];
        c.src_pitch = W;
        c.src_stride = 7 * R * W;
        for (int i = 0; i < 7; ++i) c.src_off[i] = i * R * W;
        if (lv == 0) {
            c.dst = C0.data;
            c.dst_pitch = C0.pitch;
            c.dst_stride = 0;
        } else {
            c.dst = ws + offC[lv];
            c.dst_pitch = Nw[lv];
            c.dst_stride = M[lv] * Nw[lv];
        }
        c.dst_off[0] = 0;
        c.dst_off[1] = W;
        c.dst_off[2] = R * c.dst_pitch;
        c.dst_off[3] = R * c.dst_pitch + W;
        for (int q = 0; q < 4; ++q) c.mask[q] = kSC[q];
        c.nq = 4;
        c.R = R;
        c.W = W;
        c.nprob = P[lv];
        c.accumulate = lv == 0 ? accumulate : 0;
        rc = launch_combine(c, s);
    }
    cudaFreeAsync(ws, s);
    return rc;
}

}  // namespace

// Bytes of pooled workspace strassen_core asks for at `depth` on an
// m x l x n product: the level buffers, and on a tensor engine one chunk of
// expanded leaf operands (<= 8 GiB, launch_umma_job / launch_umma_f4).
static double core_ws_bytes(int64_t m, int64_t l, int64_t n, int depth) {
    int64_t M[24], L[24], N[24], Lw[24], Nw[24], P[24];
    for (int i = 0; i <= depth; ++i) {
        M[i] = m >> i;
        L[i] = l >> i;
        N[i] = n >> i;
        Lw[i] = L[i] / kWordBits;
        Nw[i] = N[i] / kWordBits;
        P[i] = i == 0 ? 1 : P[i - 1] * 7;
    }
    if (!tc_leaves(m, l, n, depth)) {
        double words = 0;
        for (int i = 1; i <= depth; ++i)
            words += (double)P[i] * ((double)M[i] * Lw[i] + (double)L[i] * Nw[i] + (double)M[i] * Nw[i]);
        // the batched M4RM launch stages a word-major copy of every leaf's A
        // (rows padded to 256) while it runs
        words += (double)P[depth] * (double)Lw[depth] * (double)((M[depth] + 255) / 256 * 256);
        return words * 8.0;
    }
    const TcLayout ly = tc_layout(M, L, N, Lw, Nw, P, depth);
    double per;  // bytes of expanded operands per leaf
    if (g_engine == 3) {
        const double kb = (double)((L[depth] + 63) / 64 * 32), np = (double)((N[depth] + 63) / 64 * 64);
        per = ((double)M[depth] + np) * kb;
    } else {
        const double kp = (double)((L[depth] + 15) / 16 * 16), np = (double)((N[depth] + 15) / 16 * 16);
        per = (double)M[depth] * kp + (double)L[depth] * np;
    }
    return (double)ly.total * 8.0 + std::min((double)P[depth] * per, 8.0 * 1073741824.0);
}

// What the pool can hand out without going over the device: free memory plus
// the blocks the pool holds but nothing uses. GF2_WS_LIMIT (bytes) replaces
// it (tests). Negative: unknown, no limit applied.
static double ws_budget() {
    static const double env = getenv("GF2_WS_LIMIT") ? atof(getenv("GF2_WS_LIMIT")) : 0.0;
    if (env > 0) return env;
    size_t free_b = 0, total_b = 0;
    if (cudaMemGetInfo(&free_b, &total_b) != cudaSuccess) {
        cudaGetLastError();
        return -1.0;
    }
    double idle = 0;
    int dev = 0;
    cudaMemPool_t pool;
    uint64_t reserved = 0, used = 0;
    if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess &&
        cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &reserved) == cudaSuccess &&
        cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemCurrent, &used) == cudaSuccess && reserved > used)
        idle = (double)(reserved - used);
    cudaGetLastError();
    return 0.95 * ((double)free_b + idle);
}

// Deepest recursion <= depth whose workspace fits the device (HBM is
// plentiful, so every level keeps its own buffers -- until a 131072^3
// product on the M4RM engine asks for 146 GB). A shallower recursion is the
// same product with larger leaves, so it is taken instead of failing with
// out-of-memory; depth 1 is the floor (then the allocation reports OOM).
// Only products asking for more than 4 GiB pay for the query.
static int fit_depth(int64_t m, int64_t l, int64_t n, int depth, cudaStream_t s) {
    static const bool forced = getenv("GF2_WS_LIMIT") != nullptr;
    if (depth <= 1) return depth;
    if (!forced && core_ws_bytes(m, l, n, depth) <= 4.0 * 1073741824.0) return depth;
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(s, &cap) != cudaSuccess || cap != cudaStreamCaptureStatusNone) {
        cudaGetLastError();
        return depth;  // no device queries inside a graph capture
    }
    const double budget = ws_budget();
    if (budget < 0) return depth;
    while (depth > 1 && core_ws_bytes(m, l, n, depth) > budget) --depth;
    return depth;
}

// strassen.py:66-84
void peel_split(int64_t m, int64_t l, int64_t n, int64_t cutoff, int64_t out[4]) {
    out[0] = out[1] = out[2] = out[3] = 0;
    auto ok = [&](int d) {
        int64_t unit = (int64_t)kWordBits << d;
        return (m / unit) * kWordBits >= cutoff && (l / unit) * kWordBits >= cutoff &&
               (n / unit) * kWordBits >= cutoff;
    };
    if (m < 1 || l < 1 || n < 1 || !ok(1)) return;
    int depth = 1;
    while (depth < 20 && ok(depth + 1)) ++depth;
    int64_t unit = (int64_t)kWordBits << depth;
    out[0] = (m / unit) * unit;
    out[1] = (l / unit) * unit;
    out[2] = (n / unit) * unit;
    out[3] = depth;
}

// gf2_m4rm: always the M4RM kernel (the named algorithm, m4rm.py:77-121)
int m4rm_mul(const gf2_view &c, const gf2_view &a, const gf2_view &b, int accumulate, cudaStream_t s) {
    M4rmBatch mb{a.data, a.pitch, 0, b.data, b.pitch, 0, c.data, c.pitch, 0, a.nrows, a.ncols, b.ncols, 1, accumulate};
    return launch_m4rm(mb, s);
}

// gf2_mul: one product launch with the current engine, no recursion
int engine_mul(const gf2_view &c, const gf2_view &a, const gf2_view &b, int accumulate, cudaStream_t s) {
    M4rmBatch mb{a.data, a.pitch, 0, b.data, b.pitch, 0, c.data, c.pitch, 0, a.nrows, a.ncols, b.ncols, 1, accumulate};
    if (g_engine == 0) return launch_m4rm(mb, s);
    return launch_umma(mb, g_engine - 1, s);  // explicit engine: no size heuristic
}

// strassen.py:257-282 dispatch (+ peel_fixup strassen.py:219-249).
int strassen_mul(const gf2_view &C, const gf2_view &A, const gf2_view &B, int64_t cutoff, int accumulate,
                 cudaStream_t s) {
    const int64_t m = A.nrows, l = A.ncols, n = B.ncols;
    if (!m || !n) return GF2_OK;
    if (!l) return accumulate ? GF2_OK : launch_ewise(C, nullptr, nullptr, 0, s);
    // n < 64: the reference switches to mul_cubic (strassen.py:268-269); the
    // product is the same, and the M4RM kernel handles a single-word tile.
    const int64_t mn = m < l ? (m < n ? m : n) : (l < n ? l : n);
    if (n < kWordBits || mn <= cutoff) return m4rm_view(C, A, B, accumulate, s);
    int64_t ps[4];
    peel_split(m, l, n, cutoff, ps);
    if (ps[3] == 0) return m4rm_view(C, A, B, accumulate, s);
    // With a tensor engine, leaves shallower than tensor_leaf_k() in K are
    // not worth their Winograd level: 1024-deep tensor leaves are epilogue
    // bound, smaller ones fall back to M4RM, and there the recursion's
    // passes cost more than the 1/8 of lookups a level saves (2048^3 at
    // cutoff 256: 57 us against ~20 us for one M4RM product). Recurse only
    // while leaves stay >= tensor_leaf_k() -- the caller's cutoff still
    // bounds the depth -- or multiply directly. Engine 0 (M4RM) honours the
    // cutoff exactly, as the reference does.
    if (g_engine != 0 && cutoff < tensor_leaf_k() && (ps[1] >> ps[3]) < tensor_leaf_k()) {
        peel_split(m, l, n, tensor_leaf_k(), ps);
        if (ps[3] == 0) return m4rm_view(C, A, B, accumulate, s);
    }
    const int depth = fit_depth(ps[0], ps[1], ps[2], (int)ps[3], s);
    if (depth != (int)ps[3]) {  // shallower: peel to this depth's unit
        const int64_t unit = (int64_t)kWordBits << depth;
        ps[0] = (m / unit) * unit;
        ps[1] = (l / unit) * unit;
        ps[2] = (n / unit) * unit;
        ps[3] = depth;
    }
    const int64_t m2 = ps[0], l2 = ps[1], n2 = ps[2];
    GF2_TRY(strassen_core(sub_view(C, 0, 0, m2, n2), sub_view(A, 0, 0, m2, l2), sub_view(B, 0, 0, l2, n2),
                          (int)ps[3], accumulate, s));
    return peel_fixup(C, A, B, m2, l2, n2, accumulate, s);
}

// strassen.py:219-249 `peel_fixup`: complete C given that C[:m2, :n2] holds
// A[:m2, :l2] . B[:l2, :n2] -- the inner remainder accumulated into that
// block, then the bottom rows, then the right columns, each one base-case
// product (never the recursion). acc_rest = 1 XORs the bottom rows and right
// columns into C instead of overwriting them (C += A.B).
int peel_fixup(const gf2_view &C, const gf2_view &A, const gf2_view &B, int64_t m2, int64_t l2, int64_t n2,
               int acc_rest, cudaStream_t s) {
    const int64_t m = A.nrows, l = A.ncols, n = B.ncols;
    if (l2 < l && m2 && n2)
        GF2_TRY(m4rm_view(sub_view(C, 0, 0, m2, n2), sub_view(A, 0, l2, m2, l - l2), sub_view(B, l2, 0, l - l2, n2),
                          1, s));
    if (m2 < m)
        GF2_TRY(m4rm_view(sub_view(C, m2, 0, m - m2, n), sub_view(A, m2, 0, m - m2, l), B, acc_rest, s));
    if (n2 < n)
        GF2_TRY(m4rm_view(sub_view(C, 0, n2, m2, n - n2), sub_view(A, 0, 0, m2, l), sub_view(B, 0, n2, l, n - n2),
                          acc_rest, s));
    return GF2_OK;
}

// m4rm.py:124-155 as the drop-in runs it: one base-case product (no
// recursion) on the M4RM kernel, or on the selected tensor engine once the
// product is past the measured crossover -- at least tensor_min_work()
// bit-ops and every side >= tensor_min_leaf() (the M4RM kernel keeps small
// and skinny products: cfg1 1024^3 13 us on M4RM). Engine 0 forces M4RM.
int base_mul(const gf2_view &c, const gf2_view &a, const gf2_view &b, int accumulate, cudaStream_t s) {
    M4rmBatch mb{a.data, a.pitch, 0, b.data, b.pitch, 0, c.data, c.pitch, 0, a.nrows, a.ncols, b.ncols, 1, accumulate};
    const double work = (double)a.nrows * (double)a.ncols * (double)b.ncols;
    const int64_t side = std::min(a.nrows, std::min(a.ncols, b.ncols));
    if (g_engine == 0 || work < tensor_min_work() || side < tensor_min_leaf()) return launch_m4rm(mb, s);
    return launch_umma(mb, g_engine - 1, s);
}

}  // namespace gf2
