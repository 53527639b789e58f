// Structural kernels around the multiply path:
//   k_transpose  -- bit-matrix transpose (core.py:374-376), 64x64 blocks per
//                   warp with __ballot_sync: lane r holds rows r and r+32 of
//                   the block; one ballot per (column, half) yields 32 bits of
//                   a transposed row.
//   k_cubic      -- mul_cubic (cubic.py:76-102): C[i, j] = parity(A_i & (B^T)_j)
//                   over words, for narrow B (the reference's n < 64 path).
//   k_copy_cols  -- dst[:, c0 : c0+n) = src[:, 0 : n) for ANY bit offset c0
//                   (augment with a non-word-aligned split, core.py:344-358),
//                   preserving every destination bit outside the range.
#include "gf2_internal.cuh"

namespace gf2 {

namespace {

// One warp per 64x64 block: out[c][r] = in[r][c].
__global__ void k_transpose(const u64 *__restrict__ in, int64_t pin, u64 *__restrict__ out, int64_t pout,
                            int64_t rows, int64_t cols) {
    const int lane = threadIdx.x & 31;
    const int64_t wid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t wcols = words_per_row(cols), wrows = words_per_row(rows);
    const int64_t nblocks = wrows * wcols;
    if (wid >= nblocks) return;
    const int64_t br = wid / wcols, bc = wid % wcols;  // block row (input rows/64), block col (input words)
    const int64_t r0 = br * 64;
    const u64 tm = (bc == wcols - 1) ? tail_mask(cols) : ~0ULL;
    const u64 lo = (r0 + lane < rows) ? (in[(r0 + lane) * pin + bc] & tm) : 0;
    const u64 hi = (r0 + 32 + lane < rows) ? (in[(r0 + 32 + lane) * pin + bc] & tm) : 0;
    // transposed row c (= input column bc*64 + c) has input rows r0..r0+63
    // at bits 63..0: rows r0..r0+31 -> high half, r0+32..r0+63 -> low half
    u64 w0 = 0, w1 = 0;  // lane keeps transposed rows `lane` and `lane + 32`
#pragma unroll 8
    for (int c = 0; c < 64; ++c) {
        const unsigned blo = __ballot_sync(0xffffffffu, (lo >> (63 - c)) & 1);
        const unsigned bhi = __ballot_sync(0xffffffffu, (hi >> (63 - c)) & 1);
        const u64 w = ((u64)__brev(blo) << 32) | (u64)__brev(bhi);
        if (c == lane) w0 = w;
        if (c == lane + 32) w1 = w;
    }
    // bits of input rows beyond `rows` are zero, so output tails stay clean
    const int64_t oc = bc * 64 + lane;
    if (oc < cols) out[oc * pout + br] = w0;
    if (oc + 32 < cols) out[(oc + 32) * pout + br] = w1;
}

// Narrow-B cubic product: one thread per (row i, output word); BT is B^T.
__global__ void k_cubic(const u64 *__restrict__ A, int64_t pa, const u64 *__restrict__ BT, int64_t pbt,
                        u64 *__restrict__ C, int64_t pc, int64_t m, int64_t l, int64_t n, int accumulate) {
    const int64_t Wn = words_per_row(n), Wl = words_per_row(l);
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= m * Wn) return;
    const int64_t i = idx / Wn, w = idx % Wn;
    const u64 atm = tail_mask(l);
    u64 out = 0;
    const int jmax = (int)min((int64_t)64, n - w * 64);
    for (int jj = 0; jj < jmax; ++jj) {
        const u64 *bt = BT + (w * 64 + jj) * pbt;
        const u64 *ar = A + i * pa;
        u64 s = 0;
        for (int64_t x = 0; x < Wl; ++x) {
            u64 av = ar[x];
            if (x == Wl - 1) av &= atm;
            s ^= av & bt[x];
        }
        out |= (u64)(__popcll(s) & 1) << (63 - jj);
    }
    u64 *cw = C + i * pc + w;
    const u64 ctm = (w == Wn - 1) ? tail_mask(n) : ~0ULL;
    if (accumulate)
        *cw ^= out;
    else
        *cw = (*cw & ~ctm) | out;
}

// dst[:, c0:c0+n) = src[:, 0:n), any c0; one thread per destination word.
__global__ void k_copy_cols(const u64 *__restrict__ src, int64_t ps, u64 *__restrict__ dst, int64_t pd,
                            int64_t rows, int64_t c0, int64_t n) {
    const int64_t w0 = c0 / 64, w1 = (c0 + n - 1) / 64;  // destination words touched
    const int64_t nw = w1 - w0 + 1;
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= rows * nw) return;
    const int64_t r = idx / nw, k = idx % nw, wd = w0 + k;
    const int sh = (int)(c0 % 64);  // destination bit offset of source column 0
    const int64_t ws = words_per_row(n);
    const u64 stm = tail_mask(n);
    // source bits landing in destination word wd: source word (wd - w0) shifted
    // right by sh, plus the low bits of source word (wd - w0 - 1) shifted left
    auto sw = [&](int64_t j) -> u64 {
        if (j < 0 || j >= ws) return 0;
        u64 v = src[r * ps + j];
        return j == ws - 1 ? (v & stm) : v;
    };
    const int64_t j = wd - w0;
    u64 v = sh ? ((sw(j) >> sh) | (sw(j - 1) << (64 - sh))) : sw(j);
    // destination bit positions covered in this word
    const int64_t lo = max(c0, wd * 64), hi = min(c0 + n, wd * 64 + 64);  // [lo, hi)
    const int a = (int)(lo - wd * 64), b = (int)(hi - wd * 64);
    const u64 m = (b - a == 64) ? ~0ULL : (((1ULL << (b - a)) - 1) << (64 - b));
    u64 *dp = dst + r * pd + wd;
    *dp = (*dp & ~m) | (v & m);
}

}  // namespace

int launch_transpose(const gf2_view &out, const gf2_view &in, cudaStream_t s) {
    const int64_t blocks = words_per_row(in.nrows) * words_per_row(in.ncols);
    if (!blocks) return GF2_OK;
    const int64_t threads = blocks * 32;
    k_transpose<<<(unsigned)((threads + 255) / 256), 256, 0, s>>>(in.data, in.pitch, out.data, out.pitch, in.nrows,
                                                                   in.ncols);
    note_launch();
    return check_cuda(cudaGetLastError(), "k_transpose launch");
}

int launch_cubic(const gf2_view &c, const gf2_view &a, const gf2_view &bt, int accumulate, cudaStream_t s) {
    const int64_t work = c.nrows * words_per_row(c.ncols);
    if (!work) return GF2_OK;
    k_cubic<<<(unsigned)((work + 127) / 128), 128, 0, s>>>(a.data, a.pitch, bt.data, bt.pitch, c.data, c.pitch,
                                                           a.nrows, a.ncols, c.ncols, accumulate);
    note_launch();
    return check_cuda(cudaGetLastError(), "k_cubic launch");
}

int launch_copy_cols(const gf2_view &dst, int64_t c0, const gf2_view &src, cudaStream_t s) {
    if (!src.nrows || !src.ncols) return GF2_OK;
    const int64_t nw = (c0 + src.ncols - 1) / 64 - c0 / 64 + 1;
    const int64_t work = src.nrows * nw;
    k_copy_cols<<<(unsigned)((work + 255) / 256), 256, 0, s>>>(src.data, src.pitch, dst.data, dst.pitch, src.nrows,
                                                               c0, src.ncols);
    note_launch();
    return check_cuda(cudaGetLastError(), "k_copy_cols launch");
}

}  // namespace gf2
