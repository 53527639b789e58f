// Structural kernels around the multiply path:
//   k_transpose  -- bit-matrix transpose (core.py:374-376): shared-memory
//                   staged 512-row tiles, 64 x 64 blocks per warp as four
//                   warp-wide 32 x 32 butterfly transposes, staged output.
//   k_cubic      -- mul_cubic (cubic.py:76-102): C[i, j] = parity(A_i & (B^T)_j)
//                   over words, for narrow B (the reference's n < 64 path).
//   k_copy_cols  -- dst[:, c0 : c0+n) = src[:, 0 : n) for ANY bit offset c0
//                   (augment with a non-word-aligned split, core.py:344-358),
//                   preserving every destination bit outside the range.
#include "gf2_internal.cuh"

namespace gf2 {

namespace {

// out[c][r] = in[r][c]. A block stages 512 input rows x 4 words (one 32-byte
// sector per row) in shared memory; each warp transposes 64 x 64 blocks with
// four warp-wide 32 x 32 butterflies (transpose32m) into a shared output tile
// (256 rows x 8 words), written back as 16-byte stores, 64 contiguous bytes
// per output row. The kernel is bound by the L1/shared data pipe (ncu: 87 %,
// 21 M shuffle + 27 M shared wavefronts at 65536^2, 10.6 M of them bank
// conflicts of the padded pitches 5 and 9). XOR-swizzled tiles without
// padding (conflict-free on paper for all four access patterns) measured
// slower, 447 vs 392 us at 65536^2, and were not kept.
constexpr int TR_ROWS = 512, TR_WORDS = 4, TR_OUT_WORDS = TR_ROWS / 64;
__global__ void __launch_bounds__(256) k_transpose(const u64 *__restrict__ in, int64_t pin, u64 *__restrict__ out,
                                                   int64_t pout, int64_t rows, int64_t cols) {
    pdl_begin();
    __shared__ u64 tile[TR_ROWS][TR_WORDS + 1];
    __shared__ u64 stg[64 * TR_WORDS][TR_OUT_WORDS + 1];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t wcols = words_per_row(cols), wrows = words_per_row(rows);
    const int64_t w0 = (int64_t)blockIdx.x * TR_WORDS, r0 = (int64_t)blockIdx.y * TR_ROWS;
#pragma unroll
    for (int i = 0; i < TR_ROWS * TR_WORDS / 256; ++i) {
        const int idx = threadIdx.x + 256 * i;
        const int rr = idx / TR_WORDS, ww = idx % TR_WORDS;
        const int64_t r = r0 + rr, w = w0 + ww;
        u64 x = 0;
        if (r < rows && w < wcols) x = in[r * pin + w] & (w == wcols - 1 ? tail_mask(cols) : ~0ULL);
        tile[rr][ww] = x;
    }
    __syncthreads();
    // units: (word column, 64-row group); bits of rows beyond `rows` are zero.
    // Lane l takes rows 31 - l and 63 - l of the block and ends up with
    // columns 31 - l and 63 - l (transpose32m: MSB-first, no bit reversal).
    const Bfly32 bf = bfly32_init(lane);
    const int rl = 31 - lane;
#pragma unroll 2
    for (int it = 0; it < TR_WORDS * TR_OUT_WORDS / 8; ++it) {
        const int u = warp + 8 * it;
        const int ww = u % TR_WORDS, g = u / TR_WORDS;
        const u64 x0 = tile[64 * g + rl][ww], x1 = tile[64 * g + 32 + rl][ww];
        const uint32_t tp = transpose32m((uint32_t)(x0 >> 32), bf);  // rows 0..31, columns 0..31
        const uint32_t tr = transpose32m((uint32_t)(x1 >> 32), bf);  // rows 32..63, columns 0..31
        const uint32_t tq = transpose32m((uint32_t)x0, bf);          // rows 0..31, columns 32..63
        const uint32_t ts = transpose32m((uint32_t)x1, bf);          // rows 32..63, columns 32..63
        stg[64 * ww + rl][g] = ((u64)tp << 32) | tr;
        stg[64 * ww + 32 + rl][g] = ((u64)tq << 32) | ts;
    }
    __syncthreads();
    const int64_t ow0 = r0 / 64;
    const bool vec = (pout % 2 == 0) && ((uintptr_t)out % 16 == 0);
#pragma unroll
    for (int i = 0; i < 64 * TR_WORDS * TR_OUT_WORDS / 2 / 256; ++i) {
        const int idx = threadIdx.x + 256 * i;
        const int orow = idx / (TR_OUT_WORDS / 2), ch = idx % (TR_OUT_WORDS / 2);
        const int64_t oc = w0 * 64 + orow, ow = ow0 + 2 * ch;
        if (oc >= cols || ow >= wrows) continue;
        u64 *d = out + oc * pout + ow;
        if (vec && ow + 1 < wrows) {
            *reinterpret_cast<ulonglong2 *>(d) = make_ulonglong2(stg[orow][2 * ch], stg[orow][2 * ch + 1]);
        } else {
            d[0] = stg[orow][2 * ch];
            if (ow + 1 < wrows) d[1] = stg[orow][2 * ch + 1];
        }
    }
}

// Narrow-B cubic product: one thread per (row i, output word); BT is B^T.
__global__ void k_cubic(const u64 *__restrict__ A, int64_t pa, const u64 *__restrict__ BT, int64_t pbt,
                        u64 *__restrict__ C, int64_t pc, int64_t m, int64_t l, int64_t n, int accumulate) {
    pdl_begin();
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
    pdl_begin();
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
    const int64_t wcols = words_per_row(in.ncols);
    if (!wcols || !in.nrows) return GF2_OK;
    dim3 grd((unsigned)((wcols + TR_WORDS - 1) / TR_WORDS), (unsigned)((in.nrows + TR_ROWS - 1) / TR_ROWS));
    GF2_LAUNCH(launch_k(k_transpose, grd, 256, 0, s, 1, in.data, in.pitch, out.data, out.pitch, in.nrows, in.ncols));
    note_launch();
    return check_cuda(cudaGetLastError(), "k_transpose launch");
}

int launch_cubic(const gf2_view &c, const gf2_view &a, const gf2_view &bt, int accumulate, cudaStream_t s) {
    const int64_t work = c.nrows * words_per_row(c.ncols);
    if (!work) return GF2_OK;
    GF2_LAUNCH(launch_k(k_cubic, (unsigned)((work + 127) / 128), 128, 0, s, 1, a.data, a.pitch, bt.data, bt.pitch, c.data, c.pitch,
                                                           a.nrows, a.ncols, c.ncols, accumulate));
    note_launch();
    return check_cuda(cudaGetLastError(), "k_cubic launch");
}

int launch_copy_cols(const gf2_view &dst, int64_t c0, const gf2_view &src, cudaStream_t s) {
    if (!src.nrows || !src.ncols) return GF2_OK;
    const int64_t nw = (c0 + src.ncols - 1) / 64 - c0 / 64 + 1;
    const int64_t work = src.nrows * nw;
    GF2_LAUNCH(launch_k(k_copy_cols, (unsigned)((work + 255) / 256), 256, 0, s, 1, src.data, src.pitch, dst.data, dst.pitch, src.nrows,
                                                               c0, src.ncols));
    note_launch();
    return check_cuda(cudaGetLastError(), "k_copy_cols launch");
}

}  // namespace gf2
