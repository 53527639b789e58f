// Word-wise kernels: generators, masked add/copy/zero, and the batched
// XOR-combine behind the breadth-first Strassen-Winograd schedule.
// All are HBM-bound streaming kernels: one 64-bit word per thread, warps
// running along a row so every access is a coalesced 256-byte segment.
#include <type_traits>

#include <algorithm>

#include "gf2_internal.cuh"

namespace gf2 {

namespace {

constexpr u64 kGolden = 0x9E3779B97F4A7C15ULL;

__device__ __forceinline__ u64 splitmix_mix(u64 z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

// Write `v` into word j of a row of a view whose last word is `last`,
// preserving bits beyond the right edge (core.py:298-300, 320-323).
__device__ __forceinline__ void put_word(u64 *p, int64_t j, int64_t last, u64 tm, u64 v) {
    if (j == last && tm != ~0ULL)
        p[j] = (p[j] & ~tm) | (v & tm);
    else
        p[j] = v;
}

// core.py:191-208 -- word (r, j) = splitmix over flat index (row_base+r)*width+j.
__global__ void k_random(u64 *data, int64_t pitch, int64_t nrows, int64_t width, u64 tm,
                         u64 seed, int64_t row_base) {
    pdl_begin();
    int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= width) return;
    for (int64_t r = (int64_t)blockIdx.y * blockDim.y + threadIdx.y; r < nrows;
         r += (int64_t)gridDim.y * blockDim.y) {
        u64 idx = (u64)((row_base + r) * width + j) + 1ULL;
        u64 v = splitmix_mix(seed + idx * kGolden);
        put_word(data + r * pitch, j, width - 1, tm, v);
    }
}

// bit (r, c) = [splitmix(seed + (e+1)*golden) < T], e = (row_base+r)*ncols + c.
__global__ void k_bernoulli(u64 *data, int64_t pitch, int64_t nrows, int64_t ncols, int64_t width,
                            u64 tm, u64 seed, u64 thresh, int64_t row_base) {
    pdl_begin();
    int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= width) return;
    for (int64_t r = (int64_t)blockIdx.y * blockDim.y + threadIdx.y; r < nrows;
         r += (int64_t)gridDim.y * blockDim.y) {
        u64 e0 = (u64)((row_base + r) * ncols + j * kWordBits) + 1ULL;
        int nb = (int)min((int64_t)kWordBits, ncols - j * kWordBits);
        u64 v = 0;
        u64 x = seed + e0 * kGolden;
#pragma unroll 8
        for (int b = 0; b < nb; ++b) {
            u64 z = splitmix_mix(x);
            v |= (u64)(z < thresh) << (63 - b);
            x += kGolden;
        }
        put_word(data + r * pitch, j, width - 1, tm, v);
    }
}

// op 0: out = 0; op 1: out = a; op 2: out = a ^ b (core.py:278-323).
template <int OP>
__global__ void k_ewise(u64 *out, int64_t po, const u64 *a, int64_t pa, const u64 *b, int64_t pb,
                        int64_t nrows, int64_t width, u64 tm) {
    pdl_begin();
    int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= width) return;
    for (int64_t r = (int64_t)blockIdx.y * blockDim.y + threadIdx.y; r < nrows;
         r += (int64_t)gridDim.y * blockDim.y) {
        u64 v = 0;
        if (OP >= 1) v = a[r * pa + j];
        if (OP == 2) v ^= b[r * pb + j];
        put_word(out + r * po, j, width - 1, tm, v);
    }
}

// VEC words per thread (2 = 16-byte accesses when everything is 16-byte
// aligned), ROWS rows per thread with all loads issued before the stores.
template <int VEC, int ROWS>
__global__ void k_combine(CombineArgs p, int64_t wblocks) {
    pdl_begin();
    typedef typename std::conditional<VEC == 2, ulonglong2, unsigned long long>::type V;
    const int64_t o = blockIdx.x / wblocks;
    const int64_t j = ((blockIdx.x % wblocks) * blockDim.x + threadIdx.x) * VEC;
    if (j >= p.W) return;
    const int64_t prob = o / p.nq;
    const int q = (int)(o % p.nq);
    const unsigned mask = p.mask[q];
    const u64 *sbase = p.src + prob * p.src_stride;
    u64 *d = p.dst + prob * p.dst_stride + p.dst_off[q];
    for (int64_t r0 = (int64_t)blockIdx.y * blockDim.y * ROWS + threadIdx.y; r0 < p.R;
         r0 += (int64_t)gridDim.y * blockDim.y * ROWS) {
        V v[ROWS];
#pragma unroll
        for (int k = 0; k < ROWS; ++k) {
            const int64_t r = r0 + (int64_t)k * blockDim.y;
            if (VEC == 2) {
                ulonglong2 acc = make_ulonglong2(0, 0);
                if (r < p.R) {
#pragma unroll
                    for (int i = 0; i < 8; ++i)
                        if (mask & (1u << i)) {
                            const ulonglong2 x =
                                __ldg(reinterpret_cast<const ulonglong2 *>(sbase + p.src_off[i] + r * p.src_pitch + j));
                            acc.x ^= x.x;
                            acc.y ^= x.y;
                        }
                }
                reinterpret_cast<ulonglong2 *>(v)[k] = acc;
            } else {
                unsigned long long acc = 0;
                if (r < p.R) {
#pragma unroll
                    for (int i = 0; i < 8; ++i)
                        if (mask & (1u << i))
                            acc ^= __ldg(reinterpret_cast<const unsigned long long *>(sbase + p.src_off[i] +
                                                                                     r * p.src_pitch + j));
                }
                reinterpret_cast<unsigned long long *>(v)[k] = acc;
            }
        }
#pragma unroll
        for (int k = 0; k < ROWS; ++k) {
            const int64_t r = r0 + (int64_t)k * blockDim.y;
            if (r >= p.R) break;
            V *dp = reinterpret_cast<V *>(d + r * p.dst_pitch + j);
            if (VEC == 2) {
                ulonglong2 x = reinterpret_cast<ulonglong2 *>(v)[k];
                if (p.accumulate) {
                    const ulonglong2 y = *reinterpret_cast<ulonglong2 *>(dp);
                    x.x ^= y.x;
                    x.y ^= y.y;
                }
                *reinterpret_cast<ulonglong2 *>(dp) = x;
            } else {
                unsigned long long x = reinterpret_cast<unsigned long long *>(v)[k];
                if (p.accumulate) x ^= *reinterpret_cast<unsigned long long *>(dp);
                *reinterpret_cast<unsigned long long *>(dp) = x;
            }
        }
    }
}

// One Winograd level in a single pass: each thread loads its NS source
// vectors once (the 4 quadrants for the pre-additions, the 7 products for the
// post-additions) and writes all NQ outputs, instead of k_combine's one
// output per thread re-reading 1-4 sources (14 source reads per 7 outputs).
// Same CombineArgs addressing; 16-byte vectors, ROWS rows per thread.
// One row per thread and iteration, __launch_bounds__(256, 3): the earlier
// 2-row unrolled form took 112 (4 sources) / 139 (7 sources) registers, and
// the post-addition instance ran one CTA per SM (12 % of warps active) with
// too few loads in flight for HBM (cfg5: 7->4 levels at 3.9 / 2.8 TB/s).
template <int NS, int NQ>
__global__ void __launch_bounds__(256, 3) k_combine_all(CombineArgs p, int64_t wblocks) {
    pdl_begin();
    const int64_t prob = blockIdx.x / wblocks;
    const int64_t j = ((blockIdx.x % wblocks) * blockDim.x + threadIdx.x) * 2;
    if (j >= p.W) return;
    const u64 *sb = p.src + prob * p.src_stride + j;
    u64 *db = p.dst + prob * p.dst_stride + j;
    const int64_t rstep = (int64_t)gridDim.y * blockDim.y;
    for (int64_t r = (int64_t)blockIdx.y * blockDim.y + threadIdx.y; r < p.R; r += rstep) {
        const u64 *srow = sb + r * p.src_pitch;
        u64 *drow = db + r * p.dst_pitch;
        ulonglong2 in[NS];
#pragma unroll
        for (int i = 0; i < NS; ++i) in[i] = __ldg(reinterpret_cast<const ulonglong2 *>(srow + p.src_off[i]));
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
            ulonglong2 v = make_ulonglong2(0, 0);
#pragma unroll
            for (int i = 0; i < NS; ++i)
                if (p.mask[q] & (1u << i)) {
                    v.x ^= in[i].x;
                    v.y ^= in[i].y;
                }
            ulonglong2 *d = reinterpret_cast<ulonglong2 *>(drow + p.dst_off[q]);
            if (p.accumulate) {
                const ulonglong2 o = *d;
                v.x ^= o.x;
                v.y ^= o.y;
            }
            *d = v;
        }
    }
}

// Level-0 B pre-addition fused with the transpose the FP4 engine needs:
// dst_q = (XOR_{i in mask[q]} quadrant_i(src))^T, q < 7. A block stages the
// 4 quadrants' tiles (256 rows x 8 words each) in shared memory; warp w
// transposes word column w of every quadrant (transpose32m, linear, so the
// XOR commutes with it) and writes each transposed row's 4 words with two
// 16-byte stores.
// CT_ROWS = 256 (4 groups of 64 rows, 16-byte output stores); 64-row tiles
// (one group) when 256-row tiles would leave most SMs idle: cfg2 at cutoff
// 1024 transposes 2048-row quadrants into 32 tiles of 256 rows.
constexpr int CT_WORDS = 8;
template <int CT_ROWS>
constexpr int ct_smem() {
    return 4 * CT_ROWS * (CT_WORDS + 1) * 8;
}
template <int CT_ROWS>
__global__ void __launch_bounds__(256) k_combine_t(CombineArgs p) {
    constexpr int NG = CT_ROWS / 64;
    pdl_begin();
    extern __shared__ __align__(16) unsigned char ct_smem[];
    u64(*tile)[CT_ROWS][CT_WORDS + 1] = reinterpret_cast<u64(*)[CT_ROWS][CT_WORDS + 1]>(ct_smem);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t w0 = (int64_t)blockIdx.x * CT_WORDS, r0 = (int64_t)blockIdx.y * CT_ROWS;
    const u64 *sb = p.src + (int64_t)blockIdx.z * p.src_stride;
    // 16 loads in flight per thread before they are staged (the loop
    // unrolled by 4 kept 4): 652 -> 627 us at cfg5. The kernel is bound by
    // the shuffle transposes' integer work more than by its loads (a version
    // without shared memory, 32 loads in flight per lane, ran 690 us).
    constexpr int PER = 4 * CT_ROWS * CT_WORDS / 256, BATCH = PER < 16 ? PER : 16;
#pragma unroll 1
    for (int b0 = 0; b0 < PER; b0 += BATCH) {
        u64 v[BATCH];
#pragma unroll
        for (int i = 0; i < BATCH; ++i) {
            const int idx = threadIdx.x + 256 * (b0 + i);
            const int qd = idx / (CT_ROWS * CT_WORDS), rem = idx % (CT_ROWS * CT_WORDS);
            const int rr = rem / CT_WORDS, ww = rem % CT_WORDS;
            const int64_t r = r0 + rr, w = w0 + ww;
            v[i] = (r < p.R && w < p.W) ? __ldg(sb + p.src_off[qd] + r * p.src_pitch + w) : 0;
        }
#pragma unroll
        for (int i = 0; i < BATCH; ++i) {
            const int idx = threadIdx.x + 256 * (b0 + i);
            const int qd = idx / (CT_ROWS * CT_WORDS), rem = idx % (CT_ROWS * CT_WORDS);
            tile[qd][rem / CT_WORDS][rem % CT_WORDS] = v[i];
        }
    }
    __syncthreads();
    const int64_t w = w0 + warp;
    if (w >= p.W) return;
    const int ngroups = (int)min((int64_t)(CT_ROWS / 64), (p.R - r0 + 63) / 64);
    const bool vec = ngroups == 4 && (p.dst_pitch % 2 == 0) && (p.dst_stride % 2 == 0);
    u64 *db = p.dst + (int64_t)blockIdx.z * 7 * p.dst_stride;
    // one 32-byte store (STG.256) per transposed row and output when the rows
    // are sector aligned: a whole sector per lane instead of two half-sector
    // writes (ncu: 32 sectors per 16-byte store request, each written twice)
    const bool vec32 = vec && (p.dst_pitch % 4 == 0) && (p.dst_stride % 4 == 0) &&
                       ((uintptr_t)db % 32 == 0);
    // transpose32m: lane l takes rows 31 - l and 63 - l of a 64-row group and
    // ends up with column 31 - l (half 0) or 63 - l (half 1), MSB-first, with
    // no bit reversals
    const Bfly32 bf = bfly32_init(lane);
    const int rl = 31 - lane;
#pragma unroll 1
    for (int half = 0; half < 2; ++half) {
        u64 T[4][NG];  // [quadrant][64-row group]: transposed word of row 64w + 32 half + 31 - lane
#pragma unroll
        for (int qd = 0; qd < 4; ++qd)
#pragma unroll
            for (int g = 0; g < NG; ++g) {
                const u64 x0 = tile[qd][64 * g + rl][warp], x1 = tile[qd][64 * g + 32 + rl][warp];
                const uint32_t p0 = half ? (uint32_t)x0 : (uint32_t)(x0 >> 32);
                const uint32_t p1 = half ? (uint32_t)x1 : (uint32_t)(x1 >> 32);
                T[qd][g] = ((u64)transpose32m(p0, bf) << 32) | transpose32m(p1, bf);
            }
        const int64_t orow = w * 64 + half * 32 + rl;  // output row (< 64 W, always in range)
#pragma unroll
        for (int q = 0; q < 7; ++q) {
            u64 o[NG];
#pragma unroll
            for (int g = 0; g < NG; ++g) {
                o[g] = 0;
#pragma unroll
                for (int qd = 0; qd < 4; ++qd)
                    if (p.mask[q] & (1u << qd)) o[g] ^= T[qd][g];
            }
            u64 *drow = db + q * p.dst_stride + orow * p.dst_pitch + r0 / 64;
            if (NG == 4 && vec32) {
                asm volatile("st.global.v4.u64 [%0], {%1, %2, %3, %4};" ::"l"(drow), "l"(o[0]),
                             "l"(o[NG > 1 ? 1 : 0]), "l"(o[NG > 2 ? 2 : 0]), "l"(o[NG > 3 ? 3 : 0])
                             : "memory");
            } else if (NG == 4 && vec) {
                reinterpret_cast<ulonglong2 *>(drow)[0] = make_ulonglong2(o[0], o[NG > 1 ? 1 : 0]);
                reinterpret_cast<ulonglong2 *>(drow)[1] = make_ulonglong2(o[NG > 2 ? 2 : 0], o[NG > 3 ? 3 : 0]);
            } else {
#pragma unroll
                for (int g = 0; g < NG; ++g)
                    if (g < ngroups) drow[g] = o[g];
            }
        }
    }
}

inline dim3 row_grid(int64_t width, int64_t nrows, dim3 blk) {
    int64_t gx = (width + blk.x - 1) / blk.x;
    int64_t gy = (nrows + blk.y - 1) / blk.y;
    if (gy > 65535) gy = 65535;
    if (gy < 1) gy = 1;
    return dim3((unsigned)gx, (unsigned)gy, 1);
}

inline dim3 row_block(int64_t width) {
    // warps along the row; short rows get more rows per block
    if (width >= 128) return dim3(128, 2, 1);
    if (width >= 32) return dim3(32, 8, 1);
    return dim3(8, 32, 1);
}


// graycode.py:108-156 -- the 2^k-slot table of all XOR combinations of k
// source rows, slot x = XOR of rows i with bit (k-1-i) of x set (big-endian:
// bit k-1 is the first row), slot 0 = 0. Source words are masked with the
// tail mask (a window source may carry live bits beyond its right edge).
// A thread owns one word column of one group of 2^kl slots (kl = min(k, 8)):
// it XORs the group's high-bit rows once, then walks the low kl bits in Gray
// order -- one row XOR per slot, as the reference's table steps.
__global__ void k_make_table(u64 *T, int64_t tp, const u64 *src, int64_t sp, int k, int kl,
                             int64_t width, u64 tm) {
    pdl_begin();
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= width) return;
    const u64 m = j == width - 1 ? tm : ~0ULL;
    const int64_t hi = blockIdx.y;             // the slot bits above the low kl
    u64 acc = 0;
    for (int b = kl; b < k; ++b)               // bit b of the slot <-> source row k-1-b
        if ((hi >> (b - kl)) & 1) acc ^= src[(int64_t)(k - 1 - b) * sp + j] & m;
    const int64_t base = hi << kl;
    T[base * tp + j] = acc;
    for (int64_t t = 1; t < ((int64_t)1 << kl); ++t) {
        const int b = __ffsll(t) - 1;          // the bit that flips at Gray step t
        acc ^= src[(int64_t)(k - 1 - b) * sp + j] & m;
        T[(base | (t ^ (t >> 1))) * tp + j] = acc;
    }
}

}  // namespace

int launch_random(const gf2_view &v, u64 seed, int64_t row_base, cudaStream_t s) {
    int64_t width = words_per_row(v.ncols);
    if (!width || !v.nrows) return GF2_OK;
    dim3 blk = row_block(width);
    GF2_LAUNCH(launch_k(k_random, row_grid(width, v.nrows, blk), blk, 0, s, 1, v.data, v.pitch, v.nrows, width,
                                                         tail_mask(v.ncols), seed, row_base));
    note_launch();
    return check_cuda(cudaGetLastError(), "k_random launch");
}

int launch_bernoulli(const gf2_view &v, u64 seed, u64 thresh, int64_t row_base, cudaStream_t s) {
    int64_t width = words_per_row(v.ncols);
    if (!width || !v.nrows) return GF2_OK;
    dim3 blk = row_block(width);
    GF2_LAUNCH(launch_k(k_bernoulli, row_grid(width, v.nrows, blk), blk, 0, s, 1, 
        v.data, v.pitch, v.nrows, v.ncols, width, tail_mask(v.ncols), seed, thresh, row_base));
    note_launch();
    return check_cuda(cudaGetLastError(), "k_bernoulli launch");
}

int launch_ewise(const gf2_view &out, const gf2_view *a, const gf2_view *b, int op, cudaStream_t s) {
    int64_t width = words_per_row(out.ncols);
    if (!width || !out.nrows) return GF2_OK;
    dim3 blk = row_block(width);
    dim3 grd = row_grid(width, out.nrows, blk);
    u64 tm = tail_mask(out.ncols);
    if (op == 0)
        GF2_LAUNCH(launch_k(k_ewise<0>, grd, blk, 0, s, 1, out.data, out.pitch, nullptr, 0, nullptr, 0, out.nrows, width, tm));
    else if (op == 1)
        GF2_LAUNCH(launch_k(k_ewise<1>, grd, blk, 0, s, 1, out.data, out.pitch, a->data, a->pitch, nullptr, 0, out.nrows,
                                       width, tm));
    else
        GF2_LAUNCH(launch_k(k_ewise<2>, grd, blk, 0, s, 1, out.data, out.pitch, a->data, a->pitch, b->data, b->pitch,
                                       out.nrows, width, tm));
    note_launch();
    return check_cuda(cudaGetLastError(), "k_ewise launch");
}

// Zero a view: a 2-D memset when it covers whole words, else the masked
// k_ewise (bits beyond a ragged right edge belong to the parent matrix).
int launch_make_table(const gf2_view &table, const gf2_view &src, int k, cudaStream_t s) {
    const int64_t width = words_per_row(src.ncols);
    if (!width) return GF2_OK;
    const int kl = k < 8 ? k : 8;
    const dim3 blk((unsigned)(width < 128 ? ((width + 31) / 32) * 32 : 128));
    const dim3 grd((unsigned)((width + blk.x - 1) / blk.x), 1u << (k - kl));
    GF2_LAUNCH(launch_k(k_make_table, grd, blk, 0, s, 1, table.data, table.pitch, (const u64 *)src.data,
                        src.pitch, k, kl, width, tail_mask(src.ncols)));
    note_launch();
    return check_cuda(cudaGetLastError(), "k_make_table launch");
}

// narrow whole-word strips (a product target's ragged last word and
// padding): one thread per word, grid-stride
__global__ void k_zero_strip(u64 *data, int64_t pitch, int64_t nrows, int64_t w) {
    pdl_begin();
    const int64_t total = nrows * w;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x)
        data[(i / w) * pitch + i % w] = 0;
}

int launch_zero(const gf2_view &v, cudaStream_t s) {
    if (!v.nrows || !v.ncols) return GF2_OK;
    if (v.ncols % kWordBits) return launch_ewise(v, nullptr, nullptr, 0, s);
    const int64_t w = v.ncols / kWordBits;
    if (w < 64 && v.nrows > 1 && v.pitch != w) {
        // a strided 2-D memset of rows this narrow runs far below HBM speed
        // (cfg4's 16-word strips: 6.5 us); one thread per word does not
        const int64_t total = v.nrows * w;
        const int64_t blocks = std::min<int64_t>((total + 255) / 256, 4 * 148);
        GF2_LAUNCH(launch_k(k_zero_strip, dim3((unsigned)blocks), dim3(256), 0, s, 1, v.data, v.pitch, v.nrows, w));
        note_launch();
        return check_cuda(cudaGetLastError(), "k_zero_strip launch");
    }
    return check_cuda(cudaMemset2DAsync(v.data, (size_t)v.pitch * 8, 0, (size_t)w * 8, (size_t)v.nrows, s),
                      "zero");
}

int launch_combine(const CombineArgs &a, cudaStream_t s) {
    if (!a.R || !a.W || !a.nprob) return GF2_OK;
    // 16-byte path when every address the kernel forms is 16-byte aligned
    bool v2 = (a.W % 2 == 0) && ((uintptr_t)a.src % 16 == 0) && ((uintptr_t)a.dst % 16 == 0) &&
              (a.src_pitch % 2 == 0) && (a.dst_pitch % 2 == 0) && (a.src_stride % 2 == 0) &&
              (a.dst_stride % 2 == 0);
    for (int i = 0; i < 8; ++i) v2 = v2 && (a.src_off[i] % 2 == 0) && (a.dst_off[i] % 2 == 0);
    constexpr int ROWS = 4;
    const int vec = v2 ? 2 : 1;
    const int64_t wv = (a.W + vec - 1) / vec;  // vectors per row
    dim3 blk = row_block(wv);
    const int64_t wblocks = (wv + blk.x - 1) / blk.x;
    const int64_t gx = wblocks * a.nprob * a.nq;
    int64_t gy = (a.R + blk.y * ROWS - 1) / (blk.y * ROWS);
    if (gy > 65535) gy = 65535;
    int64_t gy1 = (a.R + blk.y - 1) / blk.y;
    if (gy1 > 65535) gy1 = 65535;
    unsigned used = 0;
    for (int q = 0; q < a.nq; ++q) used |= a.mask[q];
    if (v2 && a.nq == 7 && used == 0xF) {
        GF2_LAUNCH(launch_k(k_combine_all<4, 7>, dim3((unsigned)(wblocks * a.nprob), (unsigned)gy1, 1), blk, 0, s, 1, a, wblocks));
        note_launch();
        return check_cuda(cudaGetLastError(), "k_combine_all launch");
    }
    if (v2 && a.nq == 4 && used == 0x7F) {
        GF2_LAUNCH(launch_k(k_combine_all<7, 4>, dim3((unsigned)(wblocks * a.nprob), (unsigned)gy1, 1), blk, 0, s, 1, a, wblocks));
        note_launch();
        return check_cuda(cudaGetLastError(), "k_combine_all launch");
    }
    if (v2)
        GF2_LAUNCH(launch_k(k_combine<2, ROWS>, dim3((unsigned)gx, (unsigned)gy, 1), blk, 0, s, 1, a, wblocks));
    else
        GF2_LAUNCH(launch_k(k_combine<1, ROWS>, dim3((unsigned)gx, (unsigned)gy, 1), blk, 0, s, 1, a, wblocks));
    note_launch();
    return check_cuda(cudaGetLastError(), "k_combine launch");
}

}  // namespace gf2

namespace gf2 {
// CombineArgs as for launch_combine with nq = 7 and 4 source quadrants of
// R rows x W words; dst problems are 64 W rows x R / 64 words (pitch
// dst_pitch, stride dst_stride, the 7 outputs of source problem p at
// dst + (7p + q) dst_stride). R must be a multiple of 64.
int launch_combine_t(const CombineArgs &a, cudaStream_t s) {
    if (!a.R || !a.W || !a.nprob) return GF2_OK;
    if (a.R % 64) return set_error(GF2_ERR_PARAMETER, "combine_t: rows not a multiple of 64");
    static bool attr[64] = {};
    if (first_on_device(attr)) {
        GF2_TRY(check_cuda(cudaFuncSetAttribute(k_combine_t<256>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                ct_smem<256>()), "combine_t smem attr"));
        GF2_TRY(check_cuda(cudaFuncSetAttribute(k_combine_t<64>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                ct_smem<64>()), "combine_t smem attr"));
    }
    const int64_t gx = (a.W + CT_WORDS - 1) / CT_WORDS;
    const int64_t big = gx * ((a.R + 255) / 256) * a.nprob;  // 256-row tiles
    if (big >= 2 * num_sms()) {
        dim3 grd((unsigned)gx, (unsigned)((a.R + 255) / 256), (unsigned)a.nprob);
        GF2_LAUNCH(launch_k(k_combine_t<256>, grd, 256, ct_smem<256>(), s, 1, a));
    } else {
        dim3 grd((unsigned)gx, (unsigned)((a.R + 63) / 64), (unsigned)a.nprob);
        GF2_LAUNCH(launch_k(k_combine_t<64>, grd, 256, ct_smem<64>(), s, 1, a));
    }
    note_launch();
    return check_cuda(cudaGetLastError(), "k_combine_t launch");
}
}  // namespace gf2

namespace gf2 {
int side_stream(SideStream **out) {
    static SideStream sides[64] = {};
    int dev = 0;
    GF2_TRY(check_cuda(cudaGetDevice(&dev), "cudaGetDevice"));
    if (dev < 0 || dev >= 64) return set_error(GF2_ERR_CUDA, "device index out of range");
    SideStream &sd = sides[dev];
    if (!sd.s) {
        GF2_TRY(check_cuda(cudaStreamCreateWithFlags(&sd.s, cudaStreamNonBlocking), "side stream"));
        GF2_TRY(check_cuda(cudaEventCreateWithFlags(&sd.fork, cudaEventDisableTiming), "fork event"));
        GF2_TRY(check_cuda(cudaEventCreateWithFlags(&sd.join, cudaEventDisableTiming), "join event"));
        int least = 0, greatest = 0;
        GF2_TRY(check_cuda(cudaDeviceGetStreamPriorityRange(&least, &greatest), "priority range"));
        GF2_TRY(check_cuda(cudaStreamCreateWithPriority(&sd.hi, cudaStreamNonBlocking, greatest), "hi stream"));
        GF2_TRY(check_cuda(cudaEventCreateWithFlags(&sd.hi_fork, cudaEventDisableTiming), "fork event"));
        GF2_TRY(check_cuda(cudaEventCreateWithFlags(&sd.hi_join, cudaEventDisableTiming), "join event"));
    }
    *out = &sd;
    return GF2_OK;
}
}  // namespace gf2
