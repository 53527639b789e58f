// FP4 tensor-core engine (tcgen05.mma.cta_group::2.kind::mxf4, the default
// base case): bit -> e2m1 nibble expansion kernels (rows,
// rows with the 7 fused Strassen products, transposing columns), the
// persistent CTA-pair GEMM k_umma_f4 with block scales fixed at 2^0 in TMEM
// and a parity-packing epilogue, and the host launcher.
#include <stdlib.h>

#include <algorithm>

#include "gf2_tc.cuh"

namespace gf2 {

namespace {

// ------------------------------------------------------------------ FP4 (kind::mxf4)
// Entries as e2m1 nibbles (1.0 = 0x2, two per byte), both operands K-major,
// block-scaled MMA with every scale = 1.0 (UE8M0 0x7F): twice the 8-bit MMA
// rate and half the operand bytes. f32 accumulators, K chunks <= 8192 as for
// kind::f8f6f4. K order inside every 64-entry group is permuted identically
// on both sides (a fixed relabelling of the summation index): a 64-bit
// K-vector v (bit i = entry i) becomes 8 words, word t holding nibbles
// v[t], v[32+t], v[8+t], v[40+t], v[16+t], v[48+t], v[24+t], v[56+t].
constexpr int F4_BN = 224;                 // max tile N (7 x 32-bit output groups)
constexpr int F4_BNH = F4_BN / 2;          // B rows per CTA of a pair
constexpr int F4_STG = 7;
constexpr int F4_A_ST = BM * BK;           // 128 rows x 128 B (256 K entries)
constexpr int F4_B_ST = F4_BNH * BK;       // 112 rows x 128 B
constexpr int F4_EPI_OFF = 256;            // epilogue staging, after the barriers
constexpr int F4_EPI_BYTES = 4 * 32 * 4 * 8;  // 4 warps x 32 rows x 4 words
constexpr int F4_SMEM = F4_STG * (F4_A_ST + F4_B_ST) + 1024 + F4_EPI_OFF + F4_EPI_BYTES;
constexpr int F4_SF_COL = 2 * F4_BN;       // TMEM columns 448..511: constant scale factors
constexpr int64_t F4_KCHUNK = 8192;
static_assert(F4_SMEM <= 232448, "k_umma_f4 shared memory");

// word t of a K-vector's 32 nibble bytes (see the permutation above)
__device__ __forceinline__ uint32_t nib_word(u64 v, int t) {
    const uint32_t lo = (uint32_t)v, hi = (uint32_t)(v >> 32);
    return (((lo >> t) & 0x01010101u) << 1) | (((hi >> t) & 0x01010101u) << 5);
}

// A side: a warp expands 32 consecutive words of 4 rows; every store
// instruction writes 512 contiguous bytes (lane l: 16-byte chunk l + 32k of
// the warp's 1 KiB, i.e. half l & 1 of word l/2 + 16k, fetched by shuffle).
constexpr int F4_ROWS_PER_WARP = 4;
template <int LEVELS>
__global__ void __launch_bounds__(256) k_expand4_rows(ExpandArgs a) {
    pdl_begin();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t width = words_per_row(a.cols);
    const int64_t j0 = (int64_t)blockIdx.x * 32, j = j0 + lane;
    const int64_t r0 = ((int64_t)blockIdx.y * 8 + warp) * F4_ROWS_PER_WARP;
    if (r0 >= a.rows) return;
    const u64 tm = (j == width - 1) ? tail_mask(a.cols) : ~0ULL;
    const int64_t q = a.q0 + blockIdx.z;
    const int64_t p = LEVELS == 0 ? q : (LEVELS == 1 ? q / 7 : q / 49);
    const unsigned m1 = LEVELS == 0 ? 1u : a.mask[LEVELS == 1 ? q % 7 : (q / 7) % 7];
    const unsigned m2 = LEVELS == 2 ? a.mask[q % 7] : 1u;
    const u64 *s = a.src + p * a.sstride + j;
    u64 x[F4_ROWS_PER_WARP];
#pragma unroll
    for (int rr = 0; rr < F4_ROWS_PER_WARP; ++rr)
        x[rr] = (j < width && r0 + rr < a.rows) ? __brevll(gather_word<LEVELS>(a, s, r0 + rr, m1, m2) & tm) : 0;
    uint8_t *d = a.dst + (int64_t)blockIdx.z * a.dstride + j0 * 32;
    const int h = lane & 1;
#pragma unroll
    for (int rr = 0; rr < F4_ROWS_PER_WARP; ++rr) {
        if (r0 + rr >= a.rows) break;
#pragma unroll
        for (int k = 0; k < 2; ++k) {
            const int wl = (lane >> 1) + 16 * k;
            const u64 v = __shfl_sync(0xffffffffu, x[rr], wl);
            if (j0 + wl < width)
                *reinterpret_cast<uint4 *>(d + (r0 + rr) * a.dp + (lane + 32 * k) * 16) =
                    make_uint4(nib_word(v, 4 * h), nib_word(v, 4 * h + 1), nib_word(v, 4 * h + 2),
                               nib_word(v, 4 * h + 3));
        }
    }
}

// Fused level, all 7 outputs of one source problem at once: a warp loads the
// 4 quadrant words of 32 consecutive words x ROWS rows ONCE, forms the 7
// combinations (mask[i]) and writes each one's nibbles like k_expand4_rows
// (output problem 7p + i). Quadrant words are read once instead of 14
// times per 7 outputs.
// LEVELS = 2 (two fused levels, block z = 7p + i): the block first forms the
// 4 sub-quadrant words of level-0 combination i (mask[i] over the level-0
// quadrants, up to 16 source words), then writes its 7 level-1 combinations
// (output problem 49p + 7i + j = 7z + j) -- the level-0 operands are never
// materialized.
template <int ROWS, int LEVELS>
__global__ void __launch_bounds__(256) k_expand4_rows7(ExpandArgs a) {
    pdl_begin();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t width = words_per_row(a.cols);
    const int64_t j0 = (int64_t)blockIdx.x * 32, j = j0 + lane;
    const int64_t r0 = ((int64_t)blockIdx.y * 8 + warp) * ROWS;
    if (r0 >= a.rows) return;
    const u64 tm = (j == width - 1) ? tail_mask(a.cols) : ~0ULL;
    const int64_t p = LEVELS == 1 ? a.q0 / 7 + blockIdx.z : a.q0 / 49 + blockIdx.z / 7;  // source problem
    const u64 *s = a.src + p * a.sstride + j;
    const bool live = j < width;
    u64 qw[ROWS][4];
    if (LEVELS == 1) {
#pragma unroll
        for (int rr = 0; rr < ROWS; ++rr)
#pragma unroll
            for (int t = 0; t < 4; ++t)
                qw[rr][t] = (live && r0 + rr < a.rows) ? __ldg(s + a.qoff[t] + (r0 + rr) * a.sp) & tm : 0;
    } else {
        const unsigned mi = a.mask[blockIdx.z % 7];
#pragma unroll
        for (int rr = 0; rr < ROWS; ++rr)
#pragma unroll
            for (int t = 0; t < 4; ++t) {
                u64 x = 0;
                if (live && r0 + rr < a.rows) {
#pragma unroll
                    for (int Q = 0; Q < 4; ++Q)
                        if (mi & (1u << Q)) x ^= __ldg(s + a.qoff[Q] + a.qoff2[t] + (r0 + rr) * a.sp);
                }
                qw[rr][t] = x & tm;
            }
    }
    const int h = lane & 1;
#pragma unroll 1
    for (int i = 0; i < 7; ++i) {
        const unsigned m = a.mask[i];
        uint8_t *d = a.dst + ((int64_t)blockIdx.z * 7 + i) * a.dstride + j0 * 32;
#pragma unroll
        for (int rr = 0; rr < ROWS; ++rr) {
            if (r0 + rr >= a.rows) break;
            u64 x = 0;
#pragma unroll
            for (int t = 0; t < 4; ++t)
                if (m & (1u << t)) x ^= qw[rr][t];
            x = __brevll(x);
#pragma unroll
            for (int k = 0; k < 2; ++k) {
                const int wl = (lane >> 1) + 16 * k;
                const u64 v = __shfl_sync(0xffffffffu, x, wl);
                if (j0 + wl < width)
                    *reinterpret_cast<uint4 *>(d + (r0 + rr) * a.dp + (lane + 32 * k) * 16) =
                        make_uint4(nib_word(v, 4 * h), nib_word(v, 4 * h + 1), nib_word(v, 4 * h + 2),
                                   nib_word(v, 4 * h + 3));
            }
        }
    }
}

// B side, transposed. A block stages 256 K rows x 16 words (coalesced 128 B
// row segments, fused quadrant XORs) in shared memory; each warp then owns
// 2 words: per 64-row K block, four warp-wide 32 x 32 transposes turn the
// 64 x 64 bit block into 64 column K-vectors (lane: columns lane and lane + 32), and each lane writes
// its two columns' 128 contiguous bytes (256 K entries).
// WORDS = 16 source words (1024 columns) per block, or 8 when 16-word tiles
// would not give every SM a block: cfg2's 4096-column B 7.0 -> 5.3 us; the
// wider tile stays better once the grid is larger (cfg4 17.2 vs 21.0 us).
constexpr int F4T_ROWS = 256;
constexpr int F4T_STG_PITCH = 144;  // 128 B output row + 16 B pad (conflict-free)
template <int F4T_WORDS>
constexpr int f4t_tile_bytes() {
    return F4T_ROWS * (F4T_WORDS + 1) * 8;
}
template <int F4T_WORDS>
constexpr int f4t_smem() {
    return f4t_tile_bytes<F4T_WORDS>() + 8 * 32 * F4T_STG_PITCH;
}
template <int LEVELS, int F4T_WORDS>
__global__ void __launch_bounds__(256) k_expand4_cols(ExpandArgs a) {
    constexpr int F4T_TILE_BYTES = f4t_tile_bytes<F4T_WORDS>();
    pdl_begin();
    extern __shared__ __align__(16) unsigned char f4t_smem[];
    u64(*tile)[F4T_WORDS + 1] = reinterpret_cast<u64(*)[F4T_WORDS + 1]>(f4t_smem);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t width = words_per_row(a.cols);
    const int64_t w0 = (int64_t)blockIdx.x * F4T_WORDS;
    const int64_t k0 = (int64_t)blockIdx.y * F4T_ROWS;
    const int64_t q = a.q0 + blockIdx.z;
    const int64_t p = LEVELS == 0 ? q : (LEVELS == 1 ? q / 7 : q / 49);
    const unsigned m1 = LEVELS == 0 ? 1u : a.mask[LEVELS == 1 ? q % 7 : (q / 7) % 7];
    const unsigned m2 = LEVELS == 2 ? a.mask[q % 7] : 1u;
    const u64 *s = a.src + p * a.sstride;
#pragma unroll 4
    for (int i = 0; i < F4T_ROWS * F4T_WORDS / 256; ++i) {
        const int idx = threadIdx.x + 256 * i;
        const int rr = idx / F4T_WORDS, ww = idx % F4T_WORDS;
        const int64_t r = k0 + rr, w = w0 + ww;
        u64 x = 0;
        if (r < a.rows && w < width) {
            x = gather_word<LEVELS>(a, s + w, r, m1, m2);
            if (w == width - 1) x &= tail_mask(a.cols);
        }
        tile[rr][ww] = x;
    }
    __syncthreads();
    const int64_t kbytes = a.dp;  // bytes per output row
    const Bfly32 bf = bfly32_init(lane);
#pragma unroll 1
    for (int u = 0; u < F4T_WORDS / 8; ++u) {
        const int ww = warp * (F4T_WORDS / 8) + u;
        const int64_t w = w0 + ww;
        if (w >= width) break;
        // column 31 - lane / 63 - lane, K block kb (64 entries each, bit i =
        // entry i): the butterfly on the raw MSB-first halves, lane l holding
        // row l, leaves lane l with column 31 - l and rows LSB-first -- the
        // K-vector the nibble expansion wants, with no bit reversal
        u64 ca[4], cb[4];
#pragma unroll
        for (int kb = 0; kb < 4; ++kb) {
            const u64 x0 = tile[kb * 64 + lane][ww], x1 = tile[kb * 64 + 32 + lane][ww];
            const uint32_t c0a = transpose32m((uint32_t)(x0 >> 32), bf);
            const uint32_t c0b = transpose32m((uint32_t)(x1 >> 32), bf);
            const uint32_t c1a = transpose32m((uint32_t)x0, bf);
            const uint32_t c1b = transpose32m((uint32_t)x1, bf);
            ca[kb] = ((u64)c0b << 32) | c0a;
            cb[kb] = ((u64)c1b << 32) | c1a;
        }
        // stage this word's 64 output rows (128 B each) in shared memory, then
        // write them with coalesced 512-byte warp stores (8 lanes per row)
        const int64_t nbytes = kbytes - k0 / 2 < 128 ? kbytes - k0 / 2 : 128;
        uint8_t *d = a.dst + (int64_t)blockIdx.z * a.dstride + (w * 64) * a.dp + k0 / 2;
        uint8_t *stg = f4t_smem + F4T_TILE_BYTES + warp * 32 * F4T_STG_PITCH;
#pragma unroll
        for (int half = 0; half < 2; ++half) {
#pragma unroll
            for (int kb = 0; kb < 4; ++kb) {
                const u64 v = half ? cb[kb] : ca[kb];
                uint4 *o = reinterpret_cast<uint4 *>(stg + (31 - lane) * F4T_STG_PITCH + 32 * kb);
                o[0] = make_uint4(nib_word(v, 0), nib_word(v, 1), nib_word(v, 2), nib_word(v, 3));
                o[1] = make_uint4(nib_word(v, 4), nib_word(v, 5), nib_word(v, 6), nib_word(v, 7));
            }
            __syncwarp();
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const int row = 4 * i + (lane >> 3), off = (lane & 7) * 16;
                if (off < nbytes)
                    *reinterpret_cast<uint4 *>(d + (int64_t)(half * 32 + row) * a.dp + off) =
                        *reinterpret_cast<const uint4 *>(stg + row * F4T_STG_PITCH + off);
            }
            __syncwarp();
        }
    }
}

// 32 lanes x 32 columns of TMEM (this warp's lane quarter) := val
__device__ __forceinline__ void tmem_fill32(uint32_t taddr, uint32_t val) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,"
        "%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1};\n" ::"r"(taddr),
        "r"(val)
        : "memory");
}

// 32 f32 accumulators (integer sums < 2^23) -> their parities packed
// MSB-first (bit 31 - j = parity of column j). Adding 2^23 puts each sum's
// integer value in the mantissa, so bit 0 is the parity (FADD2: two columns
// per instruction). The low bytes of 4 columns j = k, 8+k, 16+k, 24+k are
// gathered into one word with two-level byte permutes (3 PRMT); the 8 words
// k = 0..7 then go to bit 7 - k of every byte with one shift and one masked
// OR each: 56 instructions per 32 columns instead of 96.
__device__ __forceinline__ uint32_t parity_pack32(const uint32_t *v) {
    uint32_t u[32];
#pragma unroll
    for (int j = 0; j < 32; j += 2)
        asm("{\n.reg .b64 a, r;\nmov.b64 a, {%2, %3};\nadd.rn.f32x2 r, a, %4;\nmov.b64 {%0, %1}, r;\n}\n"
            : "=r"(u[j]), "=r"(u[j + 1])
            : "r"(v[j]), "r"(v[j + 1]), "l"(0x4B0000004B000000ULL));
    uint32_t pk = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        const uint32_t hi = __byte_perm(u[24 + k], u[16 + k], 0x0040);  // bytes: u[24+k].b0, u[16+k].b0
        const uint32_t lo = __byte_perm(u[8 + k], u[k], 0x0040);        // bytes: u[8+k].b0, u[k].b0
        const uint32_t t = __byte_perm(hi, lo, 0x5410);                 // [u24+k, u16+k, u8+k, uk]
        pk |= (t << (7 - k)) & (0x01010101u << (7 - k));
    }
    return pk;
}

__device__ __forceinline__ void umma_f4(uint32_t taddr, uint64_t ad, uint64_t bd, uint32_t idesc, uint32_t acc,
                                        uint32_t sfa, uint32_t sfb) {
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::2.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%5], [%6], p;\n}\n" ::"r"(taddr),
        "l"(ad), "l"(bd), "r"(idesc), "r"(acc), "r"(sfa), "r"(sfb));
}

// Plain store (no accumulation) of a row's tile groups: group g (columns
// 32g..32g+31, MSB-first) is u32 index g^1 of the row's little-endian 64-bit
// words; a partial last group keeps the bits beyond n. XOR-accumulation
// (accumulate, K chunks, fused post-additions) goes through xor_rows_f4.
__device__ __forceinline__ void store_row_f4(const UArgs &p, const uint32_t *packed, int64_t row, int64_t g0,
                                             int nch, int64_t gprob) {
    if (row >= p.m) return;
    unsigned *crow = reinterpret_cast<unsigned *>(p.C + gprob * p.sc + row * p.pc);
#pragma unroll
    for (int c = 0; c < F4_BN / 32; ++c) {
        const int64_t rem = p.n - (g0 + c) * 32;
        if (c >= nch || rem <= 0) break;
        const uint32_t keep = rem < 32 ? (~0u >> rem) : 0u;
        unsigned *w = crow + ((g0 + c) ^ 1);
        *w = keep ? ((*w & keep) | (packed[c] & ~keep)) : packed[c];
    }
}

// XOR-accumulate a warp's 32 rows of a tile (packed[c] = 32-bit group g0+c
// of this lane's row) into C, coalesced: the row's 64-bit words ws..ws+3
// (ws = g0/2; a group outside the tile contributes a zero half, a no-op under
// XOR) are staged in shared memory, then each red.xor.b64 instruction covers
// 8 rows x 4 consecutive words, so the L2 sees one or two 32-byte sectors
// per row instead of 4 separate 8-byte requests. Products of the fused last
// Strassen level go to every C quadrant in their post mask.
__device__ __forceinline__ void xor_rows_f4(const UArgs &p, const uint32_t *packed, uint32_t stg, int64_t row0,
                                            int64_t g0, int nch, int64_t gprob, int lane) {
    uint32_t v[F4_BN / 32 + 1];
#pragma unroll
    for (int c = 0; c < F4_BN / 32; ++c) {
        const int64_t rem = p.n - (g0 + c) * 32;
        uint32_t x = (c < nch && rem > 0) ? packed[c] : 0u;
        if (rem > 0 && rem < 32) x &= ~(~0u >> rem);  // columns >= n stay untouched
        v[c] = x;
    }
    v[F4_BN / 32] = 0u;
    u64 w[4];
    if ((g0 & 1) == 0) {
#pragma unroll
        for (int k = 0; k < 4; ++k) w[k] = ((u64)v[2 * k] << 32) | v[2 * k + 1];
    } else {
        w[0] = v[0];
#pragma unroll
        for (int k = 1; k < 4; ++k) w[k] = ((u64)v[2 * k - 1] << 32) | v[2 * k];
    }
    asm volatile("st.shared.v2.u64 [%0], {%1, %2};\n" ::"r"(stg + lane * 32), "l"(w[0]), "l"(w[1]) : "memory");
    asm volatile("st.shared.v2.u64 [%0], {%1, %2};\n" ::"r"(stg + lane * 32 + 16), "l"(w[2]), "l"(w[3]) : "memory");
    __syncwarp();
    const int64_t ws = g0 >> 1;
    const int64_t nw = ((g0 + nch - 1) >> 1) - ws + 1;  // words this tile touches (<= 4)
    const int k = lane & 3;
    u64 x[4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
        asm volatile("ld.shared.u64 %0, [%1];\n" : "=l"(x[i]) : "r"(stg + (8 * i + (lane >> 2)) * 32 + k * 8) : "memory");
    __syncwarp();  // the next tile's staging overwrites this buffer
    auto red = [&](u64 *base) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int64_t row = row0 + 8 * i + (lane >> 2);
            if (row < p.m && k < nw && x[i])
                atomicXor(reinterpret_cast<unsigned long long *>(base + row * p.pc + ws + k), (unsigned long long)x[i]);
        }
    };
    if (p.post) {
        const unsigned dm = p.post_mask[gprob % 7];
        u64 *cbase = p.C + (gprob / 7) * p.sc;
#pragma unroll
        for (int Q = 0; Q < 4; ++Q)
            if (dm & (1u << Q)) red(cbase + p.qoffC[Q]);
    } else {
        red(p.C + gprob * p.sc);
    }
}

// Persistent CTA-pair kernel (cluster of 2, tcgen05.mma.cta_group::2), tiles
// 256 x (32..224), 128 B = 256 K entries per stage. TMEM: accumulators at columns 0 and 224, scale factors
// (all 0x7F) at 448..511 in both CTAs.
__global__ void __launch_bounds__(UMMA_THREADS, 1)
    k_umma_f4(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, UArgs p) {
    pdl_trigger();
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    const uint32_t base_u32 = (smem_u32(smem_raw) + 1023u) & ~1023u;
    const uint32_t sA = base_u32;
    const uint32_t sB = base_u32 + F4_STG * F4_A_ST;
    const uint32_t sBar = sB + F4_STG * F4_B_ST;
    const uint32_t bar_full = sBar, bar_empty = sBar + 8 * F4_STG, bar_tfull = sBar + 16 * F4_STG,
                   bar_tempty = bar_tfull + 16;
    const uint32_t tmem_holder = bar_tempty + 16;
    const uint32_t sEpi = sBar + F4_EPI_OFF;
    unsigned char *gen_base = smem_raw + (base_u32 - smem_u32(smem_raw));
    volatile uint32_t *tmem_holder_ptr = reinterpret_cast<volatile uint32_t *>(gen_base + (tmem_holder - base_u32));

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = cluster_rank();
    const int64_t unit = blockIdx.x >> 1, nunits = gridDim.x >> 1;
    if (warp == 0 && lane == 0) {
        for (int s = 0; s < F4_STG; ++s) {
            mbar_init(bar_full + 8 * s, 1);
            mbar_init(bar_empty + 8 * s, 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(bar_tfull + 8 * b, 1);
            mbar_init(bar_tempty + 8 * b, 256);
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
        asm volatile("prefetch.tensormap [%0];\n" ::"l"(&tmA) : "memory");
        asm volatile("prefetch.tensormap [%0];\n" ::"l"(&tmB) : "memory");
    }
    if (warp == 2) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(tmem_holder)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;\n" ::: "memory");
    }
    tc_fence_before();
    cluster_sync();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_holder_ptr;
    if (warp >= 4) {  // scale factors: every byte of columns 448..511 = 2^0
        const uint32_t lanes = tmem_base + ((uint32_t)((warp & 3) * 32) << 16);
#pragma unroll
        for (int h = 0; h < 2; ++h) tmem_fill32(lanes + F4_SF_COL + 32 * h, 0x7F7F7F7Fu);
        asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
    }
    tc_fence_before();
    cluster_sync();
    tc_fence_after();
    pdl_wait();  // barrier init, TMEM alloc and scale factors overlapped the previous kernel's tail

    const int64_t tiles_per_chunk = p.nprob * p.mt * p.nt;
    const int64_t ntiles = tiles_per_chunk * p.nchunks;
    // column tiles: the row's 32-column groups spread evenly over p.nt tiles
    // of <= 7 groups (4096 columns: 14 x 224 + 5 x 192), so no tile is a
    // narrow, TMA-bound remainder; starts stay 32-bit-word aligned
    const int ngroups = (int)((p.n + 31) / 32);
    const int gq = ngroups / p.nt, gr = ngroups % p.nt;
    auto tile_g0 = [&](int ntile) -> int { return ntile * gq + min(ntile, gr); };
    auto tile_width = [&](int ntile) -> int { return 32 * (gq + (ntile < gr ? 1 : 0)); };
    // position r of a problem's mt x nt tile grid -> (mtile, ntile):
    // column tiles fastest, or (order G > 0) blocks of G row tiles with the
    // row tile fastest inside a block
    auto tile_mn = [&](int64_t r, int &mtile, int &ntile) {
        if (p.order > 0) {
            const int64_t G = p.order;
            const int64_t blk = r / (G * p.nt), rem = r % (G * p.nt);
            const int64_t g = (int64_t)p.mt - blk * G < G ? (int64_t)p.mt - blk * G : G;  // rows in this (last) block
            mtile = (int)(blk * G + rem % g);
            ntile = (int)(rem / g);
        } else {
            mtile = (int)(r / p.nt);
            ntile = (int)(r % p.nt);
        }
    };

    if (warp == 0 && lane == 0) {
        int stage = 0;
        uint32_t phase = 0;
        for (int64_t t = unit; t < ntiles; t += nunits) {
            const int chunk = (int)(t / tiles_per_chunk);
            int64_t r = t % tiles_per_chunk;
            const int prob = (int)(r / (p.mt * p.nt));
            r %= (p.mt * p.nt);
            int mtile, ntile;
            tile_mn(r, mtile, ntile);
            const int kb0 = chunk * p.kchunk_blocks;
            const int kb1 = min(kb0 + p.kchunk_blocks, p.kblocks);
            const int arow = mtile * 256 + (int)rank * BM;
            const int brow = 32 * tile_g0(ntile) + (int)rank * (tile_width(ntile) / 2);
            for (int kb = kb0; kb < kb1; ++kb) {
                const uint32_t fb = bar_full + 8 * stage;
                mbar_wait(bar_empty + 8 * stage, phase ^ 1);
                if (rank == 0) mbar_expect_tx(fb, 2 * (F4_A_ST + F4_B_ST));
                tma_load_3d_2sm(sA + stage * F4_A_ST, &tmA, kb * BK, arow, prob, fb);
                tma_load_3d_2sm(sB + stage * F4_B_ST, &tmB, kb * BK, brow, prob, fb);
                if (++stage == F4_STG) {
                    stage = 0;
                    phase ^= 1;
                }
            }
        }
    } else if (warp == 1 && rank == 0) {
        // The whole warp walks the pipeline (warp-uniform control flow, so the
        // descriptors stay in uniform registers); one elected lane issues.
        // block-scaled idesc: a/b format E2M1 (1) at bits 7/10, K-major both,
        // N >> 3 at 17, scale format UE8M0 at 23, M >> 4 at 24, scale ids 0
        const uint32_t idesc0 = (1u << 7) | (1u << 10) | (1u << 23) | ((uint32_t)(256 >> 4) << 24);
        const uint32_t sfa = tmem_base + F4_SF_COL, sfb = tmem_base + F4_SF_COL + 32;
        const uint64_t adesc0 = smem_desc(sA, 16, 1024), bdesc0 = smem_desc(sB, 16, 1024);
        int stage = 0;
        uint32_t phase = 0;
        int it = 0;
        for (int64_t t = unit; t < ntiles; t += nunits, ++it) {
            const int chunk = (int)(t / tiles_per_chunk);
            int mtile_u, ntile;
            tile_mn((t % tiles_per_chunk) % (p.mt * p.nt), mtile_u, ntile);
            const uint32_t idesc = idesc0 | ((uint32_t)(tile_width(ntile) >> 3) << 17);
            const int kb0 = chunk * p.kchunk_blocks;
            const int kb1 = min(kb0 + p.kchunk_blocks, p.kblocks);
            const int acc = it & 1;
            const uint32_t acc_phase = (it >> 1) & 1;
            mbar_wait(bar_tempty + 8 * acc, acc_phase ^ 1);
            tc_fence_after();
            const uint32_t taddr = tmem_base + acc * F4_BN;
            for (int kb = kb0; kb < kb1; ++kb) {
                mbar_wait(bar_full + 8 * stage, phase);
                tc_fence_after();
                if (elect_one()) {
                    const uint64_t ad = adesc0 + (uint64_t)((stage * F4_A_ST) >> 4);
                    const uint64_t bd = bdesc0 + (uint64_t)((stage * F4_B_ST) >> 4);
#pragma unroll
                    for (int k = 0; k < BK / 32; ++k)
                        umma_f4(taddr, ad + 2 * k, bd + 2 * k, idesc,
                                (kb > kb0 || k > 0) ? 1u : 0u, sfa, sfb);
                    umma_commit_cg<2>(bar_empty + 8 * stage);
                }
                __syncwarp();
                if (++stage == F4_STG) {
                    stage = 0;
                    phase ^= 1;
                }
            }
            if (elect_one()) umma_commit_cg<2>(bar_tfull + 8 * acc);
            __syncwarp();
        }
    } else if (warp >= 4) {
        const int q = warp & 3;
        int it = 0;
        for (int64_t t = unit; t < ntiles; t += nunits, ++it) {
            int64_t r = t % tiles_per_chunk;
            const int prob = (int)(r / (p.mt * p.nt));
            r %= (p.mt * p.nt);
            int mtile, ntile;
            tile_mn(r, mtile, ntile);
            const int nch = tile_width(ntile) >> 5;
            const int acc = it & 1;
            const uint32_t acc_phase = (it >> 1) & 1;
            mbar_wait(bar_tfull + 8 * acc, acc_phase);
            tc_fence_after();
            // 32-column groups, software-pipelined: group c+1's TMEM load is
            // in flight while group c's parities are packed (parity_pack32).
            if (p.dbg == 2) {
                tc_fence_before();
                mbar_arrive_leader(bar_tempty + 8 * acc);
                continue;
            }
            const uint32_t trow = tmem_base + ((uint32_t)(q * 32) << 16) + acc * F4_BN;
            uint32_t packed[F4_BN / 32];
            uint32_t vb[2][32];
            TMEM_LD32(trow, vb[0]);
            TMEM_WAIT_LD32(vb[0]);
#pragma unroll
            for (int c = 0; c < F4_BN / 32; ++c) {
                packed[c] = 0;
                if (c < nch) {
                    if (c + 1 < nch) TMEM_LD32(trow + (c + 1) * 32, vb[(c + 1) & 1]);
                    packed[c] = parity_pack32(vb[c & 1]);
                    if (c + 1 < nch) TMEM_WAIT_LD32(vb[(c + 1) & 1]);
                }
            }
            tc_fence_before();
            mbar_arrive_leader(bar_tempty + 8 * acc);
            const int64_t row = (int64_t)mtile * 256 + (int64_t)rank * BM + q * 32 + lane;
            if (p.dbg == 1) continue;
            if (p.post || p.mode >= 1) {
                xor_rows_f4(p, packed, sEpi + q * 1024, row - lane, tile_g0(ntile), nch, p.q0 + prob, lane);
                continue;
            }
            store_row_f4(p, packed, row, (int64_t)tile_g0(ntile), nch, p.q0 + prob);
        }
    }
    tc_fence_before();
    cluster_sync();
    if (warp == 2) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;\n" ::"r"(tmem_base) : "memory");
    }
}

}  // namespace

static int launch_expand4(const ExpandArgs &a, int64_t nprob, bool cols, cudaStream_t s) {
    const int64_t width = words_per_row(a.cols);
    if (!a.rows || !width || !nprob) return GF2_OK;
    const bool g7 = a.levels == 1 && a.q0 % 7 == 0 && nprob % 7 == 0;
    const bool g49 = a.levels == 2 && a.q0 % 49 == 0 && nprob % 49 == 0;
    if (!cols && (g7 || g49)) {
        // 2 rows per warp: 48 registers, more resident blocks and a finer grid
        // than 4 (43 vs 45 us at cfg3; forcing occupancy via launch bounds spills)
        // one row per warp when two would give fewer than 4 blocks per SM
        // (cfg2 at cutoff 1024: 448 blocks; 16.8 -> 15.0 us for both sides)
        const int64_t blocks2 = (width + 31) / 32 * ((a.rows + 15) / 16) * (nprob / 7);
        if (blocks2 < 4 * num_sms()) {
            dim3 grd((unsigned)((width + 31) / 32), (unsigned)((a.rows + 8 - 1) / 8), (unsigned)(nprob / 7));
            if (g7)
                GF2_LAUNCH(launch_k(k_expand4_rows7<1, 1>, grd, 256, 0, s, 1, a));
            else
                GF2_LAUNCH(launch_k(k_expand4_rows7<1, 2>, grd, 256, 0, s, 1, a));
        } else {
            dim3 grd((unsigned)((width + 31) / 32), (unsigned)((a.rows + 8 * 2 - 1) / (8 * 2)), (unsigned)(nprob / 7));
            if (g7)
                GF2_LAUNCH(launch_k(k_expand4_rows7<2, 1>, grd, 256, 0, s, 1, a));
            else
                GF2_LAUNCH(launch_k(k_expand4_rows7<2, 2>, grd, 256, 0, s, 1, a));
        }
        note_launch();
        return check_cuda(cudaGetLastError(), "k_expand4_rows7 launch");
    }
    if (!cols) {
        dim3 grd((unsigned)((width + 31) / 32), (unsigned)((a.rows + 8 * F4_ROWS_PER_WARP - 1) / (8 * F4_ROWS_PER_WARP)),
                 (unsigned)nprob);
        if (a.levels == 0)
            GF2_LAUNCH(launch_k(k_expand4_rows<0>, grd, 256, 0, s, 1, a));
        else if (a.levels == 1)
            GF2_LAUNCH(launch_k(k_expand4_rows<1>, grd, 256, 0, s, 1, a));
        else
            GF2_LAUNCH(launch_k(k_expand4_rows<2>, grd, 256, 0, s, 1, a));
    } else {
        // a.dp = bytes per K-major row = (K rows rounded to 64) / 2
        const unsigned gy = (unsigned)((a.dp * 2 + F4T_ROWS - 1) / F4T_ROWS);
        static bool attr[64] = {};
        if (first_on_device(attr)) {
#define GF2_F4T_ATTR(L, W)                                                                                     \
    GF2_TRY(check_cuda(cudaFuncSetAttribute(k_expand4_cols<L, W>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                                            f4t_smem<W>()),                                                     \
                       "expand4 smem attr"))
            GF2_F4T_ATTR(0, 16); GF2_F4T_ATTR(1, 16); GF2_F4T_ATTR(2, 16);
            GF2_F4T_ATTR(0, 8); GF2_F4T_ATTR(1, 8); GF2_F4T_ATTR(2, 8);
#undef GF2_F4T_ATTR
        }
        const int64_t wide = (width + 15) / 16 * (int64_t)gy * nprob;  // blocks with 16-word tiles
        if (wide >= num_sms()) {
            dim3 grd((unsigned)((width + 15) / 16), gy, (unsigned)nprob);
            if (a.levels == 0)
                GF2_LAUNCH(launch_k(k_expand4_cols<0, 16>, grd, 256, f4t_smem<16>(), s, 1, a));
            else if (a.levels == 1)
                GF2_LAUNCH(launch_k(k_expand4_cols<1, 16>, grd, 256, f4t_smem<16>(), s, 1, a));
            else
                GF2_LAUNCH(launch_k(k_expand4_cols<2, 16>, grd, 256, f4t_smem<16>(), s, 1, a));
        } else {
            dim3 grd((unsigned)((width + 7) / 8), gy, (unsigned)nprob);
            if (a.levels == 0)
                GF2_LAUNCH(launch_k(k_expand4_cols<0, 8>, grd, 256, f4t_smem<8>(), s, 1, a));
            else if (a.levels == 1)
                GF2_LAUNCH(launch_k(k_expand4_cols<1, 8>, grd, 256, f4t_smem<8>(), s, 1, a));
            else
                GF2_LAUNCH(launch_k(k_expand4_cols<2, 8>, grd, 256, f4t_smem<8>(), s, 1, a));
        }
    }
    note_launch();
    return check_cuda(cudaGetLastError(), "k_expand4 launch");
}

// FP4 engine (kind::mxf4, CTA pairs): A as nibble rows (m x kb bytes), B
// transposed to nibble rows (n x kb bytes), kb = round64(l) / 2.
int launch_umma_f4(const UmmaJob &jb, int64_t nprob, cudaStream_t s) {
    static bool attr[64] = {};
    if (first_on_device(attr)) {
        GF2_TRY(check_cuda(cudaFuncSetAttribute(k_umma_f4, cudaFuncAttributeMaxDynamicSharedMemorySize, F4_SMEM),
                           "umma_f4 smem attr"));
    }
    const int64_t kb = (jb.l + 63) / 64 * 32;   // bytes per nibble row
    const int64_t np = (jb.n + 63) / 64 * 64;   // B rows (columns of B), whole words
    const int64_t per = jb.m * kb + np * kb;
    const int64_t cap = (int64_t)8 << 30;
    int64_t qchunk = std::max<int64_t>(1, std::min<int64_t>(nprob, cap / std::max<int64_t>(per, 1)));
    if (jb.fuse_pre == 1 && qchunk >= 7) qchunk -= qchunk % 7;  // whole 7-product groups (k_expand4_rows7)
    if (jb.fuse_pre == 2 && qchunk >= 49) qchunk -= qchunk % 49;  // whole 49-product groups
    uint8_t *ws = nullptr;
    GF2_TRY(pool_setup());
    cudaError_t e = cudaMallocAsync((void **)&ws, (size_t)(qchunk * per), s);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return set_error(GF2_ERR_OOM, std::string("umma workspace: ") + cudaGetErrorString(e));
    }
    uint8_t *a4 = ws, *b4 = ws + qchunk * jb.m * kb;
    const int64_t f2 = jb.fuse_pre == 2 ? 2 : 1;
    ExpandArgs ea{};
    ea.src = jb.A; ea.sp = jb.pa; ea.sstride = jb.sa; ea.levels = jb.fuse_pre;
    ea.qoff[1] = f2 * jb.l / 64; ea.qoff[2] = f2 * jb.m * jb.pa; ea.qoff[3] = ea.qoff[1] + ea.qoff[2];
    ea.qoff2[1] = jb.l / 64; ea.qoff2[2] = jb.m * jb.pa; ea.qoff2[3] = ea.qoff2[1] + ea.qoff2[2];
    for (int i = 0; i < 7; ++i) ea.mask[i] = jb.maskA[i];
    ea.dst = a4; ea.dp = kb; ea.dstride = jb.m * kb; ea.rows = jb.m; ea.cols = jb.l;
    // B side: row expansion of B^T when given transposed, else the
    // transposing column expansion of B
    const bool bt = jb.b_trans != 0;
    const int64_t brows = bt ? jb.n : jb.l, bcols = bt ? jb.l : jb.n;
    ExpandArgs eb{};
    eb.src = jb.B; eb.sp = jb.pb; eb.sstride = jb.sb; eb.levels = jb.fuse_pre;
    eb.qoff[1] = f2 * bcols / 64; eb.qoff[2] = f2 * brows * jb.pb; eb.qoff[3] = eb.qoff[1] + eb.qoff[2];
    eb.qoff2[1] = bcols / 64; eb.qoff2[2] = brows * jb.pb; eb.qoff2[3] = eb.qoff2[1] + eb.qoff2[2];
    for (int i = 0; i < 7; ++i) eb.mask[i] = jb.maskB[i];
    eb.dst = b4; eb.dp = kb; eb.dstride = np * kb; eb.rows = brows; eb.cols = bcols;

    UArgs ua{};
    ua.C = jb.C; ua.pc = jb.pc; ua.sc = jb.sc;
    ua.m = jb.m; ua.n = jb.n; ua.Wn = words_per_row(jb.n);
    ua.mt = (int)((jb.m + 255) / 256);
    // GF2_F4_BN: maximum column-tile width (tuning knob; 224 measured best)
    static const int f4bn = getenv("GF2_F4_BN") ? std::max(32, std::min(F4_BN, atoi(getenv("GF2_F4_BN")))) : F4_BN;
    ua.nt = (int)((jb.n + f4bn - 1) / f4bn);
    ua.kblocks = (int)((kb + BK - 1) / BK);
    ua.kchunk_blocks = (int)(F4_KCHUNK / (2 * BK));
    ua.nchunks = (ua.kblocks + ua.kchunk_blocks - 1) / ua.kchunk_blocks;
    ua.post = jb.fuse_post;
    static const int f4dbg = getenv("GF2_F4_DBG") ? atoi(getenv("GF2_F4_DBG")) : 0;
    ua.dbg = f4dbg;
    // tile raster: for Strassen leaves with long K (cfg3/cfg5: 7^d problems
    // of 8192^3) row tiles run fastest, so each wave of 74 pairs spans ~2.3
    // column tiles x all row tiles: the GEMM's DRAM reads drop 694 -> 590 MB
    // per cfg3 launch and the launch 0.904 -> 0.900 ms (same box, 5 runs).
    // Elsewhere column tiles stay fastest: row-tile-fastest measured slower
    // for cfg4's single 10000x7001x12345 product (233 -> 236 us) and for
    // 1024-deep leaves (37 -> 40 us). GF2_F4_ORDER = G > 0 forces blocks of
    // G row tiles (G >= mt: row tiles fastest), 0 column tiles fastest.
    static const int f4order = getenv("GF2_F4_ORDER") ? atoi(getenv("GF2_F4_ORDER")) : -1;
    ua.order = f4order >= 0 ? f4order : ((jb.fuse_post && ua.kblocks >= 16) ? ua.mt : 0);
    // G > mt is the same raster; clamping keeps G x nt small, so the kernel's
    // per-tile index divisions stay on the fast 32-bit path (a 2^30 block
    // pushed them onto 64-bit division and cost the cfg3 GEMM 1.5 %)
    if (ua.order > ua.mt) ua.order = ua.mt;
    int rc = GF2_OK;
    if (jb.fuse_post) {
        ua.qoffC[1] = jb.n / 64; ua.qoffC[2] = jb.m * jb.pc; ua.qoffC[3] = ua.qoffC[1] + ua.qoffC[2];
        for (int i = 0; i < 7; ++i) ua.post_mask[i] = jb.maskC[i];
        ua.mode = 2;
    } else if (ua.nchunks > 1) {
        if (!jb.accumulate)
            for (int64_t q = 0; q < nprob && rc == GF2_OK; ++q) {
                gf2_view v{jb.C + q * jb.sc, jb.pc, jb.m, jb.n};
                rc = launch_zero(v, s);
            }
        ua.mode = 2;
    } else {
        ua.mode = jb.accumulate ? 1 : 0;
    }
    for (int64_t q0 = 0; q0 < nprob && rc == GF2_OK; q0 += qchunk) {
        const int64_t nq = std::min<int64_t>(qchunk, nprob - q0);
        ea.q0 = eb.q0 = ua.q0 = q0;
        ua.nprob = nq;
        // with B^T produced on the side stream (depth 1), the A side expands on
        // the high-priority stream so it takes SM slots alongside the transpose
        // instead of queueing behind it (memset -> GEMM start 119 -> 110 us)
        SideStream *sd = nullptr;
        const bool hi = jb.b_ready && q0 == 0 && side_stream(&sd) == GF2_OK;
        if (hi) {
            rc = check_cuda(cudaEventRecord(sd->hi_fork, s), "hi fork");
            if (rc == GF2_OK) rc = check_cuda(cudaStreamWaitEvent(sd->hi, sd->hi_fork, 0), "hi fork wait");
            if (rc == GF2_OK) rc = launch_expand4(ea, nq, false, sd->hi);
            if (rc == GF2_OK) rc = check_cuda(cudaEventRecord(sd->hi_join, sd->hi), "hi join");
        } else {
            rc = launch_expand4(ea, nq, false, s);
        }
        if (rc == GF2_OK && jb.b_ready && q0 == 0) rc = check_cuda(cudaStreamWaitEvent(s, jb.b_ready, 0), "join wait");
        if (rc == GF2_OK) rc = launch_expand4(eb, nq, !bt, s);
        if (rc == GF2_OK && hi) rc = check_cuda(cudaStreamWaitEvent(s, sd->hi_join, 0), "hi join wait");
        CUtensorMap ta, tb;
        if (rc == GF2_OK) rc = make_map(&ta, a4, (uint64_t)kb, (uint64_t)jb.m, (uint64_t)nq, kb, jb.m * kb);
        if (rc == GF2_OK)  // rows past n (never written on the B^T path) read as zeros
            rc = make_map(&tb, b4, (uint64_t)kb, (uint64_t)jb.n, (uint64_t)nq, kb, np * kb, F4_BNH);
        if (rc != GF2_OK) break;
        const int64_t ntiles = (int64_t)ua.nchunks * nq * ua.mt * ua.nt;
        const int64_t pairs = std::min<int64_t>(ntiles, num_sms() / 2);
        const int tidx = timer_begin(s, (double)jb.m * (double)jb.l * (double)jb.n * (double)nq);
        rc = check_cuda(launch_k(k_umma_f4, dim3((unsigned)(2 * pairs)), dim3(UMMA_THREADS), F4_SMEM, s, 2, ta, tb, ua),
                        "k_umma_f4 launch");
        note_launch();
        timer_end(tidx, s);
    }
    cudaFreeAsync(ws, s);
    return rc;
}

}  // namespace gf2
