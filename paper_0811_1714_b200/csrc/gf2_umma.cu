// Tensor-core GF(2) contraction on sm_100a (north_star (c)).
//
// C (^)= A.B over GF(2) as an integer product with the sum reduced mod 2:
//   1. k_expand: packed bits -> one byte per entry (0 or ONE), A row-major
//      (K contiguous) and B row-major (N contiguous) -- no transpose needed,
//      B is consumed MN-major by the MMA.
//   2. k_umma: persistent TMA -> tcgen05.mma -> TMEM pipeline.
//        warp 0  : TMA producer (3 boxes per stage: A 128x128, B 2 x 128x128)
//        warp 1  : MMA issuer, tcgen05.mma.cta_group::1 M=128 N=256 K=32
//        warp 2  : TMEM allocator (512 columns = two 256-column accumulators)
//        warps 4-7: epilogue: tcgen05.ld 32x32b.x32 -> parity -> 32-bit packs
//                   (column c0+j -> bit 31-j, the reference's MSB-first order)
//                   -> store / XOR / red.xor into C.
//      Smem operands use the 128-byte swizzle: A K-major (8-row atoms,
//      SBO 1024), B MN-major (8-k-row atoms of 128 N bytes, SBO 1024, the two
//      128-column halves LBO = 16 KiB apart).
//   kind::i8 (u8 0/1, s32 accumulators) is exact by construction (even mod
//   2^32 the LSB is right). kind::f8f6f4 (e4m3 1.0 = 0x38, f32 accumulators)
//   is exact while partial sums stay integers representable in the
//   accumulator: K is cut into chunks of <= 8192 whose parities are XORed
//   (red.global.xor), far inside the 2^24 f32 integer range.
#include <cuda.h>

#include <stdlib.h>

#include <algorithm>
#include <vector>

#include "gf2_tc.cuh"

namespace gf2 {

namespace {

__device__ __forceinline__ void expand_store(const ExpandArgs &a, uint8_t *drow, u64 x, int lane, int64_t nbytes) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const int ci = lane + 32 * k;  // 16-byte chunk within the warp's 2 KiB
        const u64 xv = __shfl_sync(0xffffffffu, x, ci >> 2);
        if (ci * 16 >= nbytes) continue;
        const int c = ci & 3;
        const uint32_t h16 = (uint32_t)(xv >> (48 - 16 * c)) & 0xFFFFu;
        const uint32_t rv = __brev(h16) >> 16;  // entry 16c+i at bit i
        uint4 v;
        v.x = (((rv >> 0) & 0xF) * 0x00204081u & 0x01010101u) * a.one;
        v.y = (((rv >> 4) & 0xF) * 0x00204081u & 0x01010101u) * a.one;
        v.z = (((rv >> 8) & 0xF) * 0x00204081u & 0x01010101u) * a.one;
        v.w = (((rv >> 12) & 0xF) * 0x00204081u & 0x01010101u) * a.one;
        *reinterpret_cast<uint4 *>(drow + ci * 16) = v;
    }
}

template <int LEVELS>
__global__ void k_expand(ExpandArgs a) {
    pdl_begin();
    const int64_t width = words_per_row(a.cols);
    const int lane = threadIdx.x & 31;
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t j0 = j - lane;  // first word of this warp
    if (j0 >= width) return;
    const u64 tm = (j == width - 1) ? tail_mask(a.cols) : ~0ULL;
    const int64_t q = a.q0 + blockIdx.z;
    const int64_t p = LEVELS == 0 ? q : (LEVELS == 1 ? q / 7 : q / 49);
    const unsigned m1 = LEVELS == 0 ? 1u : a.mask[LEVELS == 1 ? q % 7 : (q / 7) % 7];
    const unsigned m2 = LEVELS == 2 ? a.mask[q % 7] : 1u;
    const u64 *s = a.src + p * a.sstride + j;
    uint8_t *d = a.dst + (int64_t)blockIdx.z * a.dstride + j0 * 64;
    const int64_t nbytes = min((int64_t)2048, a.dp - j0 * 64);  // bytes this warp owns in a row
    const bool live = j < width;
    for (int64_t r = blockIdx.y; r < a.rows; r += 2 * (int64_t)gridDim.y) {
        const int64_t r2 = r + gridDim.y;
        const u64 x0 = live ? gather_word<LEVELS>(a, s, r, m1, m2) & tm : 0;
        const u64 x1 = (live && r2 < a.rows) ? gather_word<LEVELS>(a, s, r2, m1, m2) & tm : 0;
        expand_store(a, d + r * a.dp, x0, lane, nbytes);
        if (r2 < a.rows) expand_store(a, d + r2 * a.dp, x1, lane, nbytes);
    }
}

__device__ __forceinline__ void store_row(const UArgs &p, const uint32_t *packed, int64_t row, int ntile,
                                          int64_t gprob) {
    if (row >= p.m) return;
    if (p.post) {
        const unsigned dm = p.post_mask[gprob % 7];
        u64 *cbase = p.C + (gprob / 7) * p.sc + row * p.pc;
#pragma unroll
        for (int Q = 0; Q < 4; ++Q) {
            if (!(dm & (1u << Q))) continue;
            u64 *crow = cbase + p.qoffC[Q];
#pragma unroll
            for (int w = 0; w < BN / 64; ++w) {
                const int64_t wi = (int64_t)ntile * (BN / 64) + w;
                if (wi >= p.Wn) break;
                const u64 v = ((u64)packed[2 * w] << 32) | (u64)packed[2 * w + 1];
                if (v) atomicXor(reinterpret_cast<unsigned long long *>(crow + wi), (unsigned long long)v);
            }
        }
        return;
    }
    u64 *crow = p.C + gprob * p.sc + row * p.pc;
    const u64 ctm = tail_mask(p.n);
#pragma unroll
    for (int w = 0; w < BN / 64; ++w) {
        const int64_t wi = (int64_t)ntile * (BN / 64) + w;
        if (wi >= p.Wn) break;
        const u64 v = ((u64)packed[2 * w] << 32) | (u64)packed[2 * w + 1];
        if (p.mode >= 1) {  // XOR-accumulate / K-chunk partials: fire-and-forget red.xor, no epilogue load
            if (v) atomicXor(reinterpret_cast<unsigned long long *>(crow + wi), (unsigned long long)v);
        } else if (wi == p.Wn - 1 && ctm != ~0ULL) {
            crow[wi] = (crow[wi] & ~ctm) | v;
        } else {
            crow[wi] = v;
        }
    }
}

template <int CG>
struct Geo {
    static constexpr int MT = BM * CG;                   // rows per (pair) tile
    static constexpr int A_ST = BM * BK;                 // 16 KiB per CTA
    static constexpr int B_ST = (BN / CG) * BK;          // this CTA's N columns x BK
    static constexpr int STG = CG == 1 ? 4 : 6;          // pipeline stages
    static constexpr int SMEM = STG * (A_ST + B_ST) + 2048;
};

// CG = 1: one CTA, tile 128 x 256. CG = 2: a CTA pair (cluster of 2) with
// tcgen05.mma.cta_group::2, tile 256 x 256; each CTA stages its 128 rows of A
// and 128 of the 256 columns of B, so per-SM operand traffic drops by 1/3.
template <int KIND, int CG>
__global__ void __launch_bounds__(UMMA_THREADS, 1)
    k_umma(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, UArgs p) {
    pdl_trigger();
    using G = Geo<CG>;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    const uint32_t base_u32 = (smem_u32(smem_raw) + 1023u) & ~1023u;  // 128-byte swizzle atoms
    const uint32_t sA = base_u32;
    const uint32_t sB = base_u32 + G::STG * G::A_ST;
    const uint32_t sBar = sB + G::STG * G::B_ST;
    const uint32_t bar_full = sBar, bar_empty = sBar + 8 * G::STG, bar_tfull = sBar + 16 * G::STG,
                   bar_tempty = bar_tfull + 16;
    const uint32_t tmem_holder = bar_tempty + 16;
    unsigned char *gen_base = smem_raw + (base_u32 - smem_u32(smem_raw));
    volatile uint32_t *tmem_holder_ptr = reinterpret_cast<volatile uint32_t *>(gen_base + (tmem_holder - base_u32));

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = CG == 1 ? 0u : cluster_rank();
    const int64_t unit = CG == 1 ? blockIdx.x : (blockIdx.x >> 1);  // CTA or pair index
    const int64_t nunits = CG == 1 ? gridDim.x : (gridDim.x >> 1);
    if (warp == 0 && lane == 0) {
        for (int s = 0; s < G::STG; ++s) {
            mbar_init(bar_full + 8 * s, 1);
            mbar_init(bar_empty + 8 * s, 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(bar_tfull + 8 * b, 1);
            mbar_init(bar_tempty + 8 * b, 128 * CG);
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
        asm volatile("prefetch.tensormap [%0];\n" ::"l"(&tmA) : "memory");
        asm volatile("prefetch.tensormap [%0];\n" ::"l"(&tmB) : "memory");
    }
    if (warp == 2) {
        if (CG == 1) {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(tmem_holder)
                         : "memory");
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
        } else {
            asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(tmem_holder)
                         : "memory");
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;\n" ::: "memory");
        }
    }
    tc_fence_before();
    if (CG == 1)
        __syncthreads();
    else
        cluster_sync();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_holder_ptr;
    pdl_wait();  // setup above overlapped the previous kernel's tail

    const int64_t tiles_per_chunk = p.nprob * p.mt * p.nt;
    const int64_t ntiles = tiles_per_chunk * p.nchunks;

    if (warp == 0 && lane == 0) {
        // ---------------- TMA producer (both CTAs of a pair)
        int stage = 0;
        uint32_t phase = 0;
        for (int64_t t = unit; t < ntiles; t += nunits) {
            const int chunk = (int)(t / tiles_per_chunk);
            int64_t r = t % tiles_per_chunk;
            const int prob = (int)(r / (p.mt * p.nt));
            r %= (p.mt * p.nt);
            const int mtile = (int)(r / p.nt), ntile = (int)(r % p.nt);
            const int kb0 = chunk * p.kchunk_blocks;
            const int kb1 = min(kb0 + p.kchunk_blocks, p.kblocks);
            const int arow = mtile * G::MT + (int)rank * BM;
            for (int kb = kb0; kb < kb1; ++kb) {
                const uint32_t fb = bar_full + 8 * stage;
                const uint32_t a_dst = sA + stage * G::A_ST, b_dst = sB + stage * G::B_ST;
                mbar_wait(bar_empty + 8 * stage, phase ^ 1);
                if (CG == 1) {
                    mbar_expect_tx(fb, G::A_ST + G::B_ST);
                    tma_load_3d(a_dst, &tmA, kb * BK, arow, prob, fb);
                    tma_load_3d(b_dst, &tmB, ntile * BN, kb * BK, prob, fb);
                    tma_load_3d(b_dst + G::B_ST / 2, &tmB, ntile * BN + 128, kb * BK, prob, fb);
                } else {
                    if (rank == 0) mbar_expect_tx(fb, 2 * (G::A_ST + G::B_ST));
                    tma_load_3d_2sm(a_dst, &tmA, kb * BK, arow, prob, fb);
                    tma_load_3d_2sm(b_dst, &tmB, ntile * BN + (int)rank * 128, kb * BK, prob, fb);
                }
                if (++stage == G::STG) {
                    stage = 0;
                    phase ^= 1;
                }
            }
        }
    } else if (warp == 1 && rank == 0) {
        // ---------------- MMA issuer (leader CTA): warp-uniform loop, one
        // elected lane issues (descriptors stay in uniform registers)
        const uint32_t idesc = (KIND == 0 ? (2u << 4) : (1u << 4)) | (1u << 16) | ((uint32_t)(BN >> 3) << 17) |
                               ((uint32_t)(G::MT >> 4) << 24);
        const uint64_t adesc0 = smem_desc(sA, 16, 1024), bdesc0 = smem_desc(sB, CG == 1 ? G::B_ST / 2 : 16, 1024);
        int stage = 0;
        uint32_t phase = 0;
        int it = 0;
        for (int64_t t = unit; t < ntiles; t += nunits, ++it) {
            const int chunk = (int)(t / tiles_per_chunk);
            const int kb0 = chunk * p.kchunk_blocks;
            const int kb1 = min(kb0 + p.kchunk_blocks, p.kblocks);
            const int acc = it & 1;
            const uint32_t acc_phase = (it >> 1) & 1;
            mbar_wait(bar_tempty + 8 * acc, acc_phase ^ 1);
            tc_fence_after();
            const uint32_t taddr = tmem_base + acc * BN;
            for (int kb = kb0; kb < kb1; ++kb) {
                mbar_wait(bar_full + 8 * stage, phase);
                tc_fence_after();
                if (elect_one()) {
                    const uint64_t ad = adesc0 + (uint64_t)((stage * G::A_ST) >> 4);
                    const uint64_t bd = bdesc0 + (uint64_t)((stage * G::B_ST) >> 4);
#pragma unroll
                    for (int k = 0; k < BK / 32; ++k)  // A: +32 B along K; B (MN-major): +32 rows of 128 B
                        umma_cg<KIND, CG>(taddr, ad + 2 * k, bd + 256 * k, idesc, (kb > kb0 || k > 0) ? 1u : 0u);
                    umma_commit_cg<CG>(bar_empty + 8 * stage);
                }
                __syncwarp();
                if (++stage == G::STG) {
                    stage = 0;
                    phase ^= 1;
                }
            }
            if (elect_one()) umma_commit_cg<CG>(bar_tfull + 8 * acc);
            __syncwarp();
        }
    } else if (warp >= 4) {
        // ---------------- epilogue: TMEM -> parity bits -> C (each CTA its rows)
        const int q = warp & 3;  // TMEM lane quadrant
        int it = 0;
        for (int64_t t = unit; t < ntiles; t += nunits, ++it) {
            int64_t r = t % tiles_per_chunk;
            const int prob = (int)(r / (p.mt * p.nt));
            r %= (p.mt * p.nt);
            const int mtile = (int)(r / p.nt), ntile = (int)(r % p.nt);
            const int acc = it & 1;
            const uint32_t acc_phase = (it >> 1) & 1;
            mbar_wait(bar_tfull + 8 * acc, acc_phase);
            tc_fence_after();
            uint32_t packed[BN / 32];
#pragma unroll
            for (int c = 0; c < BN / 32; ++c) {
                uint32_t v[32];
                TMEM_LD32(tmem_base + ((uint32_t)(q * 32) << 16) + acc * BN + c * 32, v);
                asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
                uint32_t pk = 0;
#pragma unroll
                for (int j = 0; j < 32; ++j) {
                    uint32_t bit;
                    if (KIND == 0)
                        bit = v[j] & 1u;
                    else
                        bit = __float_as_uint(__uint_as_float(v[j]) + 8388608.0f) & 1u;
                    pk = (pk << 1) | bit;
                }
                packed[c] = pk;
            }
            tc_fence_before();
            if (CG == 1)
                mbar_arrive(bar_tempty + 8 * acc);
            else
                mbar_arrive_leader(bar_tempty + 8 * acc);
            const int64_t row = (int64_t)mtile * G::MT + (int64_t)rank * BM + q * 32 + lane;
            store_row(p, packed, row, ntile, p.q0 + prob);
        }
    }
    tc_fence_before();
    if (CG == 1)
        __syncthreads();
    else
        cluster_sync();
    if (warp == 2) {
        tc_fence_after();
        if (CG == 1)
            asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem_base) : "memory");
        else
            asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;\n" ::"r"(tmem_base) : "memory");
    }
}

// ------------------------------------------------------------------ converter-fed i8
// k_umma_cv: the same 2-SM tcgen05 pipeline, but the operand tiles are built
// in shared memory straight from the PACKED bits by 8 converter warps -- no
// byte-expanded copies in HBM. Trick: with SIGNED int8 a set bit may become
// 0xFF (= -1): (-1)(-1) = +1, so the s32 dot product still counts the common
// ones. prmt(x << s, 0, 0xBA98) replicates bit 7 of each byte of (x << s),
// i.e. turns 4 bits of x into 4 bytes with 2 instructions (the shift runs on
// the FMA pipe as IMAD.SHL). The bytes come out in the order
//     K (or N) position 4s + i  <-  element 8(3 - i) + s   (within 32)
// A fixed permutation of K is harmless when B's rows are permuted alike
// (row addressing only); the permutation of N is undone for free when the
// epilogue packs parity bits (compile-time shift amounts).
struct CvArgs {
    const u64 *A;
    int64_t pa, sa;
    int64_t qoffA[4];
    unsigned maskA[7];
    const u64 *B;
    int64_t pb, sb;
    int64_t qoffB[4];
    unsigned maskB[7];
    int fuse;  // 1: product q = 7p + i reads XORs of source p's quadrants
    int64_t l, Wl;
};

__device__ __forceinline__ void cp_async_8(uint32_t saddr, const void *g, bool pred) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(saddr), "l"(g), "r"(pred ? 8 : 0)
                 : "memory");
}
__device__ __forceinline__ u64 lds64(uint32_t addr) {
    u64 v;
    asm volatile("ld.shared.u64 %0, [%1];\n" : "=l"(v) : "r"(addr));
    return v;
}

__device__ __forceinline__ uint32_t expand4(uint32_t x, int s) {
    uint32_t r;
    asm("prmt.b32 %0, %1, 0, 0xBA98;\n" : "=r"(r) : "r"(x << s));
    return r;
}

// K position of element e (0..31) in the expanded 32-block: p = 4(e & 7) + 3 - (e >> 3)
__host__ __device__ constexpr int kpos_of(int e) { return 4 * (e & 7) + 3 - (e >> 3); }
// element (output column) held at expanded position j (inverse of kpos_of)
__host__ __device__ constexpr int elem_at(int j) { return 8 * (3 - (j & 3)) + (j >> 2); }

constexpr int CV_THREADS = 512;
constexpr int CV_STG = 4;                // expanded operand stages (even: steps go in pairs)
constexpr int CV_A_ST = BM * BK;         // 16 KiB: this CTA's 128 rows x 128 K
constexpr int CV_B_ST = (BN / 2) * BK;   // 16 KiB: this CTA's 128 columns x 128 K
constexpr int CV_PST = 6;                // packed staging stages: 2 in use + 4 in flight
constexpr int CV_P_ST = 256 * 8 * 8;     // 256 threads x (4 A + 4 B terms) x 8 B = 16 KiB
constexpr int CV_SMEM = CV_STG * (CV_A_ST + CV_B_ST) + CV_PST * CV_P_ST + 2048;
static_assert(CV_SMEM <= 232448, "k_umma_cv shared memory");

__global__ void __launch_bounds__(CV_THREADS, 1) k_umma_cv(CvArgs cv, UArgs p) {
    pdl_trigger();
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    const uint32_t base_u32 = (smem_u32(smem_raw) + 1023u) & ~1023u;
    const uint32_t sA = base_u32;
    const uint32_t sB = base_u32 + CV_STG * CV_A_ST;
    const uint32_t sP = sB + CV_STG * CV_B_ST;  // packed staging ring (cp.async)
    const uint32_t sBar = sP + CV_PST * CV_P_ST;
    const uint32_t bar_full = sBar, bar_empty = sBar + 8 * CV_STG, bar_tfull = sBar + 16 * CV_STG,
                   bar_tempty = bar_tfull + 16;
    const uint32_t tmem_holder = bar_tempty + 16;
    const uint32_t bar_cfull = tmem_holder + 16;  // per-CTA: converter warps -> relay
    unsigned char *gen_base = smem_raw + (base_u32 - smem_u32(smem_raw));
    volatile uint32_t *tmem_holder_ptr = reinterpret_cast<volatile uint32_t *>(gen_base + (tmem_holder - base_u32));

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = cluster_rank();
    const int64_t unit = blockIdx.x >> 1, nunits = gridDim.x >> 1;
    if (warp == 4 && lane == 0) {
        for (int s = 0; s < CV_STG; ++s) {
            mbar_init(bar_full + 8 * s, 2);       // one relay arrival from each CTA of the pair
            mbar_init(bar_cfull + 8 * s, 8);      // the 8 converter warps of this CTA
            mbar_init(bar_empty + 8 * s, 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(bar_tfull + 8 * b, 1);
            mbar_init(bar_tempty + 8 * b, 2 * 128);
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    if (warp == 5) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(tmem_holder)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;\n" ::: "memory");
    }
    tc_fence_before();
    cluster_sync();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_holder_ptr;
    pdl_wait();  // setup above overlapped the previous kernel's tail

    const int64_t tiles = p.nprob * p.mt * p.nt;

    if (warp >= 8) {
        // ---------------- converters: packed bits -> swizzled signed bytes
        const int ct = threadIdx.x - 256;
        const int ra = ct >> 1, wa = ct & 1;                      // A: row, word of the K block
        const int l8 = ct & 7, qq = ct >> 3;                      // B: conflict-free lane map
        const int ba = l8 >> 1, wb = l8 & 1, s0 = qq & 7, g32 = qq >> 3;
        const int kr = 32 * g32 + 8 * ba + s0;                    // packed B row in the K block
        const int kp = 32 * g32 + kpos_of(8 * ba + s0);           // its smem row (K permutation)
        const u64 atm = tail_mask(cv.l), btm = tail_mask(p.n);
        // steps = (tile, K block) pairs of this pair's tiles, in MMA order;
        // step i+3's packed words are in flight (cp.async) while step i expands.
        // Two cursors walk the steps incrementally (tile decode only on a tile
        // change): `ld` issues the copies, `cs` consumes them.
        // staging is [term][thread] (8 B words): lanes touch consecutive words,
        // so the 8-byte cp.async writes and LDS.64 reads are conflict-free
        const uint32_t myslot = sP + ct * 8;
        struct Cur {
            int64_t t;
            int kb;
            const u64 *pA, *pB;  // this thread's A word / B word at kb = 0
            unsigned ma, mb;
            bool arow_ok, bword_ok;
            bool alast_possible, blast;
        };
        auto tile_setup = [&](Cur &c) {
            int64_t r = c.t;
            const int64_t prob = r / (p.mt * p.nt);
            r %= (p.mt * p.nt);
            const int mtile = (int)(r / p.nt), ntile = (int)(r % p.nt);
            const int64_t gq = p.q0 + prob;
            const int64_t src = cv.fuse ? gq / 7 : gq;
            c.ma = cv.fuse ? cv.maskA[gq % 7] : 1u;
            c.mb = cv.fuse ? cv.maskB[gq % 7] : 1u;
            const int64_t arow = (int64_t)mtile * 256 + rank * 128 + ra;
            const int64_t bword = ((int64_t)ntile * 256 + rank * 128) / 64 + wb;
            c.arow_ok = arow < p.m;
            c.bword_ok = bword < p.Wn;
            c.blast = bword == p.Wn - 1;
            c.pA = cv.A + src * cv.sa + arow * cv.pa + wa;
            c.pB = cv.B + src * cv.sb + (int64_t)kr * cv.pb + bword;
        };
        auto advance = [&](Cur &c) {
            if (++c.kb == p.kblocks) {
                c.kb = 0;
                c.t += nunits;
                if (c.t < tiles) tile_setup(c);
            }
        };
        Cur ld{unit, 0, nullptr, nullptr, 0, 0, false, false, false, false};
        if (ld.t < tiles) tile_setup(ld);
        Cur cs = ld;
        auto issue = [&](uint32_t pstage) {
            if (ld.t < tiles) {
                const int64_t aw = 2 * (int64_t)ld.kb + wa;
                const bool aok = ld.arow_ok && aw < cv.Wl;
                const int64_t krow = (int64_t)ld.kb * 128 + kr;
                const bool bok = ld.bword_ok && krow < cv.l;
                const u64 *pA = ld.pA + 2 * (int64_t)ld.kb;
                const u64 *pB = ld.pB + (int64_t)ld.kb * 128 * cv.pb;
                const uint32_t slot = myslot + pstage * CV_P_ST;
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const bool ua = aok && (ld.ma & (1u << u)), ub = bok && (ld.mb & (1u << u));
                    cp_async_8(slot + 2048 * u, ua ? (const void *)(pA + cv.qoffA[u]) : (const void *)cv.A, ua);
                    cp_async_8(slot + 2048 * (4 + u), ub ? (const void *)(pB + cv.qoffB[u]) : (const void *)cv.B, ub);
                }
                advance(ld);
            }
            asm volatile("cp.async.commit_group;\n" ::: "memory");
        };
        // two steps per iteration: their load->expand->store chains interleave,
        // one proxy fence and one warp sync cover both
        for (uint32_t k = 0; k < 4; ++k) issue(k);
        int stage = 0;
        uint32_t phase = 0;
        uint32_t pst = 0;  // packed stage of the first consumed step
        auto expand_store = [&](uint32_t stg, u64 a, u64 b) {
            const uint32_t aS = sA + stg * CV_A_ST + ra * 128;
            const uint32_t bS = sB + stg * CV_B_ST + kp * 128;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const uint32_t x = (uint32_t)(a >> (32 * (1 - h)));
                const uint32_t y = (uint32_t)(b >> (32 * (1 - h)));
                uint32_t o[8], q[8];
#pragma unroll
                for (int s = 0; s < 8; ++s) {
                    o[s] = expand4(x, s);
                    q[s] = expand4(y, s);
                }
                const int ca = 4 * wa + 2 * h, cb = 4 * wb + 2 * h;
                asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};\n" ::"r"(aS + ((ca ^ (ra & 7)) << 4)),
                             "r"(o[0]), "r"(o[1]), "r"(o[2]), "r"(o[3]) : "memory");
                asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};\n" ::"r"(aS + (((ca + 1) ^ (ra & 7)) << 4)),
                             "r"(o[4]), "r"(o[5]), "r"(o[6]), "r"(o[7]) : "memory");
                asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};\n" ::"r"(bS + ((cb ^ (kp & 7)) << 4)),
                             "r"(q[0]), "r"(q[1]), "r"(q[2]), "r"(q[3]) : "memory");
                asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};\n" ::"r"(bS + (((cb + 1) ^ (kp & 7)) << 4)),
                             "r"(q[4]), "r"(q[5]), "r"(q[6]), "r"(q[7]) : "memory");
            }
        };
        auto gather = [&](uint32_t ps, const Cur &c, u64 &a, u64 &b) {
            const uint32_t slot = myslot + ps * CV_P_ST;
            a = 0;
            b = 0;
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                a ^= lds64(slot + 2048 * u);
                b ^= lds64(slot + 2048 * (4 + u));
            }
            if (2 * c.kb + wa == cv.Wl - 1) a &= atm;
            if (c.blast) b &= btm;
        };
        while (cs.t < tiles) {
            issue(pst + 4 >= CV_PST ? pst + 4 - CV_PST : pst + 4);
            const uint32_t pst1 = pst + 1 == CV_PST ? 0 : pst + 1;
            issue(pst1 + 4 >= CV_PST ? pst1 + 4 - CV_PST : pst1 + 4);
            asm volatile("cp.async.wait_group 4;\n" ::: "memory");  // steps i, i+1 landed
            u64 a0, b0, a1 = 0, b1 = 0;
            gather(pst, cs, a0, b0);
            Cur c1 = cs;
            advance(c1);
            const bool two = c1.t < tiles;
            if (two) gather(pst1, c1, a1, b1);
            const int stage1 = stage + 1;  // CV_STG even: a pair never wraps mid-way
            mbar_wait(bar_empty + 8 * stage, phase ^ 1);
            expand_store(stage, a0, b0);
            if (two) {
                mbar_wait(bar_empty + 8 * stage1, phase ^ 1);
                expand_store(stage1, a1, b1);
            }
            asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
            __syncwarp();
            if (lane == 0) {
                mbar_arrive(bar_cfull + 8 * stage);  // CTA-scope release only
                if (two) mbar_arrive(bar_cfull + 8 * stage1);
            }
            stage += 2;
            if (stage == CV_STG) {
                stage = 0;
                phase ^= 1;
            }
            pst = pst1 + 1 == CV_PST ? 0 : pst1 + 1;
            cs = c1;
            if (two) advance(cs);
        }
        asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    } else if (warp == 6 && lane == 0) {
        // ---------------- relay: one cluster-scope arrive per stage and CTA
        // (a release.cluster per converter warp costs a GPU-wide membar each)
        int stage = 0;
        uint32_t phase = 0;
        for (int64_t t = unit; t < tiles; t += nunits) {
            for (int kb = 0; kb < p.kblocks; ++kb) {
                mbar_wait(bar_cfull + 8 * stage, phase);
                mbar_arrive_leader(bar_full + 8 * stage);
                if (++stage == CV_STG) {
                    stage = 0;
                    phase ^= 1;
                }
            }
        }
    } else if (warp == 4 && lane == 0 && rank == 0) {
        // ---------------- MMA issuer (leader CTA): signed int8, M=256 N=256
        const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | (1u << 16) | ((uint32_t)(BN >> 3) << 17) |
                               ((uint32_t)(256 >> 4) << 24);
        int stage = 0;
        uint32_t phase = 0;
        int it = 0;
        for (int64_t t = unit; t < tiles; t += nunits, ++it) {
            const int acc = it & 1;
            const uint32_t acc_phase = (it >> 1) & 1;
            mbar_wait(bar_tempty + 8 * acc, acc_phase ^ 1);
            tc_fence_after();
            const uint32_t taddr = tmem_base + acc * BN;
            for (int kb = 0; kb < p.kblocks; ++kb) {
                mbar_wait(bar_full + 8 * stage, phase);
                tc_fence_after();
#pragma unroll
                for (int k = 0; k < BK / 32; ++k) {
                    const uint64_t ad = smem_desc(sA + stage * CV_A_ST + k * 32, 16, 1024);
                    const uint64_t bd = smem_desc(sB + stage * CV_B_ST + k * 32 * 128, 16, 1024);
                    umma_cg<0, 2>(taddr, ad, bd, idesc, (kb > 0 || k > 0) ? 1u : 0u);
                }
                umma_commit_cg<2>(bar_empty + 8 * stage);
                if (++stage == CV_STG) {
                    stage = 0;
                    phase ^= 1;
                }
            }
            umma_commit_cg<2>(bar_tfull + 8 * acc);
        }
    } else if (warp < 4) {
        // ---------------- epilogue: TMEM -> parity bits (N permutation undone) -> C
        const int qd = warp;  // TMEM lane quadrant
        int it = 0;
        for (int64_t t = unit; t < tiles; t += nunits, ++it) {
            int64_t r = t;
            const int64_t prob = r / (p.mt * p.nt);
            r %= (p.mt * p.nt);
            const int mtile = (int)(r / p.nt), ntile = (int)(r % p.nt);
            const int acc = it & 1;
            const uint32_t acc_phase = (it >> 1) & 1;
            mbar_wait(bar_tfull + 8 * acc, acc_phase);
            tc_fence_after();
            uint32_t packed[BN / 32];
#pragma unroll
            for (int c = 0; c < BN / 32; ++c) {
                uint32_t pk = 0;
#pragma unroll
                for (int hf = 0; hf < 2; ++hf) {  // 16 columns at a time (register budget)
                    uint32_t v[16];
                    TMEM_LD16(tmem_base + ((uint32_t)(qd * 32) << 16) + acc * BN + c * 32 + hf * 16, v);
                    asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
                    for (int j = 0; j < 16; ++j) pk |= (v[j] & 1u) << (31 - elem_at(16 * hf + j));
                }
                packed[c] = pk;
            }
            tc_fence_before();
            mbar_arrive_leader(bar_tempty + 8 * acc);
            const int64_t row = (int64_t)mtile * 256 + (int64_t)rank * BM + qd * 32 + lane;
            store_row(p, packed, row, ntile, p.q0 + prob);
        }
    }
    tc_fence_before();
    cluster_sync();
    if (warp == 5) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;\n" ::"r"(tmem_base) : "memory");
    }
}

// ------------------------------------------------------------------ host
typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                  const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiledFn g_encode = nullptr;

int get_encode() {
    if (g_encode) return GF2_OK;
    void *fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    if (e != cudaSuccess || !fn || q != cudaDriverEntryPointSuccess)
        return set_error(GF2_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    g_encode = (EncodeTiledFn)fn;
    return GF2_OK;
}

int g_sms = 0;

}  // namespace

int num_sms() {
    if (!g_sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, dev);
        if (g_sms <= 0) g_sms = 148;
    }
    return g_sms;
}

int encode_map_3d(CUtensorMap *map, CUtensorMapDataType dt, void *base, const uint64_t dims[3],
                  const uint64_t strides[2], const uint32_t box[3], bool swizzle128) {
    GF2_TRY(get_encode());
    cuuint64_t d[3] = {dims[0], dims[1], dims[2]};
    cuuint64_t st[2] = {strides[0], strides[1]};
    cuuint32_t bx[3] = {box[0], box[1], box[2]};
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = g_encode(map, dt, 3, base, d, st, bx, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                          swizzle128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return set_error(GF2_ERR_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
    return GF2_OK;
}

int launch_expand(const ExpandArgs &a, int64_t nprob, cudaStream_t s) {
    const int64_t width = words_per_row(a.cols);
    if (!a.rows || !width || !nprob) return GF2_OK;
    dim3 blk((unsigned)(width >= 128 ? 128 : (width + 31) / 32 * 32));
    dim3 grd((unsigned)((width + blk.x - 1) / blk.x), (unsigned)std::min<int64_t>(65535, (a.rows + 1) / 2),
             (unsigned)nprob);
    if (a.levels == 0)
        GF2_LAUNCH(launch_k(k_expand<0>, grd, blk, 0, s, 1, a));
    else if (a.levels == 1)
        GF2_LAUNCH(launch_k(k_expand<1>, grd, blk, 0, s, 1, a));
    else
        GF2_LAUNCH(launch_k(k_expand<2>, grd, blk, 0, s, 1, a));
    note_launch();
    return check_cuda(cudaGetLastError(), "k_expand launch");
}

// The tensor-core product for a batch: C (^)= A.B per problem, byte expansion
// (optionally fused with the last Strassen pre-addition) + tcgen05 GEMM
// (optionally fused with the last post-addition). kind: 0 i8, 1 f8, 2 f4.
int launch_umma_job(const UmmaJob &jb, int kind, cudaStream_t s) {
    const int64_t per_src = jb.fuse_pre == 2 ? 49 : (jb.fuse_pre == 1 ? 7 : 1);
    const int64_t nprob = jb.nsrc * per_src;
    if (!jb.m || !jb.n || !nprob) return GF2_OK;
    // the expansion grids index problems in gridDim.z (<= 65535): larger
    // batches run in chunks of source problems (C problems follow sources)
    const int64_t max_src = 65535 / per_src;
    if (jb.nsrc > max_src) {
        for (int64_t s0 = 0; s0 < jb.nsrc; s0 += max_src) {
            UmmaJob c = jb;
            c.A += s0 * jb.sa;
            c.B += s0 * jb.sb;
            c.C += s0 * (jb.fuse_post ? 1 : per_src) * jb.sc;  // C per source (fused post) or per leaf
            c.nsrc = std::min<int64_t>(max_src, jb.nsrc - s0);
            GF2_TRY(launch_umma_job(c, kind, s));
        }
        return GF2_OK;
    }
    if (jb.l == 0) {
        if (jb.accumulate || jb.fuse_post) return GF2_OK;
        for (int64_t q = 0; q < nprob; ++q) {
            gf2_view v{jb.C + q * jb.sc, jb.pc, jb.m, jb.n};
            GF2_TRY(launch_zero(v, s));
        }
        return GF2_OK;
    }
    static bool umma_attr[64] = {};  // the 8-bit kernels' shared-memory opt-in, once per device
    if (first_on_device(umma_attr)) {
        GF2_TRY(check_cuda(cudaFuncSetAttribute(k_umma<0, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                Geo<1>::SMEM), "umma smem attr"));
        GF2_TRY(check_cuda(cudaFuncSetAttribute(k_umma<1, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                Geo<1>::SMEM), "umma smem attr"));
        GF2_TRY(check_cuda(cudaFuncSetAttribute(k_umma<0, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                Geo<2>::SMEM), "umma smem attr"));
        GF2_TRY(check_cuda(cudaFuncSetAttribute(k_umma<1, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                Geo<2>::SMEM), "umma smem attr"));
    }
    if (kind == 2) return launch_umma_f4(jb, nprob, s);
    // i8 with 2-SM pairs: operand tiles built in shared memory from the packed
    // bits (k_umma_cv) -- no byte expansion pass
    // opt-in (GF2_UMMA_CONV=1): shared-memory-bandwidth bound today, see DESIGN.md §4.4
    static const bool conv = getenv("GF2_UMMA_CONV") && atoi(getenv("GF2_UMMA_CONV")) == 1;
    static const int cgc = getenv("GF2_UMMA_CG") ? atoi(getenv("GF2_UMMA_CG")) : 2;
    if (kind == 0 && conv && cgc == 2 && jb.fuse_pre <= 1) {
        static bool cv_attr[64] = {};
        if (first_on_device(cv_attr)) {
            GF2_TRY(check_cuda(cudaFuncSetAttribute(k_umma_cv, cudaFuncAttributeMaxDynamicSharedMemorySize, CV_SMEM),
                               "umma_cv smem attr"));
        }
        CvArgs cv{};
        cv.A = jb.A; cv.pa = jb.pa; cv.sa = jb.sa;
        cv.B = jb.B; cv.pb = jb.pb; cv.sb = jb.sb;
        cv.fuse = jb.fuse_pre;
        cv.qoffA[1] = jb.l / 64; cv.qoffA[2] = jb.m * jb.pa; cv.qoffA[3] = cv.qoffA[1] + cv.qoffA[2];
        cv.qoffB[1] = jb.n / 64; cv.qoffB[2] = jb.l * jb.pb; cv.qoffB[3] = cv.qoffB[1] + cv.qoffB[2];
        for (int i = 0; i < 7; ++i) {
            cv.maskA[i] = jb.maskA[i];
            cv.maskB[i] = jb.maskB[i];
        }
        cv.l = jb.l;
        cv.Wl = words_per_row(jb.l);
        UArgs ua{};
        ua.C = jb.C; ua.pc = jb.pc; ua.sc = jb.sc;
        ua.m = jb.m; ua.n = jb.n; ua.Wn = words_per_row(jb.n);
        ua.mt = (int)((jb.m + 255) / 256);
        ua.nt = (int)((jb.n + BN - 1) / BN);
        ua.kblocks = (int)((jb.l + BK - 1) / BK);
        ua.kchunk_blocks = ua.kblocks;
        ua.nchunks = 1;
        ua.nprob = nprob;
        ua.q0 = 0;
        ua.post = jb.fuse_post;
        if (jb.fuse_post) {
            ua.qoffC[1] = jb.n / 64; ua.qoffC[2] = jb.m * jb.pc; ua.qoffC[3] = ua.qoffC[1] + ua.qoffC[2];
            for (int i = 0; i < 7; ++i) ua.post_mask[i] = jb.maskC[i];
            ua.mode = 2;
        } else {
            ua.mode = jb.accumulate ? 1 : 0;
        }
        const int64_t tiles = nprob * ua.mt * ua.nt;
        const int64_t pairs = std::min<int64_t>(tiles, num_sms() / 2);
        const int tidx = timer_begin(s, (double)jb.m * (double)jb.l * (double)jb.n * (double)nprob);
        int rc = check_cuda(launch_k(k_umma_cv, dim3((unsigned)(2 * pairs)), dim3(CV_THREADS), CV_SMEM, s, 2, cv, ua),
                            "k_umma_cv launch");
        note_launch();
        timer_end(tidx, s);
        return rc;
    }
    const int64_t kp = (jb.l + 15) / 16 * 16, np = (jb.n + 15) / 16 * 16;
    // byte operands for at most ~8 GiB of problems per launch (cfg5-sized
    // recursions have thousands of leaves); chunks reuse one buffer
    const int64_t per = jb.m * kp + jb.l * np;
    const int64_t cap = (int64_t)8 << 30;
    const int64_t qchunk = std::max<int64_t>(1, std::min<int64_t>(nprob, cap / std::max<int64_t>(per, 1)));
    uint8_t *ws = nullptr;
    GF2_TRY(pool_setup());
    cudaError_t e = cudaMallocAsync((void **)&ws, (size_t)(qchunk * per), s);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return set_error(GF2_ERR_OOM, std::string("umma workspace: ") + cudaGetErrorString(e));
    }
    uint8_t *a8 = ws, *b8 = ws + qchunk * jb.m * kp;
    const uint32_t one = kind == 0 ? 0x01u : 0x38u;
    // A side (rows m, cols l) and B side (rows l, cols n); quadrant offsets of
    // the source problems for the fused Strassen levels
    ExpandArgs ea{};
    const int64_t f2 = jb.fuse_pre == 2 ? 2 : 1;  // first fused level's quadrants are f2 x leaf size
    ea.src = jb.A; ea.sp = jb.pa; ea.sstride = jb.sa; ea.levels = jb.fuse_pre;
    ea.qoff[0] = 0; ea.qoff[1] = f2 * jb.l / 64; ea.qoff[2] = f2 * jb.m * jb.pa; ea.qoff[3] = ea.qoff[1] + ea.qoff[2];
    ea.qoff2[0] = 0; ea.qoff2[1] = jb.l / 64; ea.qoff2[2] = jb.m * jb.pa; ea.qoff2[3] = ea.qoff2[1] + ea.qoff2[2];
    for (int i = 0; i < 7; ++i) ea.mask[i] = jb.maskA[i];
    ea.dst = a8; ea.dp = kp; ea.dstride = jb.m * kp; ea.rows = jb.m; ea.cols = jb.l; ea.one = one;
    ExpandArgs eb{};
    eb.src = jb.B; eb.sp = jb.pb; eb.sstride = jb.sb; eb.levels = jb.fuse_pre;
    eb.qoff[0] = 0; eb.qoff[1] = f2 * jb.n / 64; eb.qoff[2] = f2 * jb.l * jb.pb; eb.qoff[3] = eb.qoff[1] + eb.qoff[2];
    eb.qoff2[0] = 0; eb.qoff2[1] = jb.n / 64; eb.qoff2[2] = jb.l * jb.pb; eb.qoff2[3] = eb.qoff2[1] + eb.qoff2[2];
    for (int i = 0; i < 7; ++i) eb.mask[i] = jb.maskB[i];
    eb.dst = b8; eb.dp = np; eb.dstride = jb.l * np; eb.rows = jb.l; eb.cols = jb.n; eb.one = one;

    UArgs ua{};
    ua.C = jb.C;
    ua.pc = jb.pc;
    ua.sc = jb.sc;
    ua.m = jb.m;
    ua.n = jb.n;
    ua.Wn = words_per_row(jb.n);
    // 2-SM (cta_group::2) pairs by default; GF2_UMMA_CG=1 selects single-CTA tiles
    static const int cg = getenv("GF2_UMMA_CG") ? atoi(getenv("GF2_UMMA_CG")) : 2;
    ua.mt = (int)((jb.m + BM * cg - 1) / (BM * cg));
    ua.nt = (int)((jb.n + BN - 1) / BN);
    ua.kblocks = (int)((jb.l + BK - 1) / BK);
    ua.kchunk_blocks = kind == 0 ? ua.kblocks : (int)(F8_KCHUNK / BK);
    ua.nchunks = (ua.kblocks + ua.kchunk_blocks - 1) / ua.kchunk_blocks;
    ua.post = jb.fuse_post;
    int rc = GF2_OK;
    if (jb.fuse_post) {
        ua.qoffC[0] = 0;
        ua.qoffC[1] = jb.n / 64;
        ua.qoffC[2] = jb.m * jb.pc;
        ua.qoffC[3] = jb.m * jb.pc + jb.n / 64;
        for (int i = 0; i < 7; ++i) ua.post_mask[i] = jb.maskC[i];
        ua.mode = 2;  // destinations pre-zeroed (or accumulated into) by the caller
    } else if (ua.nchunks > 1) {
        if (!jb.accumulate) {
            for (int64_t q = 0; q < nprob && rc == GF2_OK; ++q) {
                gf2_view v{jb.C + q * jb.sc, jb.pc, jb.m, jb.n};
                rc = launch_zero(v, s);
            }
        }
        ua.mode = 2;
    } else {
        ua.mode = jb.accumulate ? 1 : 0;
    }
    for (int64_t q0 = 0; q0 < nprob && rc == GF2_OK; q0 += qchunk) {
        const int64_t nq = std::min<int64_t>(qchunk, nprob - q0);
        ea.q0 = eb.q0 = ua.q0 = q0;
        ua.nprob = nq;
        rc = launch_expand(ea, nq, s);
        if (rc == GF2_OK) rc = launch_expand(eb, nq, s);
        CUtensorMap ta, tb;
        if (rc == GF2_OK) rc = make_map(&ta, a8, (uint64_t)jb.l, (uint64_t)jb.m, (uint64_t)nq, kp, jb.m * kp);
        if (rc == GF2_OK) rc = make_map(&tb, b8, (uint64_t)jb.n, (uint64_t)jb.l, (uint64_t)nq, np, jb.l * np);
        if (rc != GF2_OK) break;
        const int64_t ntiles = (int64_t)ua.nchunks * nq * ua.mt * ua.nt;
        const int tidx = timer_begin(s, (double)jb.m * (double)jb.l * (double)jb.n * (double)nq);
        if (cg == 1) {
            const int grid = (int)(ntiles < num_sms() ? ntiles : num_sms());
            if (kind == 0)
                GF2_LAUNCH(launch_k(k_umma<0, 1>, grid, UMMA_THREADS, Geo<1>::SMEM, s, 1, ta, tb, ua));
            else
                GF2_LAUNCH(launch_k(k_umma<1, 1>, grid, UMMA_THREADS, Geo<1>::SMEM, s, 1, ta, tb, ua));
        } else {
            const int64_t pairs = std::min<int64_t>(ntiles, num_sms() / 2);
            const dim3 g2((unsigned)(2 * pairs)), b2(UMMA_THREADS);
            if (kind == 0)
                rc = check_cuda(launch_k(k_umma<0, 2>, g2, b2, Geo<2>::SMEM, s, 2, ta, tb, ua), "k_umma 2sm launch");
            else
                rc = check_cuda(launch_k(k_umma<1, 2>, g2, b2, Geo<2>::SMEM, s, 2, ta, tb, ua), "k_umma 2sm launch");
        }
        note_launch();
        if (rc == GF2_OK) rc = check_cuda(cudaGetLastError(), "k_umma launch");
        timer_end(tidx, s);
    }
    cudaFreeAsync(ws, s);
    return rc;
}

int launch_umma(const M4rmBatch &b, int kind, cudaStream_t s) {
    UmmaJob jb{};
    jb.A = b.A; jb.pa = b.pa; jb.sa = b.sa;
    jb.B = b.B; jb.pb = b.pb; jb.sb = b.sb;
    jb.C = b.C; jb.pc = b.pc; jb.sc = b.sc;
    jb.m = b.m; jb.l = b.l; jb.n = b.n; jb.nsrc = b.nprob;
    jb.accumulate = b.accumulate;
    return launch_umma_job(jb, kind, s);
}

}  // namespace gf2
