// Shared tcgen05 / TMA / mbarrier building blocks of the tensor-core
// engines: gf2_umma.cu (0/1 bytes, kind::i8 / kind::f8f6f4) and
// gf2_umma_f4.cu (e2m1 nibbles, kind::mxf4). Device helpers are inline and
// the types live in an anonymous namespace, so each translation unit has its
// own copy.
#pragma once
#include "gf2_internal.cuh"

namespace gf2 {
namespace {

constexpr int BM = 128, BN = 256, BK = 128;
constexpr int UMMA_THREADS = 256;
constexpr int64_t F8_KCHUNK = 8192;

// ------------------------------------------------------------------ PTX
__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(bar),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void tma_load_3d(uint32_t dst, const CUtensorMap *map, int c0, int c1, int c2,
                                            uint32_t bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
        "[%5];\n" ::"r"(dst),
        "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(bar)
        : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }

// UMMA shared-memory descriptor (sm_100 "version 1"), 128-byte swizzle.
__device__ __forceinline__ uint64_t smem_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= 1ull << 46;  // version
    d |= 2ull << 61;  // SWIZZLE_128B
    return d;
}

template <int KIND>  // 0: kind::i8 (u8 x u8 -> s32), 1: kind::f8f6f4 (e4m3 -> f32)
__device__ __forceinline__ void umma(uint32_t taddr, uint64_t ad, uint64_t bd, uint32_t idesc, uint32_t acc) {
    if (KIND == 0)
        asm volatile(
            "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
            "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(taddr),
            "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
    else
        asm volatile(
            "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
            "tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], %1, %2, %3, p;\n}\n" ::"r"(taddr),
            "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ bool elect_one() {
    uint32_t pred = 0;
    asm volatile(
        "{\n.reg .pred P;\nelect.sync _|P, 0xffffffff;\n@P mov.s32 %0, 1;\n}\n"
        : "+r"(pred));
    return pred != 0;
}


#define TMEM_LD32(taddr, r)                                                                                    \
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"  \
                 "%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"              \
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),        \
                   "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),    \
                   "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), \
                   "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), \
                   "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])                                          \
                 : "r"(taddr))

// tcgen05.wait::ld that also "produces" r[0..31], so the compiler cannot
// move reads of a TMEM_LD32 destination above the wait (the load is
// asynchronous; its destination registers are only valid after the wait).
#define TMEM_WAIT_LD32(r)                                                                                      \
    asm volatile("tcgen05.wait::ld.sync.aligned;\n"                                                           \
                 : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]),        \
                   "+r"(r[7]), "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]), "+r"(r[12]), "+r"(r[13]),    \
                   "+r"(r[14]), "+r"(r[15]), "+r"(r[16]), "+r"(r[17]), "+r"(r[18]), "+r"(r[19]), "+r"(r[20]), \
                   "+r"(r[21]), "+r"(r[22]), "+r"(r[23]), "+r"(r[24]), "+r"(r[25]), "+r"(r[26]), "+r"(r[27]), \
                   "+r"(r[28]), "+r"(r[29]), "+r"(r[30]), "+r"(r[31])                                          \
                 :                                                                                             \
                 : "memory")

#define TMEM_LD16(taddr, r)                                                                                    \
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, " \
                 "[%16];\n"                                                                                     \
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),        \
                   "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),    \
                   "=r"(r[14]), "=r"(r[15])                                                                    \
                 : "r"(taddr))

// ------------------------------------------------------------------ expand
// bits -> bytes (0 or `one`), 64 entries per thread, batched over problems.
// With fuse = 1 this is also the last Strassen level's pre-addition: output
// problem q = 7p + i is the XOR of source problem p's quadrants in mask[i].
struct ExpandArgs {
    const u64 *src;
    int64_t sp, sstride;
    int64_t qoff[4];   // quadrant offsets, first fused level (2x leaf size when levels == 2)
    int64_t qoff2[4];  // quadrant offsets, second fused level (leaf size)
    unsigned mask[7];
    int levels;        // fused Strassen levels: 0, 1 (q = 7p+i) or 2 (q = 49p+7i+j)
    int64_t q0;        // first problem of this chunk (dst is indexed chunk-locally)
    uint8_t *dst;
    int64_t dp, dstride;
    int64_t rows, cols;
    uint32_t one;
};

// A warp expands 32 consecutive words (2 KiB of bytes): every lane loads one
// word, then the 128 16-byte chunks are written lane-contiguously (512 B per
// store instruction) with the source word fetched by shuffle. LEVELS = fused
// Strassen levels (0, 1, 2): up to 1, 4 or 16 source blocks XORed per word,
// all gathers issued before use; two rows per iteration for more MLP.
template <int LEVELS>
__device__ __forceinline__ u64 gather_word(const ExpandArgs &a, const u64 *s, int64_t r, unsigned m1,
                                           unsigned m2) {
    u64 x = 0;
    if (LEVELS == 0) {
        x = __ldg(s + r * a.sp);
    } else if (LEVELS == 1) {
#pragma unroll
        for (int t = 0; t < 4; ++t)
            if (m1 & (1u << t)) x ^= __ldg(s + a.qoff[t] + r * a.sp);
    } else {
#pragma unroll
        for (int k = 0; k < 16; ++k)
            if ((m1 >> (k >> 2)) & (m2 >> (k & 3)) & 1u) x ^= __ldg(s + a.qoff[k >> 2] + a.qoff2[k & 3] + r * a.sp);
    }
    return x;
}


// ------------------------------------------------------------------ gemm
struct UArgs {
    u64 *C;
    int64_t pc, sc;
    int64_t m, n, Wn;
    int mt, nt, kblocks, kchunk_blocks, nchunks;
    int64_t nprob;
    int mode;  // 0 store, 1 xor, 2 atomic xor
    // last Strassen level's post-addition fused into the epilogue: product
    // q = 7p + i is XORed (red.global.xor) into the quadrants post_mask[i] of
    // the level-(d-1) product p at C + p*sc + qoffC[Q] (C pre-zeroed).
    int64_t q0;  // global index of this launch's problem 0 (C addressing)
    int post;
    int64_t qoffC[4];
    unsigned post_mask[7];
    int dbg;  // timing experiments only (GF2_F4_DBG / GF2_UMMA_DBG): 1 no C stores, 2 no epilogue work
    int order;  // tile raster (GF2_F4_ORDER): 0 column tiles fastest, G > 0 blocks of G row tiles
};

template <int CG>
__device__ __forceinline__ void umma_commit_cg(uint32_t bar) {
    if (CG == 1)
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(bar)
                     : "memory");
    else
        asm volatile(
            "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n" ::"r"(
                bar),
            "h"((uint16_t)3)
            : "memory");
}

template <int KIND, int CG>
__device__ __forceinline__ void umma_cg(uint32_t taddr, uint64_t ad, uint64_t bd, uint32_t idesc, uint32_t acc) {
    if (CG == 1) {
        umma<KIND>(taddr, ad, bd, idesc, acc);
    } else if (KIND == 0) {
        asm volatile(
            "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
            "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(taddr),
            "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
    } else {
        asm volatile(
            "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
            "tcgen05.mma.cta_group::2.kind::f8f6f4 [%0], %1, %2, %3, p;\n}\n" ::"r"(taddr),
            "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
    }
}

// 2-SM TMA: each CTA loads its half into its own smem; the transaction bytes
// land on the leader CTA's barrier (peer bit cleared).
__device__ __forceinline__ void tma_load_3d_2sm(uint32_t dst, const CUtensorMap *map, int c0, int c1, int c2,
                                                uint32_t bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
        "%3, %4}], [%5];\n" ::"r"(dst),
        "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(bar & 0xFEFFFFFFu)
        : "memory");
}

__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}

__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
    return r;
}

// arrive on the leader CTA's copy of a barrier (cluster scope)
// Arrive on the leader CTA's copy of `bar` (accumulator-free barriers). The
// epilogue threads that arrive have already completed their TMEM reads
// (tcgen05.wait::ld) and fenced them (tcgen05.fence::before_thread_sync),
// so the arrive needs no release semantics: a release arrive would also wait
// for the thread's outstanding red.xor stores to C (MEMBAR), putting a
// global-memory round trip on every tile's accumulator hand-back.
__device__ __forceinline__ void mbar_arrive_leader(uint32_t bar) {
    uint32_t remote;
    asm volatile("mapa.shared::cluster.u32 %0, %1, 0;\n" : "=r"(remote) : "r"(bar));
    asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];\n" ::"r"(remote) : "memory");
}


// 3-D byte tensor map (inner, outer, problems), box 128 x box_outer, 128-byte
// swizzle (the operand layout both engines' MMAs read).
inline int make_map(CUtensorMap *map, void *base, uint64_t inner, uint64_t outer, uint64_t nprob, uint64_t pitch,
                    uint64_t pstride, uint32_t box_outer = 128) {
    const uint64_t dims[3] = {inner, outer, nprob};
    const uint64_t strides[2] = {pitch, pstride};
    const uint32_t box[3] = {128, box_outer, 1};
    return encode_map_3d(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, base, dims, strides, box, true);
}

}  // namespace
}  // namespace gf2
