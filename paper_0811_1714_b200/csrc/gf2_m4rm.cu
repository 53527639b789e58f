// M4RM ("Method of the Four Russians") multiply on sm_100a: C (^)= A.B.
//
// Restates m4rm.py:77-121 (`_mul_into`) + graycode.py:108-156
// (`make_table`) for the B200 memory hierarchy:
//
//   * A CTA owns a C tile of BM = 512*RPT rows x 256 columns (4 words) and
//     keeps it in registers for the whole K loop: each thread holds whole
//     256-bit rows (rows tid, tid+512, ...). Tall, narrow tiles amortise
//     every table over BM rows: the table build costs 256/BM of the lookup
//     traffic (6 % at BM = 4096).
//   * A is first rewritten word-major (A^T at word granularity, `k_words_t`:
//     At[word][row], the l-tail masked), so the A words of one K step for
//     BM rows are one dense TMA box and one dense LDS.64 per 32 rows.
//   * K advances one A word (64 rows of B) per stage. A 3-slot ring of
//     stages (the BM A words + the 64 x 256-bit B panel, both by TMA) runs
//     ahead of the consumers on full/empty mbarriers.
//   * Per A half-word (32 rows of B) the CTA needs 4 Gray-code tables of 2^8
//     slots x 256 bits. Table j, slot x holds the XOR of the rows i of its
//     8-row group with bit (7-i) of x set -- exactly the reference's
//     big-endian CombinationTable (graycode.py:78-105). The 4 tables of a
//     half-word are interleaved by 32-byte bank quarter (slot x of table j
//     at x*128 + j*32). A 3-slot ring of half-word tables is kept: half-word
//     h+2 is built by one warp pair (rotating over the 8 pairs) while all
//     warps look up half-word h; full/empty mbarriers instead of block
//     barriers let a warp run up to a half-word ahead of the slowest one.
//     A builder thread makes 32 slots of one 16-byte slice with a 5-bit
//     Gray walk in registers (one 16-byte store per slot).
//   * Lookups: the 4 bytes of a row's A half-word index the 4 tables
//     (MSB-first, m4rm.py:54-66). An LDS.128 is served in 8-lane phases;
//     in each phase the lane pairs q = 0..3 read tables (q+t)&3 -- four
//     different bank quarters -- and the two lanes of a pair start on
//     different 16-byte slices, so a phase hits all 8 bank octets once:
//     one wavefront per phase, the minimum, for any table indices.
//   * Epilogue: masked store (bits beyond the window edge preserved),
//     XOR-accumulate, or red.global.xor for split-K (order-independent, so
//     deterministic).
//
// Roofline: each lookup moves 16 B of shared memory per lane and applies 8
// rows of B to 128 columns (1024 bit-ops / 16 B = 64 bit-ops per byte). The
// kernel is bound by the 128 B/clk/SM shared-memory port.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "gf2_internal.cuh"

namespace gf2 {

namespace {

constexpr int kThreads = 512;              // 16 warps = 8 builder pairs
constexpr int kTileWords = 4;              // 256 columns per C tile
constexpr int kTabBytes = 256 * 128;       // one half-word: 4 interleaved tables, 32 KiB
constexpr int kNT = 3;                     // table ring (half-words)
constexpr int kNS = 3;                     // stage ring (A words)
constexpr int kBWordBytes = 64 * 32;       // B panel of one A word: 64 rows x 32 B

template <int RPT>
constexpr int tile_rows() {
    return kThreads * RPT;
}
// DIRECT: A staged straight from A as 2-word boxes (16 B per row, the
// stage's word is one half) instead of from the word-major copy A^T -- for
// small products, where the extra pass and launch cost more than the
// doubled A reads
template <int RPT, bool DIRECT>
constexpr int stage_bytes() {
    return tile_rows<RPT>() * (DIRECT ? 16 : 8) + kBWordBytes;
}
template <int RPT, bool DIRECT>
constexpr int smem_bytes() {
    return kNT * kTabBytes + kNS * stage_bytes<RPT, DIRECT>() + 4 * 3 * 8;
}
// rows per TMA box of A^T (the host encodes the map with the same box)
template <int RPT>
constexpr int a_box_rows() {
    return tile_rows<RPT>() < 256 ? tile_rows<RPT>() : 256;
}

struct KArgs {
    u64 *C;
    int64_t pc, sc;
    int64_t m, l, n;
    int64_t Wl, Wn;
    int64_t kws;  // A words per split
    int nsplit;
    int mode;  // 0 store, 1 xor, 2 atomic xor
    u64 atm;   // tail mask of A's last word (DIRECT; A^T is masked by k_words_t)
};

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n.reg .pred p;\nWAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n}\n" ::"r"(bar),
        "r"(parity)
        : "memory");
}
// one elected arrival per warp, after every lane's shared-memory accesses
__device__ __forceinline__ void warp_arrive(uint32_t bar, int lane) {
    __syncwarp();
    if (lane == 0) mbar_arrive(bar);
}
__device__ __forceinline__ void tma_3d(uint32_t dst, const CUtensorMap *map, int c0, int c1, int c2, uint32_t bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
        "[%5];\n" ::"r"(dst),
        "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(bar)
        : "memory");
}
__device__ __forceinline__ void sts128(uint32_t addr, u64 a, u64 b) {
    asm volatile("st.shared.v2.u64 [%0], {%1, %2};\n" ::"r"(addr), "l"(a), "l"(b) : "memory");
}
__device__ __forceinline__ void lds128(uint32_t addr, u64 &a, u64 &b) {
    asm volatile("ld.shared.v2.u64 {%0, %1}, [%2];\n" : "=l"(a), "=l"(b) : "r"(addr));
}
__device__ __forceinline__ u64 lds64(uint32_t addr) {
    u64 v;
    asm volatile("ld.shared.u64 %0, [%1];\n" : "=l"(v) : "r"(addr));
    return v;
}

// column mask of B / C word w of a row of n columns (Wn words)
__device__ __forceinline__ u64 col_mask(int64_t w, int64_t Wn, u64 tail) {
    return w < Wn - 1 ? ~0ULL : (w == Wn - 1 ? tail : 0ULL);
}

// A^T at word granularity: At[p][w][r] = A[p][r][w] (last word masked to l
// columns), rows padded to mp. 32 x 32-word tiles through shared memory.
__global__ void __launch_bounds__(256) k_words_t(const u64 *A, int64_t pa, int64_t sa, u64 *At, int64_t mp,
                                                 int64_t m, int64_t Wl, u64 atm) {
    pdl_begin();
    __shared__ u64 t[32][33];
    const int64_t prob = blockIdx.z;
    const int64_t r0 = (int64_t)blockIdx.x * 32, w0 = (int64_t)blockIdx.y * 32;
    const u64 *a = A + prob * sa;
    u64 *o = At + prob * Wl * mp;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
#pragma unroll
    for (int j = ty; j < 32; j += 8) {
        const int64_t r = r0 + j, w = w0 + tx;
        u64 v = 0;
        if (r < m && w < Wl) {
            v = a[r * pa + w];
            if (w == Wl - 1) v &= atm;
        }
        t[j][tx] = v;
    }
    __syncthreads();
#pragma unroll
    for (int j = ty; j < 32; j += 8) {
        const int64_t w = w0 + j, r = r0 + tx;
        if (w < Wl && r < m) o[w * mp + r] = t[tx][j];
    }
}

template <int RPT, bool DIRECT>
__global__ void __launch_bounds__(kThreads, 1)
    k_m4rm(KArgs p, const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB) {
    constexpr int BM = tile_rows<RPT>();
    constexpr int kABox = a_box_rows<RPT>();
    constexpr int kStage = stage_bytes<RPT, DIRECT>();
    constexpr int kABytes = BM * (DIRECT ? 16 : 8);
    extern __shared__ __align__(1024) unsigned char smem[];
    const uint32_t s_tab = (uint32_t)__cvta_generic_to_shared(smem);
    const uint32_t s_st = s_tab + kNT * kTabBytes;
    const uint32_t s_bar = s_st + kNS * kStage;
    const uint32_t b_tfull = s_bar, b_tempty = s_bar + 24, b_sfull = s_bar + 48, b_sempty = s_bar + 72;

    const int tid = threadIdx.x;
    const int lane = tid & 31;
    const int warp = tid >> 5;

    const int64_t prob = blockIdx.z / p.nsplit;
    const int split = blockIdx.z % p.nsplit;
    const int64_t col_w0 = (int64_t)blockIdx.x * kTileWords;
    const int64_t row0 = (int64_t)blockIdx.y * BM;
    u64 *C = p.C + prob * p.sc;

    const int64_t kw0 = (int64_t)split * p.kws;
    const int64_t kw1 = min(kw0 + p.kws, p.Wl);
    const int nwords = kw1 > kw0 ? (int)(kw1 - kw0) : 0;
    const int H = 2 * nwords;  // half-words
    const u64 ntm = tail_mask(p.n);

    if (tid == 0) {
        for (int i = 0; i < 3; ++i) {
            mbar_init(b_tfull + 8 * i, 2);
            mbar_init(b_tempty + 8 * i, kThreads / 32);
            mbar_init(b_sfull + 8 * i, 1);
            mbar_init(b_sempty + 8 * i, kThreads / 32);
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    pdl_begin();

    // producer (thread 0): stage of local word k -> slot k % kNS
    auto issue = [&](int k) {
        const uint32_t dst = s_st + (k % kNS) * kStage;
        const uint32_t bar = b_sfull + 8 * (k % kNS);
        mbar_expect(bar, kABytes + kBWordBytes);
#pragma unroll
        for (int i = 0; i < BM / kABox; ++i) {
            if (DIRECT)  // words (kw & ~1, +1) of kABox rows
                tma_3d(dst + i * kABox * 16, &tmA, (int)((kw0 + k) & ~int64_t(1)), (int)(row0 + i * kABox),
                       (int)prob, bar);
            else
                tma_3d(dst + i * kABox * 8, &tmA, (int)(row0 + i * kABox), (int)(kw0 + k), (int)prob, bar);
        }
        tma_3d(dst + kABytes, &tmB, (int)col_w0, (int)((kw0 + k) * 64), (int)prob, bar);
    };
    if (tid == 0)
        for (int k = 0; k < nwords && k < kNS; ++k) issue(k);

    // builder role (warp pair h & 7 builds half-word h): table tj, slice bs,
    // slots sg*32 .. sg*32+31
    const int bt = tid & 63;
    const int tj = (bt >> 1) & 3;
    const int bs = bt & 1;
    const int sg = bt >> 3;
    const u64 bm0 = col_mask(col_w0 + 2 * bs, p.Wn, ntm);
    const u64 bm1 = col_mask(col_w0 + 2 * bs + 1, p.Wn, ntm);
    auto build = [&](int h) {
        const int slot = h % kNT;
        const int k = h >> 1;
        if (h >= kNT) mbar_wait(b_tempty + 8 * slot, ((h - kNT) / kNT) & 1);
        mbar_wait(b_sfull + 8 * (k % kNS), (k / kNS) & 1);
        // rows 32*(h&1) + 8*tj + j of the word's B panel; lane tj reads row
        // (i + tj) & 7 at step i, so the 4 tables' rows sit in 4 bank quarters
        const uint32_t rb = s_st + (k % kNS) * kStage + kABytes + (32 * (h & 1) + 8 * tj) * 32 + bs * 16;
        u64 c0 = 0, c1 = 0;
        u64 x0[5], x1[5];  // slot bits 4..0 <-> rows 3..7
#pragma unroll
        for (int e = 0; e < 5; ++e) x0[e] = x1[e] = 0;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const int j = (i + tj) & 7;
            u64 y0, y1;
            lds128(rb + j * 32, y0, y1);
            y0 &= bm0;
            y1 &= bm1;
            // slot bits 7..5 (= sg bits 2..0) <-> rows 0..2
            const bool hi = (j < 3) && ((sg >> (2 - j)) & 1);
            c0 ^= hi ? y0 : 0ULL;
            c1 ^= hi ? y1 : 0ULL;
#pragma unroll
            for (int e = 0; e < 5; ++e) {
                x0[e] = (j == 3 + e) ? y0 : x0[e];
                x1[e] = (j == 3 + e) ? y1 : x1[e];
            }
        }
        const uint32_t ts = s_tab + slot * kTabBytes + (sg * 32) * 128 + tj * 32 + bs * 16;
        sts128(ts, c0, c1);
#pragma unroll
        for (int i = 1; i < 32; ++i) {
            const int b = (i & 1) ? 0 : (i & 2) ? 1 : (i & 4) ? 2 : (i & 8) ? 3 : 4;  // flipped Gray bit
            const int g = i ^ (i >> 1);
            c0 ^= x0[4 - b];  // slot bit b <-> row 7-b
            c1 ^= x1[4 - b];
            sts128(ts + g * 128, c0, c1);
        }
        warp_arrive(b_tfull + 8 * slot, lane);
    };

    // lookup role: rows tid + 512*i; lane pair q (of each 8-lane phase of
    // an LDS.128) reads table (q+t)&3 at step t, slice par first
    const int q = (lane >> 1) & 3;
    const int par = lane & 1;
    uint32_t toff[4];
#pragma unroll
    for (int t = 0; t < 4; ++t) toff[t] = s_tab + (((q + t) & 3) << 5) + (par << 4);

    u64 acc[RPT][4];  // [0..1]: slice par, [2..3]: slice 1-par
#pragma unroll
    for (int i = 0; i < RPT; ++i) acc[i][0] = acc[i][1] = acc[i][2] = acc[i][3] = 0ULL;

    const int pair = warp >> 1;
    if (pair == 0 && H > 0) build(0);
    if (pair == 1 && H > 1) build(1);

    u64 a[RPT];
    for (int h = 0; h < H; ++h) {
        const int k = h >> 1;
        if (!(h & 1)) {
            mbar_wait(b_sfull + 8 * (k % kNS), (k / kNS) & 1);
            if (DIRECT) {
                const int64_t kw = kw0 + k;
                const uint32_t sa = s_st + (k % kNS) * kStage + tid * 16 + (uint32_t)(kw & 1) * 8;
                const u64 am = (kw == p.Wl - 1) ? p.atm : ~0ULL;
#pragma unroll
                for (int i = 0; i < RPT; ++i) a[i] = lds64(sa + i * kThreads * 16) & am;
            } else {
                const uint32_t sa = s_st + (k % kNS) * kStage + tid * 8;
#pragma unroll
                for (int i = 0; i < RPT; ++i) a[i] = lds64(sa + i * kThreads * 8);
            }
            warp_arrive(b_sempty + 8 * (k % kNS), lane);
            // refill: word k-1's slot takes word k-1+kNS once every warp has
            // read word k-1 (its B panel was consumed by the builders before)
            if (tid == 0 && k >= 1 && k - 1 + kNS < nwords) {
                mbar_wait(b_sempty + 8 * ((k - 1) % kNS), ((k - 1) / kNS) & 1);
                issue(k - 1 + kNS);
            }
        }
        const int slot = h % kNT;
        mbar_wait(b_tfull + 8 * slot, (h / kNT) & 1);
        const uint32_t tb = slot * kTabBytes;
#pragma unroll
        for (int i = 0; i < RPT; ++i) {
            const uint32_t hw = (h & 1) ? (uint32_t)a[i] : (uint32_t)(a[i] >> 32);
            const uint32_t r = __funnelshift_l(hw, hw, 8 * q);  // byte 3-t <-> table (q+t)&3
#pragma unroll
            for (int t = 0; t < 4; t += 2) {
                const uint32_t ad0 = toff[t] + tb + (((r >> (24 - 8 * t)) & 0xFF) << 7);
                const uint32_t ad1 = toff[t + 1] + tb + (((r >> (16 - 8 * t)) & 0xFF) << 7);
                u64 v0, v1, v2, v3, w0, w1, w2, w3;
                lds128(ad0, v0, v1);
                lds128(ad0 ^ 16, v2, v3);
                lds128(ad1, w0, w1);
                lds128(ad1 ^ 16, w2, w3);
                acc[i][0] ^= v0 ^ w0;
                acc[i][1] ^= v1 ^ w1;
                acc[i][2] ^= v2 ^ w2;
                acc[i][3] ^= v3 ^ w3;
            }
        }
        warp_arrive(b_tempty + 8 * slot, lane);
        if (h + 2 < H && pair == ((h + 2) & 7)) build(h + 2);
    }

    // ---- epilogue: words col_w0 + 2*par + {0,1} (acc 0,1), col_w0 + 2*(1-par) + {0,1} (acc 2,3)
#pragma unroll
    for (int i = 0; i < RPT; ++i) {
        const int64_t row = row0 + i * kThreads + tid;
        if (row >= p.m) continue;
        u64 *crow = C + row * p.pc;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const int64_t wi = col_w0 + ((e < 2) ? 2 * par : 2 * (1 - par)) + (e & 1);
            if (wi >= p.Wn) continue;
            const u64 v = acc[i][e];
            if (p.mode == 2) {
                if (v) atomicXor(reinterpret_cast<unsigned long long *>(crow + wi), (unsigned long long)v);
            } else if (p.mode == 1) {
                crow[wi] ^= v;
            } else if (wi == p.Wn - 1 && ntm != ~0ULL) {
                crow[wi] = (crow[wi] & ~ntm) | v;
            } else {
                crow[wi] = v;
            }
        }
    }
}


// ------------------------------------------------------------------ BM = 8192
// Taller tile, same shared-memory budget: 16 rows per thread, 8 of them in
// registers and 8 parked in tensor memory (TMEM, 512 columns per CTA). Per
// A half-word a thread looks its register rows up, swaps them with the
// parked ones (tcgen05.st + tcgen05.ld: TMEM's own datapath, not the
// shared-memory port the lookups saturate) and looks those up. Every table
// then serves 8192 rows: the build costs 256/8192 of the lookup traffic.
// Stages are one A half-word (32 KiB of the half-word-major A^T, one 5-D TMA
// box) in a 3-slot ring, B half panels (1 KiB) in an 8-slot ring, and the
// 3-slot half-word table ring of k_m4rm.
// NG groups of 4 rows per thread (NG = 2..4): BM = 2048 NG rows per CTA
template <int NG>
constexpr int tm_rows() {
    return 2048 * NG;
}
template <int NG>
constexpr int tm_stage_a() {
    return tm_rows<NG>() * 4;  // one A half-word for BM rows
}
constexpr int kTmNA = 3;
constexpr int kTmNB = 8;
constexpr int kTmB = 32 * 32;       // 32 rows x 32 B
template <int NG>
constexpr int tm_smem() {
    return kNT * kTabBytes + kTmNA * tm_stage_a<NG>() + kTmNB * kTmB + 256;
}

__device__ __forceinline__ uint32_t lds32(uint32_t addr) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];\n" : "=r"(v) : "r"(addr));
    return v;
}
__device__ __forceinline__ void lds128v(uint32_t addr, uint32_t &a, uint32_t &b, uint32_t &c, uint32_t &d) {
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];\n" : "=r"(a), "=r"(b), "=r"(c), "=r"(d) : "r"(addr));
}
__device__ __forceinline__ void tma_5d(uint32_t dst, const CUtensorMap *map, int c0, int c1, int c2, int c3, int c4,
                                       uint32_t bar) {
    asm volatile(
        "cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, "
        "%6}], [%7];\n" ::"r"(dst),
        "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4), "r"(bar)
        : "memory");
}
// 8 rows x 8 words of accumulators <-> 64 TMEM columns of this thread's lane
__device__ __forceinline__ void tm_store(uint32_t taddr, const uint32_t (&x)[8][8]) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x64.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32, %33, %34, %35, %36, %37, %38, %39, %40, %41, %42, %43, %44, %45, %46, %47, %48, %49, %50, %51, %52, %53, %54, %55, %56, %57, %58, %59, %60, %61, %62, %63, %64};\n" ::"r"(taddr), "r"(x[0][0]), "r"(x[0][1]), "r"(x[0][2]), "r"(x[0][3]), "r"(x[0][4]), "r"(x[0][5]), "r"(x[0][6]), "r"(x[0][7]), "r"(x[1][0]), "r"(x[1][1]), "r"(x[1][2]), "r"(x[1][3]), "r"(x[1][4]), "r"(x[1][5]), "r"(x[1][6]), "r"(x[1][7]), "r"(x[2][0]), "r"(x[2][1]), "r"(x[2][2]), "r"(x[2][3]), "r"(x[2][4]), "r"(x[2][5]), "r"(x[2][6]), "r"(x[2][7]), "r"(x[3][0]), "r"(x[3][1]), "r"(x[3][2]), "r"(x[3][3]), "r"(x[3][4]), "r"(x[3][5]), "r"(x[3][6]), "r"(x[3][7]), "r"(x[4][0]), "r"(x[4][1]), "r"(x[4][2]), "r"(x[4][3]), "r"(x[4][4]), "r"(x[4][5]), "r"(x[4][6]), "r"(x[4][7]), "r"(x[5][0]), "r"(x[5][1]), "r"(x[5][2]), "r"(x[5][3]), "r"(x[5][4]), "r"(x[5][5]), "r"(x[5][6]), "r"(x[5][7]), "r"(x[6][0]), "r"(x[6][1]), "r"(x[6][2]), "r"(x[6][3]), "r"(x[6][4]), "r"(x[6][5]), "r"(x[6][6]), "r"(x[6][7]), "r"(x[7][0]), "r"(x[7][1]), "r"(x[7][2]), "r"(x[7][3]), "r"(x[7][4]), "r"(x[7][5]), "r"(x[7][6]), "r"(x[7][7]) : "memory");
    asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
}
__device__ __forceinline__ void tm_load(uint32_t taddr, uint32_t (&x)[8][8]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x64.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32, %33, %34, %35, %36, %37, %38, %39, %40, %41, %42, %43, %44, %45, %46, %47, %48, %49, %50, %51, %52, %53, %54, %55, %56, %57, %58, %59, %60, %61, %62, %63}, [%64];\n" : "=r"(x[0][0]), "=r"(x[0][1]), "=r"(x[0][2]), "=r"(x[0][3]), "=r"(x[0][4]), "=r"(x[0][5]), "=r"(x[0][6]), "=r"(x[0][7]), "=r"(x[1][0]), "=r"(x[1][1]), "=r"(x[1][2]), "=r"(x[1][3]), "=r"(x[1][4]), "=r"(x[1][5]), "=r"(x[1][6]), "=r"(x[1][7]), "=r"(x[2][0]), "=r"(x[2][1]), "=r"(x[2][2]), "=r"(x[2][3]), "=r"(x[2][4]), "=r"(x[2][5]), "=r"(x[2][6]), "=r"(x[2][7]), "=r"(x[3][0]), "=r"(x[3][1]), "=r"(x[3][2]), "=r"(x[3][3]), "=r"(x[3][4]), "=r"(x[3][5]), "=r"(x[3][6]), "=r"(x[3][7]), "=r"(x[4][0]), "=r"(x[4][1]), "=r"(x[4][2]), "=r"(x[4][3]), "=r"(x[4][4]), "=r"(x[4][5]), "=r"(x[4][6]), "=r"(x[4][7]), "=r"(x[5][0]), "=r"(x[5][1]), "=r"(x[5][2]), "=r"(x[5][3]), "=r"(x[5][4]), "=r"(x[5][5]), "=r"(x[5][6]), "=r"(x[5][7]), "=r"(x[6][0]), "=r"(x[6][1]), "=r"(x[6][2]), "=r"(x[6][3]), "=r"(x[6][4]), "=r"(x[6][5]), "=r"(x[6][6]), "=r"(x[6][7]), "=r"(x[7][0]), "=r"(x[7][1]), "=r"(x[7][2]), "=r"(x[7][3]), "=r"(x[7][4]), "=r"(x[7][5]), "=r"(x[7][6]), "=r"(x[7][7]) : "r"(taddr) : "memory");
    asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
}

// store the register group to one TMEM slot and load the other into the
// same registers, in one asm statement: the accumulators keep their
// registers across the swap (as two statements the compiler gave the
// loaded group a second register set and spilled)
__device__ __forceinline__ void tm_swap(uint32_t st_addr, uint32_t ld_addr, uint32_t (&x)[8][8]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x64.b32 [%64], {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32, %33, %34, %35, %36, %37, %38, %39, %40, %41, %42, %43, %44, %45, %46, %47, %48, %49, %50, %51, %52, %53, %54, %55, %56, %57, %58, %59, %60, %61, %62, %63};\n"
        "tcgen05.wait::st.sync.aligned;\n"
        "tcgen05.ld.sync.aligned.32x32b.x64.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32, %33, %34, %35, %36, %37, %38, %39, %40, %41, %42, %43, %44, %45, %46, %47, %48, %49, %50, %51, %52, %53, %54, %55, %56, %57, %58, %59, %60, %61, %62, %63}, [%65];\n"
        "tcgen05.wait::ld.sync.aligned;\n"
        : "+r"(x[0][0]), "+r"(x[0][1]), "+r"(x[0][2]), "+r"(x[0][3]), "+r"(x[0][4]), "+r"(x[0][5]), "+r"(x[0][6]), "+r"(x[0][7]), "+r"(x[1][0]), "+r"(x[1][1]), "+r"(x[1][2]), "+r"(x[1][3]), "+r"(x[1][4]), "+r"(x[1][5]), "+r"(x[1][6]), "+r"(x[1][7]), "+r"(x[2][0]), "+r"(x[2][1]), "+r"(x[2][2]), "+r"(x[2][3]), "+r"(x[2][4]), "+r"(x[2][5]), "+r"(x[2][6]), "+r"(x[2][7]), "+r"(x[3][0]), "+r"(x[3][1]), "+r"(x[3][2]), "+r"(x[3][3]), "+r"(x[3][4]), "+r"(x[3][5]), "+r"(x[3][6]), "+r"(x[3][7]), "+r"(x[4][0]), "+r"(x[4][1]), "+r"(x[4][2]), "+r"(x[4][3]), "+r"(x[4][4]), "+r"(x[4][5]), "+r"(x[4][6]), "+r"(x[4][7]), "+r"(x[5][0]), "+r"(x[5][1]), "+r"(x[5][2]), "+r"(x[5][3]), "+r"(x[5][4]), "+r"(x[5][5]), "+r"(x[5][6]), "+r"(x[5][7]), "+r"(x[6][0]), "+r"(x[6][1]), "+r"(x[6][2]), "+r"(x[6][3]), "+r"(x[6][4]), "+r"(x[6][5]), "+r"(x[6][6]), "+r"(x[6][7]), "+r"(x[7][0]), "+r"(x[7][1]), "+r"(x[7][2]), "+r"(x[7][3]), "+r"(x[7][4]), "+r"(x[7][5]), "+r"(x[7][6]), "+r"(x[7][7])
        : "r"(st_addr), "r"(ld_addr)
        : "memory");
}

// A^T half-word-major: At[p][w][h][r] (u32; h = 0 the high half = K rows
// 0..31 of word w), l-tail masked, rows padded to mp (a multiple of 256)
// with zeros.
__global__ void __launch_bounds__(256) k_words_th(const u64 *A, int64_t pa, int64_t sa, uint32_t *At, int64_t mp,
                                                  int64_t m, int64_t Wl, u64 atm) {
    pdl_begin();
    __shared__ u64 t[32][33];
    const int64_t prob = blockIdx.z;
    const int64_t r0 = (int64_t)blockIdx.x * 32, w0 = (int64_t)blockIdx.y * 32;
    const u64 *a = A + prob * sa;
    uint32_t *o = At + prob * Wl * 2 * mp;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
#pragma unroll
    for (int j = ty; j < 32; j += 8) {
        const int64_t r = r0 + j, w = w0 + tx;
        u64 v = 0;
        if (r < m && w < Wl) {
            v = a[r * pa + w];
            if (w == Wl - 1) v &= atm;
        }
        t[j][tx] = v;
    }
    __syncthreads();
#pragma unroll
    for (int j = ty; j < 32; j += 8) {
        const int64_t w = w0 + j, r = r0 + tx;
        if (w < Wl && r < mp) {
            const u64 v = t[tx][j];
            o[(w * 2 + 0) * mp + r] = (uint32_t)(v >> 32);
            o[(w * 2 + 1) * mp + r] = (uint32_t)v;
        }
    }
}

// 4-row register groups (32 accumulator words) <-> 32 TMEM columns
__device__ __forceinline__ void tm_swap32(uint32_t st_addr, uint32_t ld_addr, uint32_t (&x)[4][8]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%32], {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31};\n"
        "tcgen05.wait::st.sync.aligned;\n"
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%33];\n"
        "tcgen05.wait::ld.sync.aligned;\n"
        : "+r"(x[0][0]), "+r"(x[0][1]), "+r"(x[0][2]), "+r"(x[0][3]), "+r"(x[0][4]), "+r"(x[0][5]), "+r"(x[0][6]), "+r"(x[0][7]), "+r"(x[1][0]), "+r"(x[1][1]), "+r"(x[1][2]), "+r"(x[1][3]), "+r"(x[1][4]), "+r"(x[1][5]), "+r"(x[1][6]), "+r"(x[1][7]), "+r"(x[2][0]), "+r"(x[2][1]), "+r"(x[2][2]), "+r"(x[2][3]), "+r"(x[2][4]), "+r"(x[2][5]), "+r"(x[2][6]), "+r"(x[2][7]), "+r"(x[3][0]), "+r"(x[3][1]), "+r"(x[3][2]), "+r"(x[3][3]), "+r"(x[3][4]), "+r"(x[3][5]), "+r"(x[3][6]), "+r"(x[3][7])
        : "r"(st_addr), "r"(ld_addr)
        : "memory");
}
__device__ __forceinline__ void tm_store32(uint32_t taddr, const uint32_t (&x)[4][8]) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32};\n" ::"r"(taddr), "r"(x[0][0]), "r"(x[0][1]), "r"(x[0][2]), "r"(x[0][3]), "r"(x[0][4]), "r"(x[0][5]), "r"(x[0][6]), "r"(x[0][7]), "r"(x[1][0]), "r"(x[1][1]), "r"(x[1][2]), "r"(x[1][3]), "r"(x[1][4]), "r"(x[1][5]), "r"(x[1][6]), "r"(x[1][7]), "r"(x[2][0]), "r"(x[2][1]), "r"(x[2][2]), "r"(x[2][3]), "r"(x[2][4]), "r"(x[2][5]), "r"(x[2][6]), "r"(x[2][7]), "r"(x[3][0]), "r"(x[3][1]), "r"(x[3][2]), "r"(x[3][3]), "r"(x[3][4]), "r"(x[3][5]), "r"(x[3][6]), "r"(x[3][7]) : "memory");
    asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
}
__device__ __forceinline__ void tm_load32(uint32_t taddr, uint32_t (&x)[4][8]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];\n" : "=r"(x[0][0]), "=r"(x[0][1]), "=r"(x[0][2]), "=r"(x[0][3]), "=r"(x[0][4]), "=r"(x[0][5]), "=r"(x[0][6]), "=r"(x[0][7]), "=r"(x[1][0]), "=r"(x[1][1]), "=r"(x[1][2]), "=r"(x[1][3]), "=r"(x[1][4]), "=r"(x[1][5]), "=r"(x[1][6]), "=r"(x[1][7]), "=r"(x[2][0]), "=r"(x[2][1]), "=r"(x[2][2]), "=r"(x[2][3]), "=r"(x[2][4]), "=r"(x[2][5]), "=r"(x[2][6]), "=r"(x[2][7]), "=r"(x[3][0]), "=r"(x[3][1]), "=r"(x[3][2]), "=r"(x[3][3]), "=r"(x[3][4]), "=r"(x[3][5]), "=r"(x[3][6]), "=r"(x[3][7]) : "r"(taddr) : "memory");
    asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
}

template <int NG>
__global__ void __launch_bounds__(kThreads, 1)
    k_m4rm_tm(KArgs p, const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB) {
    constexpr int kTmRows = tm_rows<NG>();
    constexpr int kTmA = tm_stage_a<NG>();
    extern __shared__ __align__(1024) unsigned char smem[];
    const uint32_t s_tab = (uint32_t)__cvta_generic_to_shared(smem);
    const uint32_t s_a = s_tab + kNT * kTabBytes;
    const uint32_t s_b = s_a + kTmNA * kTmA;
    const uint32_t s_bar = s_b + kTmNB * kTmB;
    const uint32_t b_tfull = s_bar, b_tempty = s_bar + 24, b_afull = s_bar + 48, b_aempty = s_bar + 72,
                   b_bfull = s_bar + 96;  // 8 barriers
    const uint32_t s_tmem = s_bar + 160;

    const int tid = threadIdx.x;
    const int lane = tid & 31;
    const int warp = tid >> 5;

    // 32-bit coordinates (TMA coordinates are 32-bit anyway): fewer live
    // registers beside the 64 accumulator words
    const int prob = (int)(blockIdx.z / p.nsplit);
    const int split = (int)(blockIdx.z % p.nsplit);
    const int col_w0 = (int)blockIdx.x * kTileWords;
    const int rb0 = (int)blockIdx.y * (kTmRows / 256);  // first 256-row block
    const int kw0 = split * (int)p.kws;
    const int kw1 = (int)min((int64_t)kw0 + p.kws, p.Wl);
    const int nwords = kw1 > kw0 ? kw1 - kw0 : 0;
    const int H = 2 * nwords;

    if (tid == 0) {
        for (int i = 0; i < 3; ++i) {
            mbar_init(b_tfull + 8 * i, 2);
            mbar_init(b_tempty + 8 * i, kThreads / 32);
            mbar_init(b_afull + 8 * i, 1);
            mbar_init(b_aempty + 8 * i, kThreads / 32);
        }
        for (int i = 0; i < kTmNB; ++i) mbar_init(b_bfull + 8 * i, 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(s_tmem) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    const uint32_t tbase = *reinterpret_cast<volatile uint32_t *>(smem + (s_tmem - s_tab));
    pdl_begin();

    auto issue_a = [&](int h) {
        const uint32_t bar = b_afull + 8 * (h % kTmNA);
        mbar_expect(bar, kTmA);
        tma_5d(s_a + (h % kTmNA) * kTmA, &tmA, 0, rb0, h & 1, kw0 + (h >> 1), prob, bar);
    };
    auto issue_b = [&](int h) {
        const uint32_t bar = b_bfull + 8 * (h % kTmNB);
        mbar_expect(bar, kTmB);
        tma_3d(s_b + (h % kTmNB) * kTmB, &tmB, col_w0, kw0 * 64 + 32 * h, prob, bar);
    };
    if (tid == 0) {
        for (int h = 0; h < H && h < kTmNA; ++h) issue_a(h);
        for (int h = 0; h < H && h < kTmNB; ++h) issue_b(h);
    }

    // builder role (pair h & 7 builds half-word h)
    const int bt = tid & 63;
    const int tj = (bt >> 1) & 3;
    const int bs = bt & 1;
    const int sg = bt >> 3;
    auto build = [&](int h) {
        const int slot = h % kNT;
        const u64 bm0 = col_mask(col_w0 + 2 * bs, p.Wn, tail_mask(p.n));
        const u64 bm1 = col_mask(col_w0 + 2 * bs + 1, p.Wn, tail_mask(p.n));
        if (h >= kNT) mbar_wait(b_tempty + 8 * slot, ((h - kNT) / kNT) & 1);
        mbar_wait(b_bfull + 8 * (h % kTmNB), (h / kTmNB) & 1);
        const uint32_t rb = s_b + (h % kTmNB) * kTmB + (8 * tj) * 32 + bs * 16;
        u64 c0 = 0, c1 = 0;
        u64 x0[5], x1[5];
#pragma unroll
        for (int e = 0; e < 5; ++e) x0[e] = x1[e] = 0;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const int j = (i + tj) & 7;  // rows of the 4 tables in 4 bank quarters
            u64 y0, y1;
            lds128(rb + j * 32, y0, y1);
            y0 &= bm0;
            y1 &= bm1;
            const bool hi = (j < 3) && ((sg >> (2 - j)) & 1);
            c0 ^= hi ? y0 : 0ULL;
            c1 ^= hi ? y1 : 0ULL;
#pragma unroll
            for (int e = 0; e < 5; ++e) {
                x0[e] = (j == 3 + e) ? y0 : x0[e];
                x1[e] = (j == 3 + e) ? y1 : x1[e];
            }
        }
        const uint32_t ts = s_tab + slot * kTabBytes + (sg * 32) * 128 + tj * 32 + bs * 16;
        sts128(ts, c0, c1);
#pragma unroll
        for (int i = 1; i < 32; ++i) {
            const int b = (i & 1) ? 0 : (i & 2) ? 1 : (i & 4) ? 2 : (i & 8) ? 3 : 4;
            const int g = i ^ (i >> 1);
            c0 ^= x0[4 - b];
            c1 ^= x1[4 - b];
            sts128(ts + g * 128, c0, c1);
        }
        warp_arrive(b_tfull + 8 * slot, lane);
    };

    const int q = (lane >> 1) & 3;
    const int par = lane & 1;

    // accumulators of the register group: row i, u32 words 0..3 = slice par,
    // 4..7 = slice 1-par; the other group parked at TMEM columns slot*64
    // 4 groups of 4 rows (rows g*2048 + i*512 + tid): one group in
    // registers (32 words), three parked at TMEM columns g*32
    uint32_t acc[4][8];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int e = 0; e < 8; ++e) acc[i][e] = 0;
    const uint32_t tlane = tbase + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)((warp >> 2) * 128);
#pragma unroll 1
    for (int g = 1; g < NG; ++g) tm_store32(tlane + g * 32, acc);  // parked groups start at zero
    int cur = 0;

    const int pair = warp >> 1;
    if (pair == 0 && H > 0) build(0);
    if (pair == 1 && H > 1) build(1);

    auto lookups = [&](uint32_t tb, const uint32_t (&a)[4]) {
        const uint32_t tq = s_tab + tb + (par << 4);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const uint32_t hw = a[i];
            const uint32_t r = __funnelshift_l(hw, hw, 8 * q);  // byte 3-t <-> table (q+t)&3
#pragma unroll
            for (int t = 0; t < 4; ++t) {  // one lookup (two 16-byte slices) at a time: fewer live registers
                const uint32_t ad = tq + (((q + t) & 3) << 5) + (((r >> (24 - 8 * t)) & 0xFF) << 7);
                uint32_t v[8];
                lds128v(ad, v[0], v[1], v[2], v[3]);
                lds128v(ad ^ 16, v[4], v[5], v[6], v[7]);
#pragma unroll
                for (int e = 0; e < 8; ++e) acc[i][e] ^= v[e];
            }
        }
    };

    uint32_t a[4];
    for (int h = 0; h < H; ++h) {
        const int slot = h % kNT;
        const uint32_t sa = s_a + (h % kTmNA) * kTmA + tid * 4;
        mbar_wait(b_tfull + 8 * slot, (h / kNT) & 1);
        mbar_wait(b_afull + 8 * (h % kTmNA), (h / kTmNA) & 1);
        const uint32_t tb = slot * kTabBytes;
#pragma unroll 1
        for (int step = 0; step < NG; ++step) {
            if (step) {
                const int nxt = cur + 1 == NG ? 0 : cur + 1;
                tm_swap32(tlane + cur * 32, tlane + nxt * 32, acc);
                cur = nxt;
            }
#pragma unroll
            for (int i = 0; i < 4; ++i) a[i] = lds32(sa + (cur * 2048 + i * kThreads) * 4);
            if (step == NG - 1) warp_arrive(b_aempty + 8 * (h % kTmNA), lane);
            lookups(tb, a);
        }
        warp_arrive(b_tempty + 8 * slot, lane);
        if (tid == 0) {
            // A slot of half-word h-1 takes h+2 once every warp has read it;
            // B slot of h-2 (built two iterations ago: tfull(h-2) seen) takes h+6
            if (h >= 1 && h + 2 < H) {
                mbar_wait(b_aempty + 8 * ((h - 1) % kTmNA), ((h - 1) / kTmNA) & 1);
                issue_a(h + 2);
            }
            if (h >= 2 && h + 6 < H) issue_b(h + 6);
        }
        if (h + 2 < H && pair == ((h + 2) & 7)) build(h + 2);
    }

    // ---- epilogue: both groups (the register one, then the parked one)
    u64 *C = p.C + (int64_t)prob * p.sc;
    const u64 ntm = tail_mask(p.n);
    const int64_t row0 = (int64_t)rb0 * 256;
#pragma unroll 1
    for (int pass = 0; pass < NG; ++pass) {
        if (pass) {
            cur = cur + 1 == NG ? 0 : cur + 1;
            tm_load32(tlane + cur * 32, acc);
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int64_t row = row0 + cur * 2048 + i * kThreads + tid;
            if (row >= p.m) continue;
            u64 *crow = C + row * p.pc;
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int64_t wi = col_w0 + ((e < 2) ? 2 * par : 2 * (1 - par)) + (e & 1);
                if (wi >= p.Wn) continue;
                const u64 v = (u64)acc[i][2 * e] | ((u64)acc[i][2 * e + 1] << 32);
                if (p.mode == 2) {
                    if (v) atomicXor(reinterpret_cast<unsigned long long *>(crow + wi), (unsigned long long)v);
                } else if (p.mode == 1) {
                    crow[wi] ^= v;
                } else if (wi == p.Wn - 1 && ntm != ~0ULL) {
                    crow[wi] = (crow[wi] & ~ntm) | v;
                } else {
                    crow[wi] = v;
                }
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    if (warp == 0) {
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tbase) : "memory");
    }
}

template <int NG>
int launch_tm(const KArgs &ka, const CUtensorMap &ta, const CUtensorMap &tb, dim3 grid, cudaStream_t s) {
    static bool configured[64] = {};
    if (first_on_device(configured))
        GF2_TRY(check_cuda(cudaFuncSetAttribute(k_m4rm_tm<NG>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                tm_smem<NG>()),
                           "cudaFuncSetAttribute(k_m4rm_tm)"));
    GF2_LAUNCH(launch_k(k_m4rm_tm<NG>, grid, kThreads, tm_smem<NG>(), s, 1, ka, ta, tb));
    note_launch();
    g_m4rm_launches.fetch_add(1, std::memory_order_relaxed);
    return check_cuda(cudaGetLastError(), "k_m4rm_tm launch");
}

template <int RPT, bool DIRECT>
int launch_rpt(const KArgs &ka, const CUtensorMap &ta, const CUtensorMap &tb, int64_t col_tiles, int64_t row_tiles,
               int64_t zdim, cudaStream_t s) {
    static bool configured[64] = {};
    constexpr int sm = smem_bytes<RPT, DIRECT>();
    if (first_on_device(configured))
        GF2_TRY(check_cuda(cudaFuncSetAttribute(k_m4rm<RPT, DIRECT>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm),
                           "cudaFuncSetAttribute(k_m4rm)"));
    dim3 grid((unsigned)col_tiles, (unsigned)row_tiles, (unsigned)zdim);
    GF2_LAUNCH(launch_k(k_m4rm<RPT, DIRECT>, grid, kThreads, sm, s, 1, ka, ta, tb));
    note_launch();
    g_m4rm_launches.fetch_add(1, std::memory_order_relaxed);
    return check_cuda(cudaGetLastError(), "k_m4rm launch");
}

// kernel timer (gf2_timer_*): event pairs around each M4RM launch
struct TimedLaunch {
    cudaEvent_t a, b;
    double bitops;
};
bool g_timing = false;
std::vector<TimedLaunch> g_timed;
std::vector<cudaEvent_t> g_event_pool;

cudaEvent_t pool_event() {
    if (!g_event_pool.empty()) {
        cudaEvent_t e = g_event_pool.back();
        g_event_pool.pop_back();
        return e;
    }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
}

}  // namespace

int timer_enable(int on) {
    for (auto &t : g_timed) {
        g_event_pool.push_back(t.a);
        g_event_pool.push_back(t.b);
    }
    g_timed.clear();
    g_timing = on != 0;
    return GF2_OK;
}

int timer_read(double *ms, double *bitops, int64_t *launches) {
    double tot = 0, ops = 0;
    for (auto &t : g_timed) {
        GF2_TRY(check_cuda(cudaEventSynchronize(t.b), "timer sync"));
        float e = 0;
        GF2_TRY(check_cuda(cudaEventElapsedTime(&e, t.a, t.b), "timer elapsed"));
        tot += e;
        ops += t.bitops;
    }
    if (ms) *ms = tot;
    if (bitops) *bitops = ops;
    if (launches) *launches = (int64_t)g_timed.size();
    return GF2_OK;
}

int timer_begin(cudaStream_t s, double bitops) {
    if (!g_timing) return -1;
    TimedLaunch tl{pool_event(), pool_event(), bitops};
    cudaEventRecord(tl.a, s);
    g_timed.push_back(tl);
    return (int)g_timed.size() - 1;
}

void timer_end(int idx, cudaStream_t s) {
    if (idx >= 0) cudaEventRecord(g_timed[idx].b, s);
}

int launch_m4rm(const M4rmBatch &b, cudaStream_t s) {
    if (!b.m || !b.n || !b.nprob) return GF2_OK;
    // gridDim.z = K splits (<= 16) x problems must stay <= 65535: deep
    // recursions (7^6 leaves at cutoff 64) run their leaves in chunks
    constexpr int64_t kMaxBatch = 65535 / 16;
    if (b.nprob > kMaxBatch) {
        for (int64_t q0 = 0; q0 < b.nprob; q0 += kMaxBatch) {
            M4rmBatch c = b;
            c.A += q0 * b.sa;
            c.B += q0 * b.sb;
            c.C += q0 * b.sc;
            c.nprob = std::min<int64_t>(kMaxBatch, b.nprob - q0);
            GF2_TRY(launch_m4rm(c, s));
        }
        return GF2_OK;
    }
    const int64_t Wn = words_per_row(b.n), Wl = words_per_row(b.l);
    auto zero_c = [&]() -> int {
        if (b.nprob == 1 || b.sc == b.m * b.pc) {
            gf2_view v{b.C, b.pc, b.m * b.nprob, b.n};
            return launch_zero(v, s);  // a 2-D memset when whole words
        }
        for (int64_t q = 0; q < b.nprob; ++q) {
            gf2_view v{b.C + q * b.sc, b.pc, b.m, b.n};
            GF2_TRY(launch_zero(v, s));
        }
        return GF2_OK;
    };
    if (b.l == 0) return b.accumulate ? GF2_OK : zero_c();

    const int64_t col_tiles = (Wn + kTileWords - 1) / kTileWords;
    const int64_t sms = num_sms();  // one CTA per SM is resident (smem-bound)
    // Geometry from a shared-memory cost model (units: KiB of shared-memory
    // port traffic per CTA and A word, i.e. 64 rows of B): the lookups move
    // 128 KiB per RPT (512 threads x RPT rows x 8 tables x 32 B), the A
    // words 8 KiB per RPT (TMA write + LDS), the table build ~82 KiB
    // whatever the tile height (8 tables x 256 slots x 32 B of stores plus
    // the source rows). A CTA runs its K range plus a fixed cost (launch,
    // pipeline fill, first table builds, epilogue) of about two words --
    // fitted to the 7 batched 8192^3 leaves of cfg3 on the M4RM engine
    // (RPT 16: 4/5/7/8/13 splits measured 2.335/2.187/2.216/2.302/2.341 ms;
    // with half a word the model picked 13) -- and CTAs run in waves of
    // one per SM. A K split also costs the zeroing pass and red.xor. Large
    // products take RPT 16 (BM 8192, half the rows parked in TMEM) and split
    // K only to fill waves (16384^3: 128 tiles, 8 splits, 6.92 waves); small
    // ones (cfg1 1024^3) trade taller tiles for more CTAs with shorter K
    // ranges.
    int rpt = 8;
    int nsplit = 1;
    int64_t kws = Wl;
    {
        double best = 0;
        for (int r : {16, 12, 8, 4, 2, 1}) {
            const int64_t rt = (b.m + kThreads * r - 1) / (kThreads * r);
            const int64_t tiles = rt * col_tiles * b.nprob;
            for (int64_t n = 1; n <= 16 && n <= Wl; ++n) {
                const int64_t w = (Wl + n - 1) / n;
                const int64_t ns = (Wl + w - 1) / w;  // splits actually used
                if (ns != n) continue;
                const int64_t ctas = tiles * ns;
                const int64_t waves = (ctas + sms - 1) / sms;
                const double per_cta = ((double)w + 2.0) * (82.0 + 136.0 * r);
                const double cost = (double)waves * per_cta * (ns > 1 ? 1.02 : 1.0);
                if (best == 0 || cost < best * 0.999) {
                    best = cost;
                    rpt = r;
                    nsplit = (int)ns;
                    kws = w;
                }
            }
        }
    }
    {
        // tuning override, GF2_M4RM_GEOM="rpt,nsplit" (tools/ only)
        static const char *geom = getenv("GF2_M4RM_GEOM");
        int r = 0, n = 0;
        if (geom && sscanf(geom, "%d,%d", &r, &n) == 2 && (r == 1 || r == 2 || r == 4 || r == 8 || r == 12 || r == 16) && n >= 1 &&
            n <= 16) {
            rpt = r;
            kws = (Wl + n - 1) / n;
            nsplit = (int)((Wl + kws - 1) / kws);
        }
    }
    const int64_t row_tiles = (b.m + kThreads * rpt - 1) / (kThreads * rpt);
    {
        static const bool verbose = getenv("GF2_M4RM_VERBOSE") != nullptr;  // tools/ only
        if (verbose)
            fprintf(stderr, "k_m4rm geometry: m=%lld l=%lld n=%lld nprob=%lld -> rpt=%d nsplit=%d kws=%lld\n",
                    (long long)b.m, (long long)b.l, (long long)b.n, (long long)b.nprob, rpt, nsplit, (long long)kws);
    }
    if ((int64_t)nsplit * b.nprob > 65535 || row_tiles > 65535 || col_tiles > 2147483647)
        return set_error(GF2_ERR_PARAMETER, "m4rm grid too large");
    if (b.m > 2147483647 || b.l > 2147483647 / 2)
        return set_error(GF2_ERR_PARAMETER, "m4rm operand too large for a TMA map");

    // workspace: A^T at word granularity (rows padded to even) unless A is
    // staged directly (small products with a 16-byte aligned A), and B
    // copied to an aligned buffer when it is not 16-byte aligned with an
    // even pitch
    GF2_TRY(pool_setup());
    const bool direct = rpt <= 4 && (uintptr_t)b.A % 16 == 0 && b.pa % 2 == 0 && (b.nprob == 1 || b.sa % 2 == 0) &&
                        b.m * Wl * b.nprob <= (int64_t(1) << 20);
    const bool tm = rpt >= 8;  // BM 4096..8192, TMEM-parked row groups, half-word-major A^T
    const int64_t mp = tm ? (b.m + 255) & ~int64_t(255) : (b.m + 1) & ~int64_t(1);
    const bool b_ok = ((uintptr_t)b.B % 16 == 0) && (b.pb % 2 == 0) && (b.nprob == 1 || b.sb % 2 == 0);
    const int64_t wnp = (Wn + 1) & ~int64_t(1);
    const int64_t at_words = direct ? 0 : b.nprob * Wl * mp;
    const int64_t bs_words = b_ok ? 0 : b.nprob * b.l * wnp;
    u64 *ws = nullptr;
    if (at_words + bs_words) {
        cudaError_t e = cudaMallocAsync((void **)&ws, (size_t)(at_words + bs_words) * 8, s);
        if (e != cudaSuccess) return set_error(GF2_ERR_OOM, std::string("m4rm workspace: ") + cudaGetErrorString(e));
    }
    u64 *At = ws;
    const u64 *Bm = b.B;
    int64_t pb = b.pb, sb = b.sb;
    int rc = GF2_OK;
    if (tm) {
        dim3 grid((unsigned)(mp / 32), (unsigned)((Wl + 31) / 32), (unsigned)b.nprob);
        cudaError_t le = launch_k(k_words_th, grid, dim3(256), 0, s, 1, b.A, b.pa, b.sa, (uint32_t *)At, mp, b.m,
                                  Wl, tail_mask(b.l));
        if (le != cudaSuccess) rc = check_cuda(le, "k_words_th launch");
        else note_launch();
    } else if (!direct) {
        dim3 grid((unsigned)((b.m + 31) / 32), (unsigned)((Wl + 31) / 32), (unsigned)b.nprob);
        cudaError_t le = launch_k(k_words_t, grid, dim3(256), 0, s, 1, b.A, b.pa, b.sa, At, mp, b.m, Wl,
                                  tail_mask(b.l));
        if (le != cudaSuccess) rc = check_cuda(le, "k_words_t launch");
        else note_launch();
    }
    if (rc == GF2_OK && !b_ok) {
        u64 *Bs = ws + at_words;
        for (int64_t q = 0; q < b.nprob && rc == GF2_OK; ++q) {
            gf2_view dst{Bs + q * b.l * wnp, wnp, b.l, b.n};
            gf2_view src{const_cast<u64 *>(b.B + q * b.sb), b.pb, b.l, b.n};
            rc = launch_ewise(dst, &src, nullptr, 1, s);
        }
        Bm = Bs;
        pb = wnp;
        sb = b.l * wnp;
    }
    CUtensorMap ta{}, tb{};
    if (rc == GF2_OK && tm) {
        // A^T half-word-major (u32): 256 rows x row blocks x halves x words x problems
        const uint64_t da[5] = {256, (uint64_t)(mp / 256), 2, (uint64_t)Wl, (uint64_t)b.nprob};
        const uint64_t sa[4] = {1024, (uint64_t)mp * 4, (uint64_t)mp * 8, (uint64_t)(Wl * mp) * 8};
        const uint32_t ba[5] = {256, (uint32_t)(kThreads * rpt / 256), 1, 1, 1};
        rc = encode_map_nd(&ta, CU_TENSOR_MAP_DATA_TYPE_UINT32, (void *)At, 5, da, sa, ba, false);
        const uint64_t db[3] = {(uint64_t)Wn, (uint64_t)b.l, (uint64_t)b.nprob};
        const uint64_t sbb[2] = {(uint64_t)pb * 8, (uint64_t)(b.nprob > 1 ? sb : b.l * pb) * 8};
        const uint32_t bb[3] = {(uint32_t)kTileWords, 32, 1};
        if (rc == GF2_OK) rc = encode_map_3d(&tb, CU_TENSOR_MAP_DATA_TYPE_UINT64, (void *)Bm, db, sbb, bb, false);
    } else if (rc == GF2_OK) {
        // A^T: rows x words x problems (DIRECT, A: words x rows x problems);
        // B: words x rows x problems
        const uint32_t abox = (uint32_t)std::min(kThreads * rpt, 256);
        const uint64_t da[3] = {(uint64_t)(direct ? Wl : b.m), (uint64_t)(direct ? b.m : Wl), (uint64_t)b.nprob};
        const uint64_t sa[2] = {(uint64_t)(direct ? b.pa : mp) * 8,
                                (uint64_t)(direct ? (b.nprob > 1 ? b.sa : b.m * b.pa) : Wl * mp) * 8};
        const uint32_t ba[3] = {direct ? 2u : abox, direct ? abox : 1u, 1};
        const uint64_t db[3] = {(uint64_t)Wn, (uint64_t)b.l, (uint64_t)b.nprob};
        const uint64_t sbb[2] = {(uint64_t)pb * 8, (uint64_t)(b.nprob > 1 ? sb : b.l * pb) * 8};
        const uint32_t bb[3] = {(uint32_t)kTileWords, 64, 1};
        rc = encode_map_3d(&ta, CU_TENSOR_MAP_DATA_TYPE_UINT64, direct ? (void *)b.A : (void *)At, da, sa, ba, false);
        if (rc == GF2_OK) rc = encode_map_3d(&tb, CU_TENSOR_MAP_DATA_TYPE_UINT64, (void *)Bm, db, sbb, bb, false);
    }
    KArgs ka{b.C, b.pc, b.sc, b.m, b.l, b.n, Wl, Wn, kws, nsplit, 0, tail_mask(b.l)};
    if (rc == GF2_OK) {
        if (nsplit > 1) {
            if (!b.accumulate) rc = zero_c();
            ka.mode = 2;
        } else {
            ka.mode = b.accumulate ? 1 : 0;
        }
    }
    if (rc == GF2_OK) {
        const int64_t z = (int64_t)nsplit * b.nprob;
        const int tidx = timer_begin(s, (double)b.m * (double)b.l * (double)b.n * (double)b.nprob);
        if (tm) {
            dim3 grid((unsigned)col_tiles, (unsigned)row_tiles, (unsigned)z);
            rc = rpt == 16 ? launch_tm<4>(ka, ta, tb, grid, s)
                           : (rpt == 12 ? launch_tm<3>(ka, ta, tb, grid, s) : launch_tm<2>(ka, ta, tb, grid, s));
        }        else if (rpt == 4)
            rc = direct ? launch_rpt<4, true>(ka, ta, tb, col_tiles, row_tiles, z, s)
                        : launch_rpt<4, false>(ka, ta, tb, col_tiles, row_tiles, z, s);
        else if (rpt == 2)
            rc = direct ? launch_rpt<2, true>(ka, ta, tb, col_tiles, row_tiles, z, s)
                        : launch_rpt<2, false>(ka, ta, tb, col_tiles, row_tiles, z, s);
        else
            rc = direct ? launch_rpt<1, true>(ka, ta, tb, col_tiles, row_tiles, z, s)
                        : launch_rpt<1, false>(ka, ta, tb, col_tiles, row_tiles, z, s);
        timer_end(tidx, s);
    }
    if (ws) cudaFreeAsync(ws, s);
    return rc;
}

}  // namespace gf2
