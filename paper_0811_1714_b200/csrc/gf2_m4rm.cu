// M4RM ("Method of the Four Russians") multiply on sm_100a: C (^)= A.B.
//
// Restates m4rm.py:77-121 (`_mul_into`) + graycode.py:108-156
// (`make_table`) for the B200 memory hierarchy:
//
//   * A CTA owns a C tile of BM = 64*RPT rows x 1024 columns (16 words) and
//     keeps it in registers for the whole K loop: each thread holds a
//     128-bit column slice of RPT rows (8 lanes = one 128-byte row, so the
//     4 quarter-warps of a warp cover 4 rows per instruction).
//   * K advances two 64-bit words of A (128 rows of B) per stage. The B
//     panel (128 rows x 1024 columns, 16 KiB) and the A column words
//     (BM x 16 B) of the NEXT stage are prefetched (TMA, or cp.async for
//     8-byte-aligned windows) while the current stage is consumed
//     (double-buffered).
//   * Each half stage (32 rows of B) builds 4 Gray-code tables of 2^8 rows
//     x 1024 bits (4 x 32 KiB) in shared memory. Table j, slot x holds the
//     XOR of rows i of the 8-row group with bit (7-i) of x set -- exactly
//     the reference's big-endian CombinationTable (graycode.py:78-105).
//     Every thread builds 32 slots of one 128-bit column slice by a
//     Gray walk held in registers, so the build costs one 16-byte shared
//     store per slot and no shared-memory reads beyond the 8 source rows.
//   * Lookups: for every row, the 4 bytes of the A half-word index the 4
//     tables (MSB-first, m4rm.py:54-66); 8 lanes read one 128-byte table row
//     as LDS.128 -- conflict-free for any index -- and XOR it into the
//     register accumulator.
//   * Epilogue: masked store (bits beyond the window edge preserved),
//     XOR-accumulate, or red.global.xor for split-K (order-independent, so
//     deterministic).
//
// Roofline: each lookup moves 16 B of shared memory per lane and applies 8
// rows of B to 128 columns (1024 bit-ops / 16 B = 64 bit-ops per byte);
// table builds add 2^8/BM of that traffic. The kernel is bound by the
// 128 B/clk/SM shared-memory crossbar.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "gf2_internal.cuh"

namespace gf2 {

namespace {

constexpr int kThreads = 512;   // 16 warps = 64 quarter-warp row groups
constexpr int kRowGroups = kThreads / 8;
constexpr int kTables = 4;      // 8-bit tables per half stage (32 rows of B)
constexpr int kTabRows = 256;   // 2^8 slots
constexpr int kTileWords = 16;  // 1024 columns per C tile
constexpr int kRowBytes = kTileWords * 8;
constexpr int kTableBytes = kTabRows * kRowBytes;     // 32 KiB
constexpr int kStageWords = 2;                         // A words per stage
constexpr int kStageRows = 64 * kStageWords;           // rows of B per stage
constexpr int kBStageBytes = kStageRows * kRowBytes;  // 16 KiB

template <int RPT>
constexpr int smem_bytes() {
    return kTables * kTableBytes + 2 * kBStageBytes + 2 * (kRowGroups * RPT) * 8 * kStageWords + 16;
}

// rows per TMA box of A words (the host encodes the map with the same box)
template <int RPT>
constexpr int a_box_rows() {
    return kRowGroups * RPT < 256 ? kRowGroups * RPT : 256;
}

struct KArgs {
    const u64 *A;
    int64_t pa, sa;
    const u64 *B;
    int64_t pb, sb;
    u64 *C;
    int64_t pc, sc;
    int64_t m, l, n;
    int64_t Wl, Wn;
    int64_t kws;  // A words per split (even unless it is the whole row)
    int nsplit;
    int mode;  // 0 store, 1 xor, 2 atomic xor
};

// cp.async with zero-fill: copies `bytes` (0..CP) of CP and zero-fills the rest.
template <int CP>
__device__ __forceinline__ void cp_async(uint32_t saddr, const void *g, int bytes) {
    if (CP == 16)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(saddr), "l"(g), "r"(bytes)
                     : "memory");
    else
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(saddr), "l"(g), "r"(bytes)
                     : "memory");
}
__device__ __forceinline__ void mbar_init1(uint32_t bar) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_expect(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait_parity(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n.reg .pred p;\nWAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n}\n" ::"r"(bar),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void tma_3d(uint32_t dst, const CUtensorMap *map, int c0, int c1, int c2, uint32_t bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
        "[%5];\n" ::"r"(dst),
        "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(bar)
        : "memory");
}

__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }

__device__ __forceinline__ void sts128(uint32_t addr, u64 a, u64 b) {
    asm volatile("st.shared.v2.u64 [%0], {%1, %2};\n" ::"r"(addr), "l"(a), "l"(b) : "memory");
}
__device__ __forceinline__ void lds128(uint32_t addr, u64 &a, u64 &b) {
    asm volatile("ld.shared.v2.u64 {%0, %1}, [%2];\n" : "=l"(a), "=l"(b) : "r"(addr));
}
__device__ __forceinline__ uint32_t lds32(uint32_t addr) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];\n" : "=r"(v) : "r"(addr));
    return v;
}

// C tile: BM = 64*RPT rows x 1024 columns, in registers. TMA: operands are
// 16-byte aligned with 16-byte pitches, so thread 0 stages each B panel
// (128 rows x 16 words) and the A words (BM rows x 2 words, boxes of
// min(BM, 256) rows)
// with cp.async.bulk.tensor onto one mbarrier per buffer (zero fill past the
// matrix edges); otherwise every thread issues 8-byte cp.async.
template <int RPT, bool TMA>
__global__ void __launch_bounds__(kThreads, 1)
    k_m4rm(KArgs p, const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB) {
    pdl_begin();
    constexpr int BM = kRowGroups * RPT;
    constexpr int kABox = a_box_rows<RPT>();
    extern __shared__ __align__(128) unsigned char smem[];
    const uint32_t s_tab = (uint32_t)__cvta_generic_to_shared(smem);
    const uint32_t s_bst = s_tab + kTables * kTableBytes;
    const uint32_t s_ast = s_bst + 2 * kBStageBytes;
    const uint32_t s_bar = s_ast + 2 * BM * 16;

    const int tid = threadIdx.x;
    const int lane = tid & 31;
    const int s = lane & 7;                       // 128-bit column slice
    const int rg = (tid >> 5) * 4 + (lane >> 3);  // row group 0..63

    const int64_t prob = blockIdx.z / p.nsplit;
    const int split = blockIdx.z % p.nsplit;
    const int64_t col_w0 = (int64_t)blockIdx.x * kTileWords;
    const int64_t row0 = (int64_t)blockIdx.y * BM;
    const u64 *A = p.A + prob * p.sa;
    const u64 *B = p.B + prob * p.sb;
    u64 *C = p.C + prob * p.sc;

    const int64_t kw0 = (int64_t)split * p.kws;
    const int64_t kw1 = min(kw0 + p.kws, p.Wl);
    const u64 atm = tail_mask(p.l);

    // masks for this thread's two B words (tail of a ragged / windowed B)
    const int64_t wj0 = col_w0 + 2 * s;
    const u64 bm0 = (wj0 == p.Wn - 1) ? tail_mask(p.n) : ~0ULL;
    const u64 bm1 = (wj0 + 1 == p.Wn - 1) ? tail_mask(p.n) : ~0ULL;

    // stage = A words [kw, kw+2) of BM rows and the 128 matching rows of B
    auto load_stage = [&](int64_t kw, int buf) {
        const uint32_t bdst = s_bst + buf * kBStageBytes;
        if (TMA) {
            if (tid == 0) {
                const uint32_t bar = s_bar + 8 * buf;
                mbar_expect(bar, kBStageBytes + BM * 16);
                tma_3d(bdst, &tmB, (int)col_w0, (int)(kw * 64), (int)prob, bar);
#pragma unroll
                for (int i = 0; i < BM / kABox; ++i)
                    tma_3d(s_ast + (buf * BM + kABox * i) * 16, &tmA, (int)kw, (int)(row0 + kABox * i), (int)prob,
                           bar);
            }
        } else {
#pragma unroll
            for (int i = 0; i < (kStageRows * kTileWords) / kThreads; ++i) {
                const int e = tid + kThreads * i;
                const int r = e >> 4, wd = e & 15;
                const int64_t brow = kw * 64 + r;
                const bool ok = (brow < p.l) && (col_w0 + wd < p.Wn);
                const u64 *src = ok ? (B + brow * p.pb + col_w0 + wd) : B;
                cp_async<8>(bdst + r * kRowBytes + wd * 8, src, ok ? 8 : 0);
            }
#pragma unroll
            for (int i = 0; i < (2 * BM + kThreads - 1) / kThreads; ++i) {
                const int e = tid + kThreads * i;
                if (e < 2 * BM) {
                    const int r = e >> 1, wd = e & 1;
                    const bool ok = (row0 + r < p.m) && (kw + wd < kw1);
                    const u64 *src = ok ? (A + (row0 + r) * p.pa + kw + wd) : A;
                    cp_async<8>(s_ast + (buf * BM + r) * 16 + wd * 8, src, ok ? 8 : 0);
                }
            }
            cp_async_commit();
        }
    };

    u64 acc[RPT][2];
#pragma unroll
    for (int i = 0; i < RPT; ++i) acc[i][0] = acc[i][1] = 0ULL;

    // table-build role: table tj, slots [r0*16, r0*16+16), slice s
    const int tj = rg >> 4, r0 = rg & 15;

    if (TMA) {
        if (tid == 0) {
            mbar_init1(s_bar);
            mbar_init1(s_bar + 8);
            asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
        }
        __syncthreads();
    }
    if (kw0 < kw1) load_stage(kw0, 0);
    int buf = 0;
    uint32_t it = 0;
    for (int64_t kw = kw0; kw < kw1; kw += kStageWords, buf ^= 1, ++it) {
        if (TMA)
            mbar_wait_parity(s_bar + 8 * buf, (it >> 1) & 1);
        else
            cp_async_wait_all();
        __syncthreads();  // stage visible; previous lookups finished
        if (kw + kStageWords < kw1) load_stage(kw + kStageWords, buf ^ 1);
        const int nhalf = (kw + 1 < kw1) ? 4 : 2;
        for (int hs = 0; hs < nhalf; ++hs) {
            if (hs) __syncthreads();  // lookups of the previous half done before rebuild
            // ---- build table tj from B rows 32hs + 8tj + (0..7), slice s
            {
                const uint32_t srow = s_bst + buf * kBStageBytes + (32 * hs + 8 * tj) * kRowBytes + s * 16;
                u64 c0 = 0, c1 = 0, y0, y1;
#pragma unroll
                for (int i = 0; i < 4; ++i) {  // slot bits 7..4 <-> source rows 0..3
                    // only the rows in this slot group's high bits are read:
                    // the lanes of other groups skip the load, which saves
                    // shared-memory wavefronts (the kernel's binding resource)
                    if (r0 & (8 >> i)) {
                        lds128(srow + i * kRowBytes, y0, y1);
                        c0 ^= y0 & bm0;
                        c1 ^= y1 & bm1;
                    }
                }
                u64 x0[4], x1[4];  // slot bits 3..0 <-> source rows 4..7
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    lds128(srow + (4 + i) * kRowBytes, x0[i], x1[i]);
                    x0[i] &= bm0;
                    x1[i] &= bm1;
                }
                const uint32_t tbase = s_tab + tj * kTableBytes + (r0 * 16) * kRowBytes + s * 16;
                sts128(tbase, c0, c1);
#pragma unroll
                for (int i = 1; i < 16; ++i) {
                    const int b = (i & 1) ? 0 : (i & 2) ? 1 : (i & 4) ? 2 : 3;  // flipped Gray bit
                    const int g = i ^ (i >> 1);
                    c0 ^= x0[3 - b];  // slot bit b <-> source row 7-b
                    c1 ^= x1[3 - b];
                    sts128(tbase + g * kRowBytes, c0, c1);
                }
            }
            __syncthreads();
            // ---- lookups: A half-word hs of the stage (word hs/2, high half first)
            const int64_t wcur = kw + (hs >> 1);
            const uint32_t amask = (uint32_t)(((wcur == p.Wl - 1) ? atm : ~0ULL) >> ((hs & 1) ? 0 : 32));
            const uint32_t aoff = s_ast + buf * BM * 16 + (hs >> 1) * 8 + ((hs & 1) ? 0 : 4);
            const uint32_t base = s_tab + s * 16;
#pragma unroll
            for (int i = 0; i < RPT; ++i) {
                const uint32_t hw = lds32(aoff + (i * kRowGroups + rg) * 16) & amask;
                u64 v0, v1, w0, w1;
                lds128(base + 0 * kTableBytes + ((hw >> 24) & 0xFF) * kRowBytes, v0, v1);
                lds128(base + 1 * kTableBytes + ((hw >> 16) & 0xFF) * kRowBytes, w0, w1);
                acc[i][0] ^= v0 ^ w0;
                acc[i][1] ^= v1 ^ w1;
                lds128(base + 2 * kTableBytes + ((hw >> 8) & 0xFF) * kRowBytes, v0, v1);
                lds128(base + 3 * kTableBytes + (hw & 0xFF) * kRowBytes, w0, w1);
                acc[i][0] ^= v0 ^ w0;
                acc[i][1] ^= v1 ^ w1;
            }
        }
    }

    // ---- epilogue
    const u64 ctm = tail_mask(p.n);
#pragma unroll
    for (int i = 0; i < RPT; ++i) {
        const int64_t row = row0 + i * kRowGroups + rg;
        if (row >= p.m) continue;
        u64 *crow = C + row * p.pc;
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            const int64_t wi = wj0 + e;
            if (wi >= p.Wn) continue;
            const u64 v = acc[i][e];
            if (p.mode == 2) {
                if (v) atomicXor(reinterpret_cast<unsigned long long *>(crow + wi), (unsigned long long)v);
            } else if (p.mode == 1) {
                crow[wi] ^= v;
            } else if (wi == p.Wn - 1 && ctm != ~0ULL) {
                crow[wi] = (crow[wi] & ~ctm) | v;
            } else {
                crow[wi] = v;
            }
        }
    }
}

template <int RPT, bool TMA>
int launch_rpt(const KArgs &ka, const CUtensorMap &ta, const CUtensorMap &tb, int64_t col_tiles, int64_t row_tiles,
               int64_t zdim, cudaStream_t s) {
    static bool configured[64] = {};
    constexpr int sm = smem_bytes<RPT>();
    if (first_on_device(configured))
        GF2_TRY(check_cuda(cudaFuncSetAttribute(k_m4rm<RPT, TMA>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm),
                           "cudaFuncSetAttribute(k_m4rm)"));
    dim3 grid((unsigned)col_tiles, (unsigned)row_tiles, (unsigned)zdim);
    GF2_LAUNCH(launch_k(k_m4rm<RPT, TMA>, grid, kThreads, sm, s, 1, ka, ta, tb));
    note_launch();
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
            return launch_ewise(v, nullptr, nullptr, 0, s);
        }
        for (int64_t q = 0; q < b.nprob; ++q) {
            gf2_view v{b.C + q * b.sc, b.pc, b.m, b.n};
            GF2_TRY(launch_ewise(v, nullptr, nullptr, 0, s));
        }
        return GF2_OK;
    };
    if (b.l == 0) return b.accumulate ? GF2_OK : zero_c();

    const int64_t col_tiles = (Wn + kTileWords - 1) / kTileWords;
    const int64_t sms = num_sms();  // one CTA per SM is resident (smem-bound)
    // Geometry from a shared-memory cost model (units: KiB of shared traffic
    // per CTA and half stage of 32 B rows): the table build moves ~192 KiB
    // whatever the tile height (4 tables x 256 slots x 128 B of stores plus
    // the source rows), the lookups 34 KiB per RPT (RPT rows per thread:
    // one 4-byte A load and four 128 B table rows per row group). A CTA runs
    // 2 half stages per A word of its K range plus a fixed cost (launch,
    // first stage in flight, epilogue) of about one half stage; CTAs run in
    // waves of one per SM. A K split also costs the zeroing pass and
    // red.xor. Large products keep RPT 16 (BM 1024) and split K only to fill
    // waves (16384^3: 256 tiles, 4 splits, 6.92 waves); small ones
    // (cfg1 1024^3) trade taller tiles for more CTAs with shorter K ranges.
    int rpt = 16;
    int nsplit = 1;
    int64_t kws = Wl;
    {
        double best = 0;
        for (int r : {16, 8, 4, 2}) {
            const int64_t rt = (b.m + kRowGroups * r - 1) / (kRowGroups * r);
            const int64_t tiles = rt * col_tiles * b.nprob;
            for (int64_t n = 1; n <= 16 && n <= Wl; ++n) {
                // A words per split: even, so every split starts its TMA
                // boxes on a 16-byte boundary (a box at an odd word faults)
                int64_t w = (Wl + n - 1) / n;
                if (w < Wl) w = (w + 1) & ~int64_t(1);
                const int64_t ns = (Wl + w - 1) / w;  // splits actually used
                if (ns != n) continue;
                const int64_t ctas = tiles * ns;
                const int64_t waves = (ctas + sms - 1) / sms;
                const double per_cta = (2.0 * (double)w + 1.0) * (192.0 + 34.0 * r);
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
        if (geom && sscanf(geom, "%d,%d", &r, &n) == 2 && (r == 2 || r == 4 || r == 8 || r == 16) && n >= 1 &&
            n <= 16) {
            rpt = r;
            kws = (Wl + n - 1) / n;
            if (kws < Wl) kws = (kws + 1) & ~int64_t(1);
            nsplit = (int)((Wl + kws - 1) / kws);
        }
    }
    const int64_t row_tiles = (b.m + kRowGroups * rpt - 1) / (kRowGroups * rpt);
    if ((int64_t)nsplit * b.nprob > 65535 || row_tiles > 65535)
        return set_error(GF2_ERR_PARAMETER, "m4rm grid too large");

    KArgs ka{b.A, b.pa, b.sa, b.B, b.pb, b.sb, b.C, b.pc, b.sc, b.m, b.l, b.n, Wl, Wn, kws, nsplit, 0};
    if (nsplit > 1) {
        if (!b.accumulate) GF2_TRY(zero_c());
        ka.mode = 2;
    } else {
        ka.mode = b.accumulate ? 1 : 0;
    }
    const int64_t z = (int64_t)nsplit * b.nprob;
    const int tidx = timer_begin(s, (double)b.m * (double)b.l * (double)b.n * (double)b.nprob);
    bool tma = ((uintptr_t)b.A % 16 == 0) && ((uintptr_t)b.B % 16 == 0) && (b.pa % 2 == 0) && (b.pb % 2 == 0) &&
               (b.nprob == 1 || (b.sa % 2 == 0 && b.sb % 2 == 0));
    CUtensorMap ta{}, tb{};
    if (tma) {
        // words x rows x problems; the problem stride is unused when nprob == 1
        const uint64_t da[3] = {(uint64_t)Wl, (uint64_t)b.m, (uint64_t)b.nprob};
        const uint64_t sa[2] = {(uint64_t)b.pa * 8, (uint64_t)(b.nprob > 1 ? b.sa : b.m * b.pa) * 8};
        const uint32_t ba[3] = {2, (uint32_t)std::min(kRowGroups * rpt, 256), 1};
        const uint64_t db[3] = {(uint64_t)Wn, (uint64_t)b.l, (uint64_t)b.nprob};
        const uint64_t sb[2] = {(uint64_t)b.pb * 8, (uint64_t)(b.nprob > 1 ? b.sb : b.l * b.pb) * 8};
        const uint32_t bb[3] = {(uint32_t)kTileWords, (uint32_t)kStageRows, 1};
        tma = encode_map_3d(&ta, CU_TENSOR_MAP_DATA_TYPE_UINT64, (void *)b.A, da, sa, ba, false) == GF2_OK &&
              encode_map_3d(&tb, CU_TENSOR_MAP_DATA_TYPE_UINT64, (void *)b.B, db, sb, bb, false) == GF2_OK;
    }
    int rc;
    if (rpt == 16)
        rc = tma ? launch_rpt<16, true>(ka, ta, tb, col_tiles, row_tiles, z, s)
                 : launch_rpt<16, false>(ka, ta, tb, col_tiles, row_tiles, z, s);
    else if (rpt == 8)
        rc = tma ? launch_rpt<8, true>(ka, ta, tb, col_tiles, row_tiles, z, s)
                 : launch_rpt<8, false>(ka, ta, tb, col_tiles, row_tiles, z, s);
    else if (rpt == 4)
        rc = tma ? launch_rpt<4, true>(ka, ta, tb, col_tiles, row_tiles, z, s)
                 : launch_rpt<4, false>(ka, ta, tb, col_tiles, row_tiles, z, s);
    else
        rc = tma ? launch_rpt<2, true>(ka, ta, tb, col_tiles, row_tiles, z, s)
                 : launch_rpt<2, false>(ka, ta, tb, col_tiles, row_tiles, z, s);
    timer_end(tidx, s);
    return rc;
}

}  // namespace gf2
