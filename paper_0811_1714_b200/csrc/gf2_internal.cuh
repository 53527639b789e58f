// Internal declarations shared by the gf2b200 translation units.
#pragma once
#include <cstdlib>
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <string>

#include "../../include/gf2b200.h"

namespace gf2 {

typedef uint64_t u64;

constexpr int kWordBits = 64;

__host__ __device__ inline int64_t words_per_row(int64_t ncols) {
    return (ncols + kWordBits - 1) / kWordBits;
}
// core.py:49-54
__host__ __device__ inline u64 tail_mask(int64_t ncols) {
    int64_t rem = ncols % kWordBits;
    return rem == 0 ? ~0ULL : (~0ULL << (kWordBits - rem));
}

// 32 x 32 bit transpose across a warp: lane L bit P <-> lane P bit L
// (5 butterfly stages; at stage s the lanes swap the bits whose lane and
// position s-bits differ). The per-lane constants are hoisted: keep[i] = the
// bits a lane keeps at stage i, rot[i] = the left-rotation that moves the
// received half into place (32 - sh on upper lanes: a right shift, the moved
// half's complement is zero) -- 4 instructions per stage (LOP3, SHFL, SHF,
// LOP3). MSB-first words need no bit reversal around it: with lane l holding
// row 31 - l, the result is the MSB-first word of column 31 - l (reversing
// bit and lane order together maps the network onto itself); with lane l
// holding row l, it is column 31 - l with the rows LSB-first.
struct Bfly32 {
    uint32_t keep[5], rot[5];
};
__device__ __forceinline__ Bfly32 bfly32_init(int lane) {
    const uint32_t masks[5] = {0xFFFF0000u, 0xFF00FF00u, 0xF0F0F0F0u, 0xCCCCCCCCu, 0xAAAAAAAAu};
    Bfly32 c;
#pragma unroll
    for (int i = 0; i < 5; ++i) {
        const int sh = 16 >> i;
        const bool up = lane & sh;
        c.keep[i] = up ? masks[i] : ~masks[i];
        c.rot[i] = up ? 32 - sh : sh;
    }
    return c;
}
__device__ __forceinline__ uint32_t transpose32m(uint32_t x, const Bfly32 &c) {
#pragma unroll
    for (int i = 0; i < 5; ++i) {
        const uint32_t got = __shfl_xor_sync(0xffffffffu, x & ~c.keep[i], 16 >> i);
        x = (x & c.keep[i]) | __funnelshift_l(got, got, c.rot[i]);
    }
    return x;
}

// Per-device one-time setup: function attributes (the dynamic shared-memory
// opt-in) belong to the device context, so "done" is tracked per device.
// Returns true the first time it is called for `flags` on the current device.
inline bool first_on_device(bool (&flags)[64]) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) return true;
    if (flags[dev]) return false;
    flags[dev] = true;
    return true;
}

// Status plumbing ------------------------------------------------------
int set_error(int code, const std::string &msg);
int check_cuda(cudaError_t e, const char *what);
extern std::atomic<int64_t> g_launches;
extern std::atomic<int64_t> g_m4rm_launches;
inline void note_launch(int n = 1) { g_launches.fetch_add(n, std::memory_order_relaxed); }

// Programmatic dependent launch (PDL). Every library kernel is launched
// with programmatic stream serialization and executes griddepcontrol.wait
// before its first global memory access (the tensor-core GEMMs after their
// barrier/TMEM/scale-factor setup): the next kernel of the stream is
// dispatched as the previous one's CTAs exit, instead of after its
// completion has been signalled back, and waits for its memory. Ordering is
// exactly stream order. No kernel triggers its dependents early
// (GF2_PDL_TRIGGER=0, measured best: an early trigger let waiting CTAs
// crowd the primaries -- 4096^3 45.3 us with no trigger, 51.4 with a
// trigger at every kernel's start, 49.4 without PDL; 3000^3 at cutoff 512
// 109 / 113 / 142 us). GF2_PDL=0 turns the attribute off.
#ifndef GF2_PDL_TRIGGER
#define GF2_PDL_TRIGGER 0  // 0: implicit trigger at exit; 1: every kernel triggers at its start; 2: not the GEMMs
#endif
__device__ __forceinline__ void pdl_trigger() {
    if (GF2_PDL_TRIGGER == 1) asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
}
__device__ __forceinline__ void pdl_trigger_light() {  // kernels other than the persistent GEMMs
    if (GF2_PDL_TRIGGER >= 1) asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
__device__ __forceinline__ void pdl_begin() {
    pdl_trigger_light();
    pdl_wait();
}
inline int pdl_enabled() {
    static const int on = getenv("GF2_PDL") ? atoi(getenv("GF2_PDL")) : 1;
    return on;
}
// kernel<<<grid, block, smem, s>>>(args...) with the PDL attribute (and an
// optional cluster shape); returns the launch error.
template <typename... KArgs, typename... Args>
inline cudaError_t launch_k(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                            int cluster_x, Args... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[2];
    int na = 0;
    at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[na].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    ++na;
    if (cluster_x > 1) {
        at[na].id = cudaLaunchAttributeClusterDimension;
        at[na].val.clusterDim.x = (unsigned)cluster_x;
        at[na].val.clusterDim.y = 1;
        at[na].val.clusterDim.z = 1;
        ++na;
    }
    cfg.attrs = at;
    cfg.numAttrs = na;
    return cudaLaunchKernelEx(&cfg, kernel, args...);
}

#define GF2_LAUNCH(...)                                                          \
    do {                                                                         \
        cudaError_t _le = (__VA_ARGS__);                                         \
        if (_le != cudaSuccess) return check_cuda(_le, "kernel launch");         \
    } while (0)

#define GF2_TRY(expr)                  \
    do {                               \
        int _rc = (expr);              \
        if (_rc != GF2_OK) return _rc; \
    } while (0)

// A view with offsets (window of a window) resolved on the host.
inline gf2_view sub_view(const gf2_view &v, int64_t r0, int64_t c0, int64_t nr, int64_t nc) {
    gf2_view o;
    o.data = v.data + r0 * v.pitch + c0 / kWordBits;
    o.pitch = v.pitch;
    o.nrows = nr;
    o.ncols = nc;
    return o;
}

// Launchers (all asynchronous on `s`) ---------------------------------
int launch_random(const gf2_view &v, u64 seed, int64_t row_base, cudaStream_t s);
int launch_bernoulli(const gf2_view &v, u64 seed, u64 thresh, int64_t row_base, cudaStream_t s);
int launch_ewise(const gf2_view &out, const gf2_view *a, const gf2_view *b, int op, cudaStream_t s);
int launch_zero(const gf2_view &v, cudaStream_t s);
int launch_make_table(const gf2_view &table, const gf2_view &src, int k, cudaStream_t s);  // graycode.py:108-156

// Batched XOR-combine used by the breadth-first Strassen-Winograd:
// for output o = p * nq + q (p < nprob, q < nq):
//   dst(p, q) [R x W words] (^)= XOR_{i in mask[q]} src(p, i)
// with dst(p,q) = dst + p*dst_stride + dst_off[q], src(p,i) = src + p*src_stride + src_off[i].
struct CombineArgs {
    const u64 *src;
    int64_t src_pitch, src_stride;
    int64_t src_off[8];
    u64 *dst;
    int64_t dst_pitch, dst_stride;
    int64_t dst_off[8];
    unsigned mask[8];
    int nq;
    int64_t R, W;
    int64_t nprob;
    int accumulate;
};
// Per-device side stream (non-blocking) with a fork and a join event, for
// independent work that can overlap on the GPU (one user per call site at a
// time: the host thread issues fork -> side work -> join in order).
struct SideStream {
    cudaStream_t s;              // default priority
    cudaEvent_t fork, join;
    cudaStream_t hi;             // highest priority: work that should win SM slots
    cudaEvent_t hi_fork, hi_join;
};
int side_stream(SideStream **out);
int launch_combine(const CombineArgs &a, cudaStream_t s);
int launch_combine_t(const CombineArgs &a, cudaStream_t s);  // 7 transposed pre-add outputs
int pool_setup();
int launch_transpose(const gf2_view &out, const gf2_view &in, cudaStream_t s);
int launch_cubic(const gf2_view &c, const gf2_view &a, const gf2_view &bt, int accumulate, cudaStream_t s);
int launch_copy_cols(const gf2_view &dst, int64_t c0, const gf2_view &src, cudaStream_t s);

// Batched M4RM: problem q uses A + q*sa, B + q*sb, C + q*sc (same dims).
struct M4rmBatch {
    const u64 *A;
    int64_t pa, sa;
    const u64 *B;
    int64_t pb, sb;
    u64 *C;
    int64_t pc, sc;
    int64_t m, l, n;
    int64_t nprob;
    int accumulate;
};
int launch_m4rm(const M4rmBatch &b, cudaStream_t s);
int launch_umma(const M4rmBatch &b, int kind, cudaStream_t s);
// Tensor-core batch with the last Strassen level fused: fuse_pre -> product
// q = 7p + i multiplies XORs of source problem p's quadrants (maskA/maskB);
// fuse_post -> its result is XORed into quadrants maskC[i] of C problem p.
struct UmmaJob {
    const u64 *A;
    int64_t pa, sa;
    const u64 *B;
    int64_t pb, sb;
    u64 *C;
    int64_t pc, sc;
    int64_t m, l, n;  // product (leaf) dimensions
    int64_t nsrc;     // source problems (x7^fuse_pre products)
    int fuse_pre;     // Strassen levels fused into the expansion: 0, 1 or 2
    int fuse_post, accumulate;
    unsigned maskA[7], maskB[7], maskC[7];
    int b_trans;      // B given transposed (rows n, cols l, pitch pb); kind 2 only
    cudaEvent_t b_ready;  // if set: B's source is produced on another stream
};
int launch_umma_job(const UmmaJob &jb, int kind, cudaStream_t s);
// strassen.py:219-249 (acc_rest: XOR the bottom rows / right columns in)
int peel_fixup(const gf2_view &C, const gf2_view &A, const gf2_view &B, int64_t m2, int64_t l2, int64_t n2,
               int acc_rest, cudaStream_t s);
// one base-case product at the measured M4RM / tensor-engine crossover
int base_mul(const gf2_view &c, const gf2_view &a, const gf2_view &b, int accumulate, cudaStream_t s);
int launch_umma_f4(const UmmaJob &jb, int64_t nprob, cudaStream_t s);  // gf2_umma_f4.cu
int num_sms();
// multiply engine for every product (gf2_set_engine): 0 M4RM, 1 tcgen05 i8, 2 tcgen05 f8, 3 tcgen05 mxf4
extern int g_engine;
// Products below ~1e10 bit-ops run faster on the M4RM kernel than through
// operand expansion + tensor cores (fixed costs dominate). Measured with the
// tc-f4 engine (tools/crossover.py): 2048^3 (8.6e9) 40 us M4RM vs 44 us tc-f4,
// 2560^3 (1.7e10) 84 vs 53 us. The automatic dispatch (Strassen leaves,
// small non-recursive products) routes by this total work. The 8-bit
// engines move twice the operand bytes and cross over later (2^34).
// smallest product (or batch of leaves), in bit-ops, that goes to the tensor
// engine instead of M4RM; GF2_TC_MIN_WORK overrides it (tools/ crossover runs)
inline double tensor_min_work() {
    static const double env = getenv("GF2_TC_MIN_WORK") ? atof(getenv("GF2_TC_MIN_WORK")) : 0.0;
    if (env > 0) return env;
    return g_engine == 3 ? 1.0e10 : 17179869184.0;
}
// smallest leaf side for tensor-core Strassen leaves (GF2_TC_MIN_LEAF
// overrides it; tests use 256 to drive 117649 tensor leaves through chunking).
// 640: 3000^3 at cutoff 512 (736-side leaves) 104.7 -> 88.3 us on tensor
// leaves, while 4096^3 at cutoff 512 (512-side leaves) stays faster on M4RM
// (112.9 vs 121.1 us; tools/leaf_cross.py)
inline int64_t tensor_min_leaf() {
    static const int64_t env = getenv("GF2_TC_MIN_LEAF") ? atoll(getenv("GF2_TC_MIN_LEAF")) : 0;
    return env > 0 ? env : 640;
}
// shallowest tensor-core Strassen leaf in K (GF2_TC_MIN_LEAF_K overrides it;
// 0 honours the caller's cutoff exactly). A 1024-deep leaf tile is bound by
// its epilogue -- draining 224 f32 columns from TMEM (~3400 cycles) takes
// longer than its 4 K-blocks of MMA (~1900) -- so a Winograd level whose
// leaves would be shallower than this is not taken on a tensor engine: its
// product runs classically inside the accumulator (K twice as deep), which
// costs 8/7 of that level's MMAs and saves 3/7 of its epilogues. cfg2 at the
// reference's cutoff 1024: 60.6 -> ~44 us.
inline int64_t tensor_leaf_k() {
    static const int64_t env = getenv("GF2_TC_MIN_LEAF_K") ? atoll(getenv("GF2_TC_MIN_LEAF_K")) : -1;
    return env >= 0 ? env : 2048;
}
inline int launch_product(const M4rmBatch &b, cudaStream_t s) {
    const double work = (double)b.m * (double)b.l * (double)b.n * (double)b.nprob;
    if (g_engine == 0 || work < tensor_min_work()) return launch_m4rm(b, s);
    return launch_umma(b, g_engine - 1, s);
}
// cuTensorMapEncodeTiled through the runtime's driver entry point: a 3-D
// map (inner, outer, problems), byte strides for dims 1 and 2, no
// interleave, 128-byte swizzle or none, OOB elements read as zero.
// rank 1..5 (dims[0] innermost; strides[i] = bytes between steps of dim i+1)
int encode_map_nd(CUtensorMap *map, CUtensorMapDataType dt, void *base, int rank, const uint64_t *dims,
                  const uint64_t *strides, const uint32_t *box, bool swizzle128);
int encode_map_3d(CUtensorMap *map, CUtensorMapDataType dt, void *base, const uint64_t dims[3],
                  const uint64_t strides[2], const uint32_t box[3], bool swizzle128);
int timer_enable(int on);
int timer_begin(cudaStream_t s, double bitops);  // -1 when the timer is off
void timer_end(int idx, cudaStream_t s);
int timer_read(double *ms, double *bitops, int64_t *launches);

}  // namespace gf2
