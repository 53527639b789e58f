/* gf2b200 -- B200-native dense GF(2) matrix multiplication, C ABI.
 *
 * The drop-in boundary for the reference's hot path (gf2mat v0.1.0,
 * /root/reference/pkg/src/gf2mat). The reference is a pure-Python package
 * with no FFI of its own; each entry point below replaces the Python
 * function cited next to it, with the same argument meaning and the same
 * error classes (mapped from the status codes). Plain pointers and sizes
 * only; no torch types. A Python ctypes binding lives in
 * paper_0811_1714_b200/_lib.py; INTEGRATION.md shows the binding a
 * maintainer would add to gf2mat itself.
 *
 * Layout (core.py:3-11): a matrix is row-major, 64 columns per uint64 word,
 * column c of a row at bit 63 - (c % 64) of word c / 64 (MSB first). A
 * view describes a matrix or a window (core.py:110-144): `data` points at
 * word 0 of row 0 of the view (the window's word offset is folded in, so
 * windows need only 8-byte alignment), `pitch` is the word distance between
 * rows. Words per row = ceil(ncols / 64). Every write through a view keeps
 * the bits beyond its right edge (core.py:278-323); owned matrices keep
 * their trailing bits zero.
 *
 * All functions are asynchronous on `stream` (a cudaStream_t, NULL = the
 * legacy default stream) unless stated otherwise, and return a status code;
 * gf2_last_error() gives a thread-local message for the last failure.
 */
#ifndef GF2B200_H
#define GF2B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct gf2_view {
    uint64_t *data;  /* device pointer: word 0 of row 0 of the view */
    int64_t pitch;   /* words between consecutive rows (>= words per row) */
    int64_t nrows;
    int64_t ncols;   /* columns (bits) */
} gf2_view;

/* Status codes; the Python shim maps them to gf2mat's errors.py:4-21. */
enum {
    GF2_OK = 0,
    GF2_ERR_DIMENSION = 1, /* DimensionError (errors.py:8) */
    GF2_ERR_ALIGNMENT = 2, /* AlignmentError (errors.py:12) */
    GF2_ERR_PARAMETER = 3, /* ParameterError (errors.py:16) */
    GF2_ERR_CUDA = 4,      /* CUDA runtime failure (no reference analogue) */
    GF2_ERR_OOM = 5,       /* device allocation failure */
    GF2_ERR_INTERNAL = 6,
    GF2_ERR_NCCL = 7       /* NCCL missing or a collective failed */
};

const char *gf2_version(void);
const char *gf2_last_error(void);

/* row-sharded multi-GPU C_p (+)= A_p . B for hosts that
 * run NCCL themselves (one process or thread per GPU). This rank passes its
 * row shard of C and A and a device buffer `b` for all of B (its contents
 * matter only on rank `src`; with src < 0, B's rows are split into nranks
 * word-aligned blocks and rank r supplies block r, sharded.py owned_rows);
 * B is broadcast with ncclBroadcast on an internal communication stream and
 * multiplied in `npanels` word-aligned K-panels (sharded.py k_panels), each
 * (Strassen-Winograd with `cutoff`) as soon as its rows have landed.
 * `nccl_comm` is an ncclComm_t; NCCL is loaded at run time (libnccl.so.2).
 * Call it outside ncclGroupStart/End, from one host thread or process per
 * GPU: the per-panel "landed" events are recorded right after each
 * ncclBroadcast is issued, which a group would defer.
 * `b` may be any view and the ranks' pitches may differ: a B whose pitch is
 * not its width in words (a window, or a padded pitch) travels through a
 * contiguous staging buffer and is unpacked with an edge-preserving copy,
 * so no word outside B's window is written on any rank.
 * Process grid pr x pc (sharded.py ProcessGrid / mul_sharded_grid): rank
 * (i, j) calls this with the communicator of its COLUMN group (the pr ranks
 * sharing column block j), c_shard = C[rows_i, cols_j], a_shard = A[rows_i, :]
 * and b = the l x n_j column block B_j; nothing else changes, and K is never
 * split across ranks, so there is still no reduction.
 * The Python package offers the same over torch.distributed
 * (paper_0811_1714_b200.sharded.mul_sharded, mul_sharded_grid). */
int gf2_mul_sharded(const gf2_view *c_shard, const gf2_view *a_shard, const gf2_view *b, void *nccl_comm,
                    int src, int npanels, int64_t cutoff, int accumulate, void *stream);

/* Workspace (Strassen level buffers, tensor-core operands) comes from the
 * device's stream-ordered pool, which keeps freed memory cached between
 * calls (cfg5 peaks near 16 GB). This synchronizes the current device and
 * returns the cached memory to the system. */
int gf2_release_workspace(void);

/* Wait for all work queued on `stream` (NULL: the whole device). The
 * library links the CUDA runtime statically, so hosts that do not use CUDA
 * themselves synchronize through this call. */
int gf2_stream_sync(void *stream);

/* Recommended row pitch (words) for an owned device matrix of ncols
 * columns: 16-byte multiple, 128-byte multiple once a row spans 16 words. */
int64_t gf2_pitch_words(int64_t ncols);

/* Device memory for hosts without their own allocator (stream-ordered pool).
 * gf2_alloc zero-fills (core.py:176-178 `create`). */
int gf2_alloc(int64_t nrows, int64_t ncols, gf2_view *out, void *stream);
int gf2_free(gf2_view *v, void *stream);

/* Host <-> device. `host_stride` is the host row stride in words (the
 * reference's dense layout uses width = ceil(ncols/64), core.py:76-80).
 * Upload writes whole words (for owned targets); download copies raw words. */
int gf2_upload(const gf2_view *dst, const uint64_t *host, int64_t host_stride,
               void *stream);
int gf2_download(const gf2_view *src, uint64_t *host, int64_t host_stride,
                 void *stream);

/* dst = 0 on the view, preserving bits beyond its right edge. */
int gf2_zero(const gf2_view *dst, void *stream);

/* core.py:202-208 `random`: word (r, j) = splitmix64(seed + (i+1)*golden)
 * with i = (row_base + r) * width + j, last word tail-masked. row_base
 * selects rows of a taller matrix (row shards of one seeded matrix). */
int gf2_random(const gf2_view *dst, uint64_t seed, int64_t row_base,
               void *stream);

/* SURVEY.md §8(d) Bernoulli(p): entry (r, c) = 1 iff the splitmix64 output
 * at counter (row_base + r) * ncols + c + 1 is < threshold (= floor(p*2^64)). */
int gf2_bernoulli(const gf2_view *dst, uint64_t seed, uint64_t threshold,
                  int64_t row_base, void *stream);

/* core.py:278-300 `add_into`: out = a XOR b (out may alias a or b). */
int gf2_add(const gf2_view *out, const gf2_view *a, const gf2_view *b,
            void *stream);
/* core.py:312-323 `copy_into`. */
int gf2_copy(const gf2_view *out, const gf2_view *a, void *stream);

/* m4rm.py:77-121 `_mul_into` / m4rm.py:124-155 `mul_m4rm*`:
 * C = A.B (accumulate = 0) or C ^= A.B (accumulate = 1, mul_m4rm_into).
 * k is the reference's table width (1..16, validated; the device kernel
 * indexes 8-bit Gray tables -- results are independent of k). C must not
 * alias A or B. */
int gf2_m4rm(const gf2_view *c, const gf2_view *a, const gf2_view *b, int k,
             int accumulate, void *stream);

/* m4rm.py:124-155 `mul_m4rm*` as the drop-in runs them (m4rm.py:77-121
 * `_mul_into` semantics, C = A.B or C ^= A.B): one base-case product, no
 * recursion, on the M4RM kernel -- or, past the measured crossover (>= 1e10
 * bit-ops and every side >= 640), on the selected tensor engine, where the
 * same product is faster. Engine 0 (M4RM) forces the M4RM kernel. Same
 * arguments, semantics and errors as gf2_m4rm. */
int gf2_mul_base(const gf2_view *c, const gf2_view *a, const gf2_view *b, int k,
                 int accumulate, void *stream);

/* graycode.py:108-156 `make_table`: table rows [0, 2^k) = every XOR
 * combination of the k rows of `src` (pass the view of rows
 * [start_row, start_row + k) of B); slot x holds the XOR of the rows i with
 * bit k-1-i of x set (big-endian, slot 0 = zero). Bits of `src` beyond its
 * right edge are masked; the table's rows stay clean. `table` must hold at
 * least 2^k rows of src->ncols columns and must not alias src. */
int gf2_make_table(const gf2_view *table, const gf2_view *src, int k, void *stream);

/* strassen.py:219-249 `peel_fixup`: complete C = A.B given that
 * C[:m2, :n2] already holds A[:m2, :l2] . B[:l2, :n2]: the inner remainder
 * is accumulated into that block, then the bottom rows and the right
 * columns are written, each as one base-case product (never the recursion). */
int gf2_peel_fixup(const gf2_view *c, const gf2_view *a, const gf2_view *b,
                   int64_t m2, int64_t l2, int64_t n2, void *stream);

/* One product launch (no recursion) with the current engine (gf2_set_engine):
 * the dense-contraction entry of north_star (c) when a tensor engine is set.
 * Same semantics and errors as gf2_m4rm. */
int gf2_mul(const gf2_view *c, const gf2_view *a, const gf2_view *b,
            int accumulate, void *stream);

/* strassen.py:257-282 `mul_strassen` (+ peel_split strassen.py:66-84,
 * schedule strassen.py:141-204, peel_fixup strassen.py:219-249):
 * Strassen-Winograd recursion above `cutoff` over the selected base-case
 * engine (gf2_set_engine; small leaves always run M4RM).
 * accumulate = 1 gives C += A.B (cfg4/cfg5 addmul). */
int gf2_strassen(const gf2_view *c, const gf2_view *a, const gf2_view *b,
                 int64_t cutoff, int k, int accumulate, void *stream);

/* Multiply plans (CUDA graphs): capture one gf2_strassen call on fixed
 * views -- its recursion, workspace allocation, side-stream fork/join and
 * every launch -- into a graph, then replay it with a single launch. The
 * views' device buffers must outlive the plan; each launch reads their
 * current contents (accumulate = 1 adds A.B to C's current contents). This
 * removes the per-call host work (validation, planning, tensor-map encoding,
 * 4-6 launches, ~45 us) from loops that multiply the same shapes. */
typedef struct gf2_plan gf2_plan;
int gf2_plan_strassen(gf2_plan **out, const gf2_view *c, const gf2_view *a, const gf2_view *b, int64_t cutoff,
                      int k, int accumulate);
/* m4rm.py:124-155 `mul_m4rm*` / `mul_m4rm_into` (gf2_mul_base semantics,
 * accumulate = 1 for C ^= A.B) captured the same way: a small product's
 * whole host path (validation, geometry, tensor maps, 1-3 launches) becomes
 * one graph launch. */
int gf2_plan_m4rm(gf2_plan **out, const gf2_view *c, const gf2_view *a, const gf2_view *b, int k,
                  int accumulate);
int gf2_plan_launch(gf2_plan *plan, void *stream);
int gf2_plan_destroy(gf2_plan *plan);

/* core.py:374-376 `transpose`: out (a.ncols x a.nrows) = a^T (bit-matrix
 * transpose, 64x64 blocks per warp). */
int gf2_transpose(const gf2_view *out, const gf2_view *a, void *stream);

/* cubic.py:76-102 `mul_cubic`: C (^)= A.B by AND + XOR-fold + parity against
 * B^T -- the reference's narrow-B (n < 64) base case. */
int gf2_cubic(const gf2_view *c, const gf2_view *a, const gf2_view *b,
              int accumulate, void *stream);

/* dst[:, col0 : col0 + src.ncols) = src for ANY column offset (not only
 * multiples of 64), keeping every other bit of dst: the building block of
 * core.py:344-358 `augment` with a ragged left operand. */
int gf2_copy_cols(const gf2_view *dst, int64_t col0, const gf2_view *src,
                  void *stream);

/* strassen.py:66-84 `peel_split`: writes {m', l', n', depth}. Host only. */
int gf2_peel_split(int64_t m, int64_t l, int64_t n, int64_t cutoff,
                   int64_t out4[4]);

/* Number of kernels this library has launched in this process (telemetry
 * for the bench's `gpu_launches`). */
int64_t gf2_launch_count(void);

/* High-water mark (bytes) of the library's workspace in the device's
 * stream-ordered pool since the last reset (reset = 1 restarts it at the
 * current use): the device analogue of the reference CLI's peak_mem_bytes
 * (counters.py peak_live_words, cli.py:161-166). */
int gf2_workspace_peak(int64_t *bytes, int reset);

/* Of those, the launches of the M4RM kernel (k_m4rm): tells which engine
 * a product was dispatched to. */
int64_t gf2_m4rm_launch_count(void);

/* Kernel timer for the roofline: while enabled, every product launch (M4RM
 * or tensor-core GEMM) is bracketed by CUDA events recorded on the stream it
 * runs on. Enabling
 * resets the accumulators. gf2_timer_read synchronizes the recorded events
 * and returns the summed kernel milliseconds, the algorithmic bit-ops
 * (m*l*n per product) those launches computed, and the launch count. */
int gf2_timer_enable(int on);
/* Engine for Strassen leaves, non-recursive gf2_strassen calls and gf2_mul,
 * process-wide: 0 = M4RM shared-memory Gray tables, 1 = tcgen05 kind::i8
 * (u8 0/1), 2 = tcgen05 kind::f8f6f4 (e4m3 0/1), 3 = tcgen05 kind::mxf4
 * (e2m1 nibbles, unit block scales; default: measured fastest).
 * gf2_m4rm always runs the M4RM kernel; gf2_mul_base (the mul_m4rm* path)
 * uses the tensor engine past the crossover. Results are identical. */
int gf2_set_engine(int engine);
int gf2_get_engine(void);
int gf2_timer_read(double *kernel_ms, double *bitops, int64_t *launches);

#ifdef __cplusplus
}
#endif
#endif /* GF2B200_H */
