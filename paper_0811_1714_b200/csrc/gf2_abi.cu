// C-ABI entry points (include/gf2b200.h). Validation mirrors the checks and
// messages of the reference functions each entry replaces, so the Python
// shim raises the same exception classes for the same inputs.
#include <nccl.h>
#include <stdio.h>

#include <string>

#include "gf2_internal.cuh"

namespace gf2 {
int mul_sharded(const gf2_view &c, const gf2_view &a, const gf2_view &b, ncclComm_t comm, int src, int npanels,
                int64_t cutoff, int accumulate, cudaStream_t s);
int m4rm_mul(const gf2_view &c, const gf2_view &a, const gf2_view &b, int accumulate, cudaStream_t s);
int engine_mul(const gf2_view &c, const gf2_view &a, const gf2_view &b, int accumulate, cudaStream_t s);
int strassen_mul(const gf2_view &C, const gf2_view &A, const gf2_view &B, int64_t cutoff, int accumulate,
                 cudaStream_t s);
void peel_split(int64_t m, int64_t l, int64_t n, int64_t cutoff, int64_t out[4]);

std::atomic<int64_t> g_launches{0};
std::atomic<int64_t> g_m4rm_launches{0};
int g_engine = 3;  // tcgen05 kind::mxf4: measured fastest base case
static thread_local std::string t_err;

int set_error(int code, const std::string &msg) {
    t_err = msg;
    return code;
}

int check_cuda(cudaError_t e, const char *what) {
    if (e == cudaSuccess) return GF2_OK;
    return set_error(e == cudaErrorMemoryAllocation ? GF2_ERR_OOM : GF2_ERR_CUDA,
                     std::string(what) + ": " + cudaGetErrorString(e));
}

static int check_view(const gf2_view *v, const char *name) {
    if (!v) return set_error(GF2_ERR_PARAMETER, std::string(name) + ": null view");
    if (v->nrows < 0 || v->ncols < 0)
        return set_error(GF2_ERR_DIMENSION, std::string("negative dimensions ") + std::to_string(v->nrows) + "x" +
                                                std::to_string(v->ncols));
    const int64_t w = words_per_row(v->ncols);
    if (v->nrows > 1 && v->pitch < w)
        return set_error(GF2_ERR_PARAMETER, std::string(name) + ": pitch " + std::to_string(v->pitch) +
                                                " < words per row " + std::to_string(w));
    if (v->nrows > 0 && w > 0) {
        if (!v->data) return set_error(GF2_ERR_PARAMETER, std::string(name) + ": null data");
        if (reinterpret_cast<uintptr_t>(v->data) % 8)
            return set_error(GF2_ERR_ALIGNMENT, std::string(name) + ": data not 8-byte (word) aligned");
    }
    return GF2_OK;
}

static bool overlaps(const gf2_view &x, const gf2_view &y) {
    const int64_t wx = words_per_row(x.ncols), wy = words_per_row(y.ncols);
    if (!x.nrows || !wx || !y.nrows || !wy) return false;
    const uint64_t *x0 = x.data, *x1 = x.data + (x.nrows - 1) * x.pitch + wx;
    const uint64_t *y0 = y.data, *y1 = y.data + (y.nrows - 1) * y.pitch + wy;
    return x0 < y1 && y0 < x1;
}

static int check_mul(const gf2_view *c, const gf2_view *a, const gf2_view *b) {
    GF2_TRY(check_view(a, "a"));
    GF2_TRY(check_view(b, "b"));
    GF2_TRY(check_view(c, "c"));
    if (a->ncols != b->nrows)  // m4rm.py:70-73, strassen.py:260-262
        return set_error(GF2_ERR_DIMENSION, "inner dimensions " + std::to_string(a->ncols) + " and " +
                                                std::to_string(b->nrows) + " differ");
    if (c->nrows != a->nrows || c->ncols != b->ncols)  // m4rm.py:82-84
        return set_error(GF2_ERR_DIMENSION, "target " + std::to_string(c->nrows) + "x" +
                                                std::to_string(c->ncols) + " != product " +
                                                std::to_string(a->nrows) + "x" + std::to_string(b->ncols));
    if (overlaps(*c, *a) || overlaps(*c, *b))  // schedule_winograd: c must not alias a or b
        return set_error(GF2_ERR_PARAMETER, "product target aliases an operand");
    return GF2_OK;
}

static int check_same_shape(const gf2_view *out, const gf2_view *a, const char *what) {
    if (out->nrows != a->nrows || out->ncols != a->ncols)
        return set_error(GF2_ERR_DIMENSION, std::string(what) + " shapes (" + std::to_string(a->nrows) + ", " +
                                                std::to_string(a->ncols) + ") -> (" + std::to_string(out->nrows) +
                                                ", " + std::to_string(out->ncols) + ") differ");
    return GF2_OK;
}

// capture `body(stream)` into a graph on a private stream
template <typename F>
int capture_plan(cudaGraph_t *g_out, cudaGraphExec_t *e_out, F body) {
    GF2_TRY(pool_setup());
    SideStream *sd = nullptr;
    GF2_TRY(side_stream(&sd));  // created outside the capture
    cudaStream_t cs = nullptr;
    GF2_TRY(check_cuda(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking), "plan stream"));
    // relaxed: the library's one-time lazy setup (function attributes,
    // driver entry point) may run while capturing
    int rc = check_cuda(cudaStreamBeginCapture(cs, cudaStreamCaptureModeRelaxed), "begin capture");
    cudaGraph_t graph = nullptr;
    if (rc == GF2_OK) {
        rc = body(cs);
        const cudaError_t e = cudaStreamEndCapture(cs, &graph);
        if (rc == GF2_OK) rc = check_cuda(e, "end capture");
    }
    cudaGraphExec_t exec = nullptr;
    if (rc == GF2_OK) rc = check_cuda(cudaGraphInstantiate(&exec, graph, 0), "graph instantiate");
    cudaStreamDestroy(cs);
    if (rc != GF2_OK) {
        if (graph) cudaGraphDestroy(graph);
        cudaGetLastError();
        return rc;
    }
    *g_out = graph;
    *e_out = exec;
    return GF2_OK;
}

}  // namespace gf2

using namespace gf2;

extern "C" {

const char *gf2_version(void) { return "gf2b200 0.1.0 (sm_100a)"; }

const char *gf2_last_error(void) { return t_err.c_str(); }

int gf2_mul_sharded(const gf2_view *c_shard, const gf2_view *a_shard, const gf2_view *b, void *nccl_comm,
                    int src, int npanels, int64_t cutoff, int accumulate, void *stream) {
    if (!nccl_comm) return set_error(GF2_ERR_PARAMETER, "null NCCL communicator");
    if (npanels < 1) return set_error(GF2_ERR_PARAMETER, "npanels " + std::to_string(npanels) + " < 1");
    if (cutoff < 64) return set_error(GF2_ERR_PARAMETER, "cutoff " + std::to_string(cutoff) + " < 64");
    GF2_TRY(check_mul(c_shard, a_shard, b));
    return mul_sharded(*c_shard, *a_shard, *b, (ncclComm_t)nccl_comm, src, npanels, cutoff, accumulate ? 1 : 0,
                       (cudaStream_t)stream);
}

int gf2_release_workspace(void) {
    int dev = 0;
    GF2_TRY(check_cuda(cudaGetDevice(&dev), "cudaGetDevice"));
    GF2_TRY(check_cuda(cudaDeviceSynchronize(), "cudaDeviceSynchronize"));
    cudaMemPool_t pool;
    GF2_TRY(check_cuda(cudaDeviceGetDefaultMemPool(&pool, dev), "cudaDeviceGetDefaultMemPool"));
    return check_cuda(cudaMemPoolTrimTo(pool, 0), "cudaMemPoolTrimTo");
}

int gf2_stream_sync(void *stream) {
    if (!stream) return check_cuda(cudaDeviceSynchronize(), "cudaDeviceSynchronize");
    return check_cuda(cudaStreamSynchronize((cudaStream_t)stream), "cudaStreamSynchronize");
}

int64_t gf2_pitch_words(int64_t ncols) {
    int64_t w = words_per_row(ncols);
    if (w >= 16) return (w + 15) / 16 * 16;
    return (w + 1) / 2 * 2;
}

int64_t gf2_launch_count(void) { return g_launches.load(); }
int64_t gf2_m4rm_launch_count(void) { return g_m4rm_launches.load(); }

int gf2_workspace_peak(int64_t *bytes, int reset) {
    GF2_TRY(pool_setup());
    int dev = 0;
    GF2_TRY(check_cuda(cudaGetDevice(&dev), "cudaGetDevice"));
    cudaMemPool_t pool;
    GF2_TRY(check_cuda(cudaDeviceGetDefaultMemPool(&pool, dev), "cudaDeviceGetDefaultMemPool"));
    if (reset) {
        uint64_t zero = 0;
        GF2_TRY(check_cuda(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrUsedMemHigh, &zero), "reset pool peak"));
    }
    uint64_t hi = 0;
    GF2_TRY(check_cuda(cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemHigh, &hi), "pool peak"));
    if (bytes) *bytes = (int64_t)hi;
    return GF2_OK;
}

int gf2_timer_enable(int on) { return timer_enable(on); }

int gf2_set_engine(int engine) {
    if (engine < 0 || engine > 3)
        return set_error(GF2_ERR_PARAMETER, "engine must be 0 (m4rm), 1 (tc-i8), 2 (tc-f8), 3 (tc-f4)");
    g_engine = engine;
    return GF2_OK;
}

int gf2_get_engine(void) { return g_engine; }

int gf2_timer_read(double *kernel_ms, double *bitops, int64_t *launches) {
    return timer_read(kernel_ms, bitops, launches);
}

int gf2_alloc(int64_t nrows, int64_t ncols, gf2_view *out, void *stream) {
    if (!out) return set_error(GF2_ERR_PARAMETER, "null output view");
    if (nrows < 0 || ncols < 0)
        return set_error(GF2_ERR_DIMENSION,
                         "negative dimensions " + std::to_string(nrows) + "x" + std::to_string(ncols));
    const int64_t pitch = gf2_pitch_words(ncols);
    size_t bytes = (size_t)(nrows * pitch) * 8;
    void *p = nullptr;
    cudaStream_t s = (cudaStream_t)stream;
    if (bytes) {
        GF2_TRY(pool_setup());
        GF2_TRY(check_cuda(cudaMallocAsync(&p, bytes, s), "cudaMallocAsync"));
        GF2_TRY(check_cuda(cudaMemsetAsync(p, 0, bytes, s), "cudaMemsetAsync"));
    }
    out->data = (uint64_t *)p;
    out->pitch = pitch;
    out->nrows = nrows;
    out->ncols = ncols;
    return GF2_OK;
}

int gf2_free(gf2_view *v, void *stream) {
    if (!v) return GF2_OK;
    if (v->data) GF2_TRY(check_cuda(cudaFreeAsync(v->data, (cudaStream_t)stream), "cudaFreeAsync"));
    v->data = nullptr;
    return GF2_OK;
}

int gf2_upload(const gf2_view *dst, const uint64_t *host, int64_t host_stride, void *stream) {
    GF2_TRY(check_view(dst, "dst"));
    const int64_t w = words_per_row(dst->ncols);
    if (!dst->nrows || !w) return GF2_OK;
    if (!host || host_stride < w) return set_error(GF2_ERR_PARAMETER, "bad host buffer / stride");
    if (dst->pitch == w && host_stride == w)  // both dense: one linear DMA
        return check_cuda(cudaMemcpyAsync(dst->data, host, (size_t)(w * dst->nrows) * 8, cudaMemcpyHostToDevice,
                                          (cudaStream_t)stream),
                          "upload");
    return check_cuda(cudaMemcpy2DAsync(dst->data, dst->pitch * 8, host, host_stride * 8, w * 8, dst->nrows,
                                        cudaMemcpyHostToDevice, (cudaStream_t)stream),
                      "upload");
}

int gf2_download(const gf2_view *src, uint64_t *host, int64_t host_stride, void *stream) {
    GF2_TRY(check_view(src, "src"));
    const int64_t w = words_per_row(src->ncols);
    if (!src->nrows || !w) return GF2_OK;
    if (!host || host_stride < w) return set_error(GF2_ERR_PARAMETER, "bad host buffer / stride");
    if (src->pitch == w && host_stride == w)
        return check_cuda(cudaMemcpyAsync(host, src->data, (size_t)(w * src->nrows) * 8, cudaMemcpyDeviceToHost,
                                          (cudaStream_t)stream),
                          "download");
    return check_cuda(cudaMemcpy2DAsync(host, host_stride * 8, src->data, src->pitch * 8, w * 8, src->nrows,
                                        cudaMemcpyDeviceToHost, (cudaStream_t)stream),
                      "download");
}

int gf2_zero(const gf2_view *dst, void *stream) {
    GF2_TRY(check_view(dst, "dst"));
    return launch_zero(*dst, (cudaStream_t)stream);  // 2-D memset unless the right edge is ragged
}

int gf2_random(const gf2_view *dst, uint64_t seed, int64_t row_base, void *stream) {
    GF2_TRY(check_view(dst, "dst"));
    return launch_random(*dst, seed, row_base, (cudaStream_t)stream);
}

int gf2_bernoulli(const gf2_view *dst, uint64_t seed, uint64_t threshold, int64_t row_base, void *stream) {
    GF2_TRY(check_view(dst, "dst"));
    return launch_bernoulli(*dst, seed, threshold, row_base, (cudaStream_t)stream);
}

int gf2_add(const gf2_view *out, const gf2_view *a, const gf2_view *b, void *stream) {
    GF2_TRY(check_view(out, "out"));
    GF2_TRY(check_view(a, "a"));
    GF2_TRY(check_view(b, "b"));
    if (a->nrows != b->nrows || a->ncols != b->ncols || out->nrows != a->nrows || out->ncols != a->ncols)
        return set_error(GF2_ERR_DIMENSION, "add shapes (" + std::to_string(a->nrows) + ", " +
                                                std::to_string(a->ncols) + "), (" + std::to_string(b->nrows) +
                                                ", " + std::to_string(b->ncols) + ") -> (" +
                                                std::to_string(out->nrows) + ", " + std::to_string(out->ncols) +
                                                ") differ");
    return launch_ewise(*out, a, b, 2, (cudaStream_t)stream);
}

int gf2_copy(const gf2_view *out, const gf2_view *a, void *stream) {
    GF2_TRY(check_view(out, "out"));
    GF2_TRY(check_view(a, "a"));
    GF2_TRY(check_same_shape(out, a, "copy"));
    return launch_ewise(*out, a, nullptr, 1, (cudaStream_t)stream);
}

int gf2_m4rm(const gf2_view *c, const gf2_view *a, const gf2_view *b, int k, int accumulate, void *stream) {
    if (k < 1 || k > 16) return set_error(GF2_ERR_PARAMETER, "k=" + std::to_string(k) + " outside 1..16");
    GF2_TRY(check_mul(c, a, b));
    return m4rm_mul(*c, *a, *b, accumulate ? 1 : 0, (cudaStream_t)stream);
}

int gf2_mul_base(const gf2_view *c, const gf2_view *a, const gf2_view *b, int k, int accumulate, void *stream) {
    if (k < 1 || k > 16) return set_error(GF2_ERR_PARAMETER, "k=" + std::to_string(k) + " outside 1..16");
    GF2_TRY(check_mul(c, a, b));
    return base_mul(*c, *a, *b, accumulate ? 1 : 0, (cudaStream_t)stream);
}

int gf2_make_table(const gf2_view *table, const gf2_view *src, int k, void *stream) {
    GF2_TRY(check_view(table, "table"));
    GF2_TRY(check_view(src, "src"));
    if (k < 1 || k > 16) return set_error(GF2_ERR_PARAMETER, "table fill width " + std::to_string(k) +
                                                                 " outside 1..16");
    if (src->nrows != k)
        return set_error(GF2_ERR_DIMENSION, "source holds " + std::to_string(src->nrows) + " rows, k=" +
                                                std::to_string(k));
    if (table->ncols != src->ncols)  // graycode.py:128-130
        return set_error(GF2_ERR_DIMENSION, "table width " + std::to_string(table->ncols) + " != source width " +
                                                std::to_string(src->ncols));
    if (table->nrows < ((int64_t)1 << k))
        return set_error(GF2_ERR_DIMENSION, "table holds " + std::to_string(table->nrows) + " rows < 2^" +
                                                std::to_string(k));
    if (overlaps(*table, *src)) return set_error(GF2_ERR_PARAMETER, "table aliases its source rows");
    return launch_make_table(*table, *src, k, (cudaStream_t)stream);
}

int gf2_peel_fixup(const gf2_view *c, const gf2_view *a, const gf2_view *b, int64_t m2, int64_t l2, int64_t n2,
                   void *stream) {
    GF2_TRY(check_mul(c, a, b));
    if (m2 < 0 || l2 < 0 || n2 < 0 || m2 > a->nrows || l2 > a->ncols || n2 > b->ncols)  // strassen.py:234-236
        return set_error(GF2_ERR_DIMENSION, "peel dims (" + std::to_string(m2) + "," + std::to_string(l2) + "," +
                                                std::to_string(n2) + ") exceed (" + std::to_string(a->nrows) + "," +
                                                std::to_string(a->ncols) + "," + std::to_string(b->ncols) + ")");
    return peel_fixup(*c, *a, *b, m2, l2, n2, 0, (cudaStream_t)stream);
}

int gf2_mul(const gf2_view *c, const gf2_view *a, const gf2_view *b, int accumulate, void *stream) {
    GF2_TRY(check_mul(c, a, b));
    return engine_mul(*c, *a, *b, accumulate ? 1 : 0, (cudaStream_t)stream);
}

int gf2_strassen(const gf2_view *c, const gf2_view *a, const gf2_view *b, int64_t cutoff, int k, int accumulate,
                 void *stream) {
    if (cutoff < 64) return set_error(GF2_ERR_PARAMETER, "cutoff " + std::to_string(cutoff) + " < 64");
    if (k < 0 || k > 16) return set_error(GF2_ERR_PARAMETER, "k=" + std::to_string(k) + " outside 0..16");
    GF2_TRY(check_mul(c, a, b));
    return strassen_mul(*c, *a, *b, cutoff, accumulate ? 1 : 0, (cudaStream_t)stream);
}

struct gf2_plan {
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
};

int gf2_plan_strassen(gf2_plan **out, const gf2_view *c, const gf2_view *a, const gf2_view *b, int64_t cutoff,
                      int k, int accumulate) {
    if (!out) return set_error(GF2_ERR_PARAMETER, "null plan pointer");
    *out = nullptr;
    if (cutoff < 64) return set_error(GF2_ERR_PARAMETER, "cutoff " + std::to_string(cutoff) + " < 64");
    if (k < 0 || k > 16) return set_error(GF2_ERR_PARAMETER, "k=" + std::to_string(k) + " outside 0..16");
    GF2_TRY(check_mul(c, a, b));
    cudaGraph_t g = nullptr;
    cudaGraphExec_t e = nullptr;
    GF2_TRY(capture_plan(&g, &e, [&](cudaStream_t cs) { return strassen_mul(*c, *a, *b, cutoff, accumulate ? 1 : 0, cs); }));
    *out = new gf2_plan{g, e};
    return GF2_OK;
}

int gf2_plan_m4rm(gf2_plan **out, const gf2_view *c, const gf2_view *a, const gf2_view *b, int k, int accumulate) {
    if (!out) return set_error(GF2_ERR_PARAMETER, "null plan pointer");
    *out = nullptr;
    if (k < 1 || k > 16) return set_error(GF2_ERR_PARAMETER, "k=" + std::to_string(k) + " outside 1..16");
    GF2_TRY(check_mul(c, a, b));
    cudaGraph_t g = nullptr;
    cudaGraphExec_t e = nullptr;
    GF2_TRY(capture_plan(&g, &e, [&](cudaStream_t cs) { return base_mul(*c, *a, *b, accumulate ? 1 : 0, cs); }));
    *out = new gf2_plan{g, e};
    return GF2_OK;
}

int gf2_plan_launch(gf2_plan *plan, void *stream) {
    if (!plan || !plan->exec) return set_error(GF2_ERR_PARAMETER, "null plan");
    return check_cuda(cudaGraphLaunch(plan->exec, (cudaStream_t)stream), "graph launch");
}

int gf2_plan_destroy(gf2_plan *plan) {
    if (!plan) return GF2_OK;
    int rc = GF2_OK;
    if (plan->exec) rc = check_cuda(cudaGraphExecDestroy(plan->exec), "graph exec destroy");
    if (plan->graph) cudaGraphDestroy(plan->graph);
    delete plan;
    return rc;
}

int gf2_transpose(const gf2_view *out, const gf2_view *a, void *stream) {
    GF2_TRY(check_view(out, "out"));
    GF2_TRY(check_view(a, "a"));
    if (out->nrows != a->ncols || out->ncols != a->nrows)
        return set_error(GF2_ERR_DIMENSION, "transpose target " + std::to_string(out->nrows) + "x" +
                                                std::to_string(out->ncols) + " != " + std::to_string(a->ncols) +
                                                "x" + std::to_string(a->nrows));
    if (overlaps(*out, *a)) return set_error(GF2_ERR_PARAMETER, "transpose target aliases its source");
    return launch_transpose(*out, *a, (cudaStream_t)stream);
}

int gf2_cubic(const gf2_view *c, const gf2_view *a, const gf2_view *b, int accumulate, void *stream) {
    GF2_TRY(check_mul(c, a, b));
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t m = a->nrows, l = a->ncols, n = b->ncols;
    if (!m || !n) return GF2_OK;
    if (!l) return accumulate ? GF2_OK : launch_ewise(*c, nullptr, nullptr, 0, s);
    gf2_view bt{nullptr, words_per_row(l), n, l};
    GF2_TRY(pool_setup());
    GF2_TRY(check_cuda(cudaMallocAsync((void **)&bt.data, (size_t)(n * bt.pitch) * 8, s), "cubic workspace"));
    int rc = launch_transpose(bt, *b, s);
    if (rc == GF2_OK) rc = launch_cubic(*c, *a, bt, accumulate ? 1 : 0, s);
    cudaFreeAsync(bt.data, s);
    return rc;
}

int gf2_copy_cols(const gf2_view *dst, int64_t col0, const gf2_view *src, void *stream) {
    GF2_TRY(check_view(dst, "dst"));
    GF2_TRY(check_view(src, "src"));
    if (src->nrows != dst->nrows || col0 < 0 || col0 + src->ncols > dst->ncols)
        return set_error(GF2_ERR_DIMENSION, "column copy of " + std::to_string(src->nrows) + "x" +
                                                std::to_string(src->ncols) + " at column " + std::to_string(col0) +
                                                " exceeds " + std::to_string(dst->nrows) + "x" +
                                                std::to_string(dst->ncols));
    if (overlaps(*dst, *src)) return set_error(GF2_ERR_PARAMETER, "column copy target aliases its source");
    return launch_copy_cols(*dst, col0, *src, (cudaStream_t)stream);
}

int gf2_peel_split(int64_t m, int64_t l, int64_t n, int64_t cutoff, int64_t out4[4]) {
    if (!out4) return set_error(GF2_ERR_PARAMETER, "null output");
    peel_split(m, l, n, cutoff, out4);
    return GF2_OK;
}

}  // extern "C"

namespace gf2 {
// Stream-ordered pool for every workspace the library allocates: keep freed
// blocks cached so repeated calls never go back to cudaMalloc (process-wide,
// per device, idempotent).
int pool_setup() {
    static bool configured[64] = {false};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 64 && configured[dev]) return GF2_OK;
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        uint64_t thresh = UINT64_MAX;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thresh);
    }
    cudaGetLastError();
    if (dev < 64) configured[dev] = true;
    return GF2_OK;
}
}  // namespace gf2
