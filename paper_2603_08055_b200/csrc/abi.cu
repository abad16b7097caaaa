// abi.cu — the extern "C" boundary (include/gsa_sm100.h): argument validation
// with the reference's error classes, workspace carving and stream-ordered
// orchestration of the kernels. No host synchronisation in compute calls
// except where the header says so.
#include <math.h>

#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <string>

#include "kernels.h"
#include "tc.h"

using namespace gsa_sm100;

namespace gsa_sm100 {
extern std::atomic<unsigned long long> g_launch_total;
}

namespace {

thread_local std::string g_msg;
thread_local cudaEvent_t g_stage_events[7];
thread_local int g_n_stage_events = 0;


int fail(int status, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_msg = buf;
    return status;
}

int cuda_status(cudaError_t e, const char* where) {
    if (e == cudaSuccess) return GSA_OK;
    return fail(GSA_ERR_CUDA, "%s: %s", where, cudaGetErrorString(e));
}

#define GSA_TRY(expr)                 \
    do {                              \
        int _rc = (expr);             \
        if (_rc != GSA_OK) return _rc; \
    } while (0)
#define GSA_CUDA(expr) GSA_TRY(cuda_status((expr), #expr))

TensorRef ref_of(const gsa_tensor& t, int row_offset = 0) {
    TensorRef r;
    const size_t es = t.dtype == GSA_DTYPE_BF16 ? 2 : 4;
    r.data = static_cast<const char*>(t.data) + (size_t)row_offset * t.row_stride * es;
    r.dtype = t.dtype;
    r.hs = t.head_stride;
    r.rs = t.row_stride;
    return r;
}

int check_tensor(const gsa_tensor* t, const char* name, bool allow_bf16 = true) {
    if (!t) return fail(GSA_ERR_GENERIC, "%s: null tensor", name);
    if (t->dtype != GSA_DTYPE_F32 && !(allow_bf16 && t->dtype == GSA_DTYPE_BF16))
        return fail(GSA_ERR_UNSUPPORTED, "%s: dtype %d not supported here", name, t->dtype);
    if (t->heads < 0 || t->rows < 0 || t->dim < 0)
        return fail(GSA_ERR_SHAPE_MISMATCH, "%s: negative extent", name);
    if ((int64_t)t->heads * t->rows * t->dim > 0 && !t->data)
        return fail(GSA_ERR_GENERIC, "%s: null data", name);
    return GSA_OK;
}

int check_f32_out(const gsa_tensor* t, const char* name, int heads, int rows, int dim) {
    GSA_TRY(check_tensor(t, name, false));
    if (t->heads != heads || t->rows != rows || t->dim != dim)
        return fail(GSA_ERR_SHAPE_MISMATCH, "%s: expected [%d x %d x %d], got [%d x %d x %d]", name,
                    heads, rows, dim, t->heads, t->rows, t->dim);
    return GSA_OK;
}

int same_heads_dim(const gsa_tensor* a, const gsa_tensor* b, const char* what) {
    // require_same_heads_dim (tensor.hpp:60-63)
    if (a->heads != b->heads || a->dim != b->dim)
        return fail(GSA_ERR_SHAPE_MISMATCH, "%s: heads/dim disagree", what);
    return GSA_OK;
}

int check_tiling(int bm, int bn) {
    // validate_tiling (types.hpp:20-25)
    auto ok = [](int v) { return v >= 8 && v <= 256 && (v & (v - 1)) == 0; };
    if (!ok(bm) || !ok(bn))
        return fail(GSA_ERR_INVALID_TILING, "tiling blocks must be powers of two in [8, 256], got %dx%d", bm, bn);
    return GSA_OK;
}

int check_layout(const gsa_layout* l) {
    if (!l) return fail(GSA_ERR_GENERIC, "null layout");
    gsa_layout tmp;
    return gsa_make_layout(l->num_special, l->num_frames, l->grid_h, l->grid_w, l->window_s, &tmp);
}

int generic_supported(int dim, int s) {
    if (dim < 1 || dim > 128) return fail(GSA_ERR_UNSUPPORTED, "head dim %d outside [1,128]", dim);
    if (s != 1 && s != 2 && s != 4 && s != 8)
        return fail(GSA_ERR_UNSUPPORTED, "window_s=%d: the sm_100a kernels take s in {1,2,4,8}", s);
    return GSA_OK;
}

float resolved_scale(double param, int dim) {
    // reference.hpp:22-26
    return param > 0.0 ? (float)param : (float)(1.0 / sqrt((double)dim));
}

struct Carver {
    char* base;
    size_t cap, used = 0;
    bool dry;
    template <typename T>
    T* take(size_t n) {
        used = (used + 255) & ~size_t(255);
        T* p = dry ? nullptr : reinterpret_cast<T*>(base + used);
        used += n * sizeof(T);
        return p;
    }
};

int selectable_windows(const DevLayout& L, int variant, int ref_stride, int* n_forced) {
    int nf = 0;
    if (variant == 1)
        for (int f = 0; f < L.num_frames; f += ref_stride) nf += L.wins_per_frame;
    *n_forced = nf;
    return L.windows - nf;
}

}  // namespace

namespace gsa_sm100 {
// the calling thread's gsa_last_error_message() (for entry points defined in other
// translation units, e.g. comm.cu)
int report_error(int status, const char* msg) {
    g_msg = msg;
    return status;
}
// gsa_set_stage_events instrumentation: record event i on `st` when enabled
void stage_mark(int i, cudaStream_t st) {
    if (g_n_stage_events > i) cudaEventRecord(g_stage_events[i], st);
}
}  // namespace gsa_sm100

extern "C" {

int gsa_abi_version(void) { return GSA_SM100_ABI_VERSION; }

const char* gsa_status_string(int s) {
    switch (s) {
        case GSA_OK: return "ok";
        case GSA_ERR_GENERIC: return "GsaError";
        case GSA_ERR_SHAPE_MISMATCH: return "ShapeMismatch";
        case GSA_ERR_DIVISIBILITY: return "DivisibilityError";
        case GSA_ERR_ZERO_SIZE: return "ZeroSizeError";
        case GSA_ERR_INDEX_OUT_OF_RANGE: return "IndexOutOfRange";
        case GSA_ERR_NON_FINITE: return "NonFiniteInput";
        case GSA_ERR_INVALID_TILING: return "InvalidTiling";
        case GSA_ERR_INVALID_STRIDE: return "InvalidStride";
        case GSA_ERR_EMPTY_SELECTION: return "EmptySelection";
        case GSA_ERR_UNSUPPORTED: return "Unsupported";
        case GSA_ERR_CUDA: return "CudaError";
        case GSA_ERR_WORKSPACE: return "WorkspaceError";
        case GSA_ERR_NCCL: return "NcclError";
        case GSA_ERR_CONTEXT_MISMATCH: return "ContextMismatch";
        default: return "unknown";
    }
}

const char* gsa_last_error_message(void) { return g_msg.c_str(); }

int gsa_make_layout(int ns, int nf, int gh, int gw, int s, gsa_layout* out) {
    // build_token_layout (layout.cpp:7-24)
    if (ns < 0) return fail(GSA_ERR_ZERO_SIZE, "build_token_layout: num_special < 0");
    if (nf < 1) return fail(GSA_ERR_ZERO_SIZE, "build_token_layout: num_frames < 1");
    if (gh < 1 || gw < 1) return fail(GSA_ERR_ZERO_SIZE, "build_token_layout: empty grid");
    if (s < 1) return fail(GSA_ERR_ZERO_SIZE, "build_token_layout: window_s < 1");
    if (gh % s != 0 || gw % s != 0)
        return fail(GSA_ERR_DIVISIBILITY, "build_token_layout: grid %dx%d not divisible by window_s=%d", gh, gw, s);
    if ((int64_t)nf * gh * gw + ns > INT32_MAX)
        return fail(GSA_ERR_UNSUPPORTED, "build_token_layout: more than 2^31 tokens");
    if (out) *out = gsa_layout{ns, nf, gh, gw, s};
    return GSA_OK;
}

int gsa_validate_params(const gsa_params* p, const gsa_layout* l) {
    // validate_params (types.hpp:67-73) + layer.hpp:182-183
    if (!p) return fail(GSA_ERR_GENERIC, "null params");
    if (p->top_k < 1) return fail(GSA_ERR_GENERIC, "params: top_k must be >= 1");
    if (p->scale < 0.0) return fail(GSA_ERR_GENERIC, "params: scale must be > 0");
    if (p->variant == 1 && p->ref_stride < 1)
        return fail(GSA_ERR_INVALID_STRIDE, "params: ref_stride must be >= 1 for hybrid selection");
    if (p->variant != 0 && p->variant != 1) return fail(GSA_ERR_GENERIC, "params: unknown variant");
    GSA_TRY(check_tiling(p->block_m, p->block_n));
    if (l && p->window_s != l->window_s)
        return fail(GSA_ERR_SHAPE_MISMATCH, "gsa_forward: params.window_s != layout.window_s");
    return GSA_OK;
}

int gsa_avg_pool_tokens(const gsa_tensor* x, const gsa_layout* layout, const gsa_tensor* out,
                        gsa_stream_t stream) {
    GSA_TRY(check_layout(layout));
    GSA_TRY(check_tensor(x, "x_img"));
    const DevLayout L = make_dev_layout(*layout);
    if (x->rows != L.image_tokens) return fail(GSA_ERR_SHAPE_MISMATCH, "avg_pool_tokens: rows != image tokens");
    GSA_TRY(check_f32_out(out, "out", x->heads, L.windows, x->dim));
    if (out->row_stride != x->dim || out->head_stride != (int64_t)L.windows * x->dim)
        return fail(GSA_ERR_UNSUPPORTED, "avg_pool_tokens: out must be contiguous");
    PoolJob j{ref_of(*x), static_cast<float*>(out->data), nullptr, nullptr, nullptr};
    const float inv = 1.0f / (float)(L.s * L.s);  // T(1)/T(s2) (compression.hpp:25)
    GSA_CUDA(launch_pool(&j, 1, x->heads, x->dim, L, inv, (cudaStream_t)stream));
    return GSA_OK;
}

int gsa_upsample_nearest(const gsa_tensor* coarse, const gsa_layout* layout, const gsa_tensor* out,
                         gsa_stream_t stream) {
    GSA_TRY(check_layout(layout));
    GSA_TRY(check_tensor(coarse, "coarse", false));
    const DevLayout L = make_dev_layout(*layout);
    if (coarse->rows != L.windows) return fail(GSA_ERR_SHAPE_MISMATCH, "upsample_nearest: rows != num windows");
    GSA_TRY(check_f32_out(out, "out", coarse->heads, L.image_tokens, coarse->dim));
    GSA_CUDA(launch_upsample(static_cast<const float*>(coarse->data), coarse->head_stride, coarse->row_stride,
                             coarse->heads, coarse->dim, L, static_cast<float*>(out->data), out->head_stride,
                             out->row_stride, (cudaStream_t)stream));
    return GSA_OK;
}

static int dense_attention(const gsa_tensor* q, const gsa_tensor* k, const gsa_tensor* v, float scale,
                           const gsa_tensor* out, float* lse, int q_row_offset, int out_row_offset,
                           int mq, cudaStream_t st, void* ws = nullptr, size_t ws_bytes = 0,
                           const __half* v16 = nullptr, const unsigned* vmax = nullptr) {
    if (mq == 0) return GSA_OK;
    if (k->rows == 0) return fail(GSA_ERR_SHAPE_MISMATCH, "tiled_attention: empty key set");
    if (tc_dense_supported(*q, *k, *v)) {
        GSA_CUDA(tc_dense_attention(*q, *k, *v, scale, q_row_offset, mq, static_cast<float*>(out->data),
                                    out->head_stride, out->row_stride, out_row_offset, lse, ws, ws_bytes, st, v16,
                                    vmax));
        return GSA_OK;
    }
    if (q->dim == 64 && q->dtype == GSA_DTYPE_F32 && k->dtype == GSA_DTYPE_F32 && v->dtype == GSA_DTYPE_F32) {
        // f32 Q/K/V: the same tensor cores through bf16 hi/lo score splits and fp16 P.V
        GSA_CUDA(tc_dense_f32(*q, q_row_offset, mq, *k, *v, scale,
                              static_cast<float*>(out->data) + (size_t)out_row_offset * out->row_stride,
                              out->head_stride, out->row_stride, lse, ws, ws_bytes, st));
        return GSA_OK;
    }
    GSA_TRY(generic_supported(q->dim, 1));
    AttnArgs a{};
    a.q = ref_of(*q, q_row_offset);
    a.k = ref_of(*k);
    a.v = ref_of(*v);
    a.heads = q->heads;
    a.mq = mq;
    a.mk = k->rows;
    a.dim = q->dim;
    a.scale = scale;
    a.out = static_cast<float*>(out->data) + (size_t)out_row_offset * out->row_stride;
    a.out_hs = out->head_stride;
    a.out_rs = out->row_stride;
    a.lse = lse;
    GSA_CUDA(launch_attn_f32(a, st));
    return GSA_OK;
}

int gsa_tiled_attention(const gsa_tensor* q, const gsa_tensor* k, const gsa_tensor* v, float scale,
                        int bm, int bn, const gsa_tensor* out, float* lse, gsa_stream_t stream) {
    GSA_TRY(check_tensor(q, "q"));
    GSA_TRY(check_tensor(k, "k"));
    GSA_TRY(check_tensor(v, "v"));
    if (k->rows != v->rows) return fail(GSA_ERR_SHAPE_MISMATCH, "tiled_attention: K/V token counts differ");
    GSA_TRY(same_heads_dim(q, k, "tiled_attention"));
    GSA_TRY(same_heads_dim(q, v, "tiled_attention"));
    if (q->dtype != k->dtype || q->dtype != v->dtype)
        return fail(GSA_ERR_UNSUPPORTED, "tiled_attention: q/k/v dtypes differ");
    GSA_TRY(check_tiling(bm, bn));
    GSA_TRY(check_f32_out(out, "out", q->heads, q->rows, q->dim));
    return dense_attention(q, k, v, scale, out, lse, 0, 0, q->rows, (cudaStream_t)stream);
}

int gsa_special_token_attention(const gsa_tensor* q_spec, const gsa_tensor* k, const gsa_tensor* v,
                                float scale, const gsa_tensor* out, float* lse, gsa_stream_t stream) {
    if (q_spec && q_spec->rows == 0) return GSA_OK;  // layer.hpp:88-92
    return gsa_tiled_attention(q_spec, k, v, scale, 16, 16, out, lse, stream);
}

size_t gsa_compressed_attention_topk_workspace_bytes(int heads, int windows, int dim, int k) {
    return tc_compress_workspace_bytes(heads, windows, dim, k);
}

int gsa_compressed_attention_topk(const gsa_tensor* qc, const gsa_tensor* kc, const gsa_tensor* vc, int k,
                                  float scale, int bm, int bn, const uint8_t* excluded, int n_excluded,
                                  const gsa_tensor* out, float* lse, int32_t* indices, float* guide,
                                  int* k_eff_out, void* workspace, size_t ws_bytes, gsa_stream_t stream) {
    GSA_TRY(check_tensor(qc, "qc", false));
    GSA_TRY(check_tensor(kc, "kc", false));
    GSA_TRY(check_tensor(vc, "vc", false));
    // compression.hpp:185-192
    if (kc->rows != vc->rows || qc->rows != kc->rows)
        return fail(GSA_ERR_SHAPE_MISMATCH, "fused_compressed_attention_topk: Q/K/V must share the window count");
    GSA_TRY(same_heads_dim(qc, kc, "fused_compressed_attention_topk"));
    GSA_TRY(same_heads_dim(qc, vc, "fused_compressed_attention_topk"));
    GSA_TRY(check_tiling(bm, bn));
    if (k < 0) return fail(GSA_ERR_GENERIC, "fused_compressed_attention_topk: k must be >= 0");
    if (excluded && n_excluded != kc->rows)
        return fail(GSA_ERR_SHAPE_MISMATCH, "fused_compressed_attention_topk: exclusion mask size");
    GSA_TRY(check_f32_out(out, "out", qc->heads, qc->rows, qc->dim));
    const int W = qc->rows;
    // k_eff needs the number of excluded windows: the mask lives on the device
    int n_ex = 0;
    if (excluded && W > 0) {
        std::string host(W, '\0');
        GSA_CUDA(cudaMemcpyAsync(&host[0], excluded, W, cudaMemcpyDeviceToHost, (cudaStream_t)stream));
        GSA_CUDA(cudaStreamSynchronize((cudaStream_t)stream));
        for (char c : host) n_ex += c ? 1 : 0;
    }
    const int k_eff = k < W - n_ex ? k : W - n_ex;
    if (k_eff_out) *k_eff_out = k_eff;
    if (W == 0) return GSA_OK;
    GSA_TRY(generic_supported(qc->dim, 1));
    if (k_eff > kMaxTopK)
        return fail(GSA_ERR_UNSUPPORTED, "fused_compressed_attention_topk: k_eff=%d > %d (the largest per-row budget the "
                    "sm_100a selection sorts)", k_eff, kMaxTopK);
    GSA_CUDA(tc_compress_topk(*qc, *kc, *vc, k_eff, scale, excluded, static_cast<float*>(out->data),
                              out->head_stride, out->row_stride, lse, indices, guide, workspace, ws_bytes,
                              (cudaStream_t)stream));
    return GSA_OK;
}

int gsa_forced_windows(const gsa_layout* layout, int ref_stride, int32_t* forced, int* count,
                       gsa_stream_t stream) {
    GSA_TRY(check_layout(layout));
    if (ref_stride < 1) return fail(GSA_ERR_INVALID_STRIDE, "forced_frames: ref_stride must be >= 1");
    const DevLayout L = make_dev_layout(*layout);
    int nf = 0;
    selectable_windows(L, 1, ref_stride, &nf);
    if (count) *count = nf;
    if (forced) GSA_CUDA(launch_forced(L, ref_stride, forced, nullptr, (cudaStream_t)stream));
    return GSA_OK;
}

size_t gsa_build_selection_plan_workspace_bytes(int heads, int rows, int k, const gsa_layout* layout,
                                                int ref_stride) {
    (void)k;
    (void)ref_stride;
    const int64_t n = (int64_t)heads * rows;
    const int W = layout ? make_dev_layout(*layout).windows : rows;
    Carver c{nullptr, 0, 0, true};
    c.take<int64_t>(n);
    c.take<int32_t>(W);
    c.take<uint8_t>(W);
    c.take<char>(scan_offsets_tmp_bytes(n));
    c.take<int>(1);
    return c.used + 256;
}

int gsa_build_selection_plan(const int32_t* topk, int heads, int rows, int k, const gsa_layout* layout,
                             int variant, int ref_stride, int64_t* offsets, int32_t* ids,
                             int64_t ids_capacity, int64_t* n_ids, void* workspace, size_t ws_bytes,
                             gsa_stream_t stream) {
    GSA_TRY(check_layout(layout));
    const DevLayout L = make_dev_layout(*layout);
    // selection.cpp:31-32, 41-42
    if (rows != L.windows) return fail(GSA_ERR_SHAPE_MISMATCH, "build_selection_plan: topk rows != num windows");
    if (variant == 1 && ref_stride < 1)
        return fail(GSA_ERR_INVALID_STRIDE, "build_selection_plan: ref_stride must be >= 1 for hybrid");
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t n = (int64_t)heads * rows;
    Carver c{static_cast<char*>(workspace), ws_bytes, 0, false};
    int64_t* sizes = c.take<int64_t>(n);
    int32_t* forced = c.take<int32_t>(L.windows);
    uint8_t* mask = c.take<uint8_t>(L.windows);
    const size_t tmp_bytes = scan_offsets_tmp_bytes(n);
    void* tmp = c.take<char>(tmp_bytes);
    int* flag = c.take<int>(1);
    if (c.used > ws_bytes) return fail(GSA_ERR_WORKSPACE, "build_selection_plan: workspace %zu < %zu", ws_bytes, c.used);
    int nf = 0;
    if (variant == 1) {
        selectable_windows(L, 1, ref_stride, &nf);
        GSA_CUDA(launch_forced(L, ref_stride, forced, mask, st));
    }
    const uint8_t* m = variant == 1 ? mask : nullptr;
    GSA_CUDA(cudaMemsetAsync(flag, 0, sizeof(int), st));
    GSA_CUDA(launch_plan_count(topk, n, k, m, nf, L.windows, sizes, flag, st));
    GSA_CUDA(launch_scan_offsets(sizes, n, offsets, tmp, tmp_bytes, st));
    // the CSR size decides the ids capacity: one host read (the call's documented sync)
    struct { int64_t total; int flag; } hb{0, 0};
    GSA_CUDA(cudaMemcpyAsync(&hb.total, offsets + n, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    GSA_CUDA(cudaMemcpyAsync(&hb.flag, flag, sizeof(int), cudaMemcpyDeviceToHost, st));
    GSA_CUDA(cudaStreamSynchronize(st));
    if (hb.flag & 2)
        return fail(GSA_ERR_INDEX_OUT_OF_RANGE, "build_selection_plan: a top-k window id is outside [0, %d)", L.windows);
    const int64_t total = hb.total;
    if (n_ids) *n_ids = total;
    if (total > ids_capacity)
        return fail(GSA_ERR_WORKSPACE, "build_selection_plan: ids capacity %lld < %lld", (long long)ids_capacity, (long long)total);
    GSA_CUDA(launch_plan_fill(topk, n, k, m, forced, nf, L.windows, offsets, ids, st));
    return GSA_OK;
}

// A caller-supplied plan, validated before any compute (one host read: the documented
// sync of the pinned-plan entry points): EmptySelection for an empty row
// (selection.hpp:82-85), IndexOutOfRange for a window id outside [0, W) (the
// reference's tokens_of_window check, layout.cpp:37-56).
static int validate_plan(const int64_t* offsets, const int32_t* ids, int64_t rows, int W, const char* who,
                         cudaStream_t st) {
    if (!offsets) return fail(GSA_ERR_GENERIC, "%s: null plan offsets", who);
    int* flag = nullptr;
    GSA_CUDA(cudaMallocAsync(&flag, sizeof(int), st));
    GSA_CUDA(cudaMemsetAsync(flag, 0, sizeof(int), st));
    GSA_CUDA(launch_plan_check(offsets, rows, ids, W, flag, st));
    int h = 0;
    GSA_CUDA(cudaMemcpyAsync(&h, flag, sizeof(int), cudaMemcpyDeviceToHost, st));
    GSA_CUDA(cudaFreeAsync(flag, st));
    GSA_CUDA(cudaStreamSynchronize(st));
    if (h & 1) return fail(GSA_ERR_EMPTY_SELECTION, "%s: empty plan row", who);
    if (h & 4) return fail(GSA_ERR_GENERIC, "%s: null plan window ids", who);
    if (h & 2) return fail(GSA_ERR_INDEX_OUT_OF_RANGE, "%s: plan window id outside [0, %d)", who, W);
    return GSA_OK;
}

static int select_checks(const gsa_tensor* q, const gsa_tensor* k, const gsa_tensor* v, const DevLayout& L) {
    GSA_TRY(check_tensor(q, "q_img"));
    GSA_TRY(check_tensor(k, "k_img"));
    GSA_TRY(check_tensor(v, "v_img"));
    // selection.hpp:68-76
    if (q->rows != L.image_tokens) return fail(GSA_ERR_SHAPE_MISMATCH, "block_sparse_attention: Q rows != image tokens");
    if (k->rows != L.image_tokens || v->rows != L.image_tokens)
        return fail(GSA_ERR_SHAPE_MISMATCH, "block_sparse_attention: K/V rows != image tokens");
    GSA_TRY(same_heads_dim(q, k, "block_sparse_attention"));
    GSA_TRY(same_heads_dim(q, v, "block_sparse_attention"));
    if (q->dtype != k->dtype || q->dtype != v->dtype)
        return fail(GSA_ERR_UNSUPPORTED, "block_sparse_attention: q/k/v dtypes differ");
    return GSA_OK;
}

// The selection branch (block_sparse_attention, selection.hpp:63-136; with the gate and
// the gated merge fused when a.w_g is set). The tensor-core kernel's window geometry
// (d = 64, s = 4) takes every dtype: bf16 rows are TMA-gathered where they lie; f32 rows
// (and bf16 views whose strides a tensor map cannot express) are first packed into
// contiguous bf16 hi(/lo) planes allocated stream-ordered (no host sync), and the kernel
// runs 3-term products on them. Geometries outside that tile (s in {1, 2, 8}, d != 64),
// which the reference API also accepts, run the exact CUDA-core kernel.
static bool tma_rows_ok(const TensorRef& t) {
    return t.dtype == GSA_DTYPE_BF16 && t.rs >= 64 && t.rs % 8 == 0 && t.hs % 8 == 0 &&
           (reinterpret_cast<uintptr_t>(t.data) & 15) == 0;
}

static int run_select(SelectArgs a, cudaStream_t st) {
    if (!(a.dim == 64 && a.L.s == 4 && a.Lkv.s == 4)) {
        GSA_CUDA(launch_select_f32(a, st));
        return GSA_OK;
    }
    const bool f32 = a.q.dtype == GSA_DTYPE_F32;
    const bool pack_qk = f32 || !tma_rows_ok(a.q) || !tma_rows_ok(a.k);
    const bool make_v = a.v16.data == nullptr;
    const int rq = a.L.image_tokens, rkv = a.Lkv.image_tokens, H = a.heads;
    const size_t plane_q = (size_t)H * rq * 64, plane_kv = (size_t)H * rkv * 64, planes = f32 ? 2 : 1;
    size_t bytes = 0;
    if (pack_qk) bytes += (plane_q + plane_kv) * planes * 2;
    if (make_v) bytes += plane_kv * planes * 2 + 256;
    void* mem = nullptr;
    if (bytes) {
        GSA_CUDA(cudaMallocAsync(&mem, bytes, st));
        char* cur = static_cast<char*>(mem);
        auto take = [&](size_t elems) {
            void* r = cur;
            cur += elems * 2;
            return r;
        };
        auto plane = [](const void* p, int rows, int dt) { return TensorRef{p, dt, (int64_t)rows * 64, 64}; };
        if (pack_qk) {
            auto* hq = static_cast<__nv_bfloat16*>(take(plane_q));
            auto* hk = static_cast<__nv_bfloat16*>(take(plane_kv));
            auto* lq = f32 ? static_cast<__nv_bfloat16*>(take(plane_q)) : nullptr;
            auto* lk = f32 ? static_cast<__nv_bfloat16*>(take(plane_kv)) : nullptr;
            GSA_CUDA(launch_pack_rows(a.q, H, rq, hq, lq, st));
            GSA_CUDA(launch_pack_rows(a.k, H, rkv, hk, lk, st));
            a.q = plane(hq, rq, GSA_DTYPE_BF16);
            a.k = plane(hk, rkv, GSA_DTYPE_BF16);
            if (f32) {
                a.ql = plane(lq, rq, GSA_DTYPE_BF16);
                a.kl = plane(lk, rkv, GSA_DTYPE_BF16);
            }
        }
        if (make_v) {
            auto* hv = static_cast<__half*>(take(plane_kv));
            auto* lv = f32 ? static_cast<__half*>(take(plane_kv)) : nullptr;
            auto* vmax = reinterpret_cast<unsigned*>(cur);
            GSA_CUDA(launch_v16(a.v, H, rkv, vmax, hv, lv, st));
            a.v16 = plane(hv, rkv, kDtypeF16);
            if (f32) a.v16l = plane(lv, rkv, kDtypeF16);
            a.vmax = vmax;
        }
    }
    const cudaError_t e = tc_select(a, st);
    if (mem) cudaFreeAsync(mem, st);
    if (e == cudaErrorNotSupported)
        return fail(GSA_ERR_UNSUPPORTED, "block_sparse_attention: tensor-core selection rejected the operands");
    GSA_CUDA(e);
    return GSA_OK;
}

int gsa_block_sparse_attention(const gsa_tensor* q, const gsa_tensor* k, const gsa_tensor* v,
                               const int64_t* offsets, const int32_t* ids, const gsa_layout* layout,
                               float scale, const gsa_tensor* out, float* lse, gsa_stream_t stream) {
    GSA_TRY(check_layout(layout));
    const DevLayout L = make_dev_layout(*layout);
    GSA_TRY(select_checks(q, k, v, L));
    GSA_TRY(check_f32_out(out, "out", q->heads, L.image_tokens, q->dim));
    GSA_TRY(generic_supported(q->dim, L.s));
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t n = (int64_t)q->heads * L.windows;
    if (n == 0) return GSA_OK;
    GSA_TRY(validate_plan(offsets, ids, n, L.windows, "block_sparse_attention", st));
    SelectArgs a{};
    a.q = ref_of(*q);
    a.k = ref_of(*k);
    a.v = ref_of(*v);
    a.heads = q->heads;
    a.dim = q->dim;
    a.L = L;
    a.Lkv = L;
    a.rows = RowSource{offsets, ids, nullptr, 0, nullptr, 0, 0};
    a.scale = scale;
    a.out = static_cast<float*>(out->data);
    a.out_hs = out->head_stride;
    a.out_rs = out->row_stride;
    a.lse = lse;
    return run_select(a, st);
}

int gsa_gate(const gsa_tensor* q, const gsa_tensor* w_g, const gsa_tensor* g, gsa_stream_t stream) {
    GSA_TRY(check_tensor(q, "q_img"));
    GSA_TRY(check_tensor(w_g, "w_g", false));
    // layer.hpp:101-102
    if (w_g->heads != q->heads || w_g->rows != q->dim || w_g->dim != q->dim)
        return fail(GSA_ERR_SHAPE_MISMATCH, "gate: weights must be heads x dim x dim");
    if (w_g->row_stride != w_g->dim || w_g->head_stride != (int64_t)w_g->dim * w_g->dim)
        return fail(GSA_ERR_UNSUPPORTED, "gate: w_g must be contiguous");
    GSA_TRY(check_f32_out(g, "g", q->heads, q->rows, q->dim));
    GSA_CUDA(launch_gate(ref_of(*q), q->heads, q->rows, q->dim, static_cast<const float*>(w_g->data),
                         static_cast<float*>(g->data), g->head_stride, g->row_stride, (cudaStream_t)stream));
    return GSA_OK;
}

// ------------------------------------------------------------ full layer

namespace {

struct LayerPlan {
    DevLayout L;
    int heads, dim, Ms, Mi, M, W, k_eff, n_forced;
    float scale;
};

// with_plan: gsa_forward_with_plan (layer.hpp:235-262) validates the params but neither
// checks params.window_s against the layout nor runs a top-k (so no budget limit)
int layer_checks(const gsa_tensor* q, const gsa_tensor* k, const gsa_tensor* v, const gsa_tensor* w_g,
                 const gsa_layout* layout, const gsa_params* p, const gsa_tensor* out, LayerPlan* lp,
                 bool with_plan = false) {
    GSA_TRY(check_layout(layout));
    GSA_TRY(gsa_validate_params(p, with_plan ? nullptr : layout));
    GSA_TRY(check_tensor(q, "q"));
    GSA_TRY(check_tensor(k, "k"));
    GSA_TRY(check_tensor(v, "v"));
    GSA_TRY(check_tensor(w_g, "w_g", false));
    const DevLayout L = make_dev_layout(*layout);
    const int M = layout->num_special + L.image_tokens;
    // partition_qkv (layout.hpp:58-60) / layer.hpp:184-185
    if (q->rows != M || k->rows != M || v->rows != M)
        return fail(GSA_ERR_SHAPE_MISMATCH, "gsa_forward: Q/K/V rows != layout.total_tokens()");
    GSA_TRY(same_heads_dim(q, k, "partition_qkv"));
    GSA_TRY(same_heads_dim(q, v, "partition_qkv"));
    if (q->dtype != k->dtype || q->dtype != v->dtype)
        return fail(GSA_ERR_UNSUPPORTED, "gsa_forward: q/k/v dtypes differ");
    if (w_g->heads != q->heads || w_g->rows != q->dim || w_g->dim != q->dim)
        return fail(GSA_ERR_SHAPE_MISMATCH, "weights: w_g must be heads x dim x dim");
    if (w_g->row_stride != w_g->dim || w_g->head_stride != (int64_t)w_g->dim * w_g->dim)
        return fail(GSA_ERR_UNSUPPORTED, "gsa_forward: w_g must be contiguous");
    GSA_TRY(check_f32_out(out, "out", q->heads, M, q->dim));
    GSA_TRY(generic_supported(q->dim, L.s));
    lp->L = L;
    lp->heads = q->heads;
    lp->dim = q->dim;
    lp->Ms = layout->num_special;
    lp->Mi = L.image_tokens;
    lp->M = M;
    lp->W = L.windows;
    const int sel = selectable_windows(L, p->variant, p->ref_stride, &lp->n_forced);
    lp->k_eff = p->top_k < sel ? p->top_k : sel;
    lp->scale = resolved_scale(p->scale, q->dim);
    if (with_plan) {
        lp->k_eff = 0;  // no top-k on the pinned-plan path
        lp->n_forced = 0;
    } else if (lp->k_eff > kMaxTopK) {
        return fail(GSA_ERR_UNSUPPORTED, "gsa_forward: k_eff=%d > %d (the largest per-row budget the sm_100a "
                    "selection sorts)", lp->k_eff, kMaxTopK);
    }
    return GSA_OK;
}

struct LayerBufs {
    float *qc, *kc, *vc, *o_comp, *lse_comp, *lse_spec;
    // hybrid fast path: reference-frame K/V rows gathered contiguously, their dense
    // softmax (normalised output + LSE per image token) and the dense pass's workspace
    __nv_bfloat16 *kf, *vf;
    float *prior_o, *prior_lse;
    void* fa_ws;
    size_t fa_ws_bytes;
    int32_t *topk, *forced;
    uint8_t* mask;
    void* compress_ws;
    size_t compress_ws_bytes;
    uint8_t* wg_prep;
    void* dense_ws;
    size_t dense_ws_bytes;
    // V of all M rows as fp16 planes (the P.V operand of the special and selection kernels)
    __half* v16;
    unsigned* vmax;
};

size_t carve(const LayerPlan& lp, const gsa_context* ctx, char* base, size_t cap, bool dry, LayerBufs* b) {
    Carver c{base, cap, 0, dry};
    const size_t wd = (size_t)lp.heads * lp.W * lp.dim;
    auto f = [&](float* user, size_t n) { return user ? user : c.take<float>(n); };
    b->qc = f(ctx ? ctx->qc : nullptr, wd);
    b->kc = f(ctx ? ctx->kc : nullptr, wd);
    b->vc = f(ctx ? ctx->vc : nullptr, wd);
    b->o_comp = f(ctx ? ctx->o_comp : nullptr, wd);
    b->lse_comp = f(ctx ? ctx->lse_comp : nullptr, (size_t)lp.heads * lp.W);
    b->lse_spec = f(ctx ? ctx->lse_spec : nullptr, (size_t)lp.heads * lp.Ms);
    b->topk = (ctx && ctx->topk) ? ctx->topk : c.take<int32_t>((size_t)lp.heads * lp.W * lp.k_eff);
    b->forced = c.take<int32_t>(lp.W);
    b->mask = c.take<uint8_t>(lp.W);
    b->compress_ws_bytes = tc_compress_workspace_bytes(lp.heads, lp.W, lp.dim, lp.k_eff);
    b->compress_ws = c.take<char>(b->compress_ws_bytes);
    b->wg_prep = c.take<uint8_t>(tc_select_workspace_bytes(lp.heads));
    b->dense_ws_bytes = tc_dense_workspace_bytes(lp.heads, lp.Ms, lp.Ms + lp.Mi, false);
    b->dense_ws = c.take<char>(b->dense_ws_bytes);
    b->v16 = c.take<__half>((size_t)lp.heads * (lp.Ms + lp.Mi) * lp.dim);
    b->vmax = c.take<unsigned>((size_t)lp.heads);
    b->kf = b->vf = nullptr;
    b->prior_o = b->prior_lse = nullptr;
    b->fa_ws = nullptr;
    b->fa_ws_bytes = 0;
    if (lp.n_forced > 0) {  // sized whenever the plan is hybrid; used only on the tensor-core path
        const int fk = lp.n_forced / lp.L.wins_per_frame * lp.L.tokens_per_frame;  // reference-frame keys
        b->kf = c.take<__nv_bfloat16>((size_t)lp.heads * fk * lp.dim);
        b->vf = c.take<__nv_bfloat16>((size_t)lp.heads * fk * lp.dim);
        b->prior_o = c.take<float>((size_t)lp.heads * lp.Mi * lp.dim);
        b->prior_lse = c.take<float>((size_t)lp.heads * lp.Mi);
        b->fa_ws_bytes = tc_dense_workspace_bytes(lp.heads, lp.Mi, fk);
        b->fa_ws = c.take<char>(b->fa_ws_bytes);
    }
    return c.used + 256;
}


// Hybrid fast path (selection.cpp:55-59: the forced windows lead every plan row, i.e.
// every query attends ALL reference-frame keys). That part of each softmax is a dense
// attention of the queries over the reference frames' keys: one tcgen05 FA pass over a
// contiguous copy of those rows instead of gathering the same windows once per query
// window. The selection epilogue merges it with the dynamic top-k windows' partial
// softmax by log-sum-exp (identical to one softmax over forced ++ top-k up to f32
// rounding). q rows [q_row0, q_row0 + mq) are image queries; k/v image rows start at
// kv_img_row0; kf/vf [H][fk][64] bf16, prior_o [H][mq][64] f32, prior_lse [H][mq].
int hybrid_prior(const gsa_tensor* q, int q_row0, int mq, const gsa_tensor* k, const gsa_tensor* v, int kv_img_row0,
                 const DevLayout& L, int ref_stride, int n_forced, float scale, int H, __nv_bfloat16* kf,
                 __nv_bfloat16* vf, float* prior_o, float* prior_lse, void* fa_ws, size_t fa_ws_bytes, cudaStream_t st) {
    const int tpf = L.tokens_per_frame, nff = n_forced / L.wins_per_frame, fk = nff * tpf;
    for (int fi = 0; fi < nff; ++fi) {
        const int f = fi * ref_stride;  // forced frames 0, r, 2r, ... (selection.cpp:7-12)
        const size_t src_row = (size_t)kv_img_row0 + (size_t)f * tpf;
        for (int kv = 0; kv < 2; ++kv) {
            const gsa_tensor* t = kv ? v : k;
            __nv_bfloat16* dst = (kv ? vf : kf) + (size_t)fi * tpf * 64;
            const __nv_bfloat16* src = static_cast<const __nv_bfloat16*>(t->data) + src_row * t->row_stride;
            if (t->row_stride == 64) {  // contiguous rows: one 2-D copy over heads
                GSA_CUDA(cudaMemcpy2DAsync(dst, (size_t)fk * 64 * 2, src, (size_t)t->head_stride * 2,
                                           (size_t)tpf * 64 * 2, H, cudaMemcpyDeviceToDevice, st));
            } else {  // strided rows (e.g. views of a fused QKV projection): one 2-D copy per head
                for (int hh = 0; hh < H; ++hh)
                    GSA_CUDA(cudaMemcpy2DAsync(dst + (size_t)hh * fk * 64, 64 * 2, src + (size_t)hh * t->head_stride,
                                               (size_t)t->row_stride * 2, 64 * 2, tpf, cudaMemcpyDeviceToDevice, st));
            }
        }
    }
    gsa_tensor tkf{kf, GSA_DTYPE_BF16, H, fk, 64, (int64_t)fk * 64, 64};
    gsa_tensor tvf{vf, GSA_DTYPE_BF16, H, fk, 64, (int64_t)fk * 64, 64};
    gsa_tensor tpo{prior_o, GSA_DTYPE_F32, H, mq, 64, (int64_t)mq * 64, 64};
    return dense_attention(q, &tkf, &tvf, scale, &tpo, prior_lse, q_row0, 0, mq, st, fa_ws, fa_ws_bytes);
}
}  // namespace

size_t gsa_forward_workspace_bytes(const gsa_layout* layout, const gsa_params* params, int heads, int dim) {
    if (!layout || !params) return 0;
    LayerPlan lp{};
    lp.L = make_dev_layout(*layout);
    lp.heads = heads;
    lp.dim = dim;
    lp.Ms = layout->num_special;
    lp.Mi = lp.L.image_tokens;
    lp.W = lp.L.windows;
    int nf = 0;
    const int sel = selectable_windows(lp.L, params->variant, params->ref_stride > 0 ? params->ref_stride : 1, &nf);
    lp.n_forced = nf;
    lp.k_eff = params->top_k < sel ? params->top_k : sel;
    if (lp.k_eff < 0) lp.k_eff = 0;
    LayerBufs b;
    return carve(lp, nullptr, nullptr, 0, true, &b);
}

int gsa_forward(const gsa_tensor* q, const gsa_tensor* k, const gsa_tensor* v, const gsa_tensor* w_g,
                const gsa_layout* layout, const gsa_params* params, const gsa_tensor* out,
                const gsa_context* ctx, int* k_eff_out, void* workspace, size_t ws_bytes,
                gsa_stream_t stream) {
    LayerPlan lp;
    GSA_TRY(layer_checks(q, k, v, w_g, layout, params, out, &lp));
    if (k_eff_out) *k_eff_out = lp.k_eff;
    cudaStream_t st = (cudaStream_t)stream;
    LayerBufs b;
    const size_t need = carve(lp, ctx, static_cast<char*>(workspace), ws_bytes, false, &b);
    if (need > ws_bytes + 256 || (!workspace && need > 256))
        return fail(GSA_ERR_WORKSPACE, "gsa_forward: workspace %zu < %zu bytes", ws_bytes, need);
    const int H = lp.heads, d = lp.dim;
    float* outp = static_cast<float*>(out->data);

    // 1. special tokens: dense attention over all M keys (layer.hpp:201-202). bf16 inputs:
    // V is converted once to the fp16 P.V operand shared with the selection kernel
    stage_mark(0, st);
    const bool v16_made = q->dtype == GSA_DTYPE_BF16 && d == 64 && lp.L.s == 4 && tc_dense_supported(*q, *k, *v);
    if (v16_made) GSA_CUDA(launch_v16(ref_of(*v), H, lp.M, b.vmax, b.v16, nullptr, st));
    GSA_TRY(dense_attention(q, k, v, lp.scale, out, b.lse_spec, 0, 0, lp.Ms, st, b.dense_ws, b.dense_ws_bytes,
                            v16_made ? b.v16 : nullptr, v16_made ? b.vmax : nullptr));
    stage_mark(1, st);

    // 2. pool Q/K/V image rows (layer.hpp:204-206); on the tensor-core path the
    // same pass also writes Qc's bf16 hi/lo operands and row norms K2 consumes
    CompressSplits sp{};
    const bool have_sp = tc_compress_split_buffers(b.compress_ws, b.compress_ws_bytes, H, lp.W, d, lp.k_eff, &sp);
    PoolJob jobs[3] = {  // K and V get their tensor-core operands in K2 (centred K splits, fp16 V)
        {ref_of(*q, lp.Ms), b.qc, sp.qh, sp.ql, sp.qnorm},
        {ref_of(*k, lp.Ms), b.kc, nullptr, nullptr, nullptr},
        {ref_of(*v, lp.Ms), b.vc, nullptr, nullptr, nullptr},
    };
    GSA_CUDA(launch_pool(jobs, 3, H, d, lp.L, 1.0f / (float)(lp.L.s * lp.L.s), st));
    stage_mark(2, st);

    // 3. hybrid exclusion mask + forced list (layer.hpp:208-210)
    const uint8_t* excluded = nullptr;
    if (params->variant == 1) {
        GSA_CUDA(launch_forced(lp.L, params->ref_stride, b.forced, b.mask, st));
        excluded = b.mask;
    }

    // 4. compressed attention + streaming top-k (layer.hpp:211-216)
    gsa_tensor tq{b.qc, GSA_DTYPE_F32, H, lp.W, d, (int64_t)lp.W * d, d};
    gsa_tensor tk{b.kc, GSA_DTYPE_F32, H, lp.W, d, (int64_t)lp.W * d, d};
    gsa_tensor tv{b.vc, GSA_DTYPE_F32, H, lp.W, d, (int64_t)lp.W * d, d};
    GSA_CUDA(tc_compress_topk_splits(have_sp ? &sp : nullptr, tq, tk, tv, lp.k_eff, lp.scale, excluded, b.o_comp,
                                     (int64_t)lp.W * d, d, b.lse_comp, b.topk, nullptr, b.compress_ws,
                                     b.compress_ws_bytes, st));
    stage_mark(3, st);

    // 5-7. plan rows = forced ++ top-k (selection.cpp:55-59; the top-k already
    // excludes forced windows so no dedup is needed), block-sparse attention,
    // gate and gated merge fused; output rows [Ms, M) (layer.hpp:218-228)
    SelectArgs a{};
    a.q = ref_of(*q, lp.Ms);
    a.k = ref_of(*k, lp.Ms);
    a.v = ref_of(*v, lp.Ms);
    a.heads = H;
    a.dim = d;
    a.L = lp.L;
    a.Lkv = lp.L;
    a.rows = RowSource{nullptr, nullptr, b.forced, params->variant == 1 ? lp.n_forced : 0, b.topk, lp.k_eff, lp.k_eff};
    a.scale = lp.scale;
    a.out = outp + (size_t)lp.Ms * out->row_stride;
    a.out_hs = out->head_stride;
    a.out_rs = out->row_stride;
    a.lse = ctx ? ctx->lse_sel : nullptr;
    a.w_g = static_cast<const float*>(w_g->data);
    a.o_comp = b.o_comp;
    a.o_sel_ctx = ctx ? ctx->o_sel : nullptr;
    a.gate_ctx = ctx ? ctx->gate : nullptr;
    a.wg_prep = b.wg_prep;
    if (v16_made) {
        a.v16 = TensorRef{b.v16 + (size_t)lp.Ms * 64, kDtypeF16, (int64_t)lp.M * 64, 64};
        a.vmax = b.vmax;
    }
    const bool tc_sel = tc_select_supported(a);
    if (tc_sel && params->variant == 1 && lp.n_forced > 0 && lp.k_eff > 0 && b.kf && q->dim == 64 &&
        tc_dense_supported(*q, *k, *v)) {
        GSA_TRY(hybrid_prior(q, lp.Ms, lp.Mi, k, v, lp.Ms, lp.L, params->ref_stride, lp.n_forced, lp.scale, H, b.kf,
                             b.vf, b.prior_o, b.prior_lse, b.fa_ws, b.fa_ws_bytes, st));
        a.rows = RowSource{nullptr, nullptr, b.forced, 0, b.topk, lp.k_eff, lp.k_eff};
        a.prior_o = b.prior_o;
        a.prior_lse = b.prior_lse;
    }
    GSA_TRY(run_select(a, st));
    stage_mark(4, st);
    return GSA_OK;
}

int gsa_forward_with_plan(const gsa_tensor* q, const gsa_tensor* k, const gsa_tensor* v, const gsa_tensor* w_g,
                          const gsa_layout* layout, const gsa_params* params, const int64_t* offsets,
                          const int32_t* ids, const gsa_tensor* out, void* workspace, size_t ws_bytes,
                          gsa_stream_t stream) {
    LayerPlan lp;
    GSA_TRY(layer_checks(q, k, v, w_g, layout, params, out, &lp, true));
    cudaStream_t st = (cudaStream_t)stream;
    LayerBufs b;
    const size_t need = carve(lp, nullptr, static_cast<char*>(workspace), ws_bytes, false, &b);
    if (need > ws_bytes + 256) return fail(GSA_ERR_WORKSPACE, "gsa_forward_with_plan: workspace %zu < %zu", ws_bytes, need);
    const int H = lp.heads, d = lp.dim;
    GSA_TRY(validate_plan(offsets, ids, (int64_t)H * lp.W, lp.W, "gsa_forward_with_plan", st));
    GSA_TRY(dense_attention(q, k, v, lp.scale, out, b.lse_spec, 0, 0, lp.Ms, st));
    PoolJob jobs[3] = {
        {ref_of(*q, lp.Ms), b.qc, nullptr, nullptr, nullptr},
        {ref_of(*k, lp.Ms), b.kc, nullptr, nullptr, nullptr},
        {ref_of(*v, lp.Ms), b.vc, nullptr, nullptr, nullptr},
    };
    GSA_CUDA(launch_pool(jobs, 3, H, d, lp.L, 1.0f / (float)(lp.L.s * lp.L.s), st));
    // compressed branch without top-k (layer.hpp:251-253: tiled_attention)
    gsa_tensor tq{b.qc, GSA_DTYPE_F32, H, lp.W, d, (int64_t)lp.W * d, d};
    gsa_tensor tk{b.kc, GSA_DTYPE_F32, H, lp.W, d, (int64_t)lp.W * d, d};
    gsa_tensor tv{b.vc, GSA_DTYPE_F32, H, lp.W, d, (int64_t)lp.W * d, d};
    gsa_tensor to{b.o_comp, GSA_DTYPE_F32, H, lp.W, d, (int64_t)lp.W * d, d};
    GSA_TRY(dense_attention(&tq, &tk, &tv, lp.scale, &to, b.lse_comp, 0, 0, lp.W, st));
    SelectArgs a{};
    a.q = ref_of(*q, lp.Ms);
    a.k = ref_of(*k, lp.Ms);
    a.v = ref_of(*v, lp.Ms);
    a.heads = H;
    a.dim = d;
    a.L = lp.L;
    a.Lkv = lp.L;
    a.rows = RowSource{offsets, ids, nullptr, 0, nullptr, 0, 0};
    a.scale = lp.scale;
    a.out = static_cast<float*>(out->data) + (size_t)lp.Ms * out->row_stride;
    a.out_hs = out->head_stride;
    a.out_rs = out->row_stride;
    a.w_g = static_cast<const float*>(w_g->data);
    a.o_comp = b.o_comp;
    a.wg_prep = b.wg_prep;
    return run_select(a, st);
}

// ------------------------------------------------------- view-sharded layer
// One rank of a layer partitioned by query views: the
// rank owns frames [frame_begin, frame_end) and special rows [special_begin,
// special_end). K/V (all M rows) and Kc/Vc (all W windows) are completed by
// all-gathers between the three calls; window ids stay global throughout.

namespace {

struct ShardPlan {
    LayerPlan g;         // the global layer
    DevLayout Lq;        // the shard's own frames (no specials)
    int Ms_g, Mi_g, W_g, w_begin;
};

int shard_checks(const gsa_layout* layout, const gsa_params* p, const gsa_shard* sh, int heads, int dim,
                 ShardPlan* sp) {
    GSA_TRY(check_layout(layout));
    GSA_TRY(gsa_validate_params(p, layout));
    if (!sh) return fail(GSA_ERR_GENERIC, "null shard");
    if (sh->frame_begin < 0 || sh->frame_end > layout->num_frames || sh->frame_begin > sh->frame_end ||
        sh->special_begin < 0 || sh->special_end > layout->num_special || sh->special_begin > sh->special_end)
        return fail(GSA_ERR_INDEX_OUT_OF_RANGE, "shard ranges outside the layout");
    GSA_TRY(generic_supported(dim, layout->window_s));
    const DevLayout L = make_dev_layout(*layout);
    LayerPlan& lp = sp->g;
    lp.L = L;
    lp.heads = heads;
    lp.dim = dim;
    lp.Ms = layout->num_special;
    lp.Mi = L.image_tokens;
    lp.M = lp.Ms + lp.Mi;
    lp.W = L.windows;
    const int sel = selectable_windows(L, p->variant, p->ref_stride, &lp.n_forced);
    lp.k_eff = p->top_k < sel ? p->top_k : sel;
    lp.scale = resolved_scale(p->scale, dim);
    if (lp.k_eff > kMaxTopK)
        return fail(GSA_ERR_UNSUPPORTED, "k_eff=%d > %d (the largest per-row budget the sm_100a selection sorts)",
                    lp.k_eff, kMaxTopK);
    gsa_layout lq{0, sh->frame_end - sh->frame_begin, layout->grid_h, layout->grid_w, layout->window_s};
    if (lq.num_frames == 0) lq.num_frames = 1;  // placeholder geometry; an empty shard does no work
    sp->Lq = make_dev_layout(lq);
    sp->Ms_g = sh->special_end - sh->special_begin;
    sp->Mi_g = (sh->frame_end - sh->frame_begin) * L.tokens_per_frame;
    sp->W_g = (sh->frame_end - sh->frame_begin) * L.wins_per_frame;
    sp->w_begin = sh->frame_begin * L.wins_per_frame;
    return GSA_OK;
}

int check_shape(const gsa_tensor* t, const char* name, int heads, int rows, int dim, bool bf16_ok) {
    GSA_TRY(check_tensor(t, name, bf16_ok));
    if (t->heads != heads || t->rows != rows || t->dim != dim)
        return fail(GSA_ERR_SHAPE_MISMATCH, "%s: expected [%d x %d x %d], got [%d x %d x %d]", name, heads, rows, dim,
                    t->heads, t->rows, t->dim);
    return GSA_OK;
}

int contiguous_f32_windows(const gsa_tensor* t, const char* name) {
    if (t->dtype != GSA_DTYPE_F32 || t->row_stride != t->dim || t->head_stride != (int64_t)t->rows * t->dim)
        return fail(GSA_ERR_UNSUPPORTED, "%s must be contiguous f32 [H][rows][d]", name);
    return GSA_OK;
}

struct ShardBufs {
    int32_t *forced;
    uint8_t* mask;
    void* compress_ws;
    size_t compress_ws_bytes;
    uint8_t* wg_prep;
    void* dense_ws;
    size_t dense_ws_bytes;
    float* lse_spec;
    __half* v16;  // V of all M rows as fp16 planes (P.V operand of the special + selection kernels)
    unsigned* vmax;
    // hybrid fast path (hybrid_prior): reference-frame K/V copies, their dense softmax
    __nv_bfloat16 *kf, *vf;
    float *prior_o, *prior_lse;
    void* fa_ws;
    size_t fa_ws_bytes;
};

size_t shard_carve(const ShardPlan& sp, char* base, bool dry, ShardBufs* b) {
    Carver c{base, 0, 0, dry};
    const LayerPlan& g = sp.g;
    b->forced = c.take<int32_t>(g.W);
    b->mask = c.take<uint8_t>(g.W);
    b->compress_ws_bytes = tc_compress_workspace_bytes_qk(g.heads, sp.W_g, g.W, g.dim, g.k_eff);
    b->compress_ws = c.take<char>(b->compress_ws_bytes);
    b->wg_prep = c.take<uint8_t>(tc_select_workspace_bytes(g.heads));
    b->dense_ws_bytes = tc_dense_workspace_bytes(g.heads, sp.Ms_g, g.M, false);
    b->dense_ws = c.take<char>(b->dense_ws_bytes);
    b->lse_spec = c.take<float>((size_t)g.heads * sp.Ms_g);
    b->v16 = c.take<__half>((size_t)g.heads * g.M * g.dim);
    b->vmax = c.take<unsigned>((size_t)g.heads);
    b->kf = b->vf = nullptr;
    b->prior_o = b->prior_lse = nullptr;
    b->fa_ws = nullptr;
    b->fa_ws_bytes = 0;
    if (g.n_forced > 0 && sp.Mi_g > 0) {
        const int fk = g.n_forced / g.L.wins_per_frame * g.L.tokens_per_frame;  // reference-frame keys
        b->kf = c.take<__nv_bfloat16>((size_t)g.heads * fk * g.dim);
        b->vf = c.take<__nv_bfloat16>((size_t)g.heads * fk * g.dim);
        b->prior_o = c.take<float>((size_t)g.heads * sp.Mi_g * g.dim);
        b->prior_lse = c.take<float>((size_t)g.heads * sp.Mi_g);
        b->fa_ws_bytes = tc_dense_workspace_bytes(g.heads, sp.Mi_g, fk);
        b->fa_ws = c.take<char>(b->fa_ws_bytes);
    }
    return c.used + 256;
}

}  // namespace

size_t gsa_shard_workspace_bytes(const gsa_layout* layout, const gsa_params* params, const gsa_shard* shard,
                                 int heads, int dim) {
    ShardPlan sp;
    if (shard_checks(layout, params, shard, heads, dim, &sp) != GSA_OK) return 0;
    ShardBufs b;
    return shard_carve(sp, nullptr, true, &b);
}

int gsa_shard_pool(const gsa_tensor* q_own, const gsa_tensor* k_all, const gsa_tensor* v_all,
                   const gsa_layout* layout, const gsa_params* params, const gsa_shard* shard,
                   const gsa_tensor* qc_own, const gsa_tensor* kc_all, const gsa_tensor* vc_all,
                   gsa_stream_t stream) {
    GSA_TRY(check_tensor(q_own, "q_own"));
    ShardPlan sp;
    GSA_TRY(shard_checks(layout, params, shard, q_own->heads, q_own->dim, &sp));
    const LayerPlan& g = sp.g;
    const int H = g.heads, d = g.dim;
    GSA_TRY(check_shape(q_own, "q_own", H, sp.Ms_g + sp.Mi_g, d, true));
    GSA_TRY(check_shape(k_all, "k_all", H, g.M, d, true));
    GSA_TRY(check_shape(v_all, "v_all", H, g.M, d, true));
    if (k_all->dtype != q_own->dtype || v_all->dtype != q_own->dtype)
        return fail(GSA_ERR_UNSUPPORTED, "shard_pool: q/k/v dtypes differ");
    GSA_TRY(check_shape(qc_own, "qc_own", H, sp.W_g, d, false));
    GSA_TRY(check_shape(kc_all, "kc_all", H, g.W, d, false));
    GSA_TRY(check_shape(vc_all, "vc_all", H, g.W, d, false));
    GSA_TRY(contiguous_f32_windows(qc_own, "qc_own"));
    GSA_TRY(contiguous_f32_windows(kc_all, "kc_all"));
    GSA_TRY(contiguous_f32_windows(vc_all, "vc_all"));
    if (sp.W_g == 0) return GSA_OK;
    const int own_img = g.Ms + shard->frame_begin * g.L.tokens_per_frame;  // first own image row of k_all
    const int64_t wofs = (int64_t)sp.w_begin * d;
    PoolJob jobs[3] = {
        {ref_of(*q_own, sp.Ms_g), static_cast<float*>(qc_own->data), nullptr, nullptr, nullptr, 0},
        {ref_of(*k_all, own_img), static_cast<float*>(kc_all->data) + wofs, nullptr, nullptr, nullptr, (int64_t)g.W * d},
        {ref_of(*v_all, own_img), static_cast<float*>(vc_all->data) + wofs, nullptr, nullptr, nullptr, (int64_t)g.W * d},
    };
    GSA_CUDA(launch_pool(jobs, 3, H, d, sp.Lq, 1.0f / (float)(g.L.s * g.L.s), (cudaStream_t)stream));
    return GSA_OK;
}

int gsa_shard_compress(const gsa_tensor* qc_own, const gsa_tensor* kc_all, const gsa_tensor* vc_all,
                       const gsa_layout* layout, const gsa_params* params, const gsa_shard* shard,
                       const gsa_tensor* o_comp_own, float* lse_own, int32_t* topk_own, int* k_eff_out,
                       void* workspace, size_t ws_bytes, gsa_stream_t stream) {
    GSA_TRY(check_tensor(qc_own, "qc_own", false));
    ShardPlan sp;
    GSA_TRY(shard_checks(layout, params, shard, qc_own->heads, qc_own->dim, &sp));
    const LayerPlan& g = sp.g;
    const int H = g.heads, d = g.dim;
    if (k_eff_out) *k_eff_out = g.k_eff;
    GSA_TRY(check_shape(qc_own, "qc_own", H, sp.W_g, d, false));
    GSA_TRY(check_shape(kc_all, "kc_all", H, g.W, d, false));
    GSA_TRY(check_shape(vc_all, "vc_all", H, g.W, d, false));
    GSA_TRY(check_shape(o_comp_own, "o_comp_own", H, sp.W_g, d, false));
    ShardBufs b;
    const size_t need = shard_carve(sp, static_cast<char*>(workspace), workspace == nullptr, &b);
    if (!workspace || need > ws_bytes + 256)
        return fail(GSA_ERR_WORKSPACE, "shard_compress: workspace %zu < %zu bytes", ws_bytes, need);
    if (sp.W_g == 0) return GSA_OK;
    cudaStream_t st = (cudaStream_t)stream;
    const uint8_t* excluded = nullptr;
    if (params->variant == 1) {  // forced windows are global ids (selection.cpp:7-27)
        GSA_CUDA(launch_forced(g.L, params->ref_stride, b.forced, b.mask, st));
        excluded = b.mask;
    }
    GSA_CUDA(tc_compress_topk(*qc_own, *kc_all, *vc_all, g.k_eff, g.scale, excluded,
                              static_cast<float*>(o_comp_own->data), o_comp_own->head_stride,
                              o_comp_own->row_stride, lse_own, topk_own, nullptr, b.compress_ws,
                              b.compress_ws_bytes, st));
    return GSA_OK;
}

int gsa_shard_attend(const gsa_tensor* q_own, const gsa_tensor* k_all, const gsa_tensor* v_all,
                     const gsa_tensor* w_g, const gsa_layout* layout, const gsa_params* params,
                     const gsa_shard* shard, const gsa_tensor* o_comp_own, const int32_t* topk_own,
                     const gsa_tensor* out_own, void* workspace, size_t ws_bytes, gsa_stream_t stream) {
    GSA_TRY(check_tensor(q_own, "q_own"));
    ShardPlan sp;
    GSA_TRY(shard_checks(layout, params, shard, q_own->heads, q_own->dim, &sp));
    const LayerPlan& g = sp.g;
    const int H = g.heads, d = g.dim;
    GSA_TRY(check_shape(q_own, "q_own", H, sp.Ms_g + sp.Mi_g, d, true));
    GSA_TRY(check_shape(k_all, "k_all", H, g.M, d, true));
    GSA_TRY(check_shape(v_all, "v_all", H, g.M, d, true));
    if (k_all->dtype != q_own->dtype || v_all->dtype != q_own->dtype)
        return fail(GSA_ERR_UNSUPPORTED, "shard_attend: q/k/v dtypes differ");
    GSA_TRY(check_shape(o_comp_own, "o_comp_own", H, sp.W_g, d, false));
    GSA_TRY(contiguous_f32_windows(o_comp_own, "o_comp_own"));
    GSA_TRY(check_tensor(w_g, "w_g", false));
    if (w_g->heads != H || w_g->rows != d || w_g->dim != d || w_g->row_stride != d ||
        w_g->head_stride != (int64_t)d * d)
        return fail(GSA_ERR_SHAPE_MISMATCH, "weights: w_g must be contiguous heads x dim x dim");
    GSA_TRY(check_f32_out(out_own, "out_own", H, sp.Ms_g + sp.Mi_g, d));
    ShardBufs b;
    const size_t need = shard_carve(sp, static_cast<char*>(workspace), workspace == nullptr, &b);
    if (!workspace || need > ws_bytes + 256)
        return fail(GSA_ERR_WORKSPACE, "shard_attend: workspace %zu < %zu bytes", ws_bytes, need);
    cudaStream_t st = (cudaStream_t)stream;
    // V as fp16 planes over all M rows, exactly as gsa_forward makes them (same per-head
    // scale, so a sharded layer equals the unsharded one)
    const bool v16_made = q_own->dtype == GSA_DTYPE_BF16 && d == 64 && g.L.s == 4 &&
                          tc_dense_supported(*q_own, *k_all, *v_all) && (sp.Ms_g > 0 || sp.W_g > 0);
    if (v16_made) GSA_CUDA(launch_v16(ref_of(*v_all), H, g.M, b.vmax, b.v16, nullptr, st));
    // own special rows: dense attention over all M keys (layer.hpp:80-96)
    if (sp.Ms_g > 0)
        GSA_TRY(dense_attention(q_own, k_all, v_all, g.scale, out_own, b.lse_spec, 0, 0, sp.Ms_g, st, b.dense_ws,
                                b.dense_ws_bytes, v16_made ? b.v16 : nullptr, v16_made ? b.vmax : nullptr));
    if (sp.W_g == 0) return GSA_OK;
    if (params->variant == 1) GSA_CUDA(launch_forced(g.L, params->ref_stride, b.forced, b.mask, st));
    SelectArgs a{};
    a.q = ref_of(*q_own, sp.Ms_g);
    a.k = ref_of(*k_all, g.Ms);
    a.v = ref_of(*v_all, g.Ms);
    a.heads = H;
    a.dim = d;
    a.L = sp.Lq;
    a.Lkv = g.L;
    a.rows = RowSource{nullptr, nullptr, b.forced, params->variant == 1 ? g.n_forced : 0, topk_own, g.k_eff, g.k_eff};
    a.scale = g.scale;
    a.out = static_cast<float*>(out_own->data) + (size_t)sp.Ms_g * out_own->row_stride;
    a.out_hs = out_own->head_stride;
    a.out_rs = out_own->row_stride;
    a.w_g = static_cast<const float*>(w_g->data);
    a.o_comp = static_cast<const float*>(o_comp_own->data);
    a.wg_prep = b.wg_prep;
    if (v16_made) {
        a.v16 = TensorRef{b.v16 + (size_t)g.Ms * 64, kDtypeF16, (int64_t)g.M * 64, 64};
        a.vmax = b.vmax;
    }
    const bool tc_sel = tc_select_supported(a);
    if (tc_sel && params->variant == 1 && g.n_forced > 0 && g.k_eff > 0 && b.kf && d == 64 &&
        tc_dense_supported(*q_own, *k_all, *v_all)) {
        // the hybrid fast path of gsa_forward on the rank's own image queries (forced
        // frames are global: their K/V rows are complete after the K/V all-gather)
        GSA_TRY(hybrid_prior(q_own, sp.Ms_g, sp.Mi_g, k_all, v_all, g.Ms, g.L, params->ref_stride, g.n_forced,
                             g.scale, H, b.kf, b.vf, b.prior_o, b.prior_lse, b.fa_ws, b.fa_ws_bytes, st));
        a.rows = RowSource{nullptr, nullptr, b.forced, 0, topk_own, g.k_eff, g.k_eff};
        a.prior_o = b.prior_o;
        a.prior_lse = b.prior_lse;
    }
    return run_select(a, st);
}

int gsa_project_qkv_bf16(const void* x, int tokens, int model_dim, int64_t ldx, const void* w_qkv_t,
                         int n_out, void* qkv, int64_t ld_qkv, gsa_stream_t stream) {
    // the stack driver's projection on tensor cores (X . W_qkv with W_qkv stored transposed)
    if (!x || !w_qkv_t || !qkv) return fail(GSA_ERR_GENERIC, "project_qkv_bf16: null pointer");
    if (tokens < 0 || model_dim < 1 || n_out < 1) return fail(GSA_ERR_ZERO_SIZE, "project_qkv_bf16: empty shape");
    if (tokens == 0) return GSA_OK;
    if (!tc_gemm_supported(tokens, n_out, model_dim) || ldx % 8 || ld_qkv % 8 ||
        (reinterpret_cast<uintptr_t>(x) & 15) || (reinterpret_cast<uintptr_t>(w_qkv_t) & 15) ||
        (reinterpret_cast<uintptr_t>(qkv) & 15))
        return fail(GSA_ERR_UNSUPPORTED, "project_qkv_bf16: needs n_out %% 32 == 0, model_dim %% 64 == 0, 16-byte "
                    "aligned rows");
    GSA_CUDA(tc_gemm_bf16(static_cast<const __nv_bfloat16*>(x), ldx, static_cast<const __nv_bfloat16*>(w_qkv_t),
                          model_dim, static_cast<__nv_bfloat16*>(qkv), ld_qkv, tokens, n_out, model_dim,
                          (cudaStream_t)stream));
    return GSA_OK;
}

int gsa_residual_bf16(const void* x, const float* o, void* y, int64_t n, gsa_stream_t stream) {
    if (n < 0 || (n && (!x || !o || !y))) return fail(GSA_ERR_GENERIC, "residual_bf16: null pointer");
    if (n % 8 || (reinterpret_cast<uintptr_t>(x) & 15) || (reinterpret_cast<uintptr_t>(o) & 15) ||
        (reinterpret_cast<uintptr_t>(y) & 15))
        return fail(GSA_ERR_UNSUPPORTED, "residual_bf16: n %% 8 == 0 and 16-byte aligned buffers");
    GSA_CUDA(launch_residual_bf16(static_cast<const __nv_bfloat16*>(x), o, static_cast<__nv_bfloat16*>(y), n,
                                  (cudaStream_t)stream));
    return GSA_OK;
}

int gsa_convert(const void* src, int src_dtype, void* dst, int dst_dtype, int64_t n, gsa_stream_t stream) {
    if (n < 0 || (n && (!src || !dst))) return fail(GSA_ERR_GENERIC, "convert: null pointer or negative count");
    auto ok = [](int t) { return t == GSA_DTYPE_F32 || t == GSA_DTYPE_BF16; };
    if (!ok(src_dtype) || !ok(dst_dtype)) return fail(GSA_ERR_UNSUPPORTED, "convert: dtypes must be f32 or bf16");
    GSA_CUDA(launch_convert(src, src_dtype, dst, dst_dtype, n, (cudaStream_t)stream));
    return GSA_OK;
}

int gsa_project_qkv(const float* x, int tokens, int model_dim, const float* w_q, const float* w_k,
                    const float* w_v, int heads, int dim, const gsa_tensor* q, const gsa_tensor* k,
                    const gsa_tensor* v, gsa_stream_t stream) {
    // project_qkv (layer.hpp:48-76): X [1 x tokens x C], W [H x C x d]
    if (tokens < 0 || model_dim < 1 || heads < 0 || dim < 1)
        return fail(GSA_ERR_SHAPE_MISMATCH, "project_qkv: bad extents");
    if ((int64_t)tokens * model_dim > 0 && !x) return fail(GSA_ERR_GENERIC, "project_qkv: null x");
    if (!w_q || !w_k || !w_v) return fail(GSA_ERR_GENERIC, "project_qkv: null weights");
    const gsa_tensor* outs[3] = {q, k, v};
    ProjectMats m{};
    m.w[0] = w_q;
    m.w[1] = w_k;
    m.w[2] = w_v;
    int dtype = -1;
    for (int i = 0; i < 3; ++i) {
        GSA_TRY(check_tensor(outs[i], i == 0 ? "q" : (i == 1 ? "k" : "v")));
        if (outs[i]->heads != heads || outs[i]->rows != tokens || outs[i]->dim != dim)
            return fail(GSA_ERR_SHAPE_MISMATCH, "project_qkv: output must be [heads x tokens x dim]");
        if (dtype >= 0 && outs[i]->dtype != dtype) return fail(GSA_ERR_UNSUPPORTED, "project_qkv: output dtypes differ");
        dtype = outs[i]->dtype;
        m.out[i] = outs[i]->data;
        m.out_hs[i] = outs[i]->head_stride;
        m.out_rs[i] = outs[i]->row_stride;
    }
    GSA_CUDA(launch_project(x, tokens, model_dim, m, 3, heads, dim, dtype == GSA_DTYPE_BF16, (cudaStream_t)stream));
    return GSA_OK;
}

int gsa_forward_stats(const gsa_layout* layout, const gsa_params* p, int heads, uint64_t* scores,
                      uint64_t* keys) {
    GSA_TRY(check_layout(layout));
    GSA_TRY(gsa_validate_params(p, layout));
    const DevLayout L = make_dev_layout(*layout);
    const uint64_t M = (uint64_t)layout->num_special + L.image_tokens;
    int nf = 0;
    const int sel = selectable_windows(L, p->variant, p->ref_stride, &nf);
    const int k_eff = p->top_k < sel ? p->top_k : sel;
    const uint64_t s2 = (uint64_t)L.s * L.s;
    // tiled_attention counts qrows*krows per tile (compression.hpp:135-137), the
    // compressed kernel W*W per head (236-238); block_sparse adds |keys|*s2 per
    // (head, window) (selection.hpp:106-108)
    if (scores) *scores = (uint64_t)heads * ((uint64_t)layout->num_special * M + (uint64_t)L.windows * L.windows);
    if (keys) *keys = (uint64_t)heads * L.windows * (uint64_t)(nf + k_eff) * s2 * s2;
    return GSA_OK;
}

int gsa_selection_sparsity(const gsa_layout* layout, const gsa_params* p, double* sparsity) {
    GSA_TRY(check_layout(layout));
    GSA_TRY(gsa_validate_params(p, layout));
    if (!sparsity) return fail(GSA_ERR_GENERIC, "gsa_selection_sparsity: null output");
    const DevLayout L = make_dev_layout(*layout);
    int nf = 0;
    const int sel = selectable_windows(L, p->variant, p->ref_stride, &nf);
    const int k_eff = p->top_k < sel ? p->top_k : sel;
    const double attended = (double)(nf + k_eff) * L.s * L.s;  // forced ++ dynamic, deduplicated
    *sparsity = L.image_tokens > 0 ? 1.0 - attended / (double)L.image_tokens : 0.0;
    return GSA_OK;
}

// ------------------------------------------------------------------ backward

}  // extern "C"

namespace {

FMat fmat_of(const gsa_tensor& t, int row_offset = 0) {
    return FMat{static_cast<const float*>(t.data) + (int64_t)row_offset * t.row_stride, t.head_stride, t.row_stride};
}
FOut fout_of(const gsa_tensor& t, int row_offset = 0) {
    return FOut{static_cast<float*>(t.data) + (int64_t)row_offset * t.row_stride, t.head_stride, t.row_stride};
}

struct BwdBufs {
    float *q32, *k32, *v32;
    float *ds, *dz, *d_oc, *dqc, *dkc, *dvc, *d_sel, *d_comp, *d_spec;
    unsigned long long *keys, *keys_sorted;
    int64_t *counts, *inv_offsets;
    int32_t* inv_q;
    void* tmp;
    size_t tmp_bytes;
    float* part;
    int splits;
    float* spec_dq_part;  // key-split partial dQ of the special rows
    int spec_splits;
    int* check;           // plan validation flag
    // hybrid fast path (tensor cores): the forced windows' keys run as a dense pass, the
    // selection passes walk the plan without them
    int n_ff;             // forced frames (0: off)
    int64_t n_fr;         // forced rows per head
    uint8_t* fmask;
    int64_t *dyn_sizes, *dyn_offsets;
    int32_t* dyn_ids;
    __nv_bfloat16 *fk_h, *fk_l, *fv_h, *fv_l;
    float *gk, *gv;
    // tensor-core dense passes: bf16 hi (+ lo for f32 operands) planes [H][rows][64] of the
    // compressed branch (Qc, Kc, Vc, dO_comp: W rows) and the special rows (Q, dO: Ms rows;
    // K, V: M rows)
    bool tc;
    __nv_bfloat16 *c_h[4], *c_l[4], *s_h[4], *s_l[4];
    __nv_bfloat16 *ds_h, *ds_l;  // dS_sel (the selection passes' upstream gradient) [H][Mi][64]
};

// the dense backward passes run on tcgen05 at head dim 64 (bwd_tc.cu), on CUDA cores otherwise
bool bwd_use_tc(int d) { return tc_bwd_supported(d); }

// f32 rows the tensor-core epilogue writes as float4
bool aligned_rows(const gsa_tensor& t) {
    return t.row_stride % 4 == 0 && t.head_stride % 4 == 0 && (reinterpret_cast<uintptr_t>(t.data) & 15) == 0;
}

// forced frames of the hybrid fast path: reference frames every ref_stride frames, when the
// selection passes run on the tensor cores (0 otherwise)
int bwd_forced_frames(const DevLayout& L, const gsa_params* p, int d) {
    if (!p || p->variant != 1 || p->ref_stride < 1 || !tc_bwd_supported(d) || !tc_sel_bwd_supported(d, L.s)) return 0;
    return (L.num_frames + p->ref_stride - 1) / p->ref_stride;
}

size_t carve_bwd(const DevLayout& L, int Ms, int H, int d, int64_t E, bool convert, int n_ff, char* base, size_t cap,
                 bool dry, BwdBufs* b) {
    Carver c{base, cap, 0, dry};
    b->tc = bwd_use_tc(d);
    for (int i = 0; i < 4; ++i) b->c_h[i] = b->c_l[i] = b->s_h[i] = b->s_l[i] = nullptr;
    b->ds_h = b->ds_l = nullptr;
    if (b->tc) {
        const int64_t Mt = Ms + (int64_t)L.image_tokens, Wt = L.windows;
        for (int i = 0; i < 4; ++i) {
            b->c_h[i] = c.take<__nv_bfloat16>((size_t)H * Wt * 64);
            b->c_l[i] = c.take<__nv_bfloat16>((size_t)H * Wt * 64);
        }
        // Q / K / V of every row (the special rows' dense passes and the selection passes),
        // dO of the special rows; bf16 Q / K / V are exact as one plane, dO (f32) always splits
        for (int i = 0; i < 4; ++i) {
            const int64_t rows = i < 3 ? Mt : Ms;
            if (rows == 0) continue;
            b->s_h[i] = c.take<__nv_bfloat16>((size_t)H * rows * 64);
            if (convert == false || i == 3) b->s_l[i] = c.take<__nv_bfloat16>((size_t)H * rows * 64);
        }
        b->ds_h = c.take<__nv_bfloat16>((size_t)H * L.image_tokens * 64);
        b->ds_l = c.take<__nv_bfloat16>((size_t)H * L.image_tokens * 64);
    }
    const int64_t M = Ms + (int64_t)L.image_tokens, Mi = L.image_tokens, W = L.windows;
    b->q32 = b->k32 = b->v32 = nullptr;
    if (convert) {
        b->q32 = c.take<float>((size_t)H * M * d);
        b->k32 = c.take<float>((size_t)H * M * d);
        b->v32 = c.take<float>((size_t)H * M * d);
    }
    b->ds = c.take<float>((size_t)H * Mi * d);
    b->dz = c.take<float>((size_t)H * Mi * d);
    b->d_oc = c.take<float>((size_t)H * W * d);
    b->dqc = c.take<float>((size_t)H * W * d);
    b->dkc = c.take<float>((size_t)H * W * d);
    b->dvc = c.take<float>((size_t)H * W * d);
    b->d_sel = c.take<float>((size_t)H * Mi);
    b->d_comp = c.take<float>((size_t)H * W);
    b->d_spec = c.take<float>((size_t)H * (Ms > 0 ? Ms : 1));
    b->keys = c.take<unsigned long long>((size_t)E);
    b->keys_sorted = c.take<unsigned long long>((size_t)E);
    b->counts = c.take<int64_t>((size_t)H * W);
    b->inv_offsets = c.take<int64_t>((size_t)H * W + 1);
    b->inv_q = c.take<int32_t>((size_t)E);
    b->tmp_bytes = inverse_plan_tmp_bytes((int64_t)H * W, E);
    b->tmp = c.take<char>(b->tmp_bytes);
    b->splits = atb_splits(H, d, d, Mi);
    b->part = c.take<float>((size_t)H * b->splits * d * d);
    b->check = c.take<int>(4);
    b->n_ff = b->tc ? n_ff : 0;
    b->n_fr = (int64_t)b->n_ff * L.tokens_per_frame;
    b->fmask = nullptr;
    b->dyn_sizes = b->dyn_offsets = nullptr;
    b->dyn_ids = nullptr;
    b->fk_h = b->fk_l = b->fv_h = b->fv_l = nullptr;
    b->gk = b->gv = nullptr;
    if (b->n_ff > 0) {
        const size_t rows = (size_t)H * L.windows, fr = (size_t)H * b->n_fr * 64;
        b->fmask = c.take<uint8_t>((size_t)L.windows);
        b->dyn_sizes = c.take<int64_t>(rows);
        b->dyn_offsets = c.take<int64_t>(rows + 1);
        b->dyn_ids = c.take<int32_t>((size_t)(E > 0 ? E : 1));
        b->fk_h = c.take<__nv_bfloat16>(fr);
        b->fv_h = c.take<__nv_bfloat16>(fr);
        if (!convert) {
            b->fk_l = c.take<__nv_bfloat16>(fr);
            b->fv_l = c.take<__nv_bfloat16>(fr);
        }
        b->gk = c.take<float>(fr);
        b->gv = c.take<float>(fr);
    }
    b->spec_splits = Ms > 0 ? (b->tc ? tc_bwd_dq_splits(H, Ms, M) : dense_dq_splits(H, Ms, M)) : 1;
    b->spec_dq_part = b->spec_splits > 1 ? c.take<float>((size_t)b->spec_splits * H * Ms * d) : nullptr;
    return c.used;
}

}  // namespace

extern "C" {

size_t gsa_backward_workspace_bytes(const gsa_layout* layout, const gsa_params* params, int heads, int dim,
                                    int64_t plan_entries, int qkv_dtype) {
    if (check_layout(layout) != GSA_OK || heads < 0 || dim < 1 || plan_entries < 0) return 0;
    const DevLayout L = make_dev_layout(*layout);
    BwdBufs b;
    return carve_bwd(L, layout->num_special, heads, dim, plan_entries, qkv_dtype != GSA_DTYPE_F32,
                     bwd_forced_frames(L, params, dim), nullptr, 0, true,
                     &b) + 256;
}

int gsa_backward(const gsa_tensor* q, const gsa_tensor* k, const gsa_tensor* v, const gsa_tensor* w_g,
                 const gsa_layout* layout, const gsa_params* params, const gsa_saved* sv,
                 const gsa_tensor* d_out, const gsa_tensor* dq, const gsa_tensor* dk, const gsa_tensor* dv,
                 float* dw_g, void* workspace, size_t ws_bytes, gsa_stream_t stream) {
    // gsa_backward (gradients.hpp:54-75): shapes of dO and the saved context
    const gsa_tensor* o = d_out;
    GSA_TRY(check_tensor(o, "d_out", false));
    LayerPlan lp;
    GSA_TRY(layer_checks(q, k, v, w_g, layout, params, o, &lp, true));
    if (!sv) return fail(GSA_ERR_GENERIC, "gsa_backward: null saved context");
    if (!sv->qc || !sv->kc || !sv->vc || !sv->o_comp || !sv->lse_comp || !sv->o_sel || !sv->lse_sel || !sv->gate ||
        (lp.Ms > 0 && (!sv->lse_spec || !sv->o_spec.data)))
        return fail(GSA_ERR_CONTEXT_MISMATCH, "gsa_backward: saved context is incomplete");
    if (lp.Ms > 0 && (sv->o_spec.dtype != GSA_DTYPE_F32 || sv->o_spec.heads != lp.heads ||
                      sv->o_spec.rows != lp.Ms || sv->o_spec.dim != lp.dim))
        return fail(GSA_ERR_CONTEXT_MISMATCH, "gsa_backward: o_spec must be f32 [H][Ms][d]");
    GSA_TRY(check_f32_out(dq, "dq", lp.heads, lp.M, lp.dim));
    GSA_TRY(check_f32_out(dk, "dk", lp.heads, lp.M, lp.dim));
    GSA_TRY(check_f32_out(dv, "dv", lp.heads, lp.M, lp.dim));
    if (!dw_g) return fail(GSA_ERR_GENERIC, "gsa_backward: null dw_g");
    const int H = lp.heads, d = lp.dim, W = lp.W, Ms = lp.Ms;
    const int64_t rows = (int64_t)H * W;
    cudaStream_t st = (cudaStream_t)stream;
    const bool convert = q->dtype != GSA_DTYPE_F32;
    BwdBufs b;
    const size_t need = carve_bwd(lp.L, Ms, H, d, sv->plan_entries, convert, bwd_forced_frames(lp.L, params, d),
                                  static_cast<char*>(workspace), ws_bytes,
                                  false, &b);
    if (need > ws_bytes + 256) return fail(GSA_ERR_WORKSPACE, "gsa_backward: workspace %zu < %zu", ws_bytes, need);
    if (rows == 0) return GSA_OK;
    // plan validation (like gsa_forward_with_plan's) and its entry count: one round trip,
    // the flag in the caller's workspace (no allocation)
    if (!sv->plan_offsets || !sv->plan_ids) return fail(GSA_ERR_GENERIC, "gsa_backward: null plan");
    int64_t dyn_entries = 0;
    {
        GSA_CUDA(cudaMemsetAsync(b.check, 0, sizeof(int), st));
        GSA_CUDA(launch_plan_check(sv->plan_offsets, rows, sv->plan_ids, W, b.check, st));
        struct { int flag; int pad; int64_t total, dyn_total; } hb{0, 0, 0, 0};
        if (b.n_ff > 0) {
            // hybrid: the plan without the forced windows (ids outside [0, W) count as kept and
            // are reported by the check below before anything reads them)
            GSA_CUDA(launch_forced(lp.L, params->ref_stride, nullptr, b.fmask, st));
            GSA_CUDA(launch_plan_drop(sv->plan_offsets, sv->plan_ids, rows, b.fmask, W, b.dyn_sizes, b.dyn_offsets,
                                      b.dyn_ids, b.tmp, b.tmp_bytes, st));
            GSA_CUDA(cudaMemcpyAsync(&hb.dyn_total, b.dyn_offsets + rows, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
        }
        GSA_CUDA(cudaMemcpyAsync(&hb.flag, b.check, sizeof(int), cudaMemcpyDeviceToHost, st));
        GSA_CUDA(cudaMemcpyAsync(&hb.total, sv->plan_offsets + rows, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
        GSA_CUDA(cudaStreamSynchronize(st));
        dyn_entries = hb.dyn_total;
        if (hb.flag & 1) return fail(GSA_ERR_EMPTY_SELECTION, "gsa_backward: empty plan row");
        if (hb.flag & 2) return fail(GSA_ERR_INDEX_OUT_OF_RANGE, "gsa_backward: plan window id outside [0, %d)", W);
        if (hb.total != sv->plan_entries)
            return fail(GSA_ERR_CONTEXT_MISMATCH, "gsa_backward: plan holds %lld entries, saved.plan_entries = %lld",
                        (long long)hb.total, (long long)sv->plan_entries);
    }

    stage_mark(0, st);
    FMat Q = fmat_of(*q), K = fmat_of(*k), V = fmat_of(*v);
    if (convert) {
        // f32 copies for the CUDA-core kernels: Q always (dW_g = Q_img^T dz); K and V only when
        // a CUDA-core attention pass will read them (the tensor-core passes read bf16 planes)
        const bool kv32 = !b.tc || !tc_sel_bwd_supported(d, lp.L.s) || !aligned_rows(*dq) || !aligned_rows(*dk) ||
                          !aligned_rows(*dv);
        const int64_t hs = (int64_t)lp.M * d;
        GSA_CUDA(launch_to_f32(ref_of(*q), H, lp.M, d, b.q32, st));
        Q = FMat{b.q32, hs, d};
        if (kv32) {
            GSA_CUDA(launch_to_f32(ref_of(*k), H, lp.M, d, b.k32, st));
            GSA_CUDA(launch_to_f32(ref_of(*v), H, lp.M, d, b.v32, st));
            K = FMat{b.k32, hs, d};
            V = FMat{b.v32, hs, d};
        }
    }
    const FMat dO = fmat_of(*d_out);
    const FOut dQ = fout_of(*dq), dK = fout_of(*dk), dV = fout_of(*dv);
    const int64_t whs = (int64_t)W * d;

    // 1. gate fuse + upsample backward (gradients.hpp:96-128)
    GateBwdArgs g{};
    g.dout = dO;
    g.gate = sv->gate;
    g.o_sel = sv->o_sel;
    g.o_comp = sv->o_comp;
    g.w_g = static_cast<const float*>(w_g->data);
    g.L = lp.L;
    g.dim = d;
    g.ds = b.ds;
    g.dz = b.dz;
    g.d_oc = b.d_oc;
    g.d_sel = b.d_sel;
    g.d_comp = b.d_comp;
    g.dq = dQ;
    GSA_CUDA(launch_gate_bwd(g, H, st));
    if (b.tc) {
        // tensor-core operand planes of Q / K / V (all rows) and of dS_sel
        const TensorRef refs[3] = {ref_of(*q), ref_of(*k), ref_of(*v)};
        for (int i = 0; i < 3; ++i)
            GSA_CUDA(launch_pack_rows(refs[i], H, lp.M, b.s_h[i], refs[i].dtype == GSA_DTYPE_F32 ? b.s_l[i] : nullptr, st));
        GSA_CUDA(launch_pack_rows(TensorRef{b.ds, GSA_DTYPE_F32, (int64_t)lp.Mi * d, d}, H, lp.Mi, b.ds_h, b.ds_l, st));
    }
    stage_mark(1, st);

    // 2. compressed attention backward over the windows (gradients.hpp:130-155)
    DenseBwdArgs c{};
    c.q = FMat{sv->qc, whs, d};
    c.k = FMat{sv->kc, whs, d};
    c.v = FMat{sv->vc, whs, d};
    c.dout = FMat{b.d_oc, whs, d};
    c.lse = sv->lse_comp;
    c.lse_hs = W;
    c.D = b.d_comp;
    c.D_hs = W;
    c.nq = c.nk = W;
    c.dim = d;
    c.scale = lp.scale;
    c.dq = FOut{b.dqc, whs, d};
    c.dk = FOut{b.dkc, whs, d};
    c.dv = FOut{b.dvc, whs, d};
    c.accumulate = false;
    if (b.tc) {
        // operand planes (bf16 hi + lo of the f32 pooled tensors and of dO_comp)
        const float* src[4] = {sv->qc, sv->kc, sv->vc, b.d_oc};
        for (int i = 0; i < 4; ++i)
            GSA_CUDA(launch_pack_rows(TensorRef{src[i], GSA_DTYPE_F32, whs, d}, H, W, b.c_h[i], b.c_l[i], st));
        BwdTcArgs t{};
        t.heads = H;
        t.n_q = t.n_k = W;
        t.scale = lp.scale;
        t.q_hi = b.c_h[0];
        t.q_lo = b.c_l[0];
        t.k_hi = b.c_h[1];
        t.k_lo = b.c_l[1];
        t.v_hi = b.c_h[2];
        t.v_lo = b.c_l[2];
        t.do_hi = b.c_h[3];
        t.do_lo = b.c_l[3];
        t.lse = sv->lse_comp;
        t.D = b.d_comp;
        t.dq = b.dqc;
        t.dq_hs = whs;
        t.dq_rs = d;
        t.dk = b.dkc;
        t.dk_hs = whs;
        t.dk_rs = d;
        t.dv = b.dvc;
        t.dv_hs = whs;
        t.dv_rs = d;
        GSA_CUDA(launch_bwd_tc(t, st));
    } else {
        GSA_CUDA(launch_dense_bwd(c, H, st));
    }

    stage_mark(2, st);
    // 3. pooling backward into the image rows (gradients.hpp:157-169)
    PoolBwdArgs pb{};
    pb.heads = H;
    pb.rows = lp.M;
    pb.dim = d;
    pb.L = lp.L;
    pb.inv = 1.0f / (float)(lp.L.s * lp.L.s);
    pb.dqc = b.dqc;
    pb.dkc = b.dkc;
    pb.dvc = b.dvc;
    pb.dq = dQ;
    pb.dk = dK;
    pb.dv = dV;
    GSA_CUDA(launch_pool_bwd(pb, st));

    // 4. selection backward over the detached plan (gradients.hpp:171-195)
    const int64_t* sel_offsets = b.n_ff > 0 ? b.dyn_offsets : sv->plan_offsets;
    const int32_t* sel_ids = b.n_ff > 0 ? b.dyn_ids : sv->plan_ids;
    const int64_t sel_entries = b.n_ff > 0 ? dyn_entries : sv->plan_entries;
    GSA_CUDA(launch_inverse_plan(sel_offsets, sel_ids, rows, W, sel_entries, b.keys, b.keys_sorted, b.counts,
                                 b.inv_offsets, b.inv_q, b.tmp, b.tmp_bytes, st));
    SelBwdArgs sa{};
    sa.q = Q;
    sa.k = K;
    sa.v = V;
    sa.ds = b.ds;
    sa.lse = sv->lse_sel;
    sa.D = b.d_sel;
    sa.offsets = sv->plan_offsets;
    sa.ids = sv->plan_ids;
    sa.inv_offsets = b.inv_offsets;
    sa.inv_q = b.inv_q;
    sa.L = lp.L;
    sa.dim = d;
    sa.scale = lp.scale;
    sa.dq = dQ;
    sa.dk = dK;
    sa.dv = dV;
    if (b.tc && tc_sel_bwd_supported(d, lp.L.s)) {
        SelBwdTcArgs t{};
        t.L = lp.L;
        t.heads = H;
        t.scale = lp.scale;
        const int64_t phs = (int64_t)lp.M * 64, img = (int64_t)Ms * 64;  // image row 0 of the all-row planes
        auto plane = [&](const __nv_bfloat16* base) { return BwdPlane{base ? base + img : nullptr, phs, 64}; };
        t.q_hi = plane(b.s_h[0]);
        t.q_lo = plane(b.s_l[0]);
        t.k_hi = plane(b.s_h[1]);
        t.k_lo = plane(b.s_l[1]);
        t.v_hi = plane(b.s_h[2]);
        t.v_lo = plane(b.s_l[2]);
        t.ds_hi = BwdPlane{b.ds_h, (int64_t)lp.Mi * 64, 64};
        t.ds_lo = BwdPlane{b.ds_l, (int64_t)lp.Mi * 64, 64};
        t.lse = sv->lse_sel;
        t.D = b.d_sel;
        t.offsets = sel_offsets;
        t.ids = sel_ids;
        t.inv_offsets = b.inv_offsets;
        t.inv_q = b.inv_q;
        t.dq = dQ.p;
        t.dq_hs = dQ.hs;
        t.dq_rs = dQ.rs;
        t.dk = dK.p;
        t.dk_hs = dK.hs;
        t.dk_rs = dK.rs;
        t.dv = dV.p;
        t.dv_hs = dV.hs;
        t.dv_rs = dV.rs;
        GSA_CUDA(launch_sel_bwd_tc(t, st));
        if (b.n_ff > 0) {
            // the forced windows' keys: a dense pass of every image query over the forced-frame
            // rows (their P from the same total LSE rows), gathered contiguously
            const int rs = params->ref_stride;
            GSA_CUDA(launch_forced_gather(b.s_h[1], (int64_t)lp.M * 64, H, lp.L, rs, b.n_fr, b.fk_h, st));
            GSA_CUDA(launch_forced_gather(b.s_h[2], (int64_t)lp.M * 64, H, lp.L, rs, b.n_fr, b.fv_h, st));
            if (b.fk_l) {
                GSA_CUDA(launch_forced_gather(b.s_l[1], (int64_t)lp.M * 64, H, lp.L, rs, b.n_fr, b.fk_l, st));
                GSA_CUDA(launch_forced_gather(b.s_l[2], (int64_t)lp.M * 64, H, lp.L, rs, b.n_fr, b.fv_l, st));
            }
            BwdTcArgs f{};
            f.heads = H;
            f.n_q = lp.Mi;
            f.n_k = b.n_fr;
            f.scale = lp.scale;
            f.q_hi = b.s_h[0] + img;
            f.q_lo = b.s_l[0] ? b.s_l[0] + img : nullptr;
            f.q_hs = phs;
            f.do_hi = b.ds_h;
            f.do_lo = b.ds_l;
            f.do_hs = (int64_t)lp.Mi * 64;
            f.k_hi = b.fk_h;
            f.k_lo = b.fk_l;
            f.v_hi = b.fv_h;
            f.v_lo = b.fv_l;
            f.lse = sv->lse_sel;
            f.D = b.d_sel;
            f.dq = dQ.p + (int64_t)Ms * dQ.rs;  // image rows
            f.dq_hs = dQ.hs;
            f.dq_rs = dQ.rs;
            f.accumulate_q = true;
            f.dk = b.gk;
            f.dk_hs = b.n_fr * 64;
            f.dk_rs = 64;
            f.dv = b.gv;
            f.dv_hs = b.n_fr * 64;
            f.dv_rs = 64;
            f.accumulate_kv = false;
            GSA_CUDA(launch_bwd_tc(f, st));
            GSA_CUDA(launch_forced_scatter_add(b.gk, b.gv, H, lp.L, rs, b.n_fr, dK, dV, st));
        }
    } else {
        GSA_CUDA(launch_sel_bwd(sa, H, st));
    }
    stage_mark(3, st);

    // 5. special rows: dense backward over every key (gradients.hpp:197-222)
    if (Ms > 0) {
        const FMat oS = fmat_of(sv->o_spec);
        GSA_CUDA(launch_rowdot(dO, oS, H, Ms, d, b.d_spec, st));
        DenseBwdArgs sp{};
        sp.q = Q;
        sp.k = K;
        sp.v = V;
        sp.dout = dO;
        sp.lse = sv->lse_spec;
        sp.lse_hs = Ms;
        sp.D = b.d_spec;
        sp.D_hs = Ms;
        sp.nq = Ms;
        sp.nk = lp.M;
        sp.dim = d;
        sp.scale = lp.scale;
        if (b.tc && aligned_rows(*dq) && aligned_rows(*dk) && aligned_rows(*dv)) {
            // planes: Q / K / V packed after the gate; dO of the special rows here
            GSA_CUDA(launch_pack_rows(TensorRef{d_out->data, GSA_DTYPE_F32, d_out->head_stride, d_out->row_stride}, H, Ms,
                                      b.s_h[3], b.s_l[3], st));
            BwdTcArgs t{};
            t.heads = H;
            t.n_q = Ms;
            t.n_k = lp.M;
            t.scale = lp.scale;
            t.q_hs = (int64_t)lp.M * 64;  // the special rows of the all-row Q plane
            t.q_hi = b.s_h[0];
            t.q_lo = q->dtype == GSA_DTYPE_F32 ? b.s_l[0] : nullptr;
            t.k_hi = b.s_h[1];
            t.k_lo = k->dtype == GSA_DTYPE_F32 ? b.s_l[1] : nullptr;
            t.v_hi = b.s_h[2];
            t.v_lo = v->dtype == GSA_DTYPE_F32 ? b.s_l[2] : nullptr;
            t.do_hi = b.s_h[3];
            t.do_lo = b.s_l[3];
            t.lse = sv->lse_spec;
            t.D = b.d_spec;
            t.dk = dK.p;  // key side: accumulated into every row
            t.dk_hs = dK.hs;
            t.dk_rs = dK.rs;
            t.dv = dV.p;
            t.dv_hs = dV.hs;
            t.dv_rs = dV.rs;
            t.accumulate_kv = true;
            t.dq = dQ.p;  // the special rows' only dQ term: written
            t.dq_hs = dQ.hs;
            t.dq_rs = dQ.rs;
            t.dq_part = b.spec_dq_part;
            t.dq_splits = b.spec_splits;
            GSA_CUDA(launch_bwd_tc(t, st));
        } else {
            sp.dk = dK;  // key side first, accumulated into every row
            sp.dv = dV;
            sp.accumulate = true;
            GSA_CUDA(launch_dense_bwd(sp, H, st));
            sp.dk = FOut{nullptr, 0, 0};
            sp.dv = FOut{nullptr, 0, 0};
            sp.dq = dQ;  // the special rows' only dQ term: written
            sp.accumulate = false;
            sp.k_splits = b.tc ? 1 : b.spec_splits;  // (tc: the partial buffer is sized for its own splits)
            sp.dq_part = b.spec_dq_part;
            GSA_CUDA(launch_dense_bwd(sp, H, st));
        }
    }

    stage_mark(4, st);
    // 6. dW_g = Q_img^T dz per head (gradients.hpp:112-113)
    AtbArgs at{};
    at.A = Q.p + (int64_t)Ms * Q.rs;
    at.a_hs = Q.hs;
    at.a_rs = Q.rs;
    at.B = b.dz;
    at.b_hs = (int64_t)lp.Mi * d;
    at.b_rs = d;
    at.R = d;
    at.N = d;
    at.rows = lp.Mi;
    at.splits = b.splits;
    at.part = b.part;
    GSA_CUDA(launch_atb(at, H, dw_g, st));
    stage_mark(5, st);
    return GSA_OK;
}

size_t gsa_project_backward_workspace_bytes(int tokens, int model_dim, int heads, int dim) {
    if (tokens < 0 || model_dim < 1 || heads < 0 || dim < 1) return 0;
    if (tc_proj_bwd_supported(dim, model_dim)) return tc_proj_bwd_workspace_bytes(tokens, model_dim, heads) + 256;
    return (size_t)heads * atb_splits(heads, model_dim, dim, tokens) * model_dim * dim * sizeof(float) + 256;
}

int gsa_project_backward(const float* x, int tokens, int model_dim, const float* w_q, const float* w_k,
                         const float* w_v, int heads, int dim, const float* dq, const float* dk, const float* dv,
                         float* dx, float* dw_q, float* dw_k, float* dw_v, void* workspace, size_t ws_bytes,
                         gsa_stream_t stream) {
    if (tokens < 0 || model_dim < 1 || heads < 1 || dim < 1)
        return fail(GSA_ERR_SHAPE_MISMATCH, "project_backward: bad extents");
    if (!x || !w_q || !w_k || !w_v || !dq || !dk || !dv || !dx || !dw_q || !dw_k || !dw_v)
        return fail(GSA_ERR_GENERIC, "project_backward: null pointer");
    const size_t need = gsa_project_backward_workspace_bytes(tokens, model_dim, heads, dim);
    if (ws_bytes + 256 < need || (need > 256 && !workspace))
        return fail(GSA_ERR_WORKSPACE, "project_backward: workspace %zu < %zu", ws_bytes, need);
    cudaStream_t st = (cudaStream_t)stream;
    const float* g[3] = {dq, dk, dv};
    float* dw[3] = {dw_q, dw_k, dw_v};
    if (tc_proj_bwd_supported(dim, model_dim) && ((reinterpret_cast<uintptr_t>(dx) | reinterpret_cast<uintptr_t>(dw_q) |
                                                   reinterpret_cast<uintptr_t>(dw_k) | reinterpret_cast<uintptr_t>(dw_v)) &
                                                  15) == 0) {
        // tensor cores (bf16 hi / lo planes, 3-term products); the workspace holds the planes
        const float* wm[3] = {w_q, w_k, w_v};
        void* base = reinterpret_cast<void*>((reinterpret_cast<uintptr_t>(workspace) + 255) & ~uintptr_t(255));
        GSA_CUDA(launch_proj_bwd_tc(x, tokens, model_dim, wm, heads, g, dx, dw, base, st));
        return GSA_OK;
    }
    for (int i = 0; i < 3; ++i) {
        AtbArgs a{};
        a.A = x;
        a.a_hs = 0;
        a.a_rs = model_dim;
        a.B = g[i];
        a.b_hs = (int64_t)tokens * dim;
        a.b_rs = dim;
        a.R = model_dim;
        a.N = dim;
        a.rows = tokens;
        a.splits = atb_splits(heads, model_dim, dim, tokens);
        a.part = static_cast<float*>(workspace);
        GSA_CUDA(launch_atb(a, heads, dw[i], st));
    }
    DxArgs a{};
    a.g[0] = dq;
    a.g[1] = dk;
    a.g[2] = dv;
    a.w[0] = w_q;
    a.w[1] = w_k;
    a.w[2] = w_v;
    a.heads = heads;
    a.dim = dim;
    a.C = model_dim;
    a.tokens = tokens;
    a.dx = dx;
    GSA_CUDA(launch_dx_gemm(a, st));
    return GSA_OK;
}

int gsa_avg_pool_backward(const gsa_tensor* d_pooled, const gsa_layout* layout, const gsa_tensor* out,
                          gsa_stream_t stream) {
    GSA_TRY(check_layout(layout));
    GSA_TRY(check_tensor(d_pooled, "d_pooled", false));
    const DevLayout L = make_dev_layout(*layout);
    // gradients.hpp:23-24
    if (d_pooled->rows != L.windows) return fail(GSA_ERR_SHAPE_MISMATCH, "avg_pool_backward: rows != num windows");
    GSA_TRY(check_f32_out(out, "out", d_pooled->heads, L.image_tokens, d_pooled->dim));
    GSA_CUDA(launch_pool_adjoint(fmat_of(*d_pooled), d_pooled->heads, d_pooled->dim, L,
                                 1.0f / (float)(L.s * L.s), fout_of(*out), (cudaStream_t)stream));
    return GSA_OK;
}

int gsa_upsample_backward(const gsa_tensor* d_fine, const gsa_layout* layout, const gsa_tensor* out,
                          gsa_stream_t stream) {
    GSA_TRY(check_layout(layout));
    GSA_TRY(check_tensor(d_fine, "d_fine", false));
    const DevLayout L = make_dev_layout(*layout);
    // gradients.hpp:39-40
    if (d_fine->rows != L.image_tokens) return fail(GSA_ERR_SHAPE_MISMATCH, "upsample_backward: rows != image tokens");
    GSA_TRY(check_f32_out(out, "out", d_fine->heads, L.windows, d_fine->dim));
    GSA_CUDA(launch_window_sum(fmat_of(*d_fine), d_fine->heads, d_fine->dim, L, fout_of(*out), (cudaStream_t)stream));
    return GSA_OK;
}

int gsa_set_stage_events(void* const* events, int n) {
    if (n < 5 || !events) {
        g_n_stage_events = 0;
        return GSA_OK;
    }
    const int m = n >= 7 ? 7 : 5;
    for (int i = 0; i < m; ++i) g_stage_events[i] = static_cast<cudaEvent_t>(events[i]);
    g_n_stage_events = m;
    return GSA_OK;
}

int gsa_launch_count(uint64_t* count) {
    if (count) *count = gsa_sm100::g_launch_total.load();
    return GSA_OK;
}

}  // extern "C"
