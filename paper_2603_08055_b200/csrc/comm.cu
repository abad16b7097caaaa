// comm.cu — the multi-GPU layer at the C level (include/gsa_sm100.h, "Multi-GPU layer"):
// the shard of a rank, the in-place all-gather plan shared by every caller, an NCCL
// communicator resolved from libnccl.so.2 at run time, and gsa_shard_forward, which
// runs one view-sharded layer with the K/V-row gather overlapping the compressed
// branch. The reference has no multi-device code (a single-process CPU
// library); the partition is SURVEY §8(e): rank g owns views [gV/G, (g+1)V/G) and
// special rows [gMs/G, (g+1)Ms/G).
#include <dlfcn.h>
#include <nccl.h>  // types and enum values only: the symbols are resolved with dlsym

#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <vector>

#include "kernels.h"

using namespace gsa_sm100;

namespace {

int err(int status, const char* fmt, ...) __attribute__((format(printf, 2, 3)));
int err(int status, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    return report_error(status, buf);
}

#define COMM_TRY(expr)                 \
    do {                               \
        int _rc = (expr);              \
        if (_rc != GSA_OK) return _rc; \
    } while (0)
#define COMM_CUDA(expr)                                                                              \
    do {                                                                                             \
        cudaError_t _e = (expr);                                                                     \
        if (_e != cudaSuccess) return err(GSA_ERR_CUDA, "%s: %s", #expr, cudaGetErrorString(_e)); \
    } while (0)

struct NcclApi {
    ncclResult_t (*get_unique_id)(ncclUniqueId*);
    ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int);
    ncclResult_t (*comm_destroy)(ncclComm_t);
    ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t);
    ncclResult_t (*group_start)();
    ncclResult_t (*group_end)();
    const char* (*error_string)(ncclResult_t);
    bool ok = false;
    char why[256] = {0};
};

const NcclApi& nccl() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        // inside a PyTorch process this returns the libnccl torch already loaded
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            snprintf(api.why, sizeof(api.why), "libnccl.so.2 not loadable: %s", dlerror());
            return;
        }
        auto sym = [&](const char* n) {
            void* p = dlsym(h, n);
            if (!p && !api.why[0]) snprintf(api.why, sizeof(api.why), "libnccl: missing symbol %s", n);
            return p;
        };
        api.get_unique_id = reinterpret_cast<decltype(api.get_unique_id)>(sym("ncclGetUniqueId"));
        api.comm_init_rank = reinterpret_cast<decltype(api.comm_init_rank)>(sym("ncclCommInitRank"));
        api.comm_destroy = reinterpret_cast<decltype(api.comm_destroy)>(sym("ncclCommDestroy"));
        api.all_gather = reinterpret_cast<decltype(api.all_gather)>(sym("ncclAllGather"));
        api.group_start = reinterpret_cast<decltype(api.group_start)>(sym("ncclGroupStart"));
        api.group_end = reinterpret_cast<decltype(api.group_end)>(sym("ncclGroupEnd"));
        api.error_string = reinterpret_cast<decltype(api.error_string)>(sym("ncclGetErrorString"));
        api.ok = !api.why[0];
    });
    return api;
}

int nccl_status(ncclResult_t r, const char* where) {
    if (r == ncclSuccess) return GSA_OK;
    return err(GSA_ERR_NCCL, "%s: %s", where, nccl().error_string ? nccl().error_string(r) : "NCCL error");
}

int layout_ok(const gsa_layout* l) {
    if (!l) return err(GSA_ERR_GENERIC, "null layout");
    return gsa_make_layout(l->num_special, l->num_frames, l->grid_h, l->grid_w, l->window_s, nullptr);
}

size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

}  // namespace

struct gsa_comm_st {
    ncclComm_t comm = nullptr;
    int nranks = 0, rank = 0, device = 0;
    cudaStream_t cs = nullptr;  // the gathers run here, event-ordered with the caller's stream
    cudaEvent_t ev_pooled = nullptr, ev_c = nullptr, ev_kv = nullptr;
};

extern "C" {

int gsa_shard_of_rank(const gsa_layout* layout, int nranks, int rank, gsa_shard* out) {
    COMM_TRY(layout_ok(layout));
    if (nranks < 1 || rank < 0 || rank >= nranks)
        return err(GSA_ERR_INDEX_OUT_OF_RANGE, "rank %d outside a world of %d", rank, nranks);
    if (layout->num_frames % nranks || layout->num_special % nranks)
        return err(GSA_ERR_SHAPE_MISMATCH,
                   "view sharding needs num_frames (%d) and num_special (%d) divisible by the world size %d",
                   layout->num_frames, layout->num_special, nranks);
    const int fv = layout->num_frames / nranks, fs = layout->num_special / nranks;
    if (out) *out = gsa_shard{rank * fv, (rank + 1) * fv, rank * fs, (rank + 1) * fs};
    return GSA_OK;
}

int gsa_shard_gather_plan(const gsa_layout* layout, int nranks, int heads, int dim, int64_t kv_head_stride,
                          gsa_gather_op* ops, int capacity, int* n_ops) {
    gsa_shard s0;
    COMM_TRY(gsa_shard_of_rank(layout, nranks, 0, &s0));
    if (heads < 1 || dim < 1) return err(GSA_ERR_ZERO_SIZE, "gather plan: empty heads / dim");
    const int64_t tpf = (int64_t)layout->grid_h * layout->grid_w;
    const int64_t s2 = (int64_t)layout->window_s * layout->window_s;
    const int64_t W = (int64_t)layout->num_frames * tpf / s2, M = layout->num_special + layout->num_frames * tpf;
    if (kv_head_stride < M * dim) return err(GSA_ERR_SHAPE_MISMATCH, "gather plan: K/V head stride < M * dim");
    const int64_t Wg = (s0.frame_end - s0.frame_begin) * tpf / s2, Msg = s0.special_end - s0.special_begin,
                  Mig = (s0.frame_end - s0.frame_begin) * tpf;
    std::vector<gsa_gather_op> v;
    for (int b = 0; b < 2; ++b)  // Kc, Vc: rank r's windows are rows [r Wg, (r+1) Wg) of every head
        for (int h = 0; h < heads; ++h) v.push_back(gsa_gather_op{b, 0, (int64_t)h * W * dim, Wg * dim});
    for (int b = 2; b < 4; ++b)  // K, V rows: own specials, own image rows of every head
        for (int h = 0; h < heads; ++h) {
            if (Msg > 0) v.push_back(gsa_gather_op{b, 1, (int64_t)h * kv_head_stride, Msg * dim});
            v.push_back(gsa_gather_op{b, 1, (int64_t)h * kv_head_stride + (int64_t)layout->num_special * dim, Mig * dim});
        }
    if (n_ops) *n_ops = (int)v.size();
    if (ops) {
        if (capacity < (int)v.size()) return err(GSA_ERR_WORKSPACE, "gather plan: capacity %d < %d ops", capacity, (int)v.size());
        std::memcpy(ops, v.data(), v.size() * sizeof(gsa_gather_op));
    }
    return GSA_OK;
}

int gsa_comm_get_unique_id(void* id) {
    const NcclApi& n = nccl();
    if (!n.ok) return err(GSA_ERR_NCCL, "%s", n.why);
    if (!id) return err(GSA_ERR_GENERIC, "null id buffer");
    ncclUniqueId u;
    COMM_TRY(nccl_status(n.get_unique_id(&u), "ncclGetUniqueId"));
    std::memcpy(id, &u, sizeof(u));
    return GSA_OK;
}

int gsa_comm_init(gsa_comm* comm, const void* id, int nranks, int rank) {
    const NcclApi& n = nccl();
    if (!n.ok) return err(GSA_ERR_NCCL, "%s", n.why);
    if (!comm || !id) return err(GSA_ERR_GENERIC, "null comm / id");
    if (nranks < 1 || rank < 0 || rank >= nranks)
        return err(GSA_ERR_INDEX_OUT_OF_RANGE, "rank %d outside a world of %d", rank, nranks);
    auto* c = new gsa_comm_st();
    c->nranks = nranks;
    c->rank = rank;
    cudaError_t e = cudaGetDevice(&c->device);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&c->cs, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->ev_pooled, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->ev_c, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->ev_kv, cudaEventDisableTiming);
    if (e != cudaSuccess) {
        gsa_comm_destroy(c);
        return err(GSA_ERR_CUDA, "gsa_comm_init: %s", cudaGetErrorString(e));
    }
    ncclUniqueId u;
    std::memcpy(&u, id, sizeof(u));
    const int rc = nccl_status(n.comm_init_rank(&c->comm, nranks, u, rank), "ncclCommInitRank");
    if (rc != GSA_OK) {
        c->comm = nullptr;
        gsa_comm_destroy(c);
        return rc;
    }
    *comm = c;
    return GSA_OK;
}

int gsa_comm_destroy(gsa_comm c) {
    if (!c) return GSA_OK;
    int rc = GSA_OK;
    if (c->comm) rc = nccl_status(nccl().comm_destroy(c->comm), "ncclCommDestroy");
    if (c->ev_kv) cudaEventDestroy(c->ev_kv);
    if (c->ev_c) cudaEventDestroy(c->ev_c);
    if (c->ev_pooled) cudaEventDestroy(c->ev_pooled);
    if (c->cs) cudaStreamDestroy(c->cs);
    delete c;
    return rc;
}

}  // extern "C"

namespace {

// the forward's scratch: the rank's pooled / compressed buffers, then gsa_shard_* scratch
struct ShardFwdBufs {
    float *qc, *kc, *vc, *o_comp, *lse;
    int32_t* topk;
    void* ws;
    size_t ws_bytes, total;
};

int shard_fwd_carve(const gsa_layout* layout, const gsa_params* params, const gsa_shard& sh, int heads, int dim,
                    char* base, ShardFwdBufs* b) {
    const int64_t tpf = (int64_t)layout->grid_h * layout->grid_w, s2 = (int64_t)layout->window_s * layout->window_s;
    const int64_t W = layout->num_frames * tpf / s2, Wg = (sh.frame_end - sh.frame_begin) * tpf / s2;
    int nforced = 0;
    if (params->variant == 1 && params->ref_stride >= 1)
        for (int f = 0; f < layout->num_frames; f += params->ref_stride) nforced += (int)(tpf / s2);
    const int64_t sel = W - nforced;
    const int64_t k_eff = params->top_k < sel ? params->top_k : sel;
    size_t off = 0;
    auto take = [&](size_t bytes) {
        char* p = base ? base + off : nullptr;
        off = align256(off + bytes);
        return p;
    };
    b->qc = reinterpret_cast<float*>(take((size_t)heads * Wg * dim * 4));
    b->kc = reinterpret_cast<float*>(take((size_t)heads * W * dim * 4));
    b->vc = reinterpret_cast<float*>(take((size_t)heads * W * dim * 4));
    b->o_comp = reinterpret_cast<float*>(take((size_t)heads * Wg * dim * 4));
    b->lse = reinterpret_cast<float*>(take((size_t)heads * Wg * 4));
    b->topk = reinterpret_cast<int32_t*>(take((size_t)heads * Wg * (k_eff > 0 ? k_eff : 1) * 4));
    b->ws_bytes = gsa_shard_workspace_bytes(layout, params, &sh, heads, dim);
    if (b->ws_bytes == 0) return err(GSA_ERR_SHAPE_MISMATCH, "gsa_shard_forward: the shard / params were rejected");
    b->ws = take(b->ws_bytes);
    b->total = off + 256;
    return GSA_OK;
}

}  // namespace

extern "C" {

size_t gsa_shard_forward_workspace_bytes(const gsa_layout* layout, const gsa_params* params, int nranks, int rank,
                                         int heads, int dim) {
    gsa_shard sh;
    if (!params || gsa_shard_of_rank(layout, nranks, rank, &sh) != GSA_OK) return 0;
    ShardFwdBufs b{};
    if (shard_fwd_carve(layout, params, sh, heads, dim, nullptr, &b) != GSA_OK) return 0;
    return b.total;
}

int gsa_shard_forward(gsa_comm comm, const gsa_tensor* q_own, const gsa_tensor* k_all, const gsa_tensor* v_all,
                      const gsa_tensor* w_g, const gsa_layout* layout, const gsa_params* params,
                      const gsa_tensor* out_own, int32_t* topk_own, void* workspace, size_t ws_bytes,
                      gsa_stream_t stream) {
    if (!comm) return err(GSA_ERR_GENERIC, "gsa_shard_forward: null communicator");
    if (!q_own || !k_all || !v_all || !params) return err(GSA_ERR_GENERIC, "gsa_shard_forward: null argument");
    gsa_shard sh;
    COMM_TRY(gsa_shard_of_rank(layout, comm->nranks, comm->rank, &sh));
    const int H = q_own->heads, d = q_own->dim;
    // the in-place gathers need whole contiguous row blocks per head
    if (k_all->row_stride != d || v_all->row_stride != d || k_all->head_stride != v_all->head_stride ||
        k_all->dtype != v_all->dtype)
        return err(GSA_ERR_UNSUPPORTED, "gsa_shard_forward: k_all / v_all must be [H][M][d] with contiguous rows "
                                        "and equal strides");
    ShardFwdBufs b{};
    COMM_TRY(shard_fwd_carve(layout, params, sh, H, d, static_cast<char*>(workspace), &b));
    if (!workspace || b.total > ws_bytes + 256)
        return err(GSA_ERR_WORKSPACE, "gsa_shard_forward: workspace %zu < %zu bytes", ws_bytes, b.total);
    const int64_t tpf = (int64_t)layout->grid_h * layout->grid_w, s2 = (int64_t)layout->window_s * layout->window_s;
    const int W = (int)(layout->num_frames * tpf / s2), Wg = (int)((sh.frame_end - sh.frame_begin) * tpf / s2);
    gsa_tensor tqc{b.qc, GSA_DTYPE_F32, H, Wg, d, (int64_t)Wg * d, d};
    gsa_tensor tkc{b.kc, GSA_DTYPE_F32, H, W, d, (int64_t)W * d, d};
    gsa_tensor tvc{b.vc, GSA_DTYPE_F32, H, W, d, (int64_t)W * d, d};
    gsa_tensor toc{b.o_comp, GSA_DTYPE_F32, H, Wg, d, (int64_t)Wg * d, d};
    cudaStream_t st = (cudaStream_t)stream;

    // 1. own windows -> qc_own; own K/V windows at their global rows of kc_all / vc_all
    stage_mark(0, st);
    COMM_TRY(gsa_shard_pool(q_own, k_all, v_all, layout, params, &sh, &tqc, &tkc, &tvc, stream));
    // 2. the gathers, on the communicator's stream after the pooling (which also orders
    //    them after the caller's writes of its own K/V rows): Kc/Vc first, then K/V rows
    std::vector<gsa_gather_op> ops;
    int n_ops = 0;
    COMM_TRY(gsa_shard_gather_plan(layout, comm->nranks, H, d, k_all->head_stride, nullptr, 0, &n_ops));
    ops.resize(n_ops);
    COMM_TRY(gsa_shard_gather_plan(layout, comm->nranks, H, d, k_all->head_stride, ops.data(), n_ops, &n_ops));
    stage_mark(1, st);
    COMM_CUDA(cudaEventRecord(comm->ev_pooled, st));
    COMM_CUDA(cudaStreamWaitEvent(comm->cs, comm->ev_pooled, 0));
    const size_t kv_es = k_all->dtype == GSA_DTYPE_BF16 ? 2 : 4;
    char* bases[4] = {reinterpret_cast<char*>(b.kc), reinterpret_cast<char*>(b.vc), static_cast<char*>(k_all->data),
                      static_cast<char*>(v_all->data)};
    const NcclApi& n = nccl();
    for (int phase = 0; phase < 2; ++phase) {
        COMM_TRY(nccl_status(n.group_start(), "ncclGroupStart"));
        for (const gsa_gather_op& o : ops) {
            if (o.phase != phase || o.count == 0) continue;
            const size_t es = o.buffer < 2 ? 4 : kv_es;
            char* recv = bases[o.buffer] + (size_t)o.offset * es;
            const char* send = recv + (size_t)comm->rank * o.count * es;  // in place
            const ncclResult_t r = n.all_gather(send, recv, (size_t)o.count * es, ncclUint8, comm->comm, comm->cs);
            if (r != ncclSuccess) {
                n.group_end();
                return nccl_status(r, "ncclAllGather");
            }
        }
        COMM_TRY(nccl_status(n.group_end(), "ncclGroupEnd"));
        COMM_CUDA(cudaEventRecord(phase == 0 ? comm->ev_c : comm->ev_kv, comm->cs));
    }
    // 3. compressed attention + top-k of own windows vs all W (waits for Kc/Vc only)
    COMM_CUDA(cudaStreamWaitEvent(st, comm->ev_c, 0));
    stage_mark(2, st);
    int k_eff = 0;
    COMM_TRY(gsa_shard_compress(&tqc, &tkc, &tvc, layout, params, &sh, &toc, b.lse, b.topk, &k_eff, b.ws, b.ws_bytes,
                                stream));
    // 4. own specials + selection + gate + merge (waits for the K/V rows)
    stage_mark(3, st);
    COMM_CUDA(cudaStreamWaitEvent(st, comm->ev_kv, 0));
    COMM_TRY(gsa_shard_attend(q_own, k_all, v_all, w_g, layout, params, &sh, &toc, b.topk, out_own, b.ws, b.ws_bytes,
                              stream));
    stage_mark(4, st);
    if (topk_own && k_eff > 0)
        COMM_CUDA(cudaMemcpyAsync(topk_own, b.topk, (size_t)H * Wg * k_eff * 4, cudaMemcpyDeviceToDevice, st));
    return GSA_OK;
}

}  // extern "C"
