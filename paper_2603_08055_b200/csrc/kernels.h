// kernels.h — host-side launchers of the sm_100a kernels (internal to libgsa_sm100.so).
#pragma once

#include <cuda_runtime.h>

#include "common.cuh"

namespace gsa_sm100 {

// kernels launched by this library (gsa_launch_count); bumped by every launcher
void note_launch(int n = 1);
// sets the calling thread's gsa_last_error_message() and returns status
int report_error(int status, const char* msg);
// gsa_set_stage_events: records stage event i (0..4) on st when enabled on this thread
void stage_mark(int i, cudaStream_t st);

// internal dtype tag (not in the C ABI): fp16 operand planes made by launch_v16
constexpr int kDtypeF16 = 100;

struct TensorRef {  // device view, element strides
    const void* data;
    int dtype;
    int64_t hs, rs;
};

// ---- K1: window mean pooling (pool.cu) ----------------------------------
struct PoolJob {
    TensorRef in;      // image rows only (row 0 == first image token)
    float* out;        // [H][W][d] f32 (head stride W*d)
    __nv_bfloat16* hi; // optional split copies for the tensor-core path [H][W][d]
    __nv_bfloat16* lo;
    float* norm;       // optional ||row||_2 [H][W]
    int64_t out_hs;    // head stride of out (elements); 0 = W*d (contiguous). hi/lo/norm assume contiguous
};
cudaError_t launch_pool(const PoolJob* jobs, int njobs, int heads, int dim, const DevLayout& L,
                        float inv, cudaStream_t st);

// ---- dense / compressed attention on CUDA cores (attn_f32.cu) -------------
// out rows are written at out + h*out_hs + r*out_rs. TOPK variant also keeps
// per-row top-k (exact scaled_dot order) with the reference tie rule.
struct AttnArgs {
    TensorRef q, k, v;
    int heads, mq, mk, dim;
    float scale;
    float* out;
    int64_t out_hs, out_rs;
    float* lse;  // [H][mq] (nullable)
    // top-k (nullable indices => plain attention)
    int32_t* topk;
    float* guide;
    int k_eff;
    const uint8_t* excluded;  // [mk] or null
    // fallback mode for the tensor-core compressed kernel: CTA b recomputes the
    // 64-row block block_list[b] (= h * ceil(mq/64) + tile) if b < *block_count,
    // writing only top-k indices / guide scores
    const int* block_list;
    const int* block_count;
    bool topk_only;
    // set by the launcher when the per-row top-k lists do not fit in shared memory
    float* glist_s;
    int* glist_i;
};
cudaError_t launch_attn_f32(const AttnArgs& a, cudaStream_t st);

// ---- selection branch on CUDA cores (select_f32.cu) ---------------------
struct SelectArgs {
    TensorRef q, k, v;  // image rows
    TensorRef ql, kl;   // tensor-core path, f32 inputs: bf16 lo planes (q/k then hold the hi planes)
    // tensor-core path: V as fp16(v * 2^-vexp(vmax_h)) planes [H][rows][64] (v16l: the f32
    // remainder, null for bf16 inputs), image rows of the key side; made by run_select when null
    TensorRef v16, v16l;
    const unsigned* vmax;
    int heads, dim;
    DevLayout L;        // query side: windows / tokens of q, rows, o_comp, out (a view shard's own frames)
    DevLayout Lkv;      // key side: the frames k/v cover and window ids refer to (== L unsharded)
    RowSource rows;
    float scale;
    float* out;  // o_sel or merged output
    int64_t out_hs, out_rs;
    float* lse;  // [H][Mi] nullable
    // optional fused gate + merge: out = g*o_comp[w] + (1-g)*o_sel
    const float* w_g;     // [H][d][d] f32 or null
    const float* o_comp;  // [H][W][d] f32
    float* o_sel_ctx;     // optional materialised o_sel [H][Mi][d]
    float* gate_ctx;      // optional materialised gate [H][Mi][d]
    uint8_t* wg_prep;     // tensor-core path scratch: W_g hi/lo split, H * 16 KB
    // hybrid fast path: softmax already taken over the reference-frame keys by a dense
    // pass (normalised output and natural-log LSE per image token); the plan rows then
    // hold only the dynamic windows and the epilogue merges the two partial softmaxes
    const float* prior_o;    // [H][Mi][d] f32 or null
    const float* prior_lse;  // [H][Mi]
};
cudaError_t launch_select_f32(const SelectArgs& a, cudaStream_t st);

// ---- exact per-head projection (project.cu) ------------------------------
struct ProjectMats {
    const float* w[3];  // [H][C][d] f32
    void* out[3];       // [H][tokens][d] (f32 or bf16)
    int64_t out_hs[3], out_rs[3];
};
cudaError_t launch_project(const float* x, int tokens, int C, const ProjectMats& mats, int nmats, int heads, int dim,
                           bool bf16_out, cudaStream_t st);

// ---- gate, upsample, plan helpers (misc.cu) -----------------------------
// V (f32 or bf16, any strides) -> per-head max |v| (float bits, vmax zeroed by the caller's
// memset inside) and contiguous fp16 planes hi = fp16(v * 2^-e_h), lo = fp16(v * 2^-e_h - hi)
// (lo only for f32 and when non-null), e_h = ilogb(vmax_h) - 13
cudaError_t launch_v16(const TensorRef& v, int heads, int rows, unsigned* vmax, __half* hi, __half* lo,
                       cudaStream_t st);
// n contiguous elements f32 <-> bf16 (RNE) or a same-dtype copy
cudaError_t launch_convert(const void* src, int src_dtype, void* dst, int dst_dtype, int64_t n, cudaStream_t st);
// [H][rows][64] rows (f32 or bf16, any strides) -> contiguous bf16 hi (+ lo for f32) planes
cudaError_t launch_pack_rows(const TensorRef& in, int heads, int rows, __nv_bfloat16* hi, __nv_bfloat16* lo,
                             cudaStream_t st);
cudaError_t launch_gate(const TensorRef& q, int heads, int rows, int dim, const float* w_g,
                        float* g, int64_t g_hs, int64_t g_rs, cudaStream_t st);
cudaError_t launch_upsample(const float* coarse, int64_t c_hs, int64_t c_rs, int heads, int dim,
                            const DevLayout& L, float* out, int64_t o_hs, int64_t o_rs,
                            cudaStream_t st);
cudaError_t launch_forced(const DevLayout& L, int ref_stride, int32_t* forced, uint8_t* mask,
                          cudaStream_t st);
cudaError_t launch_plan_count(const int32_t* topk, int64_t rows, int k, const uint8_t* mask,
                              int n_forced, int n_windows, int64_t* sizes, int* flag, cudaStream_t st);
cudaError_t launch_plan_fill(const int32_t* topk, int64_t rows, int k, const uint8_t* mask,
                             const int32_t* forced, int n_forced, int n_windows, const int64_t* offsets,
                             int32_t* ids, cudaStream_t st);
cudaError_t launch_scan_offsets(const int64_t* sizes, int64_t n, int64_t* offsets, void* tmp,
                                size_t tmp_bytes, cudaStream_t st);
size_t scan_offsets_tmp_bytes(int64_t n);
// flag |= 1: empty plan row; flag |= 2: window id outside [0, n_windows) (ids may be null: rows only)
cudaError_t launch_plan_check(const int64_t* offsets, int64_t rows, const int32_t* ids, int n_windows, int* flag,
                              cudaStream_t st);

// ---- layer backward (backward.cu), f32 ------------------------------------
struct FMat {  // read-only f32 [H][rows][d] view, element strides
    const float* p;
    int64_t hs, rs;
};
struct FOut {  // writable f32 [H][rows][d] view
    float* p;
    int64_t hs, rs;
};
// gate fuse + upsample backward, one CTA per (head, window)
struct GateBwdArgs {
    FMat dout;                    // [H][M][d] (image rows at num_special..)
    const float *gate, *o_sel;    // [H][Mi][d]
    const float *o_comp, *w_g;    // [H][W][d], [H][d][d]
    DevLayout L;
    int dim;
    float *ds, *dz;               // [H][Mi][d]: (1-g) dO, g(1-g)(O_comp-O_sel) dO
    float *d_oc, *d_sel, *d_comp; // [H][W][d] window sums of g dO; D rows [H][Mi], [H][W]
    FOut dq;                      // image rows written with W_g dz
};
cudaError_t launch_gate_bwd(const GateBwdArgs& a, int heads, cudaStream_t st);
// FlashAttention-2 style backward of dense softmax attention from saved LSE rows;
// dq / dk (+dv) passes run when the pointer is non-null
struct DenseBwdArgs {
    FMat q, k, v, dout;
    const float *lse, *D;
    int64_t lse_hs, D_hs;
    int64_t nq, nk;
    int dim;
    float scale;
    FOut dq, dk, dv;
    bool accumulate;  // += into the outputs instead of =
    // query side split over keys (k_splits > 1): partial dQ [k_splits][H][nq][dim] in dq_part,
    // summed in split order by a reduction (dense_dq_splits picks the count)
    int k_splits;
    float* dq_part;
    int64_t k_chunk;  // set by the launcher
    int heads;        // set by the launcher
};
int dense_dq_splits(int heads, int64_t nq, int64_t nk);
cudaError_t launch_dense_bwd(const DenseBwdArgs& a, int heads, cudaStream_t st);
struct PoolBwdArgs {
    int heads;
    int64_t rows;  // all M rows of dq/dk/dv
    int dim;
    DevLayout L;
    float inv;
    const float *dqc, *dkc, *dvc;  // [H][W][d]
    FOut dq, dk, dv;
};
cudaError_t launch_pool_bwd(const PoolBwdArgs& a, cudaStream_t st);
struct SelBwdArgs {
    FMat q, k, v;                  // full rows (image rows at num_special..)
    const float *ds, *lse, *D;     // [H][Mi][d], [H][Mi], [H][Mi]
    const int64_t* offsets;        // plan CSR [H*W+1]
    const int32_t* ids;
    const int64_t* inv_offsets;    // inverse plan CSR [H*W+1]: query windows per key window
    const int32_t* inv_q;
    DevLayout L;
    int dim;
    float scale;
    FOut dq, dk, dv;               // accumulated into (image rows)
};
cudaError_t launch_sel_bwd(const SelBwdArgs& a, int heads, cudaStream_t st);
size_t inverse_plan_tmp_bytes(int64_t rows, int64_t entries);
cudaError_t launch_inverse_plan(const int64_t* offsets, const int32_t* ids, int64_t rows, int W, int64_t entries,
                                unsigned long long* keys, unsigned long long* keys_sorted, int64_t* counts,
                                int64_t* inv_offsets, int32_t* inv_q, void* tmp, size_t tmp_bytes,
                                cudaStream_t st);
// out[h] (R x N) = A[h]^T B[h] over `rows` rows, split `splits` ways with a fixed-order reduction
struct AtbArgs {
    const float *A, *B;
    int64_t a_hs, a_rs, b_hs, b_rs;
    int R, N;
    int64_t rows, chunk;
    int splits;
    float* part;  // [H][splits][R][N]
};
int atb_splits(int heads, int R, int N, int64_t rows);
cudaError_t launch_atb(AtbArgs a, int heads, float* out, cudaStream_t st);
struct DxArgs {
    const float* g[3];  // dQ, dK, dV [H][tokens][d] contiguous
    const float* w[3];  // W_q, W_k, W_v [H][C][d]
    int heads, dim, C;
    int64_t tokens;
    float* dx;          // [tokens][C]
};
cudaError_t launch_dx_gemm(const DxArgs& a, cudaStream_t st);
cudaError_t launch_to_f32(const TensorRef& in, int heads, int64_t rows, int dim, float* out, cudaStream_t st);
cudaError_t launch_pool_adjoint(const FMat& in, int heads, int dim, const DevLayout& L, float inv, const FOut& out,
                                cudaStream_t st);
cudaError_t launch_window_sum(const FMat& in, int heads, int dim, const DevLayout& L, const FOut& out, cudaStream_t st);
// hybrid backward: the plan without its forced windows (mask[w] = 1 for forced), forced-frame
// rows of bf16 planes gathered contiguously, their dK / dV added back to dk / dv
cudaError_t launch_plan_drop(const int64_t* offsets, const int32_t* ids, int64_t rows, const uint8_t* mask, int W,
                             int64_t* sizes, int64_t* out_offsets, int32_t* out_ids, void* tmp, size_t tmp_bytes,
                             cudaStream_t st);
cudaError_t launch_forced_gather(const __nv_bfloat16* src, int64_t src_hs, int heads, const DevLayout& L, int ref_stride,
                                 int64_t rows, __nv_bfloat16* dst, cudaStream_t st);
cudaError_t launch_forced_scatter_add(const float* gk, const float* gv, int heads, const DevLayout& L, int ref_stride,
                                      int64_t rows, const FOut& dk, const FOut& dv, cudaStream_t st);
cudaError_t launch_rowdot(const FMat& a, const FMat& b, int heads, int rows, int dim, float* out, cudaStream_t st);

}  // namespace gsa_sm100
