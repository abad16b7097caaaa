// tc.h — entry points of the tensor-core (tcgen05/TMEM/TMA) fast paths and
// their shape predicates. Callers fall back to the CUDA-core kernels when a
// predicate is false (f32 inputs, head dim != 64, window side != 4, ...).
#pragma once

#include "kernels.h"

namespace gsa_sm100 {

// the largest per-row top-k budget (k_eff) the selection implements: up to 128 on the
// tensor-core streaming path, up to 2048 with a shared sort buffer, up to 10240 with a
// block radix sort (compress_tc.cu, HK_KMAX)
constexpr int kMaxTopK = 10240;

// dense attention (special tokens, tiled_attention, dense baseline)
bool tc_dense_supported(const gsa_tensor& q, const gsa_tensor& k, const gsa_tensor& v);
// with_v16: room for converting V (false when the caller passes its V16 planes)
size_t tc_dense_workspace_bytes(int heads, int mq, int mk, bool with_v16 = true);
// V16/vmax: V already as fp16 planes [H][k.rows][64] (launch_v16), else converted here
cudaError_t tc_dense_attention(const gsa_tensor& q, const gsa_tensor& k, const gsa_tensor& v, float scale,
                               int q_row_offset, int mq, float* out, int64_t out_hs, int64_t out_rs,
                               int out_row_offset, float* lse, void* ws, size_t ws_bytes, cudaStream_t st,
                               const __half* v16 = nullptr, const unsigned* vmax = nullptr);

// compressed attention + top-k over pooled f32 [H][W][d] tensors: tensor-core
// approximate scores + exact re-scoring of the boundary candidates when
// supported, else the exact CUDA-core kernel. Indices are bit-exact either way.
size_t tc_compress_workspace_bytes(int heads, int windows, int dim, int k_eff);
// query rows wq (a shard's windows) against wk key windows
size_t tc_compress_workspace_bytes_qk(int heads, int wq, int wk, int dim, int k_eff);
// pre-split query operands (bf16 hi/lo of contiguous [H][W][64] Qc + row norms), written
// by the pooling kernel; carved from the compress workspace
struct CompressSplits {
    __nv_bfloat16 *qh, *ql;
    float* qnorm;
};
bool tc_compress_split_buffers(void* ws, size_t ws_bytes, int heads, int windows, int dim, int k_eff,
                               CompressSplits* out);
cudaError_t tc_compress_topk_splits(const CompressSplits* pre, const gsa_tensor& qc, const gsa_tensor& kc,
                                    const gsa_tensor& vc, int k_eff, float scale, const uint8_t* excluded,
                                    float* out, int64_t out_hs, int64_t out_rs, float* lse, int32_t* topk,
                                    float* guide, void* ws, size_t ws_bytes, cudaStream_t st);
cudaError_t tc_compress_topk(const gsa_tensor& qc, const gsa_tensor& kc, const gsa_tensor& vc, int k_eff,
                             float scale, const uint8_t* excluded, float* out, int64_t out_hs,
                             int64_t out_rs, float* lse, int32_t* topk, float* guide, void* ws,
                             size_t ws_bytes, cudaStream_t st);

// dense attention of f32 Q/K/V on tensor cores (the compressed-branch kernel without a
// top-k): the f32 special path, tiled_attention and the pinned-plan compressed branch.
// Without a large enough workspace the scratch is allocated stream-ordered.
size_t tc_dense_f32_workspace_bytes(int heads, int mq, int mk);
cudaError_t tc_dense_f32(const gsa_tensor& q, int q_row_offset, int mq, const gsa_tensor& k, const gsa_tensor& v,
                         float scale, float* out, int64_t out_hs, int64_t out_rs, float* lse, void* ws,
                         size_t ws_bytes, cudaStream_t st);

// selection branch (block_sparse_attention), with the gate + merge fused when a.w_g is set;
// bf16 Q/K/V, or f32 as bf16 hi/lo planes (a.ql/kl/vl set: 3-term products)
bool tc_select_supported(const SelectArgs& a);
size_t tc_select_workspace_bytes(int heads);
cudaError_t tc_select(const SelectArgs& a, cudaStream_t st);

// dense projection of the stack driver: C[M][N] bf16 = A[M][K] . Bt[N][K]^T (gemm.cu);
// N % 32 == 0, K % 64 == 0; and the stack's residual y = bf16(x + o)
bool tc_gemm_supported(int M, int N, int K);
cudaError_t tc_gemm_bf16(const __nv_bfloat16* a, int64_t lda, const __nv_bfloat16* bt, int64_t ldb, __nv_bfloat16* c,
                         int64_t ldc, int M, int N, int K, cudaStream_t st);
cudaError_t launch_residual_bf16(const __nv_bfloat16* x, const float* o, __nv_bfloat16* y, int64_t n, cudaStream_t st);

// dense passes of the layer backward (bwd_tc.cu), head dim 64: operands as contiguous bf16
// planes [H][rows][64] (hi, plus lo for f32 operands; lo == nullptr: the operand is exactly
// bf16); dK/dV (key side) and/or dQ (query side, optionally split over keys into dq_part
// [splits][H][n_q][64] and reduced in order) as f32 rows with 16-byte aligned strides
struct BwdTcArgs {
    int heads;
    int64_t n_q, n_k;
    float scale;
    const __nv_bfloat16 *q_hi, *q_lo, *k_hi, *k_lo, *v_hi, *v_lo, *do_hi, *do_lo;
    int64_t q_hs, k_hs, v_hs, do_hs;  // plane head strides in elements (0: rows * 64)
    const float *lse, *D;  // [H][n_q]
    float* dq;
    int64_t dq_hs, dq_rs;
    bool accumulate_q;
    float* dq_part;
    int dq_splits;
    float *dk, *dv;
    int64_t dk_hs, dk_rs, dv_hs, dv_rs;
    bool accumulate_kv;
};
bool tc_bwd_supported(int dim);
int tc_bwd_dq_splits(int heads, int64_t n_q, int64_t n_k);
cudaError_t launch_bwd_tc(const BwdTcArgs& a, cudaStream_t st);

// projection backward (proj_bwd_tc.cu), head dim 64: dX = sum G W^T and dW = X^T G with
// f32 operands as bf16 hi / lo planes (3-term products); scratch from the caller
bool tc_proj_bwd_supported(int dim, int model_dim);
size_t tc_proj_bwd_workspace_bytes(int tokens, int model_dim, int heads);
cudaError_t launch_proj_bwd_tc(const float* x, int tokens, int C, const float* const w[3], int heads,
                               const float* const g[3], float* dx, float* const dw[3], void* ws, cudaStream_t st);

// selection-branch backward (sel_bwd_tc.cu), head dim 64, window side 4: bf16 planes of the
// image rows (row 0 = image token 0; lo.p == nullptr: no lo plane), dS_sel hi / lo, the plan
// and its inverse; dq / dk / dv rows (specials first) are accumulated into
struct BwdPlane {
    const __nv_bfloat16* p;
    int64_t hs, rs;
};
struct SelBwdTcArgs {
    DevLayout L;
    int heads;
    float scale;
    BwdPlane q_hi, q_lo, k_hi, k_lo, v_hi, v_lo, ds_hi, ds_lo;
    const float *lse, *D;  // [H][Mi]
    const int64_t* offsets;
    const int32_t* ids;
    const int64_t* inv_offsets;
    const int32_t* inv_q;
    float *dq, *dk, *dv;
    int64_t dq_hs, dq_rs, dk_hs, dk_rs, dv_hs, dv_rs;
};
bool tc_sel_bwd_supported(int dim, int s);
cudaError_t launch_sel_bwd_tc(const SelBwdTcArgs& a, cudaStream_t st);

}  // namespace gsa_sm100
