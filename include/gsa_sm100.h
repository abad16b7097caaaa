/*
 * gsa_sm100.h — C ABI of the B200 (sm_100a) Global Sparse Attention library
 * (libgsa_sm100.so). This is the drop-in boundary: the C++ operator API in
 * include/gsa/ (same names and signatures as the reference's
 * proj/include/gsa) forwards to these entry points, and so can any FFI.
 *
 * Conventions
 *  - Plain C: no exceptions, no torch types. Every entry point returns a
 *    gsa_status; gsa_last_error_message() gives the detail of the last failure
 *    on the calling thread. Status values mirror the reference's exception
 *    classes (proj/include/gsa/errors.hpp:8-58).
 *  - All tensor data pointers are DEVICE pointers. Compute calls are
 *    stream-ordered on `stream`, do no allocation and no host synchronisation
 *    unless the comment says so. Scratch memory is caller-owned (`workspace`);
 *    query its size with the matching *_workspace_bytes function.
 *  - Deterministic: no floating-point atomics reach any output; repeated calls
 *    on the same inputs are bitwise identical.
 *  - Top-k indices are bit-exact with the reference CPU implementation:
 *    pooled Qc/Kc are summed in ascending member order (compression.hpp:29-35),
 *    guide scores follow scaled_dot's 4-lane order without FMA (dot.hpp:11-23),
 *    rows are ordered by (score desc, index asc) (compression.hpp:67-73).
 *
 * Reference interface replaced by each entry point (file:line under
 * /root/reference/proj) is cited on the declaration.
 */
#ifndef GSA_SM100_H
#define GSA_SM100_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GSA_SM100_ABI_VERSION 1

typedef struct CUstream_st* gsa_stream_t; /* == cudaStream_t */

typedef enum {
    GSA_OK = 0,
    GSA_ERR_GENERIC = 1,            /* GsaError           errors.hpp:8   */
    GSA_ERR_SHAPE_MISMATCH = 2,     /* ShapeMismatch      errors.hpp:12  */
    GSA_ERR_DIVISIBILITY = 3,       /* DivisibilityError  errors.hpp:16  */
    GSA_ERR_ZERO_SIZE = 4,          /* ZeroSizeError      errors.hpp:20  */
    GSA_ERR_INDEX_OUT_OF_RANGE = 5, /* IndexOutOfRange    errors.hpp:24  */
    GSA_ERR_NON_FINITE = 6,         /* NonFiniteInput     errors.hpp:28  */
    GSA_ERR_INVALID_TILING = 7,     /* InvalidTiling      errors.hpp:32  */
    GSA_ERR_INVALID_STRIDE = 8,     /* InvalidStride      errors.hpp:36  */
    GSA_ERR_EMPTY_SELECTION = 9,    /* EmptySelection     errors.hpp:40  */
    GSA_ERR_UNSUPPORTED = 10,       /* shape outside what the sm_100a kernels implement */
    GSA_ERR_CUDA = 11,              /* CUDA runtime / launch failure */
    GSA_ERR_WORKSPACE = 12,         /* workspace too small or misaligned */
    GSA_ERR_NCCL = 13,              /* NCCL failure in the multi-GPU layer (gsa_comm_*, gsa_shard_forward) */
    GSA_ERR_CONTEXT_MISMATCH = 14   /* ContextMismatch    errors.hpp:44  (gsa_backward's saved state) */
} gsa_status;

typedef enum { GSA_DTYPE_F32 = 0, GSA_DTYPE_BF16 = 1 } gsa_dtype;

/* A [heads x rows x dim] view of device memory (tensor.hpp:15-42 Tensor<T>,
 * head-major). Strides are in ELEMENTS; dim is contiguous. */
typedef struct {
    void* data;
    int32_t dtype; /* gsa_dtype */
    int32_t heads, rows, dim;
    int64_t head_stride, row_stride;
} gsa_tensor;

/* layout.hpp:13-40 TokenLayout */
typedef struct {
    int32_t num_special, num_frames, grid_h, grid_w, window_s;
} gsa_layout;

/* types.hpp:58-65 GsaParams (+ KernelTiling 13-16). variant: 0 plain, 1 hybrid. */
typedef struct {
    int32_t window_s, top_k;
    double scale; /* 0 => 1/sqrt(dim) (reference.hpp:22-26) */
    int32_t variant, ref_stride;
    int32_t block_m, block_n; /* validated like validate_tiling (types.hpp:20-25) */
} gsa_params;

/* Device pointers for the ForwardContext fields (layer.hpp:124-142) the
 * caller wants materialised; any may be NULL. Shapes: qc/kc/vc/o_comp
 * [H][W][d] f32, lse_comp [H][W], topk [H][W][k_eff] int32, o_sel/gate
 * [H][Mi][d] f32, lse_sel [H][Mi], lse_spec [H][Ms]. */
typedef struct {
    float *qc, *kc, *vc, *o_comp, *lse_comp;
    int32_t* topk;
    float *o_sel, *lse_sel, *gate, *lse_spec;
} gsa_context;

int gsa_abi_version(void);
const char* gsa_status_string(int status);
const char* gsa_last_error_message(void);

/* build_token_layout (layout.cpp:7-24): validates and fills *out. */
int gsa_make_layout(int num_special, int num_frames, int grid_h, int grid_w, int window_s,
                    gsa_layout* out);
/* validate_params (types.hpp:67-73) + window_s consistency (layer.hpp:182-183). */
int gsa_validate_params(const gsa_params* params, const gsa_layout* layout);

/* avg_pool_tokens (compression.hpp:20-38). x_img: rows == image tokens (f32 or
 * bf16). out: f32 [H][W][d]. Bit-exact with the reference. */
int gsa_avg_pool_tokens(const gsa_tensor* x_img, const gsa_layout* layout, const gsa_tensor* out,
                        gsa_stream_t stream);

/* upsample_nearest (compression.hpp:42-53). coarse f32 [H][W][d] -> out f32 [H][Mi][d]. */
int gsa_upsample_nearest(const gsa_tensor* coarse, const gsa_layout* layout, const gsa_tensor* out,
                         gsa_stream_t stream);

/* tiled_attention (compression.hpp:99-165): out = softmax(q k^T * scale) v (f32),
 * lse [H][mq] = m + log(l). q/k/v f32 or bf16. */
int gsa_tiled_attention(const gsa_tensor* q, const gsa_tensor* k, const gsa_tensor* v, float scale,
                        int block_m, int block_n, const gsa_tensor* out, float* lse,
                        gsa_stream_t stream);

/* special_token_attention (layer.hpp:80-96): dense attention of the special
 * queries over ALL keys. Empty q_spec is a no-op. */
int gsa_special_token_attention(const gsa_tensor* q_spec, const gsa_tensor* k, const gsa_tensor* v,
                                float scale, const gsa_tensor* out, float* lse,
                                gsa_stream_t stream);

/* fused_compressed_attention_topk (compression.hpp:180-297). qc/kc/vc f32
 * [H][W][d]; excluded: device byte mask [W] or NULL; out f32 [H][W][d]; lse
 * [H][W]; indices [H][W][k_eff]; guide_scores (nullable) [H][W][k_eff] f32.
 * *k_eff_out (host) = min(k, selectable). Indices are bit-exact; k_eff up to
 * 10240 (above 128 the selection runs on exact CUDA-core scores; above 10240 the
 * call returns GSA_ERR_UNSUPPORTED). With an
 * exclusion mask the call synchronises `stream` (k_eff needs the mask's count). */
size_t gsa_compressed_attention_topk_workspace_bytes(int heads, int windows, int dim, int k);
int gsa_compressed_attention_topk(const gsa_tensor* qc, const gsa_tensor* kc, const gsa_tensor* vc,
                                  int k, float scale, int block_m, int block_n,
                                  const uint8_t* excluded, int n_excluded, const gsa_tensor* out,
                                  float* lse, int32_t* indices, float* guide_scores, int* k_eff_out,
                                  void* workspace, size_t workspace_bytes, gsa_stream_t stream);

/* forced_windows_of (selection.cpp:14-21): writes the ascending forced window
 * ids into forced (device, capacity >= count) and their count (host). */
int gsa_forced_windows(const gsa_layout* layout, int ref_stride, int32_t* forced, int* count,
                       gsa_stream_t stream);

/* build_selection_plan (selection.cpp:29-67): device CSR plan from device
 * top-k rows [H][rows][k]. offsets [H*rows+1] int64; window_ids capacity
 * ids_capacity (plain: H*rows*k; hybrid: H*rows*(F+k) suffices). *n_ids
 * (host) is the realised size; this call synchronises `stream`. A top-k id
 * outside [0, W) is IndexOutOfRange. */
int gsa_build_selection_plan(const int32_t* topk, int heads, int rows, int k,
                             const gsa_layout* layout, int variant, int ref_stride,
                             int64_t* offsets, int32_t* window_ids, int64_t ids_capacity,
                             int64_t* n_ids, void* workspace, size_t workspace_bytes,
                             gsa_stream_t stream);
size_t gsa_build_selection_plan_workspace_bytes(int heads, int rows, int k,
                                                const gsa_layout* layout, int ref_stride);

/* block_sparse_attention (selection.hpp:63-136) over a device CSR plan.
 * Validates the plan before any compute (synchronises `stream`): an empty row
 * is EmptySelection (selection.hpp:82-85), a window id outside [0, W) is
 * IndexOutOfRange (tokens_of_window, layout.cpp:37-56). The 4-byte flag for it
 * is a stream-ordered cudaMallocAsync, the one allocation in the library
 * (gsa_forward builds its own plan and needs no check).
 * out f32 [H][Mi][d], lse [H][Mi]. */
int gsa_block_sparse_attention(const gsa_tensor* q_img, const gsa_tensor* k_img,
                               const gsa_tensor* v_img, const int64_t* offsets,
                               const int32_t* window_ids, const gsa_layout* layout, float scale,
                               const gsa_tensor* out, float* lse, gsa_stream_t stream);

/* gate (layer.hpp:99-119): g = sigmoid(q . w_g[h]); w_g f32 [H][d][d]; g f32. */
int gsa_gate(const gsa_tensor* q_img, const gsa_tensor* w_g, const gsa_tensor* g,
             gsa_stream_t stream);

/* gsa_forward (layer.hpp:177-230) from projected Q/K/V: special path, pooling,
 * compressed attention + top-k, selection plan, block-sparse attention, gate,
 * gated merge and concat, all on the device, no host sync. q/k/v [H][M][d]
 * (bf16 is the fast path); w_g f32 [H][d][d]; out f32 [H][M][d]. ctx may be NULL. */
size_t gsa_forward_workspace_bytes(const gsa_layout* layout, const gsa_params* params, int heads,
                                   int dim);
int gsa_forward(const gsa_tensor* q, const gsa_tensor* k, const gsa_tensor* v,
                const gsa_tensor* w_g, const gsa_layout* layout, const gsa_params* params,
                const gsa_tensor* out, const gsa_context* ctx, int* k_eff_out, void* workspace,
                size_t workspace_bytes, gsa_stream_t stream);

/* gsa_forward_with_plan (layer.hpp:235-262): selection pinned to a device CSR
 * plan; the compressed branch is plain tiled attention (no top-k, so no budget
 * limit and no params.window_s check, as in the reference). The plan is
 * validated like gsa_block_sparse_attention's (synchronises `stream`). */
int gsa_forward_with_plan(const gsa_tensor* q, const gsa_tensor* k, const gsa_tensor* v,
                          const gsa_tensor* w_g, const gsa_layout* layout,
                          const gsa_params* params, const int64_t* offsets,
                          const int32_t* window_ids, const gsa_tensor* out, void* workspace,
                          size_t workspace_bytes, gsa_stream_t stream);

/* ---------------------------------------------------------------------------
 * View-sharded layer (multi-GPU; no reference counterpart — the reference is a
 * single-process CPU library). A rank owns frames [frame_begin, frame_end) and
 * special rows [special_begin, special_end) of the global layout. Per layer:
 *   1. gsa_shard_pool: own Q windows -> qc_own; own K/V windows written at their
 *      global rows of kc_all / vc_all ([H][W][d] f32), ready for an in-place
 *      all-gather. k_all / v_all hold the rank's own rows at their global
 *      positions (the K/V all-gather may run concurrently: pooling only reads
 *      own rows).
 *   2. (all-gather kc_all, vc_all) gsa_shard_compress: own query windows against
 *      all W windows; topk_own [H][W_g][k_eff] holds GLOBAL window ids, bit-exact
 *      with the unsharded layer.
 *   3. (all-gather k_all, v_all) gsa_shard_attend: own special rows over all M
 *      keys, own windows' selection + gate + merge; out_own [H][Ms_g + Mi_g][d]
 *      f32 = the rank's rows of the unsharded output (specials first).
 * q_own: [H][Ms_g + Mi_g][d] (own specials, then own image rows). */
typedef struct {
    int32_t frame_begin, frame_end, special_begin, special_end;
} gsa_shard;

size_t gsa_shard_workspace_bytes(const gsa_layout* layout, const gsa_params* params, const gsa_shard* shard,
                                 int heads, int dim);
int gsa_shard_pool(const gsa_tensor* q_own, const gsa_tensor* k_all, const gsa_tensor* v_all,
                   const gsa_layout* layout, const gsa_params* params, const gsa_shard* shard,
                   const gsa_tensor* qc_own, const gsa_tensor* kc_all, const gsa_tensor* vc_all,
                   gsa_stream_t stream);
int gsa_shard_compress(const gsa_tensor* qc_own, const gsa_tensor* kc_all, const gsa_tensor* vc_all,
                       const gsa_layout* layout, const gsa_params* params, const gsa_shard* shard,
                       const gsa_tensor* o_comp_own, float* lse_own, int32_t* topk_own, int* k_eff_out,
                       void* workspace, size_t workspace_bytes, gsa_stream_t stream);
int gsa_shard_attend(const gsa_tensor* q_own, const gsa_tensor* k_all, const gsa_tensor* v_all,
                     const gsa_tensor* w_g, const gsa_layout* layout, const gsa_params* params,
                     const gsa_shard* shard, const gsa_tensor* o_comp_own, const int32_t* topk_own,
                     const gsa_tensor* out_own, void* workspace, size_t workspace_bytes,
                     gsa_stream_t stream);

/* ---------------------------------------------------------------------------
 * Multi-GPU layer at the C level (one process per GPU, NCCL over NVLink/NVSwitch).
 *
 * gsa_shard_of_rank: the rank's shard -- equal contiguous blocks of views and of
 * special rows (num_frames and num_special must divide by nranks: every gather is
 * then a plain equal-count all-gather).
 *
 * gsa_shard_gather_plan: the in-place all-gathers that complete a rank's buffers,
 * identical on every rank. Op i gathers `count` elements per rank into buffer
 * `buffer` at element offset `offset` (rank r's block at offset + r * count); buffers
 * 0/1 = kc_all/vc_all (f32 [H][W][d]), 2/3 = k_all/v_all ([H][M][d], rows contiguous,
 * head stride kv_head_stride elements). phase 0 (Kc/Vc) gates gsa_shard_compress,
 * phase 1 (K/V rows) gates gsa_shard_attend. torch.distributed callers (dist.py)
 * and gsa_shard_forward run the same plan.
 *
 * gsa_comm_*: an NCCL communicator. libnccl.so.2 is resolved at run time (inside a
 * PyTorch process that is the library torch already loaded); the id is
 * NCCL_UNIQUE_ID_BYTES = 128 bytes, made by rank 0 and broadcast by the caller.
 * The communicator binds to the device current at gsa_comm_init. Failures are
 * GSA_ERR_NCCL.
 *
 * gsa_shard_forward: the whole view-sharded layer on this rank: pool own windows ->
 * Kc/Vc all-gather -> compressed attention + top-k of own windows vs all W (global
 * ids) -> own specials + selection + gate + merge, with the K/V-row all-gather on
 * the communicator's own stream overlapping the compressed branch (event-ordered,
 * no host sync). q_own [H][Ms_g + Mi_g][d] (own specials, then own image rows);
 * k_all / v_all [H][M][d] hold the rank's own rows, the rest is filled in place;
 * out_own f32 = the rank's rows of the unsharded output; topk_own (nullable, device,
 * [H][W_g][k_eff]) receives the rank's top-k rows. Bit-exact top-k with gsa_forward. */
typedef struct {
    int32_t buffer, phase;
    int64_t offset, count;
} gsa_gather_op;
typedef struct gsa_comm_st* gsa_comm;

int gsa_shard_of_rank(const gsa_layout* layout, int nranks, int rank, gsa_shard* out);
int gsa_shard_gather_plan(const gsa_layout* layout, int nranks, int heads, int dim, int64_t kv_head_stride,
                          gsa_gather_op* ops, int capacity, int* n_ops);
int gsa_comm_get_unique_id(void* id /* 128 bytes */);
int gsa_comm_init(gsa_comm* comm, const void* id /* 128 bytes */, int nranks, int rank);
int gsa_comm_destroy(gsa_comm comm);
size_t gsa_shard_forward_workspace_bytes(const gsa_layout* layout, const gsa_params* params, int nranks, int rank,
                                         int heads, int dim);
int gsa_shard_forward(gsa_comm comm, const gsa_tensor* q_own, const gsa_tensor* k_all, const gsa_tensor* v_all,
                      const gsa_tensor* w_g, const gsa_layout* layout, const gsa_params* params,
                      const gsa_tensor* out_own, int32_t* topk_own, void* workspace, size_t workspace_bytes,
                      gsa_stream_t stream);

/* project_qkv (layer.hpp:48-76): q/k/v[h][t][j] = sum_a x[t][a] * w[h][a][j], a
 * ascending, products and sums rounded separately (the reference's arithmetic,
 * so f32 outputs are bit-identical to it). x: device [tokens][model_dim] f32;
 * w_*: device [heads][model_dim][dim] f32; outputs f32 (exact) or bf16 (RNE of
 * the exact value). Adjacent to the hot path. */
int gsa_project_qkv(const float* x, int tokens, int model_dim, const float* w_q, const float* w_k,
                    const float* w_v, int heads, int dim, const gsa_tensor* q, const gsa_tensor* k,
                    const gsa_tensor* v, gsa_stream_t stream);

/* The L-layer stack driver's per-layer maps (BASELINE configs[2]), on
 * tensor cores. gsa_project_qkv_bf16: qkv[t][n] = sum_a x[t][a] * W[a][n] with bf16
 * x [tokens][model_dim] (row stride ldx), the weight given TRANSPOSED w_qkv_t
 * [n_out][model_dim] (K-major, stored once per layer), f32 accumulation, bf16 qkv
 * [tokens][n_out] (row stride ld_qkv) -- e.g. n_out = 3 * heads * dim for a fused
 * [Q | K | V] projection whose head views feed gsa_forward as strided tensors.
 * n_out % 32 == 0, model_dim % 64 == 0. gsa_residual_bf16: y = bf16(x + o) over n
 * elements (x, y bf16; o f32), the residual connection between stacked layers. */
int gsa_project_qkv_bf16(const void* x, int tokens, int model_dim, int64_t ldx, const void* w_qkv_t, int n_out,
                         void* qkv, int64_t ld_qkv, gsa_stream_t stream);
int gsa_residual_bf16(const void* x, const float* o, void* y, int64_t n, gsa_stream_t stream);

/* Element-wise dtype conversion of n contiguous elements on the device (f32 <-> bf16 with
 * round-to-nearest-even, or a plain copy for equal dtypes): the host API converts its
 * operands on the GPU instead of in host loops (Precision::kBf16 uploads, bf16 downloads). */
int gsa_convert(const void* src, int src_dtype, void* dst, int dst_dtype, int64_t n, gsa_stream_t stream);

/* KernelStats (types.hpp:78-86) in closed form for a gsa_forward call:
 * scores_computed = H*(Ms*M + W*W); keys_attended = sum over rows of
 * |row| * s^2 * s^2 (rows have width F + k_eff). */
int gsa_forward_stats(const gsa_layout* layout, const gsa_params* params, int heads,
                      uint64_t* scores_computed, uint64_t* keys_attended);

/* selection_sparsity (declared at the reference's proj/include/gsa/workload.hpp:112 but
 * never defined there): 1 - attended fine keys per image query /
 * image_tokens, attended = (|forced windows| + k_eff) * s^2 with k_eff = min(k,
 * selectable windows) (plain: min(k, num_windows) * s^2). Host arithmetic only. */
int gsa_selection_sparsity(const gsa_layout* layout, const gsa_params* params, double* sparsity);

/* ---------------------------------------------------------------------------
 * Backward (gradients.hpp:14-265): the layer's manual backward with
 * the top-k selection held constant, on CUDA cores in f32. Deterministic (every
 * gradient element has one writer per kernel; no floating-point atomics).
 *
 * gsa_saved: the ForwardContext fields (layer.hpp:124-142) the backward reads, as
 * device f32 arrays in gsa_context's shapes: qc/kc/vc/o_comp [H][W][d], lse_comp
 * [H][W], o_sel/gate [H][Mi][d], lse_sel [H][Mi], lse_spec [H][Ms]; o_spec the
 * special rows of the forward output ([H][Ms][d] view, e.g. the first Ms rows of
 * gsa_forward's `out`); the selection plan as device CSR (gsa_build_selection_plan)
 * with plan_entries = offsets[H*W]. */
typedef struct {
    const float *qc, *kc, *vc, *o_comp, *lse_comp;
    const int64_t* plan_offsets;
    const int32_t* plan_ids;
    int64_t plan_entries;
    const float *o_sel, *lse_sel, *gate;
    gsa_tensor o_spec;
    const float* lse_spec;
} gsa_saved;

/* gsa_backward (gradients.hpp:54-243, up to the projection): from the projected
 * q/k/v (f32 or bf16, [H][M][d]), w_g f32 [H][d][d], the saved context and d_out f32
 * [H][M][d], writes dq/dk/dv f32 [H][M][d] and dw_g f32 [H][d][d]. The plan is
 * validated first (synchronises `stream`, like gsa_forward_with_plan). */
size_t gsa_backward_workspace_bytes(const gsa_layout* layout, const gsa_params* params, int heads, int dim,
                                    int64_t plan_entries, int qkv_dtype);
int gsa_backward(const gsa_tensor* q, const gsa_tensor* k, const gsa_tensor* v, const gsa_tensor* w_g,
                 const gsa_layout* layout, const gsa_params* params, const gsa_saved* saved,
                 const gsa_tensor* d_out, const gsa_tensor* dq, const gsa_tensor* dk, const gsa_tensor* dv,
                 float* dw_g, void* workspace, size_t workspace_bytes, gsa_stream_t stream);

/* Projection backward (gradients.hpp:226-263): dw_q[h] = x^T dq[h] (likewise k, v) and
 * dx = sum_h dq[h] w_q[h]^T + dk[h] w_k[h]^T + dv[h] w_v[h]^T. All device f32,
 * contiguous: x / dx [tokens][model_dim], w_* / dw_* [H][model_dim][dim], dq/dk/dv
 * [H][tokens][dim]. Row reductions are split and summed in a fixed order. */
size_t gsa_project_backward_workspace_bytes(int tokens, int model_dim, int heads, int dim);
int gsa_project_backward(const float* x, int tokens, int model_dim, const float* w_q, const float* w_k,
                         const float* w_v, int heads, int dim, const float* dq, const float* dk, const float* dv,
                         float* dx, float* dw_q, float* dw_k, float* dw_v, void* workspace, size_t workspace_bytes,
                         gsa_stream_t stream);

/* avg_pool_backward (gradients.hpp:21-34): out[h][t] = d_pooled[h][window_of(t)] / s^2;
 * upsample_backward (gradients.hpp:37-49): out[h][w] = sum of d_fine over w's members
 * in ascending token order. f32, bit-identical to the reference. */
int gsa_avg_pool_backward(const gsa_tensor* d_pooled, const gsa_layout* layout, const gsa_tensor* out,
                          gsa_stream_t stream);
int gsa_upsample_backward(const gsa_tensor* d_fine, const gsa_layout* layout, const gsa_tensor* out,
                          gsa_stream_t stream);

/* Instrumentation (bench.py, profiling). gsa_set_stage_events: when n >= 5,
 * subsequent gsa_forward calls on this thread record cudaEvent_t events[0..4]
 * on `stream` at: start, after the special path, after pooling, after the
 * compressed attention + top-k, after selection/gate/merge (gsa_shard_forward: start,
 * after pooling, after the Kc/Vc gather, after the compressed branch, done). With
 * n >= 7, events[5] and events[6] also bracket the compressed-attention kernel launch
 * itself (compress_tc_kernel), so its duration is measured on its own stream. n = 0
 * disables. gsa_backward records events[0..5]: start (after validation), after the gate
 * fuse, after the compressed-branch dense passes, after pooling + selection backward,
 * after the special rows, done (dW_g).
 * gsa_launch_count: kernels this library has launched since it was loaded. */
int gsa_set_stage_events(void* const* events, int n);
int gsa_launch_count(uint64_t* count);

#ifdef __cplusplus
}
#endif
#endif /* GSA_SM100_H */
