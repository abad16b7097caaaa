/*
 * gsa_oracle.h — TEST INFRASTRUCTURE ONLY.
 *
 * CPU restatement (plain C11) of the reference's Global Sparse Attention
 * forward path (arxiv 2603.08055, /root/reference/proj). It exists to CHECK
 * the sm_100a kernels: only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg may load it. The product path never links or calls it.
 *
 * Every function cites the reference file:line whose arithmetic it follows.
 * Arithmetic that decides top-k indices (pooling order, the 4-lane scaled_dot,
 * the tie rule) is reproduced operation for operation; this file must be
 * compiled with -ffp-contract=off and without -ffast-math (see oracle/Makefile).
 *
 * Pinning: the restatement is checked against the reference itself (compiled
 * unmodified into oracle/_ref by oracle/Makefile) and against the committed
 * fixtures in tests/golden/ that oracle/_ref generated (tests/golden/make_golden.py).
 */
#ifndef GSA_ORACLE_H
#define GSA_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* layout.hpp:13-40 TokenLayout */
typedef struct {
    int num_special, num_frames, grid_h, grid_w, window_s;
} orc_layout;

/* 0 = ok, 2 = DivisibilityError, 3 = ZeroSizeError (errors.hpp numbering of the C-ABI) */
int orc_build_layout(int num_special, int num_frames, int grid_h, int grid_w, int window_s,
                     orc_layout* out);
int orc_num_windows(const orc_layout* l);
int orc_image_tokens(const orc_layout* l);
int orc_total_tokens(const orc_layout* l);
/* layout.cpp:26-35 */
int orc_window_of_token(const orc_layout* l, int image_token);
/* layout.cpp:37-56: writes s*s ascending image-token indices (dr outer, dc inner) */
void orc_tokens_of_window(const orc_layout* l, int window, int* members);

/* dot.hpp:11-23 — the bit-exactness contract */
float orc_scaled_dot(const float* a, const float* b, int n, float scale);

/* helpers for synthetic inputs (prng.hpp:13-47 CounterRng, SplitMix64 + Box-Muller) */
uint64_t orc_rng_derive(uint64_t seed, uint64_t tag);
double orc_rng_normal(uint64_t stream_seed, uint64_t counter);
float orc_bf16_round(float x);
/* fill[i] = normal(stream, i) * mul (double -> float, then optional bf16 RNE) */
void orc_fill_normal(uint64_t seed, uint64_t tag, int64_t n, float mul, int round_bf16, float* out);
/* integer-exact uniform in [-1,1): ((bits>>40) - 2^23) * 2^-23, then bf16 RNE */
void orc_fill_uniform_bf16(uint64_t seed, uint64_t tag, int64_t n, float* out);

/* compression.hpp:20-38 avg_pool_tokens: x_img [H][Mi][d] -> out [H][W][d] */
void orc_pool(const float* x_img, int heads, int dim, const orc_layout* l, float* out);

/* naive_topk / naive_topk_excluding (reference.hpp:79-109): indices of the k best,
 * score desc, ties to the lower index; excluded may be NULL. Returns count. */
int orc_topk_row(const float* scores, int n, const uint8_t* excluded, int k, int32_t* out_idx);

/* Compressed branch (reference.hpp:238-253 with the fused kernel's k_eff rule,
 * compression.hpp:195-199): for each requested (h,wq) row: guide scores with
 * scaled_dot, top-k_eff indices, softmax over ALL windows, P.Vc, lse = m+log(l).
 * rows: flat h*W+wq list, NULL = all H*W rows (outputs then full-size).
 * Outputs are compact [n_rows][...]. guide may be NULL. Returns k_eff. */
int orc_compress_topk(const float* qc, const float* kc, const float* vc, int heads, int windows,
                      int dim, int k, float scale, const uint8_t* excluded, const int64_t* rows,
                      int64_t n_rows, float* out, float* lse, int32_t* idx, float* guide);

/* selection.cpp:7-67: forced windows of the hybrid variant, ascending. Returns count;
 * writes up to cap ids when out != NULL. */
int orc_forced_windows(const orc_layout* l, int ref_stride, int32_t* out, int cap);
/* build_selection_plan: offsets [H*W+1], ids. variant 0 = plain, 1 = hybrid.
 * Returns total ids (call with ids == NULL to size). */
int64_t orc_build_plan(const int32_t* topk, int heads, int windows, int k_eff, const orc_layout* l,
                       int variant, int ref_stride, int64_t* offsets, int32_t* ids);

/* selection.hpp:63-136 block_sparse_attention for the windows in rows (flat h*W+w,
 * NULL = all). q/k/v_img [H][Mi][d]. With rows == NULL, out/lse use the reference
 * layout [H][Mi][d] / [H][Mi]; otherwise compact [n_rows][s*s][d] / [n_rows][s*s]. */
void orc_block_sparse(const float* q_img, const float* k_img, const float* v_img, int heads,
                      int dim, const orc_layout* l, const int64_t* offsets, const int32_t* ids,
                      float scale, const int64_t* rows, int64_t n_rows, float* out, float* lse);

/* tiled_attention (compression.hpp:99-165) semantics: softmax(q k^T scale) v and lse,
 * q [H][mq][d], k/v [H][mk][d]. */
void orc_dense_attention(const float* q, const float* k, const float* v, int heads, int mq, int mk,
                         int dim, float scale, float* out, float* lse);

/* layer.hpp:99-119 gate: g = sigmoid(sum_a q[a] * w_g[h][a][j]) */
void orc_gate(const float* q_img, const float* w_g, int heads, int rows, int dim, float* g);

/* gsa_forward body after project_qkv (layer.hpp:194-229). q/k/v [H][M][d]; w_g [H][d][d].
 * out [H][M][d]. Any ctx_* pointer may be NULL. Returns k_eff, or -status on error. */
int orc_gsa_forward(const float* q, const float* k, const float* v, const float* w_g, int heads,
                    int dim, const orc_layout* l, int top_k, double scale_param, int variant,
                    int ref_stride, float* out, int32_t* ctx_topk, float* ctx_o_comp,
                    float* ctx_lse_comp, float* ctx_lse_sel);

#ifdef __cplusplus
}
#endif
#endif
