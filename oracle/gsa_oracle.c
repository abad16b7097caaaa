/*
 * gsa_oracle.c — TEST INFRASTRUCTURE ONLY (see gsa_oracle.h).
 *
 * Plain-C restatement of the reference GSA forward (post-projection). The
 * per-row work is parallelised with OpenMP; every row is independent, so the
 * results are identical for any thread count (as parallel.hpp:12-29 promises
 * for the reference).
 *
 * Build: oracle/Makefile (gcc -O2 -ffp-contract=off -fopenmp). No -ffast-math.
 */
#include "gsa_oracle.h"

#include <float.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ layout */

int orc_build_layout(int ns, int nf, int gh, int gw, int s, orc_layout* out) {
    /* layout.cpp:7-24 */
    if (ns < 0 || nf < 1 || gh < 1 || gw < 1 || s < 1) return 3;
    if (gh % s != 0 || gw % s != 0) return 2;
    out->num_special = ns;
    out->num_frames = nf;
    out->grid_h = gh;
    out->grid_w = gw;
    out->window_s = s;
    return 0;
}

static int wins_w(const orc_layout* l) { return l->grid_w / l->window_s; }
static int wins_per_frame(const orc_layout* l) {
    return (l->grid_h / l->window_s) * (l->grid_w / l->window_s);
}
int orc_num_windows(const orc_layout* l) { return l->num_frames * wins_per_frame(l); }
int orc_image_tokens(const orc_layout* l) { return l->num_frames * l->grid_h * l->grid_w; }
int orc_total_tokens(const orc_layout* l) { return l->num_special + orc_image_tokens(l); }

int orc_window_of_token(const orc_layout* l, int t) {
    /* layout.cpp:26-35 */
    const int tpf = l->grid_h * l->grid_w;
    const int frame = t / tpf, in_frame = t % tpf;
    const int row = in_frame / l->grid_w, col = in_frame % l->grid_w;
    return frame * wins_per_frame(l) + (row / l->window_s) * wins_w(l) + col / l->window_s;
}

void orc_tokens_of_window(const orc_layout* l, int w, int* members) {
    /* layout.cpp:37-56: dr outer, dc inner -> ascending token order */
    const int wpf = wins_per_frame(l);
    const int frame = w / wpf, in_frame = w % wpf;
    const int wrow = in_frame / wins_w(l), wcol = in_frame % wins_w(l);
    const int base = frame * l->grid_h * l->grid_w;
    int n = 0;
    for (int dr = 0; dr < l->window_s; ++dr)
        for (int dc = 0; dc < l->window_s; ++dc)
            members[n++] = base + (wrow * l->window_s + dr) * l->grid_w + wcol * l->window_s + dc;
}

/* ------------------------------------------------------------- primitives */

float orc_scaled_dot(const float* a, const float* b, int n, float scale) {
    /* dot.hpp:11-23: four stride-4 lane sums, ((s0+s1)+(s2+s3))*scale.
     * Separate multiply and add (no contraction; -ffp-contract=off). */
    float s0 = 0.0f, s1 = 0.0f, s2 = 0.0f, s3 = 0.0f;
    int i = 0;
    for (; i + 4 <= n; i += 4) {
        s0 += a[i] * b[i];
        s1 += a[i + 1] * b[i + 1];
        s2 += a[i + 2] * b[i + 2];
        s3 += a[i + 3] * b[i + 3];
    }
    for (; i < n; ++i) s0 += a[i] * b[i];
    return ((s0 + s1) + (s2 + s3)) * scale;
}

/* prng.hpp:17-43 */
static uint64_t mix64(uint64_t z) {
    z += 0x9e3779b97f4a7c15ULL;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}
uint64_t orc_rng_derive(uint64_t seed, uint64_t tag) { return mix64(seed ^ mix64(tag)); }
static uint64_t rng_bits(uint64_t s, uint64_t c) { return mix64(s + c * 0x9e3779b97f4a7c15ULL); }
static double rng_uniform(uint64_t s, uint64_t c) {
    return ((double)(rng_bits(s, c) >> 11) + 1.0) * 0x1.0p-53;
}
double orc_rng_normal(uint64_t s, uint64_t c) {
    const double u1 = rng_uniform(s, 2 * c), u2 = rng_uniform(s, 2 * c + 1);
    const double r = sqrt(-2.0 * log(u1));
    return r * cos(2.0 * 3.141592653589793238462643383279502884 * u2);
}

float orc_bf16_round(float x) {
    uint32_t u;
    memcpy(&u, &x, 4);
    if ((u & 0x7f800000u) == 0x7f800000u) return x; /* inf/nan untouched */
    u += 0x7fffu + ((u >> 16) & 1u);
    u &= 0xffff0000u;
    float r;
    memcpy(&r, &u, 4);
    return r;
}

void orc_fill_normal(uint64_t seed, uint64_t tag, int64_t n, float mul, int round_bf16,
                     float* out) {
    const uint64_t s = orc_rng_derive(seed, tag);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) {
        float v = (float)orc_rng_normal(s, (uint64_t)i) * mul;
        out[i] = round_bf16 ? orc_bf16_round(v) : v;
    }
}

void orc_fill_uniform_bf16(uint64_t seed, uint64_t tag, int64_t n, float* out) {
    const uint64_t s = orc_rng_derive(seed, tag);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) {
        const int64_t top = (int64_t)(rng_bits(s, (uint64_t)i) >> 40); /* 24 bits */
        const float v = (float)(top - (1 << 23)) * 0x1.0p-23f;           /* exact */
        out[i] = orc_bf16_round(v);
    }
}

/* ---------------------------------------------------------------- pooling */

static void pool_heads(const float* x_img, int64_t head_stride, int heads, int dim,
                       const orc_layout* l, float* out) {
    /* compression.hpp:20-38: dst starts at +0, members added in ascending
     * order, then multiplied by inv = T(1)/T(s2) (a float division). */
    const int W = orc_num_windows(l), s2 = l->window_s * l->window_s;
    const float inv = 1.0f / (float)s2;
#pragma omp parallel for schedule(static)
    for (int64_t hw = 0; hw < (int64_t)heads * W; ++hw) {
        const int h = (int)(hw / W), w = (int)(hw % W);
        int members[1024];
        orc_tokens_of_window(l, w, members);
        float* dst = out + ((int64_t)h * W + w) * dim;
        for (int d = 0; d < dim; ++d) dst[d] = 0.0f;
        for (int m = 0; m < s2; ++m) {
            const float* src = x_img + h * head_stride + (int64_t)members[m] * dim;
            for (int d = 0; d < dim; ++d) dst[d] += src[d];
        }
        for (int d = 0; d < dim; ++d) dst[d] *= inv;
    }
}

void orc_pool(const float* x_img, int heads, int dim, const orc_layout* l, float* out) {
    pool_heads(x_img, (int64_t)orc_image_tokens(l) * dim, heads, dim, l, out);
}

/* ------------------------------------------------------------------ top-k */

int orc_topk_row(const float* scores, int n, const uint8_t* excluded, int k, int32_t* out_idx) {
    /* naive_topk (reference.hpp:79-91): stable sort by score desc keeps the
     * lower index first among equal scores; equivalently insert in index
     * order after every entry whose score is >= the newcomer's. */
    int cnt = 0;
    if (k <= 0) return 0;
    float* best = (float*)malloc(sizeof(float) * (size_t)k);
    for (int i = 0; i < n; ++i) {
        if (!isfinite(scores[i])) { free(best); return -1; } /* NonFiniteInput */
        if (excluded && excluded[i]) continue;
        const float s = scores[i];
        if (cnt == k && !(s > best[k - 1])) continue;
        int pos = cnt < k ? cnt : k - 1;
        while (pos > 0 && s > best[pos - 1]) {
            best[pos] = best[pos - 1];
            out_idx[pos] = out_idx[pos - 1];
            --pos;
        }
        best[pos] = s;
        out_idx[pos] = i;
        if (cnt < k) ++cnt;
    }
    free(best);
    return cnt;
}

static int k_effective(int k, int windows, const uint8_t* excluded) {
    /* compression.hpp:195-199 */
    int selectable = windows;
    if (excluded)
        for (int i = 0; i < windows; ++i)
            if (excluded[i]) --selectable;
    return k < selectable ? k : selectable;
}

int orc_compress_topk(const float* qc, const float* kc, const float* vc, int heads, int windows,
                      int dim, int k, float scale, const uint8_t* excluded, const int64_t* rows,
                      int64_t n_rows, float* out, float* lse, int32_t* idx, float* guide) {
    const int k_eff = k_effective(k, windows, excluded);
    if (!rows) n_rows = (int64_t)heads * windows;
    int bad = 0;
#pragma omp parallel
    {
        float* srow = (float*)malloc(sizeof(float) * (size_t)windows);
#pragma omp for schedule(dynamic, 4)
        for (int64_t r = 0; r < n_rows; ++r) {
            const int64_t flat = rows ? rows[r] : r;
            const int h = (int)(flat / windows), wq = (int)(flat % windows);
            const float* qrow = qc + ((int64_t)h * windows + wq) * dim;
            const float* kh = kc + (int64_t)h * windows * dim;
            const float* vh = vc + (int64_t)h * windows * dim;
            /* reference.hpp:241-247 */
            for (int wk = 0; wk < windows; ++wk)
                srow[wk] = orc_scaled_dot(qrow, kh + (int64_t)wk * dim, dim, scale);
            int32_t* irow = idx + r * k_eff;
            if (k_eff > 0 && orc_topk_row(srow, windows, excluded, k_eff, irow) < 0) bad = 1;
            if (guide)
                for (int j = 0; j < k_eff; ++j) guide[r * k_eff + j] = srow[irow[j]];
            /* reference.hpp:29-40 softmax_inplace, then P.Vc (248-253) */
            float m = -INFINITY;
            for (int wk = 0; wk < windows; ++wk) m = srow[wk] > m ? srow[wk] : m;
            float sum = 0.0f;
            for (int wk = 0; wk < windows; ++wk) {
                srow[wk] = expf(srow[wk] - m);
                sum += srow[wk];
            }
            const float inv = 1.0f / sum;
            float* orow = out + r * dim;
            for (int d = 0; d < dim; ++d) orow[d] = 0.0f;
            for (int wk = 0; wk < windows; ++wk) {
                const float p = srow[wk] * inv;
                const float* vrow = vh + (int64_t)wk * dim;
                for (int d = 0; d < dim; ++d) orow[d] += p * vrow[d];
            }
            lse[r] = m + logf(sum);
        }
        free(srow);
    }
    return bad ? -5 : k_eff;
}

/* ------------------------------------------------------------------ plan */

int orc_forced_windows(const orc_layout* l, int ref_stride, int32_t* out, int cap) {
    /* selection.cpp:7-21: frames {0, r, 2r, ...}; all their windows ascending */
    if (ref_stride < 1) return -7; /* InvalidStride */
    const int wpf = wins_per_frame(l);
    int n = 0;
    for (int f = 0; f < l->num_frames; f += ref_stride)
        for (int w = 0; w < wpf; ++w) {
            if (out && n < cap) out[n] = f * wpf + w;
            ++n;
        }
    return n;
}

int64_t orc_build_plan(const int32_t* topk, int heads, int windows, int k_eff, const orc_layout* l,
                       int variant, int ref_stride, int64_t* offsets, int32_t* ids) {
    /* selection.cpp:29-67 */
    int nf = 0;
    int32_t* forced = NULL;
    uint8_t* mask = NULL;
    if (variant == 1) {
        nf = orc_forced_windows(l, ref_stride, NULL, 0);
        if (nf < 0) return nf;
        forced = (int32_t*)malloc(sizeof(int32_t) * (size_t)(nf > 0 ? nf : 1));
        orc_forced_windows(l, ref_stride, forced, nf);
        mask = (uint8_t*)calloc((size_t)windows, 1);
        for (int i = 0; i < nf; ++i) mask[forced[i]] = 1;
    }
    int64_t pos = 0;
    if (offsets) offsets[0] = 0;
    for (int64_t r = 0; r < (int64_t)heads * windows; ++r) {
        const int32_t* src = topk + r * k_eff;
        if (variant == 1) {
            for (int i = 0; i < nf; ++i) {
                if (ids) ids[pos] = forced[i];
                ++pos;
            }
            for (int j = 0; j < k_eff; ++j)
                if (!mask[src[j]]) {
                    if (ids) ids[pos] = src[j];
                    ++pos;
                }
        } else {
            for (int j = 0; j < k_eff; ++j) {
                if (ids) ids[pos] = src[j];
                ++pos;
            }
        }
        if (offsets) offsets[r + 1] = pos;
    }
    free(forced);
    free(mask);
    return pos;
}

/* ------------------------------------------------------- block-sparse attn */

static void block_sparse_heads(const float* q_img, const float* k_img, const float* v_img,
                               int64_t head_stride, int heads, int dim, const orc_layout* l,
                               const int64_t* offsets, const int32_t* ids, float scale,
                               const int64_t* rows, int64_t n_rows, float* out, float* lse) {
    /* selection.hpp:63-136: keys = members of each plan-row window in row
     * order; per query an online softmax that rescales only when the
     * running max grows (lines 112-133). */
    const int W = orc_num_windows(l), Mi = orc_image_tokens(l), s2 = l->window_s * l->window_s;
    if (!rows) n_rows = (int64_t)heads * W;
#pragma omp parallel
    {
        float* acc = (float*)malloc(sizeof(float) * (size_t)dim);
        int qmem[1024], kmem[1024];
#pragma omp for schedule(dynamic, 4)
        for (int64_t r = 0; r < n_rows; ++r) {
            const int64_t flat = rows ? rows[r] : r;
            const int h = (int)(flat / W), w = (int)(flat % W);
            const int64_t b = offsets[flat], e = offsets[flat + 1];
            const float* qh = q_img + h * head_stride;
            const float* kh = k_img + h * head_stride;
            const float* vh = v_img + h * head_stride;
            orc_tokens_of_window(l, w, qmem);
            for (int qi = 0; qi < s2; ++qi) {
                const float* qrow = qh + (int64_t)qmem[qi] * dim;
                float m = -INFINITY, lsum = 0.0f;
                for (int d = 0; d < dim; ++d) acc[d] = 0.0f;
                for (int64_t j = b; j < e; ++j) {
                    orc_tokens_of_window(l, ids[j], kmem);
                    for (int kk = 0; kk < s2; ++kk) {
                        const float s = orc_scaled_dot(qrow, kh + (int64_t)kmem[kk] * dim, dim, scale);
                        if (s > m) {
                            const float alpha = expf(m - s);
                            for (int d = 0; d < dim; ++d) acc[d] *= alpha;
                            lsum *= alpha;
                            m = s;
                        }
                        const float p = expf(s - m);
                        lsum += p;
                        const float* vrow = vh + (int64_t)kmem[kk] * dim;
                        for (int d = 0; d < dim; ++d) acc[d] += p * vrow[d];
                    }
                }
                float* orow;
                float* lrow;
                if (rows) {
                    orow = out + (r * s2 + qi) * dim;
                    lrow = lse + r * s2 + qi;
                } else {
                    orow = out + ((int64_t)h * Mi + qmem[qi]) * dim;
                    lrow = lse + (int64_t)h * Mi + qmem[qi];
                }
                const float inv = 1.0f / lsum;
                for (int d = 0; d < dim; ++d) orow[d] = acc[d] * inv;
                *lrow = m + logf(lsum);
            }
        }
        free(acc);
    }
}

void orc_block_sparse(const float* q_img, const float* k_img, const float* v_img, int heads,
                      int dim, const orc_layout* l, const int64_t* offsets, const int32_t* ids,
                      float scale, const int64_t* rows, int64_t n_rows, float* out, float* lse) {
    block_sparse_heads(q_img, k_img, v_img, (int64_t)orc_image_tokens(l) * dim, heads, dim, l,
                       offsets, ids, scale, rows, n_rows, out, lse);
}

/* --------------------------------------------------------------- dense attn */

static void dense_heads(const float* q, int64_t q_hs, const float* k, const float* v, int64_t kv_hs,
                        int heads, int mq, int mk, int dim, float scale, float* out,
                        int64_t out_hs, float* lse, int64_t lse_hs) {
    /* tiled_attention (compression.hpp:99-165) computes softmax(scaled_dot)
     * V with an online max; restated as max pass + exp/sum pass. */
#pragma omp parallel
    {
        float* srow = (float*)malloc(sizeof(float) * (size_t)(mk > 0 ? mk : 1));
#pragma omp for schedule(dynamic, 2)
        for (int64_t hq = 0; hq < (int64_t)heads * mq; ++hq) {
            const int h = (int)(hq / mq), t = (int)(hq % mq);
            const float* qrow = q + h * q_hs + (int64_t)t * dim;
            float m = -INFINITY;
            for (int j = 0; j < mk; ++j) {
                srow[j] = orc_scaled_dot(qrow, k + h * kv_hs + (int64_t)j * dim, dim, scale);
                m = srow[j] > m ? srow[j] : m;
            }
            float* orow = out + h * out_hs + (int64_t)t * dim;
            for (int d = 0; d < dim; ++d) orow[d] = 0.0f;
            float sum = 0.0f;
            for (int j = 0; j < mk; ++j) {
                const float p = expf(srow[j] - m);
                sum += p;
                const float* vrow = v + h * kv_hs + (int64_t)j * dim;
                for (int d = 0; d < dim; ++d) orow[d] += p * vrow[d];
            }
            const float inv = 1.0f / sum;
            for (int d = 0; d < dim; ++d) orow[d] *= inv;
            lse[h * lse_hs + t] = m + logf(sum);
        }
        free(srow);
    }
}

void orc_dense_attention(const float* q, const float* k, const float* v, int heads, int mq, int mk,
                         int dim, float scale, float* out, float* lse) {
    dense_heads(q, (int64_t)mq * dim, k, v, (int64_t)mk * dim, heads, mq, mk, dim, scale, out,
                (int64_t)mq * dim, lse, mq);
}

/* ------------------------------------------------------------------- gate */

static void gate_heads(const float* q, int64_t q_hs, const float* w_g, int heads, int rows, int dim,
                       float* g) {
    /* layer.hpp:99-119: grow[j] += q[a] * w[a][j] for a ascending, then sigmoid */
#pragma omp parallel for schedule(static)
    for (int64_t ht = 0; ht < (int64_t)heads * rows; ++ht) {
        const int h = (int)(ht / rows), t = (int)(ht % rows);
        const float* qrow = q + h * q_hs + (int64_t)t * dim;
        const float* wh = w_g + (int64_t)h * dim * dim;
        float* grow = g + ((int64_t)h * rows + t) * dim;
        for (int j = 0; j < dim; ++j) grow[j] = 0.0f;
        for (int a = 0; a < dim; ++a) {
            const float qa = qrow[a];
            const float* wrow = wh + (int64_t)a * dim;
            for (int j = 0; j < dim; ++j) grow[j] += qa * wrow[j];
        }
        for (int j = 0; j < dim; ++j) grow[j] = 1.0f / (1.0f + expf(-grow[j]));
    }
}

void orc_gate(const float* q_img, const float* w_g, int heads, int rows, int dim, float* g) {
    gate_heads(q_img, (int64_t)rows * dim, w_g, heads, rows, dim, g);
}

/* ------------------------------------------------------------ full forward */

int orc_gsa_forward(const float* q, const float* k, const float* v, const float* w_g, int heads,
                    int dim, const orc_layout* l, int top_k, double scale_param, int variant,
                    int ref_stride, float* out, int32_t* ctx_topk, float* ctx_o_comp,
                    float* ctx_lse_comp, float* ctx_lse_sel) {
    /* layer.hpp:177-230 minus project_qkv; resolved_scale reference.hpp:22-26 */
    if (top_k < 1) return -11;
    if (variant == 1 && ref_stride < 1) return -7;
    const float scale = scale_param > 0.0 ? (float)scale_param
                                          : (float)(1.0 / sqrt((double)dim));
    const int Ms = l->num_special, Mi = orc_image_tokens(l), M = Ms + Mi;
    const int W = orc_num_windows(l);
    const int64_t hs = (int64_t)M * dim;
    const float* q_img = q + (int64_t)Ms * dim;
    const float* k_img = k + (int64_t)Ms * dim;
    const float* v_img = v + (int64_t)Ms * dim;

    /* special_token_attention over ALL keys (layer.hpp:80-96) */
    if (Ms > 0) {
        float* lse_spec = (float*)malloc(sizeof(float) * (size_t)heads * Ms);
        dense_heads(q, hs, k, v, hs, heads, Ms, M, dim, scale, out, hs, lse_spec, Ms);
        free(lse_spec);
    }
    const size_t wsz = (size_t)heads * W * dim;
    float* qc = (float*)malloc(sizeof(float) * wsz);
    float* kc = (float*)malloc(sizeof(float) * wsz);
    float* vc = (float*)malloc(sizeof(float) * wsz);
    pool_heads(q_img, hs, heads, dim, l, qc);
    pool_heads(k_img, hs, heads, dim, l, kc);
    pool_heads(v_img, hs, heads, dim, l, vc);

    uint8_t* excluded = NULL;
    if (variant == 1) {
        const int nf = orc_forced_windows(l, ref_stride, NULL, 0);
        int32_t* fw = (int32_t*)malloc(sizeof(int32_t) * (size_t)(nf > 0 ? nf : 1));
        orc_forced_windows(l, ref_stride, fw, nf);
        excluded = (uint8_t*)calloc((size_t)W, 1);
        for (int i = 0; i < nf; ++i) excluded[fw[i]] = 1;
        free(fw);
    }
    const int k_eff = k_effective(top_k, W, excluded);
    float* o_comp = (float*)malloc(sizeof(float) * wsz);
    float* lse_comp = (float*)malloc(sizeof(float) * (size_t)heads * W);
    int32_t* topk = (int32_t*)malloc(sizeof(int32_t) * (size_t)heads * W * (k_eff > 0 ? k_eff : 1));
    int rc = orc_compress_topk(qc, kc, vc, heads, W, dim, top_k, scale, excluded, NULL, 0, o_comp,
                               lse_comp, topk, NULL);
    if (rc < 0) {
        free(qc); free(kc); free(vc); free(excluded); free(o_comp); free(lse_comp); free(topk);
        return rc;
    }
    const int64_t nids = orc_build_plan(topk, heads, W, k_eff, l, variant, ref_stride, NULL, NULL);
    int64_t* offsets = (int64_t*)malloc(sizeof(int64_t) * ((size_t)heads * W + 1));
    int32_t* ids = (int32_t*)malloc(sizeof(int32_t) * (size_t)(nids > 0 ? nids : 1));
    orc_build_plan(topk, heads, W, k_eff, l, variant, ref_stride, offsets, ids);
    for (int64_t r = 0; r < (int64_t)heads * W; ++r)
        if (offsets[r + 1] == offsets[r]) { /* EmptySelection (selection.hpp:82-85) */
            rc = -8;
            break;
        }
    float* o_sel = (float*)malloc(sizeof(float) * (size_t)heads * Mi * dim);
    float* lse_sel = (float*)malloc(sizeof(float) * (size_t)heads * Mi);
    float* g = (float*)malloc(sizeof(float) * (size_t)heads * Mi * dim);
    if (rc >= 0) {
        block_sparse_heads(q_img, k_img, v_img, hs, heads, dim, l, offsets, ids, scale, NULL, 0,
                           o_sel, lse_sel);
        gate_heads(q_img, hs, w_g, heads, Mi, dim, g);
        /* detail::assemble_image_output (layer.hpp:154-170) */
#pragma omp parallel for schedule(static)
        for (int64_t ht = 0; ht < (int64_t)heads * Mi; ++ht) {
            const int h = (int)(ht / Mi), t = (int)(ht % Mi);
            const float* comp = o_comp + ((int64_t)h * W + orc_window_of_token(l, t)) * dim;
            const float* sel = o_sel + ht * dim;
            const float* gg = g + ht * dim;
            float* orow = out + h * hs + (int64_t)(Ms + t) * dim;
            for (int d = 0; d < dim; ++d) orow[d] = gg[d] * comp[d] + (1.0f - gg[d]) * sel[d];
        }
        if (ctx_topk) memcpy(ctx_topk, topk, sizeof(int32_t) * (size_t)heads * W * k_eff);
        if (ctx_o_comp) memcpy(ctx_o_comp, o_comp, sizeof(float) * wsz);
        if (ctx_lse_comp) memcpy(ctx_lse_comp, lse_comp, sizeof(float) * (size_t)heads * W);
        if (ctx_lse_sel) memcpy(ctx_lse_sel, lse_sel, sizeof(float) * (size_t)heads * Mi);
    }
    free(qc); free(kc); free(vc); free(excluded); free(o_comp); free(lse_comp); free(topk);
    free(offsets); free(ids); free(o_sel); free(lse_sel); free(g);
    return rc < 0 ? rc : k_eff;
}
