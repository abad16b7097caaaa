// ref_harness.cpp — TEST INFRASTRUCTURE ONLY.
//
// extern "C" wrappers around the UNMODIFIED reference implementation
// (/root/reference/proj/include + src/{layout,selection}.cpp). oracle/Makefile
// compiles this file together with the reference sources where they lie into
// oracle/_ref/libgsa_ref.so; nothing from the reference is copied into the repo.
// Used (1) to pin the C restatement in gsa_oracle.c, (2) to generate the
// committed golden fixtures (tests/golden/make_golden.py) and (3) as the timed
// CPU baseline (bench.py cpu_baseline / --impl reference, kind "reference").
//
// Every wrapper returns 0 or a negative status mirroring the exception class:
// -1 GsaError, -2 ShapeMismatch, -3 DivisibilityError, -4 ZeroSizeError,
// -5 IndexOutOfRange, -6 NonFiniteInput, -7 InvalidTiling, -8 InvalidStride,
// -9 EmptySelection, -99 other.
#include <chrono>
#include <cstdint>
#include <cstring>
#include <limits>
#include <cmath>
#include <algorithm>
#include <string>
#include <vector>

#include "gsa/compression.hpp"
#include "gsa/gradients.hpp"
#include "gsa/layer.hpp"
#include "gsa/layout.hpp"
#include "gsa/reference.hpp"
#include "gsa/selection.hpp"
#include "gsa/tensor.hpp"
#include "gsa/types.hpp"
#include "gsa/workload.hpp"

namespace {

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const gsa::ShapeMismatch& e) {
        g_err = e.what();
        return -2;
    } catch (const gsa::DivisibilityError& e) {
        g_err = e.what();
        return -3;
    } catch (const gsa::ZeroSizeError& e) {
        g_err = e.what();
        return -4;
    } catch (const gsa::IndexOutOfRange& e) {
        g_err = e.what();
        return -5;
    } catch (const gsa::NonFiniteInput& e) {
        g_err = e.what();
        return -6;
    } catch (const gsa::InvalidTiling& e) {
        g_err = e.what();
        return -7;
    } catch (const gsa::InvalidStride& e) {
        g_err = e.what();
        return -8;
    } catch (const gsa::EmptySelection& e) {
        g_err = e.what();
        return -9;
    } catch (const gsa::GsaError& e) {
        g_err = e.what();
        return -1;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -99;
    }
}

gsa::Tensor<float> to_tensor(const float* p, int h, int t, int d) {
    gsa::Tensor<float> x(h, t, d);
    if (p) std::memcpy(x.data.data(), p, sizeof(float) * x.data.size());
    return x;
}

void from_tensor(const gsa::Tensor<float>& x, float* p) {
    if (p) std::memcpy(p, x.data.data(), sizeof(float) * x.data.size());
}

gsa::GsaParams make_params(int s, int top_k, double scale, int variant, int ref_stride, int bm,
                           int bn) {
    gsa::GsaParams p;
    p.window_s = s;
    p.top_k = top_k;
    p.scale = scale;
    p.variant = variant ? gsa::SelectionVariant::kHybrid : gsa::SelectionVariant::kPlain;
    p.ref_stride = ref_stride;
    p.tiling.block_m = bm;
    p.tiling.block_n = bn;
    return p;
}

double ms_since(std::chrono::steady_clock::time_point t0) {
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
}

}  // namespace

extern "C" {

const char* gsa_ref_last_error() { return g_err.c_str(); }

int gsa_ref_build_layout(int ns, int nf, int gh, int gw, int s, int* windows, int* image_tokens) {
    return guarded([&] {
        gsa::TokenLayout l = gsa::build_token_layout(ns, nf, gh, gw, s);
        if (windows) *windows = l.num_windows();
        if (image_tokens) *image_tokens = l.image_tokens();
    });
}

int gsa_ref_window_of_token(int ns, int nf, int gh, int gw, int s, int t, int* out) {
    return guarded([&] { *out = gsa::build_token_layout(ns, nf, gh, gw, s).window_of_token(t); });
}

int gsa_ref_tokens_of_window(int ns, int nf, int gh, int gw, int s, int w, int* out) {
    return guarded([&] {
        auto m = gsa::build_token_layout(ns, nf, gh, gw, s).tokens_of_window(w);
        std::copy(m.begin(), m.end(), out);
    });
}

float gsa_ref_scaled_dot(const float* a, const float* b, int n, float scale) {
    return gsa::scaled_dot(a, b, n, scale);
}

int gsa_ref_naive_topk(const float* scores, int n, const uint8_t* excluded, int k, int32_t* out,
                       int* count) {
    return guarded([&] {
        std::vector<float> s(scores, scores + n);
        std::vector<int32_t> r;
        if (excluded) {
            std::vector<uint8_t> ex(excluded, excluded + n);
            r = gsa::naive_topk_excluding(s, ex, k);
        } else {
            r = gsa::naive_topk(s, k);
        }
        std::copy(r.begin(), r.end(), out);
        *count = static_cast<int>(r.size());
    });
}

int gsa_ref_pool(const float* x_img, int heads, int dim, int ns, int nf, int gh, int gw, int s,
                 float* out) {
    return guarded([&] {
        auto l = gsa::build_token_layout(ns, nf, gh, gw, s);
        auto y = gsa::avg_pool_tokens(to_tensor(x_img, heads, l.image_tokens(), dim), l);
        from_tensor(y, out);
    });
}

int gsa_ref_upsample(const float* coarse, int heads, int dim, int ns, int nf, int gh, int gw, int s,
                     float* out) {
    return guarded([&] {
        auto l = gsa::build_token_layout(ns, nf, gh, gw, s);
        from_tensor(gsa::upsample_nearest(to_tensor(coarse, heads, l.num_windows(), dim), l), out);
    });
}

// fused_compressed_attention_topk (compression.hpp:180-297). excluded may be NULL.
int gsa_ref_compress(const float* qc, const float* kc, const float* vc, int heads, int windows,
                     int dim, int k, float scale, int bm, int bn, const uint8_t* excluded,
                     int threads, float* out, float* lse, int32_t* idx, double* guide, int* k_eff) {
    return guarded([&] {
        gsa::KernelTiling t{bm, bn};
        std::vector<uint8_t> ex;
        if (excluded) ex.assign(excluded, excluded + windows);
        auto r = gsa::fused_compressed_attention_topk(
            to_tensor(qc, heads, windows, dim), to_tensor(kc, heads, windows, dim),
            to_tensor(vc, heads, windows, dim), k, scale, t, excluded ? &ex : nullptr,
            guide != nullptr, nullptr, threads);
        from_tensor(r.out, out);
        if (lse) std::copy(r.lse.begin(), r.lse.end(), lse);
        if (idx) std::copy(r.topk.indices.begin(), r.topk.indices.end(), idx);
        if (guide) std::copy(r.topk.guide_scores.begin(), r.topk.guide_scores.end(), guide);
        *k_eff = r.topk.k;
    });
}

// build_selection_plan (selection.cpp:29-67). Call with ids == NULL to get *n_ids.
int gsa_ref_plan(const int32_t* topk, int heads, int rows, int k, int ns, int nf, int gh, int gw,
                 int s, int variant, int ref_stride, int64_t* offsets, int32_t* ids,
                 int64_t* n_ids) {
    return guarded([&] {
        auto l = gsa::build_token_layout(ns, nf, gh, gw, s);
        gsa::TopkResult t(heads, rows, k);
        std::copy(topk, topk + static_cast<size_t>(heads) * rows * k, t.indices.begin());
        auto p = gsa::build_selection_plan(
            t, l, variant ? gsa::SelectionVariant::kHybrid : gsa::SelectionVariant::kPlain,
            ref_stride);
        *n_ids = static_cast<int64_t>(p.window_ids.size());
        if (offsets) std::copy(p.offsets.begin(), p.offsets.end(), offsets);
        if (ids) std::copy(p.window_ids.begin(), p.window_ids.end(), ids);
    });
}

int gsa_ref_forced_windows(int ns, int nf, int gh, int gw, int s, int ref_stride, int32_t* out,
                           int* count) {
    return guarded([&] {
        auto l = gsa::build_token_layout(ns, nf, gh, gw, s);
        auto f = gsa::forced_windows_of(l, ref_stride);
        if (out) std::copy(f.begin(), f.end(), out);
        *count = static_cast<int>(f.size());
    });
}

// block_sparse_attention (selection.hpp:63-136) on a CSR plan.
int gsa_ref_block_sparse(const float* q_img, const float* k_img, const float* v_img, int heads,
                         int dim, int ns, int nf, int gh, int gw, int s, const int64_t* offsets,
                         const int32_t* ids, float scale, int threads, float* out, float* lse) {
    return guarded([&] {
        auto l = gsa::build_token_layout(ns, nf, gh, gw, s);
        gsa::SelectionPlan p;
        p.heads = heads;
        p.rows = l.num_windows();
        const size_t nr = static_cast<size_t>(heads) * p.rows;
        p.offsets.assign(offsets, offsets + nr + 1);
        p.window_ids.assign(ids, ids + offsets[nr]);
        const int mi = l.image_tokens();
        auto r = gsa::block_sparse_attention(to_tensor(q_img, heads, mi, dim),
                                             to_tensor(k_img, heads, mi, dim),
                                             to_tensor(v_img, heads, mi, dim), p, l, scale,
                                             gsa::KernelTiling{}, nullptr, threads);
        from_tensor(r.out, out);
        if (lse) std::copy(r.lse.begin(), r.lse.end(), lse);
    });
}

// masked_image_attention (reference.hpp:120-170): the -inf-masked dense selection oracle,
// with the per-query denominators sum_j exp(score_j) (SPEC.md:576 gather/mask equivalence).
int gsa_ref_masked_attention(const float* q_img, const float* k_img, const float* v_img, int heads, int dim,
                             int ns, int nf, int gh, int gw, int s, const int64_t* offsets, const int32_t* ids,
                             float scale, float* out, double* denominators) {
    return guarded([&] {
        auto l = gsa::build_token_layout(ns, nf, gh, gw, s);
        gsa::SelectionPlan p;
        p.heads = heads;
        p.rows = l.num_windows();
        const size_t nr = static_cast<size_t>(heads) * p.rows;
        p.offsets.assign(offsets, offsets + nr + 1);
        p.window_ids.assign(ids, ids + offsets[nr]);
        const int mi = l.image_tokens();
        auto r = gsa::masked_image_attention(to_tensor(q_img, heads, mi, dim), to_tensor(k_img, heads, mi, dim),
                                             to_tensor(v_img, heads, mi, dim), p, l, scale);
        from_tensor(r.out, out);
        if (denominators) std::copy(r.denominators.begin(), r.denominators.end(), denominators);
    });
}

int gsa_ref_tiled_attention(const float* q, const float* k, const float* v, int heads, int mq,
                            int mk, int dim, float scale, int bm, int bn, int threads, float* out,
                            float* lse) {
    return guarded([&] {
        gsa::Tensor<float> o;
        std::vector<float> l;
        gsa::tiled_attention(to_tensor(q, heads, mq, dim), to_tensor(k, heads, mk, dim),
                             to_tensor(v, heads, mk, dim), scale, gsa::KernelTiling{bm, bn}, o, l,
                             nullptr, threads);
        from_tensor(o, out);
        if (lse) std::copy(l.begin(), l.end(), lse);
    });
}

int gsa_ref_full_attention(const float* q, const float* k, const float* v, int heads, int mq,
                           int mk, int dim, float scale, float* out) {
    return guarded([&] {
        from_tensor(gsa::full_attention(to_tensor(q, heads, mq, dim), to_tensor(k, heads, mk, dim),
                                        to_tensor(v, heads, mk, dim), scale),
                    out);
    });
}

int gsa_ref_gate(const float* q_img, const float* w_g, int heads, int rows, int dim, float* g) {
    return guarded([&] {
        from_tensor(gsa::gate(to_tensor(q_img, heads, rows, dim), to_tensor(w_g, heads, dim, dim)),
                    g);
    });
}

// The reference's fused CPU layer (gsa_forward, layer.hpp:194-229) starting from
// projected Q/K/V: partition, special path, pool x3, compress+top-k, plan,
// block-sparse, gate, assemble, concat — each stage timed into stage_ms[0..6]:
// 0 partition, 1 special, 2 pool, 3 compress, 4 plan, 5 select, 6 gate+merge+concat.
// Context pointers may be NULL.
int gsa_ref_forward(const float* q, const float* k, const float* v, const float* w_g, int heads,
                    int dim, int ns, int nf, int gh, int gw, int s, int top_k, double scale_param,
                    int variant, int ref_stride, int bm, int bn, int threads, float* out,
                    float* ctx_qc, float* ctx_kc, float* ctx_vc, float* ctx_o_comp,
                    float* ctx_lse_comp, int32_t* ctx_topk, int* k_eff, float* ctx_o_sel,
                    float* ctx_lse_sel, float* ctx_gate, float* ctx_lse_spec, double* stage_ms) {
    return guarded([&] {
        using clk = std::chrono::steady_clock;
        auto l = gsa::build_token_layout(ns, nf, gh, gw, s);
        gsa::GsaParams params = make_params(s, top_k, scale_param, variant, ref_stride, bm, bn);
        gsa::validate_params(params);
        const int m = l.total_tokens();
        auto Q = to_tensor(q, heads, m, dim);
        auto K = to_tensor(k, heads, m, dim);
        auto V = to_tensor(v, heads, m, dim);
        auto Wg = to_tensor(w_g, heads, dim, dim);
        const float scale = gsa::resolved_scale<float>(params, dim);
        double t[7] = {0, 0, 0, 0, 0, 0, 0};

        auto t0 = clk::now();
        auto parts = gsa::partition_qkv(Q, K, V, l);
        t[0] = ms_since(t0);

        t0 = clk::now();
        std::vector<float> lse_spec;
        auto o_spec = gsa::special_token_attention(parts.q_spec, K, V, scale, params.tiling,
                                                   &lse_spec, nullptr, threads);
        t[1] = ms_since(t0);

        t0 = clk::now();
        auto qc = gsa::avg_pool_tokens(parts.q_img, l);
        auto kc = gsa::avg_pool_tokens(parts.k_img, l);
        auto vc = gsa::avg_pool_tokens(parts.v_img, l);
        t[2] = ms_since(t0);

        t0 = clk::now();
        std::vector<uint8_t> excluded;
        if (params.variant == gsa::SelectionVariant::kHybrid)
            excluded = gsa::forced_window_mask(l, params.ref_stride);
        auto comp = gsa::fused_compressed_attention_topk(
            qc, kc, vc, params.top_k, scale, params.tiling,
            excluded.empty() ? nullptr : &excluded, false, nullptr, threads);
        t[3] = ms_since(t0);

        t0 = clk::now();
        auto plan = gsa::build_selection_plan(comp.topk, l, params.variant, params.ref_stride);
        t[4] = ms_since(t0);

        t0 = clk::now();
        auto sel = gsa::block_sparse_attention(parts.q_img, parts.k_img, parts.v_img, plan, l,
                                               scale, params.tiling, nullptr, threads);
        t[5] = ms_since(t0);

        t0 = clk::now();
        auto g = gsa::gate(parts.q_img, Wg);
        auto o_img = gsa::detail::assemble_image_output(parts, comp.out, sel.out, g, l);
        auto o = gsa::concat_rows(o_spec, o_img);
        t[6] = ms_since(t0);

        from_tensor(o, out);
        from_tensor(qc, ctx_qc);
        from_tensor(kc, ctx_kc);
        from_tensor(vc, ctx_vc);
        from_tensor(comp.out, ctx_o_comp);
        if (ctx_lse_comp) std::copy(comp.lse.begin(), comp.lse.end(), ctx_lse_comp);
        if (ctx_topk) std::copy(comp.topk.indices.begin(), comp.topk.indices.end(), ctx_topk);
        if (k_eff) *k_eff = comp.topk.k;
        from_tensor(sel.out, ctx_o_sel);
        if (ctx_lse_sel) std::copy(sel.lse.begin(), sel.lse.end(), ctx_lse_sel);
        from_tensor(g, ctx_gate);
        if (ctx_lse_spec) std::copy(lse_spec.begin(), lse_spec.end(), ctx_lse_spec);
        if (stage_ms) std::copy(t, t + 7, stage_ms);
    });
}

// The brute-force oracle reference_gsa (reference.hpp:203-280).
int gsa_ref_reference_gsa(const float* q, const float* k, const float* v, const float* w_g,
                          int heads, int dim, int ns, int nf, int gh, int gw, int s, int top_k,
                          double scale_param, int variant, int ref_stride, float* out) {
    return guarded([&] {
        auto l = gsa::build_token_layout(ns, nf, gh, gw, s);
        gsa::GsaParams params = make_params(s, top_k, scale_param, variant, ref_stride, 16, 16);
        const int m = l.total_tokens();
        from_tensor(gsa::reference_gsa(to_tensor(q, heads, m, dim), to_tensor(k, heads, m, dim),
                                       to_tensor(v, heads, m, dim), l, params,
                                       to_tensor(w_g, heads, dim, dim)),
                    out);
    });
}

// generate_workload (workload.hpp:63-106) + project_qkv (layer.hpp:48-76): the
// reference's own "random init" instance. q/k/v [heads][tokens][dim], w_g [heads][dim][dim].
int gsa_ref_random_init(uint64_t seed, int ns, int nf, int gh, int gw, int s, int heads, int dim,
                        int model_dim, int clustered, float* q, float* k, float* v, float* w_g) {
    return guarded([&] {
        gsa::WorkloadConfig c;
        c.seed = seed;
        c.layout = gsa::build_token_layout(ns, nf, gh, gw, s);
        c.heads = heads;
        c.dim = dim;
        c.model_dim = model_dim;
        c.precision = gsa::Precision::kF32;
        c.distribution = clustered ? gsa::Distribution::kClustered : gsa::Distribution::kGaussian;
        auto w = gsa::generate_workload<float>(c);
        auto p = gsa::project_qkv(w.x, w.weights);
        from_tensor(p.q, q);
        from_tensor(p.k, k);
        from_tensor(p.v, v);
        from_tensor(w.weights.w_g, w_g);
    });
}

// Sampled-row parity at scale ("For V >= 500, use sampled-row parity"),
// ONE head at a time: the reference's per-row path for a subset of query windows and
// special rows, with the reference's own functions wherever they exist:
//   pooling         avg_pool_tokens (compression.hpp:20-38, what gsa_forward uses)
//   guide scores    scaled_dot (dot.hpp:11-23) over every key window, then
//                   naive_topk / naive_topk_excluding (reference.hpp:79-109), exactly the
//                   row body of reference_gsa (reference.hpp:236-247)
//   compressed out  softmax_inplace + P.Vc (reference.hpp:248-253); lse = m + log(sum)
//   plan row        build_selection_plan (selection.cpp:29-67) on a TopkResult holding
//                   the sampled rows
//   selection       the fused block_sparse_attention loop body (selection.hpp:100-133)
//                   for the sampled window's s^2 queries (the masked O(M_i) oracle would
//                   be O(M_i) per query: infeasible at 1.3M tokens)
//   gate + merge    gate (layer.hpp:99-119) on the sampled query rows, then the
//                   assemble_image_output formula (layer.hpp:154-170)
//   special rows    special_token_attention -> tiled_attention (layer.hpp:80-96) of the
//                   sampled special queries over all M keys
// q/k/v: this head's rows [M][d] (specials first, then image tokens); w_g [d][d].
// Outputs per sampled window i: topk [i][k_eff], guide [i][k_eff] (nullable), o_comp
// [i][d], lse_comp [i], out_img / o_sel [i][s^2][d] (window member order), lse_sel
// [i][s^2]; per sampled special j: out_spec [j][d].
int gsa_ref_sampled_head(const float* q, const float* k, const float* v, const float* w_g, int dim, int ns,
                         int nf, int gh, int gw, int s, int top_k, double scale_param, int variant,
                         int ref_stride, const int32_t* wins, int n_wins, const int32_t* specs, int n_specs,
                         int threads, int32_t* topk_out, float* guide_out, float* o_comp_out,
                         float* lse_comp_out, float* out_img, float* o_sel_out, float* lse_sel_out,
                         float* out_spec, int* k_eff_out) {
    return guarded([&] {
        auto l = gsa::build_token_layout(ns, nf, gh, gw, s);
        gsa::GsaParams params = make_params(s, top_k, scale_param, variant, ref_stride, 16, 16);
        gsa::validate_params(params);
        const int m = l.total_tokens(), W = l.num_windows(), s2 = s * s;
        const float scale = gsa::resolved_scale<float>(params, dim);
        auto Q = to_tensor(q, 1, m, dim);
        auto K = to_tensor(k, 1, m, dim);
        auto V = to_tensor(v, 1, m, dim);
        auto parts = gsa::partition_qkv(Q, K, V, l);
        auto qc = gsa::avg_pool_tokens(parts.q_img, l);
        auto kc = gsa::avg_pool_tokens(parts.k_img, l);
        auto vc = gsa::avg_pool_tokens(parts.v_img, l);
        std::vector<uint8_t> excluded;
        if (params.variant == gsa::SelectionVariant::kHybrid)
            excluded = gsa::forced_window_mask(l, params.ref_stride);
        int selectable = W;
        for (uint8_t e : excluded)
            if (e) --selectable;
        const int k_eff = std::min(params.top_k, selectable);
        *k_eff_out = k_eff;
        for (int i = 0; i < n_wins; ++i)
            if (wins[i] < 0 || wins[i] >= W) throw gsa::IndexOutOfRange("sampled window out of range");

        // per sampled row: guide scores, top-k, compressed softmax row (reference.hpp:236-253)
        gsa::TopkResult topk(1, W, k_eff);
        std::fill(topk.indices.begin(), topk.indices.end(), 0);
        gsa::parallel_for(n_wins, threads, [&](int i) {
            const int wq = wins[i];
            std::vector<float> row(W);
            const float* qrow = qc.row(0, wq);
            for (int wk = 0; wk < W; ++wk) row[wk] = gsa::scaled_dot(qrow, kc.row(0, wk), dim, scale);
            std::vector<int32_t> top =
                excluded.empty() ? gsa::naive_topk(row, k_eff) : gsa::naive_topk_excluding(row, excluded, k_eff);
            std::copy(top.begin(), top.end(), topk_out + (size_t)i * k_eff);
            std::copy(top.begin(), top.end(), topk.row(0, wq));  // distinct rows: no race
            if (guide_out)
                for (int j = 0; j < k_eff; ++j) guide_out[(size_t)i * k_eff + j] = row[top[j]];
            float mx = -std::numeric_limits<float>::infinity();
            for (int wk = 0; wk < W; ++wk) mx = std::max(mx, row[wk]);
            double sum = 0.0;
            for (int wk = 0; wk < W; ++wk) sum += std::exp((double)row[wk] - mx);
            lse_comp_out[i] = (float)(mx + std::log(sum));
            gsa::softmax_inplace(row.data(), W);
            float* orow = o_comp_out + (size_t)i * dim;
            std::fill(orow, orow + dim, 0.0f);
            for (int wk = 0; wk < W; ++wk) {
                const float* vrow = vc.row(0, wk);
                for (int d = 0; d < dim; ++d) orow[d] += row[wk] * vrow[d];
            }
        });

        // plan rows (selection.cpp:29-67), then the fused selection loop per sampled window
        auto plan = gsa::build_selection_plan(topk, l, params.variant, params.ref_stride);
        gsa::Tensor<float> qsel(1, n_wins * s2, dim);  // the sampled windows' query rows, member order
        for (int i = 0; i < n_wins; ++i) {
            const auto members = l.tokens_of_window(wins[i]);
            for (int j = 0; j < s2; ++j)
                std::copy(parts.q_img.row(0, members[j]), parts.q_img.row(0, members[j]) + dim, qsel.row(0, i * s2 + j));
        }
        gsa::parallel_for(n_wins, threads, [&](int i) {
            const int w = wins[i];
            const int nsel = plan.row_size(0, w);
            const int32_t* sel = plan.row(0, w);
            std::vector<int> keys;  // selection.hpp:100-105
            keys.reserve((size_t)nsel * s2);
            for (int j = 0; j < nsel; ++j)
                for (int member : l.tokens_of_window(sel[j])) keys.push_back(member);
            std::vector<float> acc(dim);
            for (int qi = 0; qi < s2; ++qi) {  // selection.hpp:112-133
                const float* qrow = qsel.row(0, i * s2 + qi);
                float mm = -std::numeric_limits<float>::infinity(), ll = 0.0f;
                std::fill(acc.begin(), acc.end(), 0.0f);
                for (int key : keys) {
                    const float sc = gsa::scaled_dot(qrow, parts.k_img.row(0, key), dim, scale);
                    if (sc > mm) {
                        const float alpha = std::exp(mm - sc);
                        for (int d = 0; d < dim; ++d) acc[d] *= alpha;
                        ll *= alpha;
                        mm = sc;
                    }
                    const float p = std::exp(sc - mm);
                    ll += p;
                    const float* vrow = parts.v_img.row(0, key);
                    for (int d = 0; d < dim; ++d) acc[d] += p * vrow[d];
                }
                float* orow = o_sel_out + ((size_t)i * s2 + qi) * dim;
                const float inv = 1.0f / ll;
                for (int d = 0; d < dim; ++d) orow[d] = acc[d] * inv;
                lse_sel_out[(size_t)i * s2 + qi] = mm + std::log(ll);
            }
        });
        // gate (layer.hpp:99-119) + merge (layer.hpp:154-170)
        auto Wg = to_tensor(w_g, 1, dim, dim);
        auto g = gsa::gate(qsel, Wg);
        for (int i = 0; i < n_wins; ++i)
            for (int qi = 0; qi < s2; ++qi) {
                const float* gr = g.row(0, i * s2 + qi);
                const float* comp = o_comp_out + (size_t)i * dim;
                const float* selr = o_sel_out + ((size_t)i * s2 + qi) * dim;
                float* orow = out_img + ((size_t)i * s2 + qi) * dim;
                for (int d = 0; d < dim; ++d) orow[d] = gr[d] * comp[d] + (1.0f - gr[d]) * selr[d];
            }
        // special rows over all M keys (layer.hpp:80-96)
        if (n_specs > 0) {
            gsa::Tensor<float> qs(1, n_specs, dim);
            for (int j = 0; j < n_specs; ++j) {
                if (specs[j] < 0 || specs[j] >= ns) throw gsa::IndexOutOfRange("sampled special row out of range");
                std::copy(Q.row(0, specs[j]), Q.row(0, specs[j]) + dim, qs.row(0, j));
            }
            std::vector<float> lse;
            auto os = gsa::special_token_attention(qs, K, V, scale, params.tiling, &lse, nullptr, threads);
            from_tensor(os, out_spec);
        }
    });
}

// project_qkv (layer.hpp:48-76) on given X [tokens][C] and W_q/W_k/W_v [heads][C][dim].
int gsa_ref_project(const float* x, int tokens, int model_dim, const float* wq, const float* wk, const float* wv,
                    int heads, int dim, float* q, float* k, float* v) {
    return guarded([&] {
        gsa::LayerWeights<float> w;
        w.w_q = to_tensor(wq, heads, model_dim, dim);
        w.w_k = to_tensor(wk, heads, model_dim, dim);
        w.w_v = to_tensor(wv, heads, model_dim, dim);
        w.w_g = gsa::Tensor<float>(heads, dim, dim);
        auto p = gsa::project_qkv(to_tensor(x, 1, tokens, model_dim), w);
        from_tensor(p.q, q);
        from_tensor(p.k, k);
        from_tensor(p.v, v);
    });
}

// gsa_forward (layer.hpp:177-230) then gsa_backward (gradients.hpp:54-265) on X / weights,
// in f32 (f64 = 0) or in double (f64 = 1; inputs widened, results rounded back to f32).
// Returns the forward output, the ForwardContext fields the device backward consumes (any
// pointer may be NULL; topk holds H*W*k_eff ids) and the gradients GsaGradients. ms[0] /
// ms[1]: forward / backward wall time.
int gsa_ref_backward(const float* x, int model_dim, const float* wq, const float* wk, const float* wv,
                     const float* wg, int heads, int dim, int ns, int nf, int gh, int gw, int s, int top_k,
                     double scale_param, int variant, int ref_stride, int threads, int f64, const float* d_out,
                     float* out, float* q, float* k, float* v, float* qc, float* kc, float* vc, float* o_comp,
                     float* lse_comp, int32_t* topk, int* k_eff, float* o_sel, float* lse_sel, float* gate,
                     float* lse_spec, float* dx, float* dwq, float* dwk, float* dwv, float* dwg, double* ms) {
    auto run = [&](auto zero) {
        using T = decltype(zero);
        auto in = [](const float* p, int h, int t, int d) {
            gsa::Tensor<T> r(h, t, d);
            for (size_t i = 0; i < r.data.size(); ++i) r.data[i] = static_cast<T>(p[i]);
            return r;
        };
        auto put = [](const gsa::Tensor<T>& t, float* p) {
            if (p)
                for (size_t i = 0; i < t.data.size(); ++i) p[i] = static_cast<float>(t.data[i]);
        };
        auto putv = [](const std::vector<T>& t, float* p) {
            if (p)
                for (size_t i = 0; i < t.size(); ++i) p[i] = static_cast<float>(t[i]);
        };
        auto l = gsa::build_token_layout(ns, nf, gh, gw, s);
        gsa::GsaParams params = make_params(s, top_k, scale_param, variant, ref_stride, 16, 16);
        const int m = l.total_tokens();
        gsa::LayerWeights<T> w;
        w.w_q = in(wq, heads, model_dim, dim);
        w.w_k = in(wk, heads, model_dim, dim);
        w.w_v = in(wv, heads, model_dim, dim);
        w.w_g = in(wg, heads, dim, dim);
        auto t0 = std::chrono::steady_clock::now();
        auto fwd = gsa::gsa_forward(in(x, 1, m, model_dim), l, params, w, nullptr, threads);
        if (ms) ms[0] = ms_since(t0);
        t0 = std::chrono::steady_clock::now();
        auto g = gsa::gsa_backward(fwd.saved, in(d_out, heads, m, dim), threads);
        if (ms) ms[1] = ms_since(t0);
        const auto& c = fwd.saved;
        put(fwd.out, out);
        put(c.q, q);
        put(c.k, k);
        put(c.v, v);
        put(c.qc, qc);
        put(c.kc, kc);
        put(c.vc, vc);
        put(c.o_comp_coarse, o_comp);
        putv(c.lse_comp, lse_comp);
        if (topk) std::copy(c.topk.indices.begin(), c.topk.indices.end(), topk);
        if (k_eff) *k_eff = c.topk.k;
        put(c.o_sel, o_sel);
        putv(c.lse_sel, lse_sel);
        put(c.gate_vals, gate);
        putv(c.lse_spec, lse_spec);
        put(g.dx, dx);
        put(g.dw_q, dwq);
        put(g.dw_k, dwk);
        put(g.dw_v, dwv);
        put(g.dw_g, dwg);
    };
    return guarded([&] {
        if (f64) run(0.0);
        else run(0.0f);
    });
}

}  // extern "C"
