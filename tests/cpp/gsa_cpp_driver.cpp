// gsa_cpp_driver.cpp — exercises the C++ drop-in API (include/gsa/*.hpp, the
// reference's operator signatures) on the GPU and dumps every result for the
// pytest side (tests/test_cpp_api.py) to compare against the reference
// compiled unmodified (oracle/_ref). It is written the way a user of the
// reference would call it: build a layout, make weights and X, call
// gsa_forward / the per-branch operators, catch gsa:: exceptions.
//
//   gsa_cpp_driver <out_dir> <num_special> <frames> <grid_h> <grid_w> <s> <heads> <model_dim> <top_k> <variant> [f32|bf16]
//   gsa_cpp_driver --time <views> <iters> [f32|bf16]
//       times gsa::gsa_forward(Tensor<float> X, ...) host -> host (upload, projection, layer,
//       context download: everything the reference API returns) at V views of 5 specials +
//       36x36 patches, 16 heads, C = 1024, top-32; prints one JSON line
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <string>
#include <vector>

#include "gsa/gsa.hpp"

namespace {

std::ofstream g_manifest;
std::string g_dir;

template <typename U>
void dump(const std::string& name, const std::vector<U>& v, const char* dtype, std::vector<long> shape) {
    std::ofstream f(g_dir + "/" + name + ".bin", std::ios::binary);
    f.write(reinterpret_cast<const char*>(v.data()), static_cast<std::streamsize>(v.size() * sizeof(U)));
    g_manifest << name << " " << dtype;
    for (long s : shape) g_manifest << " " << s;
    g_manifest << "\n";
}

void dump(const std::string& name, const gsa::Tensor<float>& t) {
    dump(name, t.data, "f32", {t.heads, t.tokens, t.dim});
}

// deterministic N(0, 1)-ish values (sum of uniforms), independent of the reference's RNG
struct Lcg {
    uint64_t s;
    float uniform() {
        s = s * 6364136223846793005ull + 1442695040888963407ull;
        return static_cast<float>((s >> 40) & 0xffffff) / 16777216.0f;
    }
    float normal() {
        float a = 0.0f;
        for (int i = 0; i < 12; ++i) a += uniform();
        return a - 6.0f;
    }
};

gsa::Tensor<float> random_tensor(int h, int t, int d, float mul, uint64_t seed) {
    gsa::Tensor<float> x(h, t, d);
    Lcg r{seed};
    for (float& v : x.data) v = r.normal() * mul;
    return x;
}

template <typename E, typename F>
void expect_throw(const char* what, F&& f) {
    try {
        f();
    } catch (const E&) {
        g_manifest << "# ok " << what << "\n";
        return;
    } catch (const std::exception& e) {
        std::fprintf(stderr, "%s: wrong exception: %s\n", what, e.what());
        std::exit(3);
    }
    std::fprintf(stderr, "%s: no exception\n", what);
    std::exit(3);
}

int time_forward(int views, int iters, bool bf16) {
    gsa::device::compute_precision() = bf16 ? gsa::device::Precision::kBf16 : gsa::device::Precision::kF32;
    const int heads = 16, dim = 64, model_dim = heads * dim;
    const gsa::TokenLayout layout = gsa::build_token_layout(5 * views, views, 36, 36, 4);
    gsa::LayerWeights<float> w;
    const float wscale = 1.0f / std::sqrt(static_cast<float>(model_dim));
    w.w_q = random_tensor(heads, model_dim, dim, wscale, 2);
    w.w_k = random_tensor(heads, model_dim, dim, wscale, 3);
    w.w_v = random_tensor(heads, model_dim, dim, wscale, 4);
    w.w_g = random_tensor(heads, dim, dim, 1.0f / 8.0f, 5);
    const gsa::Tensor<float> x = random_tensor(1, layout.total_tokens(), model_dim, 1.0f, 1);
    gsa::GsaParams p;
    { auto warm = gsa::gsa_forward(x, layout, p, w); }
    double best = 1e30, sum = 0.0;
    for (int i = 0; i < iters; ++i) {
        const auto t0 = std::chrono::steady_clock::now();
        auto r = gsa::gsa_forward(x, layout, p, w);
        const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
        best = std::min(best, ms);
        sum += ms;
    }
    // where the host->host time goes: the pinned staging rates, host allocation (the
    // zero-filled std::vector every returned Tensor owns) and project_qkv (X up, Q/K/V down)
    auto ms_of = [](auto&& f) {
        const auto t0 = std::chrono::steady_clock::now();
        f();
        return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    };
    const size_t nb = x.data.size() * sizeof(float);
    gsa::device::Buffer dbuf(nb);
    std::vector<float> hbuf(x.data.size());
    const double h2d = ms_of([&] { gsa::device::Staging::get().h2d(dbuf.get(), x.data.data(), nb); });
    const double d2h = ms_of([&] { gsa::device::Staging::get().d2h(hbuf.data(), dbuf.get(), nb); });
    const double alloc = ms_of([&] { gsa::Tensor<float> t(1, layout.total_tokens(), model_dim); });
    const double proj = ms_of([&] { auto pr = gsa::project_qkv(x, w); });
    std::printf("{\"views\": %d, \"tokens\": %d, \"precision\": \"%s\", \"iters\": %d, \"ms_mean\": %.3f, "
                "\"ms_best\": %.3f, \"tokens_per_s\": %.1f, \"staging_h2d_gbs\": %.1f, \"staging_d2h_gbs\": %.1f, "
                "\"host_alloc_gbs\": %.1f, \"project_qkv_ms\": %.1f}\n",
                views, layout.total_tokens(), bf16 ? "bf16" : "f32", iters, sum / iters, best,
                layout.total_tokens() / (sum / iters / 1e3), nb / h2d / 1e6, nb / d2h / 1e6, nb / alloc / 1e6, proj);
    return 0;
}

}  // namespace

int main(int argc, char** argv) {
    if (argc >= 4 && std::string(argv[1]) == "--time") {
        try {
            return time_forward(std::atoi(argv[2]), std::atoi(argv[3]), argc >= 5 && std::string(argv[4]) == "bf16");
        } catch (const gsa::GsaError& e) {
            std::fprintf(stderr, "gsa error: %s\n", e.what());
            return 1;
        }
    }
    if (argc < 11) {
        std::fprintf(stderr, "usage: %s out_dir ns frames gh gw s heads model_dim top_k variant\n", argv[0]);
        return 2;
    }
    g_dir = argv[1];
    const int ns = std::atoi(argv[2]), nf = std::atoi(argv[3]), gh = std::atoi(argv[4]), gw = std::atoi(argv[5]);
    const int s = std::atoi(argv[6]), heads = std::atoi(argv[7]), model_dim = std::atoi(argv[8]);
    const int top_k = std::atoi(argv[9]), variant = std::atoi(argv[10]);
    const bool bf16 = argc >= 12 && std::string(argv[11]) == "bf16";
    gsa::device::compute_precision() = bf16 ? gsa::device::Precision::kBf16 : gsa::device::Precision::kF32;
    const int dim = 64;
    g_manifest.open(g_dir + "/manifest.txt");
    try {
        // ---- geometry and error convention (errors.hpp)
        const gsa::TokenLayout layout = gsa::build_token_layout(ns, nf, gh, gw, s);
        expect_throw<gsa::DivisibilityError>("divisibility", [] { gsa::build_token_layout(0, 1, 5, 5, 4); });
        expect_throw<gsa::InvalidTiling>("tiling", [] {
            gsa::KernelTiling t;
            t.block_m = 12;
            gsa::validate_tiling(t);
        });
        expect_throw<gsa::Unsupported>("double", [&] {
            gsa::avg_pool_tokens(gsa::Tensor<double>(1, layout.image_tokens(), 8), layout);
        });

        // ---- weights and X as a reference user would make them (layer.hpp:17-25)
        gsa::LayerWeights<float> w;
        const float wscale = 1.0f / std::sqrt(static_cast<float>(model_dim));
        w.w_q = random_tensor(heads, model_dim, dim, wscale, 2);
        w.w_k = random_tensor(heads, model_dim, dim, wscale, 3);
        w.w_v = random_tensor(heads, model_dim, dim, wscale, 4);
        w.w_g = random_tensor(heads, dim, dim, 1.0f / 8.0f, 5);
        const gsa::Tensor<float> x = random_tensor(1, layout.total_tokens(), model_dim, 1.0f, 1);
        dump("x", x);
        dump("w_q", w.w_q);
        dump("w_k", w.w_k);
        dump("w_v", w.w_v);
        dump("w_g", w.w_g);

        gsa::GsaParams p;
        p.window_s = s;
        p.top_k = top_k;
        p.variant = variant ? gsa::SelectionVariant::kHybrid : gsa::SelectionVariant::kPlain;
        p.ref_stride = 2;

        // ---- the full layer (layer.hpp:177-230)
        gsa::KernelStats stats;
        gsa::GsaOutput<float> r = gsa::gsa_forward(x, layout, p, w, &stats, 8);
        dump("out", r.out);
        dump("q", r.saved.q);
        dump("k", r.saved.k);
        dump("v", r.saved.v);
        dump("qc", r.saved.qc);
        dump("o_comp", r.saved.o_comp_coarse);
        dump("gate", r.saved.gate_vals);
        dump("o_sel", r.saved.o_sel);
        dump("topk", r.saved.topk.indices, "i32", {r.saved.topk.heads, r.saved.topk.rows, r.saved.topk.k});
        dump("plan_offsets", r.saved.plan.offsets, "i64", {static_cast<long>(r.saved.plan.offsets.size())});
        dump("plan_ids", r.saved.plan.window_ids, "i32", {static_cast<long>(r.saved.plan.window_ids.size())});
        dump("lse_comp", r.saved.lse_comp, "f32", {static_cast<long>(r.saved.lse_comp.size())});
        const std::vector<int64_t> st = {static_cast<int64_t>(stats.scores_computed.load()),
                                         static_cast<int64_t>(stats.keys_attended.load())};
        dump("stats", st, "i64", {2});

        // ---- the layer backward (gradients.hpp:54-265) with a random upstream gradient
        {
            const gsa::Tensor<float> d_out = random_tensor(heads, layout.total_tokens(), dim, 1.0f, 6);
            const gsa::GsaGradients<float> g = gsa::gsa_backward(r.saved, d_out, 8);
            dump("d_out", d_out);
            dump("dx", g.dx);
            dump("dw_q", g.dw_q);
            dump("dw_k", g.dw_k);
            dump("dw_v", g.dw_v);
            dump("dw_g", g.dw_g);
            expect_throw<gsa::ContextMismatch>("backward_shape", [&] {
                gsa::gsa_backward(r.saved, gsa::Tensor<float>(heads, layout.total_tokens() - 1, dim));
            });
        }

        // ---- the per-branch operators on the projected tensors
        const float scale = gsa::resolved_scale<float>(p, dim);
        auto parts = gsa::partition_qkv(r.saved.q, r.saved.k, r.saved.v, layout);
        const auto qc = gsa::avg_pool_tokens(parts.q_img, layout);
        const auto kc = gsa::avg_pool_tokens(parts.k_img, layout);
        const auto vc = gsa::avg_pool_tokens(parts.v_img, layout);
        dump("op_kc", kc);
        std::vector<uint8_t> excluded;
        if (variant) excluded = gsa::forced_window_mask(layout, p.ref_stride);
        const auto comp = gsa::fused_compressed_attention_topk(qc, kc, vc, top_k, scale, p.tiling,
                                                               variant ? &excluded : nullptr, true);
        dump("op_topk", comp.topk.indices, "i32", {comp.topk.heads, comp.topk.rows, comp.topk.k});
        std::vector<float> guide(comp.topk.guide_scores.begin(), comp.topk.guide_scores.end());
        dump("op_guide", guide, "f32", {static_cast<long>(guide.size())});
        dump("op_o_comp", comp.out);
        const auto plan = gsa::build_selection_plan(comp.topk, layout, p.variant, p.ref_stride);
        dump("op_plan_ids", plan.window_ids, "i32", {static_cast<long>(plan.window_ids.size())});
        const auto sel = gsa::block_sparse_attention(parts.q_img, parts.k_img, parts.v_img, plan, layout, scale, p.tiling);
        dump("op_o_sel", sel.out);
        dump("op_gate", gsa::gate(parts.q_img, w.w_g));
        dump("op_up", gsa::upsample_nearest(comp.out, layout));
        std::vector<float> lse_spec;
        const auto ospec = gsa::special_token_attention(parts.q_spec, r.saved.k, r.saved.v, scale, p.tiling, &lse_spec);
        dump("op_o_spec", ospec);
        dump("op_out_with_plan", gsa::gsa_forward_with_plan(x, layout, p, w, plan));

        // ---- error paths of the operators
        gsa::SelectionPlan empty = plan;
        std::fill(empty.offsets.begin(), empty.offsets.end(), 0);
        empty.window_ids.clear();
        expect_throw<gsa::EmptySelection>("empty_selection", [&] {
            gsa::block_sparse_attention(parts.q_img, parts.k_img, parts.v_img, empty, layout, scale, p.tiling);
        });
        expect_throw<gsa::ShapeMismatch>("forward_rows", [&] {
            gsa::gsa_forward(gsa::Tensor<float>(1, layout.total_tokens() + 1, model_dim), layout, p, w);
        });
        expect_throw<gsa::NonFiniteInput>("nonfinite", [&] {
            gsa::Tensor<float> bad = x;
            bad.data[0] = NAN;
            gsa::project_qkv(bad, w);
        });
    } catch (const gsa::GsaError& e) {
        std::fprintf(stderr, "gsa error: %s\n", e.what());
        return 1;
    }
    g_manifest << "# done\n";
    return 0;
}
