// gsa/layer.hpp — the GSA layer (drop-in for the reference's
// proj/include/gsa/layer.hpp:17-262) on the sm_100a library:
//   project_qkv             -> gsa_project_qkv (exact f32 arithmetic of layer.hpp:48-76)
//   special_token_attention -> gsa_special_token_attention
//   gate                    -> gsa_gate
//   gsa_forward             -> gsa_project_qkv + gsa_forward (special path, pooling,
//                              compressed attention + top-k, selection, gate and merge
//                              fused; Q/K/V stay on the device between the two calls)
//   gsa_forward_with_plan   -> gsa_project_qkv + gsa_forward_with_plan
// With the default f32 precision the projected Q/K/V are bit-identical to the
// reference's, so TopkResult indices match it bit for bit end to end.
#pragma once

#include <algorithm>
#include <cmath>
#include <future>
#include <vector>

#include "gsa/compression.hpp"

#include "gsa/device.hpp"
#include "gsa/layout.hpp"
#include "gsa/selection.hpp"
#include "gsa/tensor.hpp"
#include "gsa/types.hpp"

namespace gsa {

// w_q/w_k/w_v: [heads x model_dim x dim], applied as x . W per head; w_g: [heads x dim x dim]
template <typename T>
struct LayerWeights {
    Tensor<T> w_q, w_k, w_v;
    Tensor<T> w_g;

    int heads() const { return w_q.heads; }
    int model_dim() const { return w_q.tokens; }
    int dim() const { return w_q.dim; }
};

template <typename T>
void validate_weights(const LayerWeights<T>& w) {
    const int h = w.w_q.heads, c = w.w_q.tokens, d = w.w_q.dim;
    const auto shaped = [](const Tensor<T>& t, int a, int b, int e) { return t.heads == a && t.tokens == b && t.dim == e; };
    if (!shaped(w.w_k, h, c, d) || !shaped(w.w_v, h, c, d)) throw ShapeMismatch("weights: w_q/w_k/w_v shapes disagree");
    if (!shaped(w.w_g, h, d, d)) throw ShapeMismatch("weights: w_g must be heads x dim x dim");
    require_finite(w.w_q, "w_q");
    require_finite(w.w_k, "w_k");
    require_finite(w.w_v, "w_v");
    require_finite(w.w_g, "w_g");
}

template <typename T>
struct Projected {
    Tensor<T> q, k, v;
};

namespace detail {

struct DeviceQkv {
    device::DeviceTensor q, k, v;
};

// X [1 x tokens x model_dim] -> device Q/K/V [heads x tokens x dim] (f32, or bf16 when
// the compute precision asks for it: the RNE rounding of the exact f32 projection)
template <typename T>
DeviceQkv project_on_device(const Tensor<T>& x, const LayerWeights<T>& weights) {
    validate_weights(weights);
    if (x.heads != 1 || x.dim != weights.model_dim()) throw ShapeMismatch("project_qkv: X must be [1 x tokens x model_dim]");
    require_finite(x, "X");
    device::require_float<T>("project_qkv");
    const int H = weights.heads(), tokens = x.tokens, d = weights.dim();
    const int dt = device::compute_precision() == device::Precision::kBf16 ? GSA_DTYPE_BF16 : GSA_DTYPE_F32;
    const auto xd = device::upload(x), wq = device::upload(weights.w_q), wk = device::upload(weights.w_k),
               wv = device::upload(weights.w_v);
    DeviceQkv r{device::alloc(H, tokens, d, dt), device::alloc(H, tokens, d, dt), device::alloc(H, tokens, d, dt)};
    const gsa_tensor a = r.q.desc(), b = r.k.desc(), c = r.v.desc();
    device::check(gsa_project_qkv(xd.buf.f(), tokens, weights.model_dim(), wq.buf.f(),
                                  wk.buf.f(), wv.buf.f(), H, d, &a, &b, &c, nullptr));
    return r;
}

}  // namespace detail

template <typename T>
Projected<T> project_qkv(const Tensor<T>& x, const LayerWeights<T>& weights) {
    auto d = detail::project_on_device(x, weights);
    return Projected<T>{device::download<T>(d.q), device::download<T>(d.k), device::download<T>(d.v)};
}

// Dense attention of the special tokens over the whole sequence (layer.hpp:80-96).
template <typename T>
Tensor<T> special_token_attention(const Tensor<T>& q_spec, const Tensor<T>& k, const Tensor<T>& v, T scale,
                                  const KernelTiling& tiling = {}, std::vector<T>* lse_out = nullptr,
                                  KernelStats* stats = nullptr, int threads = 1) {
    if (q_spec.tokens == 0) {
        if (lse_out) lse_out->clear();
        return Tensor<T>(q_spec.heads, 0, q_spec.dim);
    }
    Tensor<T> out;
    std::vector<T> lse;
    tiled_attention(q_spec, k, v, scale, tiling, out, lse, stats, threads);
    if (lse_out) *lse_out = std::move(lse);
    return out;
}

// g = sigmoid(q . W_g[h]) elementwise (layer.hpp:99-119)
template <typename T>
Tensor<T> gate(const Tensor<T>& q_img, const Tensor<T>& w_g) {
    if (w_g.heads != q_img.heads || w_g.tokens != q_img.dim || w_g.dim != q_img.dim)
        throw ShapeMismatch("gate: weights must be heads x dim x dim");
    device::require_float<T>("gate");
    const auto q = device::upload(q_img, true), w = device::upload(w_g);
    auto g = device::alloc(q_img.heads, q_img.tokens, q_img.dim);
    const gsa_tensor a = q.desc(), b = w.desc(), c = g.desc();
    device::check(gsa_gate(&a, &b, &c, nullptr));
    return device::download<T>(g);
}

// Everything a backward pass would need (layer.hpp:124-142).
template <typename T>
struct ForwardContext {
    TokenLayout layout;
    GsaParams params;
    LayerWeights<T> weights;
    Tensor<T> x;

    Tensor<T> q, k, v;
    Tensor<T> qc, kc, vc;
    Tensor<T> o_comp_coarse;
    std::vector<T> lse_comp;
    TopkResult topk;
    SelectionPlan plan;
    Tensor<T> o_sel;
    std::vector<T> lse_sel;
    Tensor<T> gate_vals;
    Tensor<T> o_spec;
    std::vector<T> lse_spec;
};

template <typename T>
struct GsaOutput {
    Tensor<T> out;
    ForwardContext<T> saved;
};

// The full layer (layer.hpp:177-230): project, dense special path, pooled
// compressed attention with fused top-k, plan, block-sparse selection, gated
// merge, concatenation — one device call after the projection.
template <typename T>
GsaOutput<T> gsa_forward(const Tensor<T>& x, const TokenLayout& layout, const GsaParams& params,
                         const LayerWeights<T>& weights, KernelStats* stats = nullptr, int threads = 1) {
    (void)threads;
    validate_params(params);
    if (params.window_s != layout.window_s) throw ShapeMismatch("gsa_forward: params.window_s != layout.window_s");
    if (x.tokens != layout.total_tokens()) throw ShapeMismatch("gsa_forward: X rows != layout.total_tokens()");
    device::require_float<T>("gsa_forward");
    GsaOutput<T> r;
    ForwardContext<T>& ctx = r.saved;
    ctx.layout = layout;
    ctx.params = params;
    ctx.weights = weights;
    ctx.x = Tensor<T>(x.heads, x.tokens, x.dim);  // the reference keeps a copy of X (layer.hpp:124-142)
    device::Staging::host_copy(ctx.x.data.data(), x.data.data(), x.data.size() * sizeof(T));

    // the host tensors this call returns (~38 GB at 1000 views) are allocated and zero-filled
    // on worker threads while X uploads and the GPU projects and runs the layer
    const int H = weights.heads(), d = weights.dim(), M = layout.total_tokens();
    const int Ms = layout.num_special, Mi = layout.image_tokens(), W = layout.num_windows();
    auto host = [](int a, int b, int c) {
        return std::async(std::launch::async, [=] { return Tensor<T>(a, b, c); });
    };
    auto h_q = host(H, M, d), h_k = host(H, M, d), h_v = host(H, M, d), h_out = host(H, M, d);
    auto h_osel = host(H, Mi, d), h_gate = host(H, Mi, d);
    auto h_qc = host(H, W, d), h_kc = host(H, W, d), h_vc = host(H, W, d), h_oc = host(H, W, d);
    auto qkv = detail::project_on_device(x, weights);
    const int forced = params.variant == SelectionVariant::kHybrid
                           ? static_cast<int>(forced_frames(layout, params.ref_stride).size()) * layout.windows_per_frame()
                           : 0;
    const int k_cap = std::max(0, std::min(params.top_k, W - forced));
    const auto wg = device::upload(weights.w_g);
    auto out = device::alloc(H, M, d);
    auto qc = device::alloc(H, W, d), kc = device::alloc(H, W, d), vc = device::alloc(H, W, d);
    auto oc = device::alloc(H, W, d), osel = device::alloc(H, Mi, d), gv = device::alloc(H, Mi, d);
    device::Buffer lse_comp(static_cast<size_t>(H) * W * 4), lse_sel(static_cast<size_t>(H) * Mi * 4),
        lse_spec(static_cast<size_t>(H) * std::max(Ms, 1) * 4),
        topk(static_cast<size_t>(H) * W * std::max(k_cap, 1) * 4);
    gsa_context cx{qc.buf.f(), kc.buf.f(), vc.buf.f(), oc.buf.f(),
                   lse_comp.f(), topk.i32(), osel.buf.f(), lse_sel.f(),
                   gv.buf.f(), lse_spec.f()};
    const gsa_layout lc = device::c_layout(layout);
    const gsa_params pc = device::c_params(params);
    const size_t ws_bytes = gsa_forward_workspace_bytes(&lc, &pc, H, d);
    device::Buffer ws(ws_bytes);
    const gsa_tensor a = qkv.q.desc(), b = qkv.k.desc(), c = qkv.v.desc(), w = wg.desc(), o = out.desc();
    int k_eff = 0;
    device::check(gsa_forward(&a, &b, &c, &w, &lc, &pc, &o, &cx, &k_eff, ws.get(), ws_bytes, nullptr));

    ctx.q = h_q.get();
    device::download_into(ctx.q, qkv.q);
    ctx.k = h_k.get();
    device::download_into(ctx.k, qkv.k);
    ctx.v = h_v.get();
    device::download_into(ctx.v, qkv.v);
    ctx.qc = h_qc.get();
    device::download_into(ctx.qc, qc);
    ctx.kc = h_kc.get();
    device::download_into(ctx.kc, kc);
    ctx.vc = h_vc.get();
    device::download_into(ctx.vc, vc);
    ctx.o_comp_coarse = h_oc.get();
    device::download_into(ctx.o_comp_coarse, oc);
    ctx.lse_comp = device::download_f32<T>(lse_comp, static_cast<size_t>(H) * W);
    ctx.topk = TopkResult(H, W, k_eff);
    ctx.topk.indices = device::download_vector<int32_t>(topk.get(), static_cast<size_t>(H) * W * k_eff);
    ctx.plan = build_selection_plan(ctx.topk, layout, params.variant, params.ref_stride);
    ctx.o_sel = h_osel.get();
    device::download_into(ctx.o_sel, osel);
    ctx.lse_sel = device::download_f32<T>(lse_sel, static_cast<size_t>(H) * Mi);
    ctx.gate_vals = h_gate.get();
    device::download_into(ctx.gate_vals, gv);
    r.out = h_out.get();
    device::download_into(r.out, out);
    ctx.o_spec = slice_rows(r.out, 0, Ms);
    ctx.lse_spec = device::download_f32<T>(lse_spec, static_cast<size_t>(H) * Ms);
    if (stats) {
        uint64_t scores = 0, keys = 0;
        device::check(gsa_forward_stats(&lc, &pc, H, &scores, &keys));
        stats->scores_computed.fetch_add(scores);
        stats->keys_attended.fetch_add(keys);
    }
    return r;
}

// Forward with the selection pinned to `plan` (layer.hpp:235-262); the
// compressed branch is plain tiled attention over the pooled tensors.
template <typename T>
Tensor<T> gsa_forward_with_plan(const Tensor<T>& x, const TokenLayout& layout, const GsaParams& params,
                                const LayerWeights<T>& weights, const SelectionPlan& plan) {
    validate_params(params);
    if (x.tokens != layout.total_tokens()) throw ShapeMismatch("gsa_forward_with_plan: X rows != layout.total_tokens()");
    device::require_float<T>("gsa_forward_with_plan");
    if (plan.heads != weights.heads() || plan.rows != layout.num_windows() ||
        plan.offsets.size() != static_cast<size_t>(plan.heads) * plan.rows + 1)
        throw ShapeMismatch("block_sparse_attention: plan shape does not match layout/heads");
    for (int h = 0; h < plan.heads; ++h)
        for (int w = 0; w < plan.rows; ++w)
            if (plan.row_size(h, w) == 0) throw EmptySelection("block_sparse_attention: empty plan row");
    auto qkv = detail::project_on_device(x, weights);
    const int H = weights.heads(), d = weights.dim(), M = layout.total_tokens();
    const auto wg = device::upload(weights.w_g);
    auto out = device::alloc(H, M, d);
    device::Buffer offs_d = device::upload_vector(plan.offsets), ids_d = device::upload_vector(plan.window_ids);
    const gsa_layout lc = device::c_layout(layout);
    const gsa_params pc = device::c_params(params);
    const size_t ws_bytes = gsa_forward_workspace_bytes(&lc, &pc, H, d);
    device::Buffer ws(ws_bytes);
    const gsa_tensor a = qkv.q.desc(), b = qkv.k.desc(), c = qkv.v.desc(), w = wg.desc(), o = out.desc();
    device::check(gsa_forward_with_plan(&a, &b, &c, &w, &lc, &pc, offs_d.i64(), ids_d.i32(), &o,
                                        ws.get(), ws_bytes, nullptr));
    return device::download<T>(out);
}

}  // namespace gsa
