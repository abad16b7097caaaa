// gsa/gradients.hpp — the layer backward (drop-in for the reference's
// proj/include/gsa/gradients.hpp:14-320) on the sm_100a library:
//   avg_pool_backward   -> gsa_avg_pool_backward   (bit-identical)
//   upsample_backward   -> gsa_upsample_backward   (bit-identical)
//   gsa_backward        -> gsa_backward (gate fuse, upsample / pooling adjoints, compressed,
//                          selection and special attention backward from the saved LSE
//                          rows, dW_g) + gsa_project_backward (dW_q/k/v, dX), all f32 on
//                          the device with the selection detached, as in the reference
//   kahan_inner, finite_difference_check: host numerics utilities (same contracts)
#pragma once

#include <algorithm>
#include <cmath>
#include <cstring>
#include <functional>
#include <vector>

#include "gsa/layer.hpp"

namespace gsa {

template <typename T>
struct GsaGradients {
    Tensor<T> dx;                // [1 x tokens x model_dim]
    Tensor<T> dw_q, dw_k, dw_v;  // [heads x model_dim x dim]
    Tensor<T> dw_g;              // [heads x dim x dim]
};

// Adjoint of avg_pool_tokens (gradients.hpp:21-34): member rows get their window's row / s^2.
template <typename T>
Tensor<T> avg_pool_backward(const Tensor<T>& d_pooled, const TokenLayout& layout) {
    if (d_pooled.tokens != layout.num_windows()) throw ShapeMismatch("avg_pool_backward: rows != num windows");
    device::require_float<T>("avg_pool_backward");
    const auto in = device::upload(d_pooled);
    auto out = device::alloc(d_pooled.heads, layout.image_tokens(), d_pooled.dim);
    const gsa_layout lc = device::c_layout(layout);
    const gsa_tensor a = in.desc(), b = out.desc();
    device::check(gsa_avg_pool_backward(&a, &lc, &b, nullptr));
    return device::download<T>(out);
}

// Adjoint of upsample_nearest (gradients.hpp:37-49): member rows summed into their window.
template <typename T>
Tensor<T> upsample_backward(const Tensor<T>& d_fine, const TokenLayout& layout) {
    if (d_fine.tokens != layout.image_tokens()) throw ShapeMismatch("upsample_backward: rows != image tokens");
    device::require_float<T>("upsample_backward");
    const auto in = device::upload(d_fine);
    auto out = device::alloc(d_fine.heads, layout.num_windows(), d_fine.dim);
    const gsa_layout lc = device::c_layout(layout);
    const gsa_tensor a = in.desc(), b = out.desc();
    device::check(gsa_upsample_backward(&a, &lc, &b, nullptr));
    return device::download<T>(out);
}

// Backward of gsa_forward with the top-k selection held constant (gradients.hpp:54-265):
// the saved context goes to the device once, the layer backward and the projection
// backward run there, and the five gradients come back. `threads` is accepted for
// signature compatibility (the device decides its own parallelism).
template <typename T>
GsaGradients<T> gsa_backward(const ForwardContext<T>& ctx, const Tensor<T>& d_out, int threads = 1) {
    (void)threads;
    device::require_float<T>("gsa_backward");
    const TokenLayout& layout = ctx.layout;
    const int H = ctx.weights.heads(), d = ctx.weights.dim(), C = ctx.weights.model_dim();
    const int M = layout.total_tokens(), Ms = layout.num_special, W = layout.num_windows();
    if (d_out.heads != H || d_out.tokens != M || d_out.dim != d)
        throw ContextMismatch("gsa_backward: dO shape does not match the saved forward");
    if (ctx.q.tokens != M || ctx.x.tokens != M || ctx.o_spec.tokens != Ms)
        throw ContextMismatch("gsa_backward: saved context is inconsistent");
    if (ctx.plan.heads != H || ctx.plan.rows != W)
        throw ContextMismatch("gsa_backward: saved plan does not match the layout");

    // saved tensors as the forward left them (f32; bf16-precision runs saved the rounded values)
    const auto q = device::upload(ctx.q), k = device::upload(ctx.k), v = device::upload(ctx.v);
    const auto wg = device::upload(ctx.weights.w_g);
    const auto qc = device::upload(ctx.qc), kc = device::upload(ctx.kc), vc = device::upload(ctx.vc);
    const auto oc = device::upload(ctx.o_comp_coarse), osel = device::upload(ctx.o_sel);
    const auto gv = device::upload(ctx.gate_vals), ospec = device::upload(ctx.o_spec);
    const auto go = device::upload(d_out);
    auto f32_vector = [](const std::vector<T>& s) { return device::upload_vector(std::vector<float>(s.begin(), s.end())); };
    const device::Buffer lse_comp = f32_vector(ctx.lse_comp), lse_sel = f32_vector(ctx.lse_sel),
                         lse_spec = f32_vector(ctx.lse_spec);
    const device::Buffer offs = device::upload_vector(ctx.plan.offsets), ids = device::upload_vector(ctx.plan.window_ids);

    gsa_saved sv{};
    sv.qc = qc.buf.f();
    sv.kc = kc.buf.f();
    sv.vc = vc.buf.f();
    sv.o_comp = oc.buf.f();
    sv.lse_comp = lse_comp.f();
    sv.plan_offsets = offs.i64();
    sv.plan_ids = ids.i32();
    sv.plan_entries = static_cast<int64_t>(ctx.plan.window_ids.size());
    sv.o_sel = osel.buf.f();
    sv.lse_sel = lse_sel.f();
    sv.gate = gv.buf.f();
    sv.o_spec = ospec.desc();
    sv.lse_spec = lse_spec.f();

    auto dq = device::alloc(H, M, d), dk = device::alloc(H, M, d), dv = device::alloc(H, M, d);
    auto dwg = device::alloc(H, d, d);
    const gsa_layout lc = device::c_layout(layout);
    const gsa_params pc = device::c_params(ctx.params);
    const size_t ws_bytes = gsa_backward_workspace_bytes(&lc, &pc, H, d, sv.plan_entries, GSA_DTYPE_F32);
    {
        device::Buffer ws(ws_bytes);
        const gsa_tensor a = q.desc(), b = k.desc(), c = v.desc(), w = wg.desc(), o = go.desc();
        const gsa_tensor tq = dq.desc(), tk = dk.desc(), tv = dv.desc();
        device::check(gsa_backward(&a, &b, &c, &w, &lc, &pc, &sv, &o, &tq, &tk, &tv, dwg.buf.f(), ws.get(), ws_bytes,
                                   nullptr));
    }

    // projection backward (gradients.hpp:226-263)
    const auto x = device::upload(ctx.x), wq = device::upload(ctx.weights.w_q), wk = device::upload(ctx.weights.w_k),
               wv = device::upload(ctx.weights.w_v);
    auto dx = device::alloc(1, M, C), dwq = device::alloc(H, C, d), dwk = device::alloc(H, C, d),
         dwv = device::alloc(H, C, d);
    const size_t pws_bytes = gsa_project_backward_workspace_bytes(M, C, H, d);
    device::Buffer pws(pws_bytes);
    device::check(gsa_project_backward(x.buf.f(), M, C, wq.buf.f(), wk.buf.f(), wv.buf.f(), H, d, dq.buf.f(),
                                       dk.buf.f(), dv.buf.f(), dx.buf.f(), dwq.buf.f(), dwk.buf.f(), dwv.buf.f(),
                                       pws.get(), pws_bytes, nullptr));
    GsaGradients<T> g;
    g.dx = device::download<T>(dx);
    g.dw_q = device::download<T>(dwq);
    g.dw_k = device::download<T>(dwk);
    g.dw_v = device::download<T>(dwv);
    g.dw_g = device::download<T>(dwg);
    return g;
}

// Kahan-compensated inner product in double (gradients.hpp:269-281).
template <typename T>
double kahan_inner(const Tensor<T>& a, const Tensor<T>& b) {
    if (!a.same_shape(b)) throw ShapeMismatch("kahan_inner: shapes differ");
    double total = 0.0, lost = 0.0;
    for (size_t i = 0; i < a.data.size(); ++i) {
        const double y = static_cast<double>(a.data[i]) * static_cast<double>(b.data[i]) - lost;
        const double next = total + y;
        lost = (next - total) - y;
        total = next;
    }
    return total;
}

// Central differences against an analytic gradient (gradients.hpp:287-320): the worst
// relative error over the probed coordinates (all, or `coords`), denominator
// max(|analytic|, |numeric|, 1e-12); `forward` must be bitwise deterministic.
inline double finite_difference_check(const std::function<double(const std::vector<double>&)>& forward,
                                      const std::vector<double>& point, const std::vector<double>& analytic_grad,
                                      double epsilon, const std::vector<int>* coords = nullptr) {
    if (point.size() != analytic_grad.size())
        throw ShapeMismatch("finite_difference_check: gradient size != point size");
    const double base = forward(point), again = forward(point);
    if (std::memcmp(&base, &again, sizeof(double)) != 0)
        throw NonDeterministicForward("finite_difference_check: forward is not deterministic");
    std::vector<double> probe = point;
    double worst = 0.0;
    auto check_one = [&](size_t j) {
        const double x0 = probe[j];
        probe[j] = x0 + epsilon;
        const double up = forward(probe);
        probe[j] = x0 - epsilon;
        const double down = forward(probe);
        probe[j] = x0;
        const double numeric = (up - down) / (2.0 * epsilon);
        const double denom = std::max({std::abs(analytic_grad[j]), std::abs(numeric), 1e-12});
        worst = std::max(worst, std::abs(analytic_grad[j] - numeric) / denom);
    };
    if (coords) {
        for (int j : *coords) check_one(static_cast<size_t>(j));
    } else {
        for (size_t j = 0; j < point.size(); ++j) check_one(j);
    }
    return worst;
}

}  // namespace gsa
