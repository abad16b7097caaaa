// gsa/compression.hpp — the compression branch (drop-in for the reference's
// proj/include/gsa/compression.hpp:20-297), executed by the sm_100a kernels:
//   avg_pool_tokens                 -> gsa_avg_pool_tokens   (K1, HBM-bound, bit-exact)
//   upsample_nearest                -> gsa_upsample_nearest
//   tiled_attention                 -> gsa_tiled_attention   (K5, tcgen05 flash attention)
//   fused_compressed_attention_topk -> gsa_compressed_attention_topk (K2, tcgen05 scores +
//                                      exact re-score: indices bit-exact with the reference)
// `tiling` is validated like the reference's and otherwise ignored (the kernels
// pick their own tiles; results are tiling-independent in both). `threads` is
// accepted and ignored: there is no CPU path.
#pragma once

#include <algorithm>
#include <cstdint>
#include <vector>

#include "gsa/device.hpp"
#include "gsa/layout.hpp"
#include "gsa/tensor.hpp"
#include "gsa/types.hpp"

namespace gsa {

template <typename T>
Tensor<T> avg_pool_tokens(const Tensor<T>& x_img, const TokenLayout& layout) {
    if (x_img.tokens != layout.image_tokens()) throw ShapeMismatch("avg_pool_tokens: rows != image tokens");
    device::require_float<T>("avg_pool_tokens");
    const auto x = device::upload(x_img);
    auto out = device::alloc(x_img.heads, layout.num_windows(), x_img.dim);
    const gsa_layout lc = device::c_layout(layout);
    const gsa_tensor xd = x.desc(), od = out.desc();
    device::check(gsa_avg_pool_tokens(&xd, &lc, &od, nullptr));
    return device::download<T>(out);
}

template <typename T>
Tensor<T> upsample_nearest(const Tensor<T>& coarse, const TokenLayout& layout) {
    if (coarse.tokens != layout.num_windows()) throw ShapeMismatch("upsample_nearest: rows != num windows");
    device::require_float<T>("upsample_nearest");
    const auto c = device::upload(coarse);
    auto out = device::alloc(coarse.heads, layout.image_tokens(), coarse.dim);
    const gsa_layout lc = device::c_layout(layout);
    const gsa_tensor cd = c.desc(), od = out.desc();
    device::check(gsa_upsample_nearest(&cd, &lc, &od, nullptr));
    return device::download<T>(out);
}

// out = softmax(q k^T * scale) v, lse[h*mq + i] = m + log(l)  (compression.hpp:99-165)
template <typename T>
void tiled_attention(const Tensor<T>& q, const Tensor<T>& k, const Tensor<T>& v, T scale, const KernelTiling& tiling,
                     Tensor<T>& out, std::vector<T>& lse, KernelStats* stats = nullptr, int threads = 1) {
    (void)threads;
    require_same_heads_dim(q, k, "tiled_attention");
    require_same_heads_dim(q, v, "tiled_attention");
    if (k.tokens != v.tokens) throw ShapeMismatch("tiled_attention: K/V token counts differ");
    validate_tiling(tiling);
    device::require_float<T>("tiled_attention");
    const auto qd = device::upload(q, true), kd = device::upload(k, true), vd = device::upload(v, true);
    auto od = device::alloc(q.heads, q.tokens, q.dim);
    device::Buffer lse_d(static_cast<size_t>(q.heads) * q.tokens * sizeof(float));
    const gsa_tensor a = qd.desc(), b = kd.desc(), c = vd.desc(), o = od.desc();
    device::check(gsa_tiled_attention(&a, &b, &c, static_cast<float>(scale), tiling.block_m, tiling.block_n, &o,
                                      lse_d.f(), nullptr));
    out = device::download<T>(od);
    lse = device::download_f32<T>(lse_d, static_cast<size_t>(q.heads) * q.tokens);
    if (stats) stats->scores_computed.fetch_add(static_cast<uint64_t>(q.heads) * q.tokens * k.tokens);
}

template <typename T>
struct CompressedResult {
    Tensor<T> out;       // coarse attention output, one row per window
    std::vector<T> lse;  // heads * windows
    TopkResult topk;
};

// compression.hpp:180-297. Excluded windows count in the softmax but are never
// top-k candidates; the realised width is min(k, selectable windows).
template <typename T>
CompressedResult<T> fused_compressed_attention_topk(const Tensor<T>& qc, const Tensor<T>& kc, const Tensor<T>& vc,
                                                    int k, T scale, const KernelTiling& tiling,
                                                    const std::vector<uint8_t>* excluded = nullptr,
                                                    bool keep_guide_scores = false, KernelStats* stats = nullptr,
                                                    int threads = 1) {
    (void)threads;
    if (kc.tokens != vc.tokens || qc.tokens != kc.tokens)
        throw ShapeMismatch("fused_compressed_attention_topk: Q/K/V must share the window count");
    require_same_heads_dim(qc, kc, "fused_compressed_attention_topk");
    require_same_heads_dim(qc, vc, "fused_compressed_attention_topk");
    validate_tiling(tiling);
    if (k < 0) throw GsaError("fused_compressed_attention_topk: k must be >= 0");
    if (excluded && static_cast<int>(excluded->size()) != kc.tokens)
        throw ShapeMismatch("fused_compressed_attention_topk: exclusion mask size");
    device::require_float<T>("fused_compressed_attention_topk");
    const int H = qc.heads, W = qc.tokens, d = qc.dim;
    int selectable = W;
    if (excluded)
        for (uint8_t e : *excluded) selectable -= e ? 1 : 0;
    const int k_cap = std::max(0, std::min(k, selectable));
    const auto q = device::upload(qc), kk = device::upload(kc), v = device::upload(vc);
    auto od = device::alloc(H, W, d);
    device::Buffer lse_d(static_cast<size_t>(H) * W * sizeof(float));
    device::Buffer idx_d(static_cast<size_t>(H) * W * std::max(1, k_cap) * sizeof(int32_t));
    device::Buffer guide_d(keep_guide_scores ? static_cast<size_t>(H) * W * std::max(1, k_cap) * sizeof(float) : 0);
    device::Buffer ex_d = excluded ? device::upload_vector(*excluded) : device::Buffer();
    const size_t ws_bytes = gsa_compressed_attention_topk_workspace_bytes(H, W, d, k_cap);
    device::Buffer ws(ws_bytes);
    const gsa_tensor a = q.desc(), b = kk.desc(), c = v.desc(), o = od.desc();
    int k_eff = 0;
    device::check(gsa_compressed_attention_topk(&a, &b, &c, k, static_cast<float>(scale), tiling.block_m,
                                                tiling.block_n, excluded ? ex_d.u8() : nullptr,
                                                excluded ? W : 0, &o, lse_d.f(), idx_d.i32(),
                                                keep_guide_scores ? guide_d.f() : nullptr, &k_eff, ws.get(),
                                                ws_bytes, nullptr));
    CompressedResult<T> r;
    r.out = device::download<T>(od);
    r.lse = device::download_f32<T>(lse_d, static_cast<size_t>(H) * W);
    r.topk = TopkResult(H, W, k_eff);
    r.topk.indices = device::download_vector<int32_t>(idx_d.get(), static_cast<size_t>(H) * W * k_eff);
    if (keep_guide_scores) {
        const auto g = device::download_vector<float>(guide_d.get(), static_cast<size_t>(H) * W * k_eff);
        r.topk.guide_scores.assign(g.begin(), g.end());
    }
    if (stats) stats->scores_computed.fetch_add(static_cast<uint64_t>(H) * W * W);
    return r;
}

}  // namespace gsa
