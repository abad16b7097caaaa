// gsa/selection.hpp — the selection branch (drop-in for the reference's
// proj/include/gsa/selection.hpp:19-136 and proj/src/selection.cpp:7-67):
//   forced_frames / forced_windows_of / forced_window_mask  (hybrid variant)
//   build_selection_plan   -> gsa_build_selection_plan (device CSR build)
//   block_sparse_attention -> gsa_block_sparse_attention (K4 gather attention)
#pragma once

#include <cstdint>
#include <vector>

#include "gsa/device.hpp"
#include "gsa/layout.hpp"
#include "gsa/tensor.hpp"
#include "gsa/types.hpp"

namespace gsa {

// Per (head, query window) key-window lists, CSR-packed (selection.hpp:19-33).
struct SelectionPlan {
    int heads = 0;
    int rows = 0;                         // num_windows
    std::vector<int64_t> offsets;         // heads * rows + 1
    std::vector<int32_t> window_ids;      // row payloads
    std::vector<int32_t> forced_windows;  // ascending; empty for plain

    int row_size(int h, int r) const {
        const size_t i = static_cast<size_t>(h) * rows + r;
        return static_cast<int>(offsets[i + 1] - offsets[i]);
    }
    const int32_t* row(int h, int r) const { return window_ids.data() + offsets[static_cast<size_t>(h) * rows + r]; }
};

// Reference frame 0 and every ref_stride-th frame after it (selection.cpp:7-12).
inline std::vector<int> forced_frames(const TokenLayout& layout, int ref_stride) {
    if (ref_stride < 1) throw InvalidStride("forced_frames: ref_stride must be >= 1");
    std::vector<int> frames;
    for (int f = 0; f < layout.num_frames; f += ref_stride) frames.push_back(f);
    return frames;
}

// All windows of the forced frames, ascending (selection.cpp:14-21), from the device library.
inline std::vector<int32_t> forced_windows_of(const TokenLayout& layout, int ref_stride) {
    const gsa_layout lc = device::c_layout(layout);
    int n = 0;
    device::check(gsa_forced_windows(&lc, ref_stride, nullptr, &n, nullptr));
    device::Buffer d(static_cast<size_t>(n) * sizeof(int32_t));
    device::check(gsa_forced_windows(&lc, ref_stride, d.i32(), &n, nullptr));
    return device::download_vector<int32_t>(d.get(), static_cast<size_t>(n));
}

inline std::vector<uint8_t> forced_window_mask(const TokenLayout& layout, int ref_stride) {
    std::vector<uint8_t> mask(static_cast<size_t>(layout.num_windows()), 0);
    for (int32_t w : forced_windows_of(layout, ref_stride)) mask[static_cast<size_t>(w)] = 1;
    return mask;
}

// plain: the top-k rows; hybrid: forced windows (ascending) then the dynamic
// entries in score order, forced duplicates dropped (selection.cpp:29-67).
inline SelectionPlan build_selection_plan(const TopkResult& topk, const TokenLayout& layout, SelectionVariant variant,
                                          int ref_stride) {
    const gsa_layout lc = device::c_layout(layout);
    const int H = topk.heads, R = topk.rows, K = topk.k;
    const int v = variant == SelectionVariant::kHybrid ? 1 : 0;
    const int64_t rows = static_cast<int64_t>(H) * R;
    device::Buffer top_d = device::upload_vector(topk.indices);
    device::Buffer offs_d(static_cast<size_t>(rows + 1) * sizeof(int64_t));
    const int64_t cap = rows * (K + (v ? layout.num_windows() : 0));
    device::Buffer ids_d(static_cast<size_t>(std::max<int64_t>(cap, 1)) * sizeof(int32_t));
    const size_t ws_bytes = gsa_build_selection_plan_workspace_bytes(H, R, K, &lc, ref_stride > 0 ? ref_stride : 1);
    device::Buffer ws(ws_bytes);
    int64_t n_ids = 0;
    device::check(gsa_build_selection_plan(top_d.i32(), H, R, K, &lc, v, ref_stride, offs_d.i64(),
                                           ids_d.i32(), cap, &n_ids, ws.get(), ws_bytes, nullptr));
    SelectionPlan plan;
    plan.heads = H;
    plan.rows = R;
    plan.offsets = device::download_vector<int64_t>(offs_d.get(), static_cast<size_t>(rows + 1));
    plan.window_ids = device::download_vector<int32_t>(ids_d.get(), static_cast<size_t>(n_ids));
    if (v) plan.forced_windows = forced_windows_of(layout, ref_stride);
    return plan;
}

template <typename T>
struct SelectionResult {
    Tensor<T> out;       // one row per image token
    std::vector<T> lse;  // heads * image_tokens
};

// Fine attention restricted to the plan: the s^2 queries of window w attend the
// s^2 members of every window in row (h, w) (selection.hpp:63-136).
template <typename T>
SelectionResult<T> block_sparse_attention(const Tensor<T>& q_img, const Tensor<T>& k_img, const Tensor<T>& v_img,
                                          const SelectionPlan& plan, const TokenLayout& layout, T scale,
                                          const KernelTiling& tiling, KernelStats* stats = nullptr, int threads = 1) {
    (void)threads;
    if (q_img.tokens != layout.image_tokens()) throw ShapeMismatch("block_sparse_attention: Q rows != image tokens");
    if (k_img.tokens != layout.image_tokens() || v_img.tokens != layout.image_tokens())
        throw ShapeMismatch("block_sparse_attention: K/V rows != image tokens");
    require_same_heads_dim(q_img, k_img, "block_sparse_attention");
    require_same_heads_dim(q_img, v_img, "block_sparse_attention");
    validate_tiling(tiling);
    if (plan.heads != q_img.heads || plan.rows != layout.num_windows())
        throw ShapeMismatch("block_sparse_attention: plan shape does not match layout/heads");
    if (plan.offsets.size() != static_cast<size_t>(plan.heads) * plan.rows + 1)
        throw ShapeMismatch("block_sparse_attention: plan offsets size");
    device::require_float<T>("block_sparse_attention");
    const auto q = device::upload(q_img, true), k = device::upload(k_img, true), v = device::upload(v_img, true);
    device::Buffer offs_d = device::upload_vector(plan.offsets);
    device::Buffer ids_d = device::upload_vector(plan.window_ids);
    auto od = device::alloc(q_img.heads, layout.image_tokens(), q_img.dim);
    device::Buffer lse_d(static_cast<size_t>(q_img.heads) * layout.image_tokens() * sizeof(float));
    const gsa_layout lc = device::c_layout(layout);
    const gsa_tensor a = q.desc(), b = k.desc(), c = v.desc(), o = od.desc();
    device::check(gsa_block_sparse_attention(&a, &b, &c, offs_d.i64(), ids_d.i32(), &lc,
                                             static_cast<float>(scale), &o, lse_d.f(), nullptr));
    SelectionResult<T> r;
    r.out = device::download<T>(od);
    r.lse = device::download_f32<T>(lse_d, static_cast<size_t>(q_img.heads) * layout.image_tokens());
    if (stats) {
        const uint64_t s2 = static_cast<uint64_t>(layout.window_s) * layout.window_s;
        stats->keys_attended.fetch_add(static_cast<uint64_t>(plan.window_ids.size()) * s2 * s2);
    }
    return r;
}

}  // namespace gsa
