// gsa/layout.hpp — token geometry (drop-in for the reference's
// proj/include/gsa/layout.hpp:13-69 and proj/src/layout.cpp:7-56).
// Sequence order: [special tokens][frame 0 grid, row-major][frame 1]...; each
// frame's grid is tiled by non-overlapping s x s windows. Header-only: the
// integer geometry is the same closed form the sm_100a kernels evaluate.
#pragma once

#include <vector>

#include "gsa/errors.hpp"
#include "gsa/tensor.hpp"
#include "gsa_sm100.h"

namespace gsa {

struct TokenLayout {
    int num_special = 0;
    int num_frames = 1;
    int grid_h = 0;
    int grid_w = 0;
    int window_s = 1;

    int tokens_per_frame() const { return grid_h * grid_w; }
    int image_tokens() const { return num_frames * tokens_per_frame(); }
    int total_tokens() const { return num_special + image_tokens(); }
    int wins_h() const { return grid_h / window_s; }
    int wins_w() const { return grid_w / window_s; }
    int windows_per_frame() const { return wins_h() * wins_w(); }
    int num_windows() const { return num_frames * windows_per_frame(); }

    // image_token_index counts from the first image token (layout.cpp:26-35)
    int window_of_token(int image_token_index) const {
        if (image_token_index < 0 || image_token_index >= image_tokens())
            throw IndexOutOfRange("window_of_token: image token index out of range");
        const int f = image_token_index / tokens_per_frame(), r = image_token_index % tokens_per_frame();
        return f * windows_per_frame() + (r / grid_w / window_s) * wins_w() + (r % grid_w) / window_s;
    }

    // the s^2 member image tokens, ascending: window rows outer, columns inner (layout.cpp:37-56)
    std::vector<int> tokens_of_window(int window_index) const {
        if (window_index < 0 || window_index >= num_windows())
            throw IndexOutOfRange("tokens_of_window: window index out of range");
        const int f = window_index / windows_per_frame(), r = window_index % windows_per_frame();
        const int top = (r / wins_w()) * window_s, left = (r % wins_w()) * window_s;
        std::vector<int> members;
        members.reserve(static_cast<size_t>(window_s) * window_s);
        for (int dr = 0; dr < window_s; ++dr)
            for (int dc = 0; dc < window_s; ++dc)
                members.push_back(f * tokens_per_frame() + (top + dr) * grid_w + left + dc);
        return members;
    }

    int frame_of_window(int window_index) const {
        if (window_index < 0 || window_index >= num_windows())
            throw IndexOutOfRange("frame_of_window: window index out of range");
        return window_index / windows_per_frame();
    }
};

// layout.cpp:7-24 validation, evaluated by the device library's gsa_make_layout
inline TokenLayout build_token_layout(int num_special, int num_frames, int grid_h, int grid_w, int window_s) {
    gsa_layout l;
    const int rc = gsa_make_layout(num_special, num_frames, grid_h, grid_w, window_s, &l);
    if (rc == GSA_ERR_DIVISIBILITY) throw DivisibilityError(gsa_last_error_message());
    if (rc == GSA_ERR_ZERO_SIZE) throw ZeroSizeError(gsa_last_error_message());
    if (rc == GSA_ERR_UNSUPPORTED) throw Unsupported(gsa_last_error_message());
    if (rc != GSA_OK) throw GsaError(gsa_last_error_message());
    TokenLayout t;
    t.num_special = num_special;
    t.num_frames = num_frames;
    t.grid_h = grid_h;
    t.grid_w = grid_w;
    t.window_s = window_s;
    return t;
}

template <typename T>
struct QkvPartition {
    Tensor<T> q_spec, k_spec, v_spec;
    Tensor<T> q_img, k_img, v_img;
};

// layout.hpp:54-69: special rows [0, Ms) and image rows [Ms, M) of each tensor
template <typename T>
QkvPartition<T> partition_qkv(const Tensor<T>& q, const Tensor<T>& k, const Tensor<T>& v, const TokenLayout& layout) {
    const int total = layout.total_tokens();
    if (q.tokens != total || k.tokens != total || v.tokens != total)
        throw ShapeMismatch("partition_qkv: token count does not match layout");
    require_same_heads_dim(q, k, "partition_qkv");
    require_same_heads_dim(q, v, "partition_qkv");
    const int ms = layout.num_special, mi = layout.image_tokens();
    return QkvPartition<T>{slice_rows(q, 0, ms), slice_rows(k, 0, ms), slice_rows(v, 0, ms),
                           slice_rows(q, ms, mi), slice_rows(k, ms, mi), slice_rows(v, ms, mi)};
}

}  // namespace gsa
