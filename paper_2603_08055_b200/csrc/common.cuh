// common.cuh — shared device helpers for the sm_100a GSA kernels.
#pragma once

#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "gsa_sm100.h"

namespace gsa_sm100 {

// ---------------------------------------------------------------- loads
template <typename T>
__device__ __forceinline__ float to_f32(T x);
template <>
__device__ __forceinline__ float to_f32<float>(float x) {
    return x;
}
template <>
__device__ __forceinline__ float to_f32<__nv_bfloat16>(__nv_bfloat16 x) {
    return __bfloat162float(x);
}

// 8 consecutive elements -> 8 floats (16-byte aligned bf16, 32-byte aligned f32)
__device__ __forceinline__ void load8(const __nv_bfloat16* p, float* o) {
    const uint4 u = __ldg(reinterpret_cast<const uint4*>(p));
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const float2 f = __bfloat1622float2(h[i]);
        o[2 * i] = f.x;
        o[2 * i + 1] = f.y;
    }
}
__device__ __forceinline__ void load8(const float* p, float* o) {
    const float4 a = __ldg(reinterpret_cast<const float4*>(p));
    const float4 b = __ldg(reinterpret_cast<const float4*>(p) + 1);
    o[0] = a.x; o[1] = a.y; o[2] = a.z; o[3] = a.w;
    o[4] = b.x; o[5] = b.y; o[6] = b.z; o[7] = b.w;
}

// ------------------------------------------------------ exact score order
// scaled_dot (dot.hpp:11-23): four stride-4 lane sums, each product and sum
// rounded separately (no FMA contraction), combined ((s0+s1)+(s2+s3))*scale.
struct ExactDot4 {
    float s0, s1, s2, s3;
    __device__ __forceinline__ void zero() { s0 = s1 = s2 = s3 = 0.0f; }
    __device__ __forceinline__ void step(float a0, float a1, float a2, float a3, float b0, float b1,
                                         float b2, float b3) {
        s0 = __fadd_rn(s0, __fmul_rn(a0, b0));
        s1 = __fadd_rn(s1, __fmul_rn(a1, b1));
        s2 = __fadd_rn(s2, __fmul_rn(a2, b2));
        s3 = __fadd_rn(s3, __fmul_rn(a3, b3));
    }
    __device__ __forceinline__ void tail(float a, float b) { s0 = __fadd_rn(s0, __fmul_rn(a, b)); }
    __device__ __forceinline__ float finish(float scale) const {
        return __fmul_rn(__fadd_rn(__fadd_rn(s0, s1), __fadd_rn(s2, s3)), scale);
    }
};

__device__ __forceinline__ float exact_scaled_dot(const float* a, const float* b, int n,
                                                  float scale) {
    ExactDot4 acc;
    acc.zero();
    int i = 0;
    for (; i + 4 <= n; i += 4) acc.step(a[i], a[i + 1], a[i + 2], a[i + 3], b[i], b[i + 1], b[i + 2], b[i + 3]);
    for (; i < n; ++i) acc.tail(a[i], b[i]);
    return acc.finish(scale);
}

// topk_better (compression.hpp:67-73) for real entries (index >= 0)
__device__ __forceinline__ bool topk_better(float sa, int ia, float sb, int ib) {
    if (ib < 0) return ia >= 0;
    if (ia < 0) return false;
    if (sa != sb) return sa > sb;
    return ia < ib;
}

// --------------------------------------------------------- layout helpers
struct DevLayout {
    int num_special, num_frames, grid_h, grid_w, s;
    int wins_w, wins_per_frame, tokens_per_frame, windows, image_tokens;
    __host__ __device__ __forceinline__ int window_of_token(int t) const {
        const int f = t / tokens_per_frame, r = t - f * tokens_per_frame;
        const int row = r / grid_w, col = r - row * grid_w;
        return f * wins_per_frame + (row / s) * wins_w + col / s;
    }
    // member m (0..s*s-1) of window w, in the reference's ascending order
    __host__ __device__ __forceinline__ int member(int w, int m) const {
        const int f = w / wins_per_frame, r = w - f * wins_per_frame;
        const int wr = r / wins_w, wc = r - wr * wins_w;
        const int dr = m / s, dc = m - dr * s;
        return f * tokens_per_frame + (wr * s + dr) * grid_w + wc * s + dc;
    }
};

inline DevLayout make_dev_layout(const gsa_layout& l) {
    DevLayout d;
    d.num_special = l.num_special;
    d.num_frames = l.num_frames;
    d.grid_h = l.grid_h;
    d.grid_w = l.grid_w;
    d.s = l.window_s;
    d.wins_w = l.grid_w / l.window_s;
    d.wins_per_frame = (l.grid_h / l.window_s) * d.wins_w;
    d.tokens_per_frame = l.grid_h * l.grid_w;
    d.windows = d.wins_per_frame * l.num_frames;
    d.image_tokens = d.tokens_per_frame * l.num_frames;
    return d;
}

// A selection row: CSR (offsets/ids) or "forced list ++ dynamic top-k row".
struct RowSource {
    const int64_t* offsets;  // CSR form when non-null
    const int32_t* ids;
    const int32_t* forced;  // otherwise: forced[0..n_forced) then dyn[r*dyn_stride ..+dyn_count)
    int n_forced;
    const int32_t* dyn;
    int dyn_stride, dyn_count;
    __device__ __forceinline__ int64_t size(int64_t r) const {
        return offsets ? offsets[r + 1] - offsets[r] : (int64_t)n_forced + dyn_count;
    }
    __device__ __forceinline__ int window(int64_t r, int64_t j) const {
        if (offsets) return ids[offsets[r] + j];
        return j < n_forced ? forced[j] : dyn[r * dyn_stride + (j - n_forced)];
    }
};

}  // namespace gsa_sm100
