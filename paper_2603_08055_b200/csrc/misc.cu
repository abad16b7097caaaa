// misc.cu — small device kernels around the hot path: the stand-alone gate
// (layer.hpp:99-119), nearest upsampling (compression.hpp:42-53), the hybrid
// forced-window set (selection.cpp:7-27) and the CSR selection plan
// (selection.cpp:29-67).
#include <algorithm>
#include <cub/device/device_scan.cuh>

#include "kernels.h"

namespace gsa_sm100 {
namespace {

// g[h][t][j] = sigmoid(sum_a q[h][t][a] * w[h][a][j]); one warp per row, a
// thread per (up to 4) output features; a ascending like the reference loop.
template <typename T>
__global__ void gate_kernel(TensorRef q, int heads, int rows, int dim, const float* __restrict__ w,
                            float* g, int64_t g_hs, int64_t g_rs) {
    const int64_t row = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
    const int lane = threadIdx.x & 31;
    if (row >= (int64_t)heads * rows) return;
    const int h = (int)(row / rows), t = (int)(row % rows);
    const T* qr = reinterpret_cast<const T*>(q.data) + (int64_t)h * q.hs + (int64_t)t * q.rs;
    const float* wh = w + (int64_t)h * dim * dim;
    float* gr = g + (int64_t)h * g_hs + (int64_t)t * g_rs;
    for (int j = lane; j < dim; j += 32) {
        float z = 0.0f;
        for (int a = 0; a < dim; ++a) z = fmaf(to_f32(qr[a]), wh[(int64_t)a * dim + j], z);
        gr[j] = 1.0f / (1.0f + expf(-z));
    }
}

// rows of a [H][rows][64] tensor (any strides; f32 or bf16) -> contiguous bf16 planes
// [H][rows][64]: hi = RN(x), lo = RN(x - hi) (f32 only; lo may be null). One thread = 8
// features. Feeds the tensor-core selection with TMA-loadable operands.
template <typename T>
__global__ void pack_rows_kernel(TensorRef in, int heads, int rows, __nv_bfloat16* __restrict__ hi,
                                 __nv_bfloat16* __restrict__ lo) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;  // over heads*rows*8
    if (i >= (int64_t)heads * rows * 8) return;
    const int c = (int)(i & 7);
    const int64_t hr = i >> 3;
    const int h = (int)(hr / rows), r = (int)(hr - (int64_t)h * rows);
    const T* src = reinterpret_cast<const T*>(in.data) + (int64_t)h * in.hs + (int64_t)r * in.rs + 8 * c;
    __align__(16) __nv_bfloat16 vh[8], vl[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
        const float x = to_f32(src[e]);
        vh[e] = __float2bfloat16_rn(x);
        vl[e] = __float2bfloat16_rn(x - __bfloat162float(vh[e]));
    }
    *reinterpret_cast<uint4*>(hi + 8 * i) = *reinterpret_cast<const uint4*>(vh);
    if (lo) *reinterpret_cast<uint4*>(lo + 8 * i) = *reinterpret_cast<const uint4*>(vl);
}

__device__ __forceinline__ int v16_exp(float vmax) { return vmax > 0.0f ? ilogbf(vmax) - 13 : 0; }

// max |v| per head (blockIdx.y): |x| bit patterns order like the values
template <typename T>
__global__ void vmax_kernel(TensorRef v, int rows, unsigned* vmax_bits) {
    const int h = blockIdx.y;
    unsigned mx = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < (int64_t)rows * 8;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int r = (int)(i >> 3), c = (int)(i & 7);
        const T* src = reinterpret_cast<const T*>(v.data) + h * v.hs + r * v.rs + 8 * c;
#pragma unroll
        for (int e = 0; e < 8; ++e) mx = max(mx, __float_as_uint(fabsf(to_f32(src[e]))));
    }
    mx = __reduce_max_sync(0xffffffffu, mx);
    if ((threadIdx.x & 31) == 0) atomicMax(&vmax_bits[h], mx);
}

template <typename T>
__global__ void v16_kernel(TensorRef v, int heads, int rows, const unsigned* __restrict__ vmax_bits,
                           __half* __restrict__ hi, __half* __restrict__ lo) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;  // over heads*rows*8
    if (i >= (int64_t)heads * rows * 8) return;
    const int c = (int)(i & 7);
    const int64_t hr = i >> 3;
    const int h = (int)(hr / rows), r = (int)(hr - (int64_t)h * rows);
    const float sc = ldexpf(1.0f, -v16_exp(__uint_as_float(vmax_bits[h])));
    const T* src = reinterpret_cast<const T*>(v.data) + h * v.hs + (int64_t)r * v.rs + 8 * c;
    __align__(16) __half vh[8], vl[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
        const float x = to_f32(src[e]) * sc;  // exact: power-of-two scale
        vh[e] = __float2half_rn(x);
        vl[e] = __float2half_rn(x - __half2float(vh[e]));
    }
    *reinterpret_cast<uint4*>(hi + 8 * i) = *reinterpret_cast<const uint4*>(vh);
    if (lo) *reinterpret_cast<uint4*>(lo + 8 * i) = *reinterpret_cast<const uint4*>(vl);
}

__global__ void upsample_kernel(const float* __restrict__ c, int64_t c_hs, int64_t c_rs, int heads,
                                int dim, DevLayout L, float* o, int64_t o_hs, int64_t o_rs) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t n = (int64_t)heads * L.image_tokens * dim;
    if (i >= n) return;
    const int j = (int)(i % dim);
    const int64_t ht = i / dim;
    const int h = (int)(ht / L.image_tokens), t = (int)(ht % L.image_tokens);
    o[(int64_t)h * o_hs + (int64_t)t * o_rs + j] = c[(int64_t)h * c_hs + (int64_t)L.window_of_token(t) * c_rs + j];
}

// forced frames {0, r, 2r, ...}; their windows in ascending order (selection.cpp:7-21)
__global__ void forced_kernel(DevLayout L, int ref_stride, int32_t* forced, uint8_t* mask) {
    const int w = blockIdx.x * blockDim.x + threadIdx.x;
    if (w >= L.windows) return;
    const int f = w / L.wins_per_frame;
    const bool is_forced = (f % ref_stride) == 0;
    if (mask) mask[w] = is_forced ? 1 : 0;
    if (forced && is_forced) {
        const int rank = (f / ref_stride) * L.wins_per_frame + (w - f * L.wins_per_frame);
        forced[rank] = w;
    }
}

// flag bit 2: a top-k id outside [0, W) (the reference would index its forced mask /
// tokens_of_window with it: IndexOutOfRange, layout.cpp:37-56); such ids are counted as
// dynamic so the plan stays well-formed, and the caller reports the error
__global__ void plan_count_kernel(const int32_t* __restrict__ topk, int64_t rows, int k,
                                  const uint8_t* __restrict__ mask, int n_forced, int W, int64_t* sizes,
                                  int* flag) {
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= rows) return;
    int n = 0;
    bool bad = false;
    for (int j = 0; j < k; ++j) {
        const int32_t w = topk[r * k + j];
        const bool ok = w >= 0 && w < W;
        bad |= !ok;
        n += (ok && mask && mask[w]) ? 0 : 1;
    }
    if (bad && flag) atomicOr(flag, 2);
    sizes[r] = n + (mask ? n_forced : 0);
}

__global__ void plan_fill_kernel(const int32_t* __restrict__ topk, int64_t rows, int k,
                                 const uint8_t* __restrict__ mask, const int32_t* __restrict__ forced,
                                 int n_forced, int n_windows, const int64_t* __restrict__ offsets, int32_t* ids) {
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= rows) return;
    int64_t o = offsets[r];
    if (mask)
        for (int i = 0; i < n_forced; ++i) ids[o++] = forced[i];
    for (int j = 0; j < k; ++j) {
        const int32_t w = topk[r * k + j];
        if (!(mask && w >= 0 && w < n_windows && mask[w])) ids[o++] = w;
    }
}

// plan validation (block_sparse_attention, selection.hpp:82-85 + tokens_of_window's range
// check): flag bit 1 = an empty (or negative-size) row, bit 2 = a window id outside [0, W)
__global__ void plan_check_kernel(const int64_t* __restrict__ offsets, int64_t rows, const int32_t* __restrict__ ids,
                                  int W, int* flag) {
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= rows) return;
    const int64_t a = offsets[r], b = offsets[r + 1];
    if (b <= a) atomicOr(flag, 1);
    if (!ids) {
        if (b > a) atomicOr(flag, 4);  // non-empty rows but no id array
        return;
    }
    bool bad = a < 0;
    for (int64_t i = a; i < b && !bad; ++i) bad = ids[i] < 0 || ids[i] >= W;
    if (bad) atomicOr(flag, 2);
}

__global__ void set_zero_kernel(int64_t* p) { *p = 0; }

}  // namespace

cudaError_t launch_gate(const TensorRef& q, int heads, int rows, int dim, const float* w_g, float* g,
                        int64_t g_hs, int64_t g_rs, cudaStream_t st) {
    const int64_t n = (int64_t)heads * rows;
    if (n == 0) return cudaSuccess;
    const int wpb = 8;
    const unsigned blocks = (unsigned)((n + wpb - 1) / wpb);
    if (q.dtype == GSA_DTYPE_BF16)
        { gate_kernel<__nv_bfloat16><<<blocks, 32 * wpb, 0, st>>>(q, heads, rows, dim, w_g, g, g_hs, g_rs); note_launch(); }
    else
        { gate_kernel<float><<<blocks, 32 * wpb, 0, st>>>(q, heads, rows, dim, w_g, g, g_hs, g_rs); note_launch(); }
    return cudaGetLastError();
}

cudaError_t launch_pack_rows(const TensorRef& in, int heads, int rows, __nv_bfloat16* hi, __nv_bfloat16* lo,
                             cudaStream_t st) {
    const int64_t n = (int64_t)heads * rows * 8;
    if (n == 0) return cudaSuccess;
    const unsigned blocks = (unsigned)((n + 255) / 256);
    if (in.dtype == GSA_DTYPE_F32)
        pack_rows_kernel<float><<<blocks, 256, 0, st>>>(in, heads, rows, hi, lo);
    else
        pack_rows_kernel<__nv_bfloat16><<<blocks, 256, 0, st>>>(in, heads, rows, hi, nullptr);
    note_launch();
    return cudaGetLastError();
}

__global__ void f32_to_bf16_kernel(const float* __restrict__ x, __nv_bfloat16* __restrict__ y, int64_t n) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        y[i] = __float2bfloat16_rn(x[i]);
}
__global__ void bf16_to_f32_kernel(const __nv_bfloat16* __restrict__ x, float* __restrict__ y, int64_t n) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        y[i] = __bfloat162float(x[i]);
}

cudaError_t launch_convert(const void* src, int src_dtype, void* dst, int dst_dtype, int64_t n, cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    if (src_dtype == dst_dtype)
        return cudaMemcpyAsync(dst, src, (size_t)n * (src_dtype == GSA_DTYPE_BF16 ? 2 : 4), cudaMemcpyDeviceToDevice, st);
    const unsigned blocks = (unsigned)std::min<int64_t>((n + 255) / 256, 148 * 32);
    if (src_dtype == GSA_DTYPE_F32)
        f32_to_bf16_kernel<<<blocks, 256, 0, st>>>(static_cast<const float*>(src), static_cast<__nv_bfloat16*>(dst), n);
    else
        bf16_to_f32_kernel<<<blocks, 256, 0, st>>>(static_cast<const __nv_bfloat16*>(src), static_cast<float*>(dst), n);
    note_launch();
    return cudaGetLastError();
}

cudaError_t launch_v16(const TensorRef& v, int heads, int rows, unsigned* vmax, __half* hi, __half* lo,
                       cudaStream_t st) {
    cudaMemsetAsync(vmax, 0, (size_t)heads * 4, st);
    if ((int64_t)heads * rows == 0) return cudaSuccess;
    const int blocks = (int)std::min<int64_t>(((int64_t)rows * 8 + 255) / 256, 512);
    const unsigned cb = (unsigned)(((int64_t)heads * rows * 8 + 255) / 256);
    if (v.dtype == GSA_DTYPE_F32) {
        vmax_kernel<float><<<dim3(blocks, heads), 256, 0, st>>>(v, rows, vmax);
        v16_kernel<float><<<cb, 256, 0, st>>>(v, heads, rows, vmax, hi, lo);
    } else {
        vmax_kernel<__nv_bfloat16><<<dim3(blocks, heads), 256, 0, st>>>(v, rows, vmax);
        v16_kernel<__nv_bfloat16><<<cb, 256, 0, st>>>(v, heads, rows, vmax, hi, nullptr);
    }
    note_launch(2);
    return cudaGetLastError();
}

cudaError_t launch_upsample(const float* coarse, int64_t c_hs, int64_t c_rs, int heads, int dim,
                            const DevLayout& L, float* out, int64_t o_hs, int64_t o_rs,
                            cudaStream_t st) {
    const int64_t n = (int64_t)heads * L.image_tokens * dim;
    if (n == 0) return cudaSuccess;
    { upsample_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(coarse, c_hs, c_rs, heads, dim, L, out, o_hs, o_rs); note_launch(); }
    return cudaGetLastError();
}

cudaError_t launch_forced(const DevLayout& L, int ref_stride, int32_t* forced, uint8_t* mask,
                          cudaStream_t st) {
    if (L.windows == 0) return cudaSuccess;
    { forced_kernel<<<(L.windows + 255) / 256, 256, 0, st>>>(L, ref_stride, forced, mask); note_launch(); }
    return cudaGetLastError();
}

cudaError_t launch_plan_count(const int32_t* topk, int64_t rows, int k, const uint8_t* mask,
                              int n_forced, int n_windows, int64_t* sizes, int* flag, cudaStream_t st) {
    if (rows == 0) return cudaSuccess;
    { plan_count_kernel<<<(unsigned)((rows + 255) / 256), 256, 0, st>>>(topk, rows, k, mask, n_forced, n_windows, sizes, flag); note_launch(); }
    return cudaGetLastError();
}

cudaError_t launch_plan_fill(const int32_t* topk, int64_t rows, int k, const uint8_t* mask,
                             const int32_t* forced, int n_forced, int n_windows, const int64_t* offsets,
                             int32_t* ids, cudaStream_t st) {
    if (rows == 0) return cudaSuccess;
    { plan_fill_kernel<<<(unsigned)((rows + 255) / 256), 256, 0, st>>>(topk, rows, k, mask, forced, n_forced, n_windows, offsets, ids); note_launch(); }
    return cudaGetLastError();
}

size_t scan_offsets_tmp_bytes(int64_t n) {
    size_t bytes = 0;
    cub::DeviceScan::InclusiveSum(nullptr, bytes, (const int64_t*)nullptr, (int64_t*)nullptr, (int)n);
    return bytes;
}

// offsets[0] = 0, offsets[i+1] = sizes[0] + ... + sizes[i]
cudaError_t launch_scan_offsets(const int64_t* sizes, int64_t n, int64_t* offsets, void* tmp,
                                size_t tmp_bytes, cudaStream_t st) {
    { set_zero_kernel<<<1, 1, 0, st>>>(offsets); note_launch(); }
    if (n == 0) return cudaGetLastError();
    return cub::DeviceScan::InclusiveSum(tmp, tmp_bytes, sizes, offsets + 1, (int)n, st);
}

cudaError_t launch_plan_check(const int64_t* offsets, int64_t rows, const int32_t* ids, int n_windows, int* flag,
                              cudaStream_t st) {
    if (rows == 0) return cudaSuccess;
    { plan_check_kernel<<<(unsigned)((rows + 255) / 256), 256, 0, st>>>(offsets, rows, ids, n_windows, flag); note_launch(); }
    return cudaGetLastError();
}

}  // namespace gsa_sm100
