// gsa/device.hpp — plumbing between the host operator API (Tensor<T>,
// exceptions) and the sm_100a C ABI (include/gsa_sm100.h): RAII device
// buffers, host<->device transfer, descriptor construction, and the mapping of
// gsa_status codes onto the reference's exception classes (errors.hpp).
//
// Every operator of this API runs on the GPU; there is no CPU fallback. Calls
// are synchronous at the API boundary (results are host tensors, as in the
// reference) and use the CUDA legacy default stream.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>
#include <string>
#include <type_traits>
#include <vector>

#include "gsa/errors.hpp"
#include "gsa/layout.hpp"
#include "gsa/tensor.hpp"
#include "gsa/types.hpp"
#include "gsa_sm100.h"

namespace gsa {
namespace device {

// Arithmetic type the Q/K/V operands are uploaded in. kF32 (default) keeps the
// caller's values exactly; kBf16 rounds them to bf16 on upload and takes the
// tensor-core fast paths. Pooled / compressed / gate / output tensors are f32
// either way.
enum class Precision { kF32, kBf16 };

inline Precision& compute_precision() {
    static Precision p = Precision::kF32;
    return p;
}

[[noreturn]] inline void raise(int status) {
    const std::string msg = gsa_last_error_message();
    switch (status) {
        case GSA_ERR_SHAPE_MISMATCH: throw ShapeMismatch(msg);
        case GSA_ERR_DIVISIBILITY: throw DivisibilityError(msg);
        case GSA_ERR_ZERO_SIZE: throw ZeroSizeError(msg);
        case GSA_ERR_INDEX_OUT_OF_RANGE: throw IndexOutOfRange(msg);
        case GSA_ERR_NON_FINITE: throw NonFiniteInput(msg);
        case GSA_ERR_INVALID_TILING: throw InvalidTiling(msg);
        case GSA_ERR_INVALID_STRIDE: throw InvalidStride(msg);
        case GSA_ERR_EMPTY_SELECTION: throw EmptySelection(msg);
        case GSA_ERR_UNSUPPORTED: throw Unsupported(msg);
        case GSA_ERR_CUDA: throw CudaError(msg);
        default: throw GsaError(std::string(gsa_status_string(status)) + ": " + msg);
    }
}

inline void check(int status) {
    if (status != GSA_OK) raise(status);
}

inline void check_cuda(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw CudaError(std::string(what) + ": " + cudaGetErrorString(e));
}

inline void sync() { check_cuda(cudaStreamSynchronize(nullptr), "cudaStreamSynchronize"); }

// Owning device allocation (move-only).
class Buffer {
  public:
    Buffer() = default;
    explicit Buffer(size_t bytes) : bytes_(bytes) {
        if (bytes_) check_cuda(cudaMalloc(&ptr_, bytes_), "cudaMalloc");
    }
    ~Buffer() {
        if (ptr_) cudaFree(ptr_);
    }
    Buffer(Buffer&& o) noexcept : ptr_(o.ptr_), bytes_(o.bytes_) {
        o.ptr_ = nullptr;
        o.bytes_ = 0;
    }
    Buffer& operator=(Buffer&& o) noexcept {
        if (this != &o) {
            if (ptr_) cudaFree(ptr_);
            ptr_ = o.ptr_;
            bytes_ = o.bytes_;
            o.ptr_ = nullptr;
            o.bytes_ = 0;
        }
        return *this;
    }
    Buffer(const Buffer&) = delete;
    Buffer& operator=(const Buffer&) = delete;

    void* get() const { return ptr_; }
    template <typename U>
    U* as() const {
        return static_cast<U*>(ptr_);
    }
    size_t bytes() const { return bytes_; }
    float* f() const { return static_cast<float*>(ptr_); }
    int32_t* i32() const { return static_cast<int32_t*>(ptr_); }
    int64_t* i64() const { return static_cast<int64_t*>(ptr_); }
    uint8_t* u8() const { return static_cast<uint8_t*>(ptr_); }

  private:
    void* ptr_ = nullptr;
    size_t bytes_ = 0;
};

// bf16 round-to-nearest-even of a finite float (NaN kept quiet)
inline uint16_t bf16_bits(float x) {
    uint32_t u;
    std::memcpy(&u, &x, 4);
    if ((u & 0x7f800000u) == 0x7f800000u) return static_cast<uint16_t>((u >> 16) | ((u & 0xffffu) ? 0x40u : 0u));
    u += 0x7fffu + ((u >> 16) & 1u);
    return static_cast<uint16_t>(u >> 16);
}

inline float bf16_to_float(uint16_t b) {
    const uint32_t u = static_cast<uint32_t>(b) << 16;
    float f;
    std::memcpy(&f, &u, 4);
    return f;
}

// The sm_100a kernels compute in f32 / bf16: Tensor<double> is rejected.
template <typename T>
inline void require_float(const char* what) {
    if (!std::is_same<T, float>::value)
        throw Unsupported(std::string(what) + ": the sm_100a implementation takes Tensor<float> only");
}

// A device copy of a host tensor, as f32 or (operands only) bf16.
struct DeviceTensor {
    Buffer buf;
    int dtype = GSA_DTYPE_F32;
    int heads = 0, rows = 0, dim = 0;

    gsa_tensor desc() const {
        return gsa_tensor{buf.get(), dtype, heads, rows, dim, static_cast<int64_t>(rows) * dim, dim};
    }
    gsa_tensor rows_view(int begin, int count) const {
        const size_t es = dtype == GSA_DTYPE_BF16 ? 2 : 4;
        return gsa_tensor{static_cast<char*>(buf.get()) + static_cast<size_t>(begin) * dim * es, dtype, heads, count,
                          dim, static_cast<int64_t>(rows) * dim, dim};
    }
};

inline DeviceTensor alloc(int heads, int rows, int dim, int dtype = GSA_DTYPE_F32) {
    DeviceTensor d;
    d.dtype = dtype;
    d.heads = heads;
    d.rows = rows;
    d.dim = dim;
    d.buf = Buffer(static_cast<size_t>(heads) * rows * dim * (dtype == GSA_DTYPE_BF16 ? 2 : 4));
    return d;
}

template <typename T>
DeviceTensor upload(const Tensor<T>& t, bool operand = false) {
    require_float<T>("upload");
    const bool bf16 = operand && compute_precision() == Precision::kBf16;
    DeviceTensor d = alloc(t.heads, t.tokens, t.dim, bf16 ? GSA_DTYPE_BF16 : GSA_DTYPE_F32);
    if (t.data.empty()) return d;
    if (bf16) {
        std::vector<uint16_t> tmp(t.data.size());
        for (size_t i = 0; i < tmp.size(); ++i) tmp[i] = bf16_bits(static_cast<float>(t.data[i]));
        check_cuda(cudaMemcpy(d.buf.get(), tmp.data(), tmp.size() * 2, cudaMemcpyHostToDevice), "upload");
    } else {
        check_cuda(cudaMemcpy(d.buf.get(), t.data.data(), t.data.size() * 4, cudaMemcpyHostToDevice), "upload");
    }
    return d;
}

template <typename U>
Buffer upload_vector(const std::vector<U>& v) {
    Buffer b(v.size() * sizeof(U));
    if (!v.empty()) check_cuda(cudaMemcpy(b.get(), v.data(), v.size() * sizeof(U), cudaMemcpyHostToDevice), "upload");
    return b;
}

template <typename U>
std::vector<U> download_vector(const void* src, size_t n) {
    std::vector<U> v(n);
    if (n) check_cuda(cudaMemcpy(v.data(), src, n * sizeof(U), cudaMemcpyDeviceToHost), "download");
    return v;
}

template <typename T>
Tensor<T> download(const DeviceTensor& d) {
    Tensor<T> t(d.heads, d.rows, d.dim);
    if (t.data.empty()) return t;
    if (d.dtype == GSA_DTYPE_BF16) {
        const auto bits = download_vector<uint16_t>(d.buf.get(), t.data.size());
        for (size_t i = 0; i < bits.size(); ++i) t.data[i] = static_cast<T>(bf16_to_float(bits[i]));
    } else {
        check_cuda(cudaMemcpy(t.data.data(), d.buf.get(), t.data.size() * 4, cudaMemcpyDeviceToHost), "download");
    }
    return t;
}

template <typename T>
std::vector<T> download_f32(const Buffer& b, size_t n) {
    const auto f = download_vector<float>(b.get(), n);
    return std::vector<T>(f.begin(), f.end());
}

inline gsa_layout c_layout(const TokenLayout& l) {
    return gsa_layout{l.num_special, l.num_frames, l.grid_h, l.grid_w, l.window_s};
}

inline gsa_params c_params(const GsaParams& p) {
    return gsa_params{p.window_s, p.top_k, p.scale, p.variant == SelectionVariant::kHybrid ? 1 : 0, p.ref_stride,
                      p.tiling.block_m, p.tiling.block_n};
}

}  // namespace device
}  // namespace gsa
