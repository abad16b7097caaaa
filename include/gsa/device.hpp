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

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <string>
#include <thread>
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
        case GSA_ERR_CONTEXT_MISMATCH: throw ContextMismatch(msg);
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

// Large host <-> device copies of pageable host memory: chunks cycle through two pinned
// staging buffers so the DMA of one chunk overlaps the host-side copy of the other, and
// each host-side copy is split over worker threads (one thread copies ~10 GB/s; PCIe moves
// ~50). Small copies go straight through cudaMemcpy.
class Staging {
  public:
    static constexpr size_t kChunk = size_t(64) << 20;
    static constexpr size_t kDirect = size_t(8) << 20;  // below this: plain cudaMemcpy

    static Staging& get() {
        static Staging s;
        return s;
    }
    void h2d(void* dev, const void* host, size_t bytes) {
        if (bytes < kDirect) {
            check_cuda(cudaMemcpy(dev, host, bytes, cudaMemcpyHostToDevice), "upload");
            return;
        }
        init();
        const char* src = static_cast<const char*>(host);
        char* dst = static_cast<char*>(dev);
        for (size_t off = 0, i = 0; off < bytes; off += kChunk, ++i) {
            const size_t n = std::min(kChunk, bytes - off);
            const int b = static_cast<int>(i & 1);
            check_cuda(cudaEventSynchronize(done_[b]), "upload");  // the slot's previous DMA
            par_copy(pinned_[b], src + off, n);
            check_cuda(cudaMemcpyAsync(dst + off, pinned_[b], n, cudaMemcpyHostToDevice, stream_), "upload");
            check_cuda(cudaEventRecord(done_[b], stream_), "upload");
        }
        check_cuda(cudaStreamSynchronize(stream_), "upload");
    }
    void d2h(void* host, const void* dev, size_t bytes) {
        if (bytes < kDirect) {
            check_cuda(cudaMemcpy(host, dev, bytes, cudaMemcpyDeviceToHost), "download");
            return;
        }
        init();
        check_cuda(cudaStreamSynchronize(nullptr), "download");  // results of the legacy stream
        const char* src = static_cast<const char*>(dev);
        char* dst = static_cast<char*>(host);
        const size_t chunks = (bytes + kChunk - 1) / kChunk;
        auto issue = [&](size_t i) {
            const size_t off = i * kChunk, n = std::min(kChunk, bytes - off);
            check_cuda(cudaMemcpyAsync(pinned_[i & 1], src + off, n, cudaMemcpyDeviceToHost, stream_), "download");
            check_cuda(cudaEventRecord(done_[i & 1], stream_), "download");
        };
        issue(0);
        for (size_t i = 0; i < chunks; ++i) {
            if (i + 1 < chunks) issue(i + 1);  // (its slot's host copy finished in iteration i - 1)
            check_cuda(cudaEventSynchronize(done_[i & 1]), "download");
            const size_t off = i * kChunk;
            par_copy(dst + off, pinned_[i & 1], std::min(kChunk, bytes - off));
        }
    }

    // host-side copy split over worker threads
    static void host_copy(void* dst, const void* src, size_t n) { par_copy(dst, src, n); }

  private:
    Staging() = default;
    ~Staging() {
        for (int b = 0; b < 2; ++b) {
            if (pinned_[b]) cudaFreeHost(pinned_[b]);
            if (done_[b]) cudaEventDestroy(done_[b]);
        }
        if (stream_) cudaStreamDestroy(stream_);
    }
    void init() {
        if (stream_) return;
        check_cuda(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking), "staging stream");
        for (int b = 0; b < 2; ++b) {
            check_cuda(cudaMallocHost(&pinned_[b], kChunk), "staging buffer");
            check_cuda(cudaEventCreateWithFlags(&done_[b], cudaEventDisableTiming), "staging event");
            check_cuda(cudaEventRecord(done_[b], stream_), "staging event");
        }
    }
    static void par_copy(void* dst, const void* src, size_t n) {
        const unsigned hw = std::max(1u, std::min(8u, std::thread::hardware_concurrency()));
        const size_t part = (n / hw + 4095) & ~size_t(4095);
        std::vector<std::thread> th;
        for (unsigned t = 1; t < hw && t * part < n; ++t)
            th.emplace_back([=] {
                std::memcpy(static_cast<char*>(dst) + t * part, static_cast<const char*>(src) + t * part,
                            std::min(part, n - t * part));
            });
        std::memcpy(dst, src, std::min(part, n));
        for (auto& x : th) x.join();
    }
    cudaStream_t stream_ = nullptr;
    void* pinned_[2] = {nullptr, nullptr};
    cudaEvent_t done_[2] = {nullptr, nullptr};
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
    if (bf16) {  // f32 over the bus, rounded to bf16 (RNE) on the device
        Buffer tmp(t.data.size() * 4);
        Staging::get().h2d(tmp.get(), t.data.data(), t.data.size() * 4);
        check(gsa_convert(tmp.get(), GSA_DTYPE_F32, d.buf.get(), GSA_DTYPE_BF16, static_cast<int64_t>(t.data.size()),
                          nullptr));
        sync();
    } else {
        Staging::get().h2d(d.buf.get(), t.data.data(), t.data.size() * 4);
    }
    return d;
}

template <typename U>
Buffer upload_vector(const std::vector<U>& v) {
    Buffer b(v.size() * sizeof(U));
    if (!v.empty()) Staging::get().h2d(b.get(), v.data(), v.size() * sizeof(U));
    return b;
}

template <typename U>
std::vector<U> download_vector(const void* src, size_t n) {
    std::vector<U> v;
    gsa::detail::zero_vector(v, n);
    if (n) Staging::get().d2h(v.data(), src, n * sizeof(U));
    return v;
}

// into a host tensor of d's shape the caller already holds (e.g. allocated on a worker thread)
template <typename T>
void download_into(Tensor<T>& t, const DeviceTensor& d) {
    if (t.heads != d.heads || t.tokens != d.rows || t.dim != d.dim) t = Tensor<T>(d.heads, d.rows, d.dim);
    if (t.data.empty()) return;
    if (d.dtype == GSA_DTYPE_BF16) {  // widened to f32 on the device
        Buffer tmp(t.data.size() * 4);
        check(gsa_convert(d.buf.get(), GSA_DTYPE_BF16, tmp.get(), GSA_DTYPE_F32, static_cast<int64_t>(t.data.size()),
                          nullptr));
        Staging::get().d2h(t.data.data(), tmp.get(), t.data.size() * 4);
    } else {
        Staging::get().d2h(t.data.data(), d.buf.get(), t.data.size() * 4);
    }
}

template <typename T>
Tensor<T> download(const DeviceTensor& d) {
    Tensor<T> t(d.heads, d.rows, d.dim);
    if (t.data.empty()) return t;
    if (d.dtype == GSA_DTYPE_BF16) {  // widened to f32 on the device
        Buffer tmp(t.data.size() * 4);
        check(gsa_convert(d.buf.get(), GSA_DTYPE_BF16, tmp.get(), GSA_DTYPE_F32, static_cast<int64_t>(t.data.size()),
                          nullptr));
        Staging::get().d2h(t.data.data(), tmp.get(), t.data.size() * 4);
    } else {
        Staging::get().d2h(t.data.data(), d.buf.get(), t.data.size() * 4);
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
