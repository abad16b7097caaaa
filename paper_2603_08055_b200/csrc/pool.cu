// pool.cu — K1: s x s window mean pooling (avg_pool_tokens, compression.hpp:20-38).
//
// HBM-bound: every image row of Q/K/V is read once (bf16: 2*d bytes) and one
// f32 row per window is written (optionally plus the hi/lo bf16 split the
// tensor-core compressed-attention kernel consumes, and the row norm used by
// its error bound). Each thread owns 8 consecutive features of one window and
// adds the s*s member rows in the reference's ascending member order with
// round-to-nearest adds, then multiplies by 1/s^2: bit-identical to the CPU.
// A cross-member warp-shuffle tree would reorder the sum and move top-k
// indices (SURVEY §0 finding 1), so shuffles are used only for the norm.
#include "kernels.h"

namespace gsa_sm100 {
namespace {

struct PoolJobs {
    PoolJob j[3];
};

template <typename T, bool VEC8>
__global__ void __launch_bounds__(256) pool_kernel(PoolJobs jobs, int njobs, int heads, int dim,
                                                   DevLayout L, float inv) {
    const int chunk = VEC8 ? 8 : 1;
    const int chunks = dim / chunk;
    const int64_t per_job = (int64_t)heads * L.windows * chunks;
    const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const bool active = gid < per_job * njobs;
    int64_t rem = active ? gid : 0;
    const int jb = (int)(rem / per_job);
    rem -= (int64_t)jb * per_job;
    const int c = (int)(rem % chunks);
    rem /= chunks;
    const int w = (int)(rem % L.windows);
    const int h = (int)(rem / L.windows);
    const PoolJob& J = jobs.j[jb];
    const T* base = reinterpret_cast<const T*>(J.in.data) + (int64_t)h * J.in.hs + c * chunk;

    float acc[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[i] = 0.0f;
    const int s2 = L.s * L.s;
    if (active) {
        for (int m = 0; m < s2; ++m) {
            const T* src = base + (int64_t)L.member(w, m) * J.in.rs;
            float x[8];
            if (VEC8) {
                load8(src, x);
            } else {
                x[0] = to_f32(src[0]);
            }
#pragma unroll
            for (int i = 0; i < chunk; ++i) acc[i] = __fadd_rn(acc[i], x[i]);
        }
    }
    float sq = 0.0f;
#pragma unroll
    for (int i = 0; i < chunk; ++i) {
        acc[i] = __fmul_rn(acc[i], inv);
        sq = fmaf(acc[i], acc[i], sq);
    }
    const int64_t ohs = J.out_hs ? J.out_hs : (int64_t)L.windows * dim;
    const int64_t orow = (int64_t)h * ohs + (int64_t)w * dim + c * chunk;
    if (active) {
        if (VEC8) {
            float4* o = reinterpret_cast<float4*>(J.out + orow);
            o[0] = make_float4(acc[0], acc[1], acc[2], acc[3]);
            o[1] = make_float4(acc[4], acc[5], acc[6], acc[7]);
        } else {
            J.out[orow] = acc[0];
        }
        if (J.hi) {
            __nv_bfloat16 hi[8], lo[8];
#pragma unroll
            for (int i = 0; i < chunk; ++i) {
                hi[i] = __float2bfloat16_rn(acc[i]);
                lo[i] = __float2bfloat16_rn(acc[i] - __bfloat162float(hi[i]));
            }
            if (VEC8) {
                *reinterpret_cast<uint4*>(J.hi + orow) = *reinterpret_cast<uint4*>(hi);
                *reinterpret_cast<uint4*>(J.lo + orow) = *reinterpret_cast<uint4*>(lo);
            } else {
                J.hi[orow] = hi[0];
                J.lo[orow] = lo[0];
            }
        }
    }
    // ||row||_2 for the tensor-core path's error bound. The `chunks` lanes of a
    // window are consecutive and aligned, so the xor-tree never mixes windows;
    // every lane takes part (the condition is grid-uniform).
    if (VEC8 && chunks <= 32 && (32 % chunks) == 0) {
        for (int o = chunks / 2; o > 0; o >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o);
        if (J.norm && active && c == 0) J.norm[(int64_t)h * L.windows + w] = sqrtf(sq);
    }
}

}  // namespace

cudaError_t launch_pool(const PoolJob* jobs, int njobs, int heads, int dim, const DevLayout& L,
                        float inv, cudaStream_t st) {
    if (njobs <= 0 || njobs > 3) return cudaErrorInvalidValue;
    PoolJobs pj{};
    bool vec = (dim % 8) == 0;
    int dtype = jobs[0].in.dtype;
    for (int i = 0; i < njobs; ++i) {
        pj.j[i] = jobs[i];
        if (jobs[i].in.dtype != dtype) return cudaErrorInvalidValue;
        const int align = dtype == GSA_DTYPE_BF16 ? 8 : 4;
        if (jobs[i].in.rs % align || jobs[i].in.hs % align ||
            (reinterpret_cast<uintptr_t>(jobs[i].in.data) & 15))
            vec = false;
        if (reinterpret_cast<uintptr_t>(jobs[i].out) & 15) vec = false;
    }
    const int chunks = vec ? dim / 8 : dim;
    const int64_t total = (int64_t)njobs * heads * L.windows * chunks;
    if (total == 0) return cudaSuccess;
    // grid: the block count is rounded up; a thread past the end is inactive
    // but still joins the norm shuffle so the warp stays converged.
    const int64_t blocks = (total + 255) / 256;
    if (dtype == GSA_DTYPE_BF16) {
        if (vec) pool_kernel<__nv_bfloat16, true><<<blocks, 256, 0, st>>>(pj, njobs, heads, dim, L, inv);
        else pool_kernel<__nv_bfloat16, false><<<blocks, 256, 0, st>>>(pj, njobs, heads, dim, L, inv);
    } else {
        if (vec) pool_kernel<float, true><<<blocks, 256, 0, st>>>(pj, njobs, heads, dim, L, inv);
        else pool_kernel<float, false><<<blocks, 256, 0, st>>>(pj, njobs, heads, dim, L, inv);
    }
    note_launch();
    return cudaGetLastError();
}

}  // namespace gsa_sm100
