// project.cu — per-head Q/K/V projection (project_qkv, layer.hpp:48-76) with
// the reference's exact arithmetic: out[h][t][j] = sum over a = 0..C-1, in
// ascending order, of x[t][a] * w[h][a][j], each product and sum rounded
// separately (the canonical reference build has no FMA). The projection is an
// adjacent stage, not the hot path; this kernel lets the C++
// drop-in's gsa_forward(x, ...) reproduce the reference's Q/K/V bit for bit so
// the top-k parity contract holds end to end. A tensor-core bf16 projection
// would be ~50x faster but moves indices; it is out of scope here.
//
// Tiling: one CTA = 64 tokens x 64 output features of one (matrix, head); 256
// threads each own a 4 x 4 register tile; x and w stream through shared memory
// in 16-wide slices of the reduction axis, consumed in ascending order.
#include "kernels.h"

namespace gsa_sm100 {
namespace {

constexpr int BT = 64, BJ = 64, BA = 16;

template <typename OutT>
__global__ void __launch_bounds__(256) project_kernel(const float* __restrict__ x, int tokens, int C,
                                                      ProjectMats mats, int heads, int dim) {
    __shared__ float xs[BA][BT + 4];  // [a][t]
    __shared__ float wsm[BA][BJ];     // [a][j]
    const int t0 = blockIdx.x * BT, j0 = blockIdx.y * BJ;
    const int hm = blockIdx.z, m = hm / heads, h = hm % heads;
    const float* w = mats.w[m] + (size_t)h * C * dim;
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;  // 16 x 16 threads, 4 x 4 each
    float acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) acc[i][jj] = 0.0f;
    for (int a0 = 0; a0 < C; a0 += BA) {
        for (int e = threadIdx.x; e < BA * BT; e += 256) {
            const int t = e / BA, a = e % BA;
            xs[a][t] = (t0 + t < tokens && a0 + a < C) ? x[(size_t)(t0 + t) * C + a0 + a] : 0.0f;
        }
        for (int e = threadIdx.x; e < BA * BJ; e += 256) {
            const int a = e / BJ, j = e % BJ;
            wsm[a][j] = (a0 + a < C && j0 + j < dim) ? w[(size_t)(a0 + a) * dim + j0 + j] : 0.0f;
        }
        __syncthreads();
        const int na = min(BA, C - a0);
        for (int a = 0; a < na; ++a) {
            float xv[4], wv[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) xv[i] = xs[a][ty * 4 + i];
#pragma unroll
            for (int jj = 0; jj < 4; ++jj) wv[jj] = wsm[a][tx * 4 + jj];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int jj = 0; jj < 4; ++jj) acc[i][jj] = __fadd_rn(acc[i][jj], __fmul_rn(xv[i], wv[jj]));
        }
        __syncthreads();
    }
    OutT* out = static_cast<OutT*>(mats.out[m]);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int t = t0 + ty * 4 + i;
        if (t >= tokens) continue;
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) {
            const int j = j0 + tx * 4 + jj;
            if (j >= dim) continue;
            const int64_t o = (int64_t)h * mats.out_hs[m] + (int64_t)t * mats.out_rs[m] + j;
            if constexpr (sizeof(OutT) == 4) out[o] = acc[i][jj];
            else out[o] = __float2bfloat16_rn(acc[i][jj]);
        }
    }
}

}  // namespace

cudaError_t launch_project(const float* x, int tokens, int C, const ProjectMats& mats, int nmats, int heads, int dim,
                           bool bf16_out, cudaStream_t st) {
    if (tokens == 0 || heads == 0 || dim == 0 || nmats == 0) return cudaSuccess;
    dim3 grid((tokens + BT - 1) / BT, (dim + BJ - 1) / BJ, heads * nmats);
    if (bf16_out)
        project_kernel<__nv_bfloat16><<<grid, 256, 0, st>>>(x, tokens, C, mats, heads, dim);
    else
        project_kernel<float><<<grid, 256, 0, st>>>(x, tokens, C, mats, heads, dim);
    note_launch();
    return cudaGetLastError();
}

}  // namespace gsa_sm100
