// proj_bwd_tc.cu — the projection backward (gradients.hpp:226-263) on tcgen05 tensor
// cores, head dim 64:
//   dX[m][c]      = sum over (mat, h) of sum_j G_mat[h][m][j] W_mat[h][c][j]     (dx_tc_kernel)
//   dW_mat[h][c][j] = sum_m X[m][c] G_mat[h][m][j]                                (dw_tc_kernel)
// with G = dQ, dK, dV. f32 operands enter as bf16 hi + lo planes and every product takes
// the hi.hi + hi.lo + lo.hi terms (|x - hi - lo| <= 2^-18 |x|): f32-level results,
// accumulated in TMEM, one CTA per output tile (deterministic).
//
// dx: tile 128 m x 128 c; the reduction runs over the 3H head blocks of 64 features, each
//     a K-major TMA box of G (rows m) and of W (rows c) -- no transposes.
// dw: tile 128 c x 64 j for one (mat, h); the reduction runs over m in blocks of 128: A =
//     X^T (a transposed bf16 copy, K-major along m), B = the G head block as an MN-major
//     operand (rows m, 64 contiguous features), like V in the attention P.V products.
// Warp roles (192 threads): warps 0-3 epilogue (one thread per TMEM lane), warp 4 TMA,
// warp 5 MMA issue.
#include <cuda.h>

#include "tc.h"
#include "tc_ptx.cuh"
#include "tma_util.cuh"

namespace gsa_sm100 {
namespace {

using namespace ptx;

constexpr int PT_THREADS = 192;
constexpr int BOX = 16384;  // 128 rows x 64 bf16

// ----------------------------------------------------------------- dX
constexpr int DX_NS = 3;
struct __align__(1024) DxSmem {
    uint8_t st[DX_NS][4][BOX];  // G hi, G lo, W hi, W lo of one (mat, h) block
    uint64_t full[DX_NS], empty[DX_NS], done;
    uint32_t tmem_base;
};

__global__ void __launch_bounds__(PT_THREADS, 1)
    dx_tc_kernel(const __grid_constant__ CUtensorMap tg_h, const __grid_constant__ CUtensorMap tg_l,
                 const __grid_constant__ CUtensorMap tw_h, const __grid_constant__ CUtensorMap tw_l, int nblocks,
                 int64_t M, int C, float* dx) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    DxSmem& sm = *reinterpret_cast<DxSmem*>(smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u));
    const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
    const int c0 = blockIdx.x * 128;
    const int m0 = blockIdx.y * 128;
    if (threadIdx.x == 0) {
        for (int i = 0; i < DX_NS; ++i) {
            mbar_init(&sm.full[i], 1);
            mbar_init(&sm.empty[i], 1);
        }
        mbar_init(&sm.done, 1);
        fence_barrier_init();
    }
    if (warp == 5) tmem_alloc(&sm.tmem_base, 128);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = sm.tmem_base;
    if (warp == 4) {
        if (elect_one()) {
            for (int kb = 0; kb < nblocks; ++kb) {
                const int s = kb % DX_NS;
                mbar_wait(&sm.empty[s], (uint32_t)(((kb / DX_NS) & 1) ^ 1));
                mbar_arrive_expect_tx(&sm.full[s], 4 * BOX);
                tma_load_3d(sm.st[s][0], &tg_h, &sm.full[s], 0, m0, kb);
                tma_load_3d(sm.st[s][1], &tg_l, &sm.full[s], 0, m0, kb);
                tma_load_3d(sm.st[s][2], &tw_h, &sm.full[s], 0, c0, kb);
                tma_load_3d(sm.st[s][3], &tw_l, &sm.full[s], 0, c0, kb);
            }
        }
        __syncwarp();
    } else if (warp == 5) {
        const uint32_t id = idesc_bf16(128, 128, 0, 0);
        auto kd = [](const uint8_t* t) { return umma_desc(smem_u32(t), 16, 1024, 2); };
        for (int kb = 0; kb < nblocks; ++kb) {
            const int s = kb % DX_NS;
            mbar_wait(&sm.full[s], (uint32_t)((kb / DX_NS) & 1));
            tc_fence_after();
            const uint64_t gh = kd(sm.st[s][0]), gl = kd(sm.st[s][1]), wh = kd(sm.st[s][2]), wl = kd(sm.st[s][3]);
            if (elect_one()) {
                for (int ks = 0; ks < 4; ++ks) {
                    mma_bf16(tmem, gh + 2 * ks, wh + 2 * ks, id, (kb | ks) != 0);
                    mma_bf16(tmem, gh + 2 * ks, wl + 2 * ks, id, 1);
                    mma_bf16(tmem, gl + 2 * ks, wh + 2 * ks, id, 1);
                }
                mma_commit(&sm.empty[s]);
                if (kb == nblocks - 1) mma_commit(&sm.done);
            }
            __syncwarp();
        }
    } else {
        mbar_wait(&sm.done, 0);
        __syncwarp();
        tc_fence_after();
        const int row = 32 * warp + lane;
        const uint32_t lb = tmem + ((uint32_t)(32 * warp) << 16);
        const int64_t m = m0 + row;
#pragma unroll 1
        for (int c = 0; c < 4; ++c) {
            uint32_t v[32];
            tmem_ld_32x32b_x32(lb + 32 * c, v);
            tmem_wait_ld();
            if (m < M) {
                float* dst = dx + m * C + c0 + 32 * c;
                const int valid = C - (c0 + 32 * c);
#pragma unroll
                for (int e = 0; e < 32; e += 4)
                    if (e + 4 <= valid)
                        *reinterpret_cast<float4*>(dst + e) =
                            make_float4(__uint_as_float(v[e]), __uint_as_float(v[e + 1]), __uint_as_float(v[e + 2]),
                                        __uint_as_float(v[e + 3]));
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 5) {
        tc_fence_after();
        tmem_dealloc(tmem, 128);
    }
}

// ----------------------------------------------------------------- dW
constexpr int DW_NS = 2;
struct __align__(1024) DwSmem {
    uint8_t a[DW_NS][2][2][BOX];  // X^T hi / lo, two 64-row halves of the 128-m block
    uint8_t b[DW_NS][2][BOX];     // G hi / lo, 128 m rows x 64 features
    uint64_t full[DW_NS], empty[DW_NS], done;
    uint32_t tmem_base;
};

__global__ void __launch_bounds__(PT_THREADS, 1)
    dw_tc_kernel(const __grid_constant__ CUtensorMap tx_h, const __grid_constant__ CUtensorMap tx_l,
                 const __grid_constant__ CUtensorMap tg_h, const __grid_constant__ CUtensorMap tg_l, int64_t M, int C,
                 int heads, float* dw0, float* dw1, float* dw2) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    DwSmem& sm = *reinterpret_cast<DwSmem*>(smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u));
    const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
    const int c0 = blockIdx.x * 128, blk = blockIdx.y;  // blk = mat * H + h
    const int nk = (int)((M + 127) / 128);
    if (threadIdx.x == 0) {
        for (int i = 0; i < DW_NS; ++i) {
            mbar_init(&sm.full[i], 1);
            mbar_init(&sm.empty[i], 1);
        }
        mbar_init(&sm.done, 1);
        fence_barrier_init();
    }
    if (warp == 5) tmem_alloc(&sm.tmem_base, 64);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = sm.tmem_base;
    if (warp == 4) {
        if (elect_one()) {
            for (int kb = 0; kb < nk; ++kb) {
                const int s = kb % DW_NS;
                mbar_wait(&sm.empty[s], (uint32_t)(((kb / DW_NS) & 1) ^ 1));
                mbar_arrive_expect_tx(&sm.full[s], 6 * BOX);
                const int m0 = kb * 128;
                tma_load_2d(sm.a[s][0][0], &tx_h, &sm.full[s], m0, c0);
                tma_load_2d(sm.a[s][0][1], &tx_h, &sm.full[s], m0 + 64, c0);
                tma_load_2d(sm.a[s][1][0], &tx_l, &sm.full[s], m0, c0);
                tma_load_2d(sm.a[s][1][1], &tx_l, &sm.full[s], m0 + 64, c0);
                tma_load_3d(sm.b[s][0], &tg_h, &sm.full[s], 0, m0, blk);
                tma_load_3d(sm.b[s][1], &tg_l, &sm.full[s], 0, m0, blk);
            }
        }
        __syncwarp();
    } else if (warp == 5) {
        const uint32_t id = idesc_bf16(128, 64, 0, 1);  // B (G) MN-major
        auto kd = [](const uint8_t* t) { return umma_desc(smem_u32(t), 16, 1024, 2); };
        for (int kb = 0; kb < nk; ++kb) {
            const int s = kb % DW_NS;
            mbar_wait(&sm.full[s], (uint32_t)((kb / DW_NS) & 1));
            tc_fence_after();
            if (elect_one()) {
                const uint64_t gh = kd(sm.b[s][0]), gl = kd(sm.b[s][1]);
                for (int ks = 0; ks < 8; ++ks) {
                    const uint64_t xh = kd(sm.a[s][0][ks >> 2]) + 2 * (ks & 3);
                    const uint64_t xl = kd(sm.a[s][1][ks >> 2]) + 2 * (ks & 3);
                    mma_bf16(tmem, xh, gh + 128 * ks, id, (kb | ks) != 0);
                    mma_bf16(tmem, xh, gl + 128 * ks, id, 1);
                    mma_bf16(tmem, xl, gh + 128 * ks, id, 1);
                }
                mma_commit(&sm.empty[s]);
                if (kb == nk - 1) mma_commit(&sm.done);
            }
            __syncwarp();
        }
    } else {
        mbar_wait(&sm.done, 0);
        __syncwarp();
        tc_fence_after();
        const int row = 32 * warp + lane;
        const uint32_t lb = tmem + ((uint32_t)(32 * warp) << 16);
        const int c = c0 + row;
#pragma unroll 1
        for (int half = 0; half < 2; ++half) {
            uint32_t v[32];
            tmem_ld_32x32b_x32(lb + 32 * half, v);
            tmem_wait_ld();
            if (c < C) {
                const int mat = blk / heads, h = blk - mat * heads;
                float* dw = mat == 0 ? dw0 : mat == 1 ? dw1 : dw2;
                float* dst = dw + ((int64_t)h * C + c) * 64 + 32 * half;
#pragma unroll
                for (int e = 0; e < 32; e += 4)
                    *reinterpret_cast<float4*>(dst + e) = make_float4(
                        __uint_as_float(v[e]), __uint_as_float(v[e + 1]), __uint_as_float(v[e + 2]), __uint_as_float(v[e + 3]));
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 5) {
        tc_fence_after();
        tmem_dealloc(tmem, 64);
    }
}

// X f32 [M][C] -> X^T bf16 hi / lo [C][ldt] (32 x 32 tiles through shared memory)
__global__ void transpose_split_kernel(const float* __restrict__ x, int64_t M, int C, int64_t ldt, __nv_bfloat16* hi,
                                       __nv_bfloat16* lo) {
    __shared__ float t[32][33];
    const int64_t m0 = (int64_t)blockIdx.x * 32;
    const int c0 = blockIdx.y * 32;
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {
        const int64_t m = m0 + r;
        const int c = c0 + threadIdx.x;
        t[r][threadIdx.x] = (m < M && c < C) ? x[m * C + c] : 0.0f;
    }
    __syncthreads();
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {
        const int c = c0 + r;
        const int64_t m = m0 + threadIdx.x;
        if (c < C && m < M) {
            const float v = t[threadIdx.x][r];
            const __nv_bfloat16 h = __float2bfloat16_rn(v);
            hi[(int64_t)c * ldt + m] = h;
            lo[(int64_t)c * ldt + m] = __float2bfloat16_rn(v - __bfloat162float(h));
        }
    }
}

// [rows][cols] bf16 row-major with row stride ld (elements, ld % 8 == 0), boxes of 128 rows x
// 64 columns (128B swizzle); columns past cols read as zeros
bool make_2d_map(CUtensorMap* m, const void* base, int64_t rows, int64_t cols, int64_t ld) {
    TmapEncodeFn enc = tmap_encode_fn();
    if (!enc) return false;
    cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)ld * 2};
    cuuint32_t box[2] = {64, 128};
    cuuint32_t es[2] = {1, 1};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, es,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace

bool tc_proj_bwd_supported(int dim, int model_dim) {
    // dX rows are written as float4 (model_dim % 4)
    return dim == 64 && model_dim % 4 == 0 && tmap_encode_fn() != nullptr;
}

static int64_t xt_ld(int64_t tokens) { return (tokens + 7) / 8 * 8; }  // X^T row stride: 16-byte TMA rows

size_t tc_proj_bwd_workspace_bytes(int tokens, int model_dim, int heads) {
    const size_t g = (size_t)3 * heads * tokens * 64 * 2, w = (size_t)3 * heads * model_dim * 64 * 2,
                 xt = (size_t)model_dim * xt_ld(tokens) * 2;
    return 2 * (g + w + xt) + 6 * 256;
}

cudaError_t launch_proj_bwd_tc(const float* x, int tokens, int C, const float* const w[3], int heads,
                               const float* const g[3], float* dx, float* const dw[3], void* ws, cudaStream_t st) {
    const int64_t M = tokens;
    if (M == 0) return cudaSuccess;
    char* p = static_cast<char*>(ws);
    auto take = [&](size_t bytes) {
        char* r = p;
        p += (bytes + 255) / 256 * 256;
        return reinterpret_cast<__nv_bfloat16*>(r);
    };
    const int64_t ldt = xt_ld(M);
    const size_t gsz = (size_t)3 * heads * M * 64 * 2, wsz = (size_t)3 * heads * C * 64 * 2, xsz = (size_t)C * ldt * 2;
    __nv_bfloat16 *gh = take(gsz), *gl = take(gsz), *wh = take(wsz), *wl = take(wsz), *xh = take(xsz), *xl = take(xsz);
    // operand planes: G and W as [3H][rows][64] hi / lo, X^T as [C][M] hi / lo
    for (int i = 0; i < 3; ++i) {
        cudaError_t e = launch_pack_rows(TensorRef{g[i], GSA_DTYPE_F32, M * 64, 64}, heads, tokens,
                                         gh + (size_t)i * heads * M * 64, gl + (size_t)i * heads * M * 64, st);
        if (e != cudaSuccess) return e;
        e = launch_pack_rows(TensorRef{w[i], GSA_DTYPE_F32, (int64_t)C * 64, 64}, heads, C,
                             wh + (size_t)i * heads * C * 64, wl + (size_t)i * heads * C * 64, st);
        if (e != cudaSuccess) return e;
    }
    transpose_split_kernel<<<dim3((unsigned)((M + 31) / 32), (C + 31) / 32), dim3(32, 8), 0, st>>>(x, M, C, ldt, xh, xl);
    note_launch();
    CUtensorMap tg_h, tg_l, tw_h, tw_l, tx_h, tx_l;
    if (!make_rows_tmap(&tg_h, gh, 3 * heads, (int)M, M * 64, 64) ||
        !make_rows_tmap(&tg_l, gl, 3 * heads, (int)M, M * 64, 64) ||
        !make_rows_tmap(&tw_h, wh, 3 * heads, C, (int64_t)C * 64, 64) ||
        !make_rows_tmap(&tw_l, wl, 3 * heads, C, (int64_t)C * 64, 64) || !make_2d_map(&tx_h, xh, C, M, ldt) ||
        !make_2d_map(&tx_l, xl, C, M, ldt))
        return cudaErrorNotSupported;
    const size_t dx_smem = sizeof(DxSmem) + 1024, dw_smem = sizeof(DwSmem) + 1024;
    cudaError_t e = cudaFuncSetAttribute(dx_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dx_smem);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(dw_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dw_smem);
    if (e != cudaSuccess) return e;
    dx_tc_kernel<<<dim3((unsigned)((C + 127) / 128), (unsigned)((M + 127) / 128)), PT_THREADS, dx_smem, st>>>(
        tg_h, tg_l, tw_h, tw_l, 3 * heads, M, C, dx);
    note_launch();
    // dW: one CTA per (128 model features, matrix x head) block
    dw_tc_kernel<<<dim3((unsigned)((C + 127) / 128), 3 * heads), PT_THREADS, dw_smem, st>>>(tx_h, tx_l, tg_h, tg_l, M, C,
                                                                                        heads, dw[0], dw[1], dw[2]);
    note_launch();
    return cudaGetLastError();
}

}  // namespace gsa_sm100
