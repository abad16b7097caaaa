// gemm.cu — the stack driver's dense projection on tcgen05 tensor cores (sm_100a):
// QKV[M][N] (bf16) = X[M][K] (bf16) . W[K][N] with W given transposed (Wt[N][K],
// K-major, the layout a static weight is stored in once), f32 accumulation in TMEM.
// N % 32 == 0 (a ragged last N tile reads zero rows of Wt), K % 64 == 0, any M.
// This is the per-layer X -> Q/K/V projection of the L-layer stack (BASELINE
// configs[2]; the reference's project_qkv, layer.hpp:48-76, does the same map in
// exact f32 on the CPU). Plus the residual X_{l+1} = bf16(X_l + O_l) of the stack.
//
// Persistent CTAs (one per SM), tiles of 128 x 256 output elements walked M-major
// so the ~12 N-tiles of one 128-row block of X run at the same time and share it in
// L2; W (6 MB) stays L2-resident. Warp roles:
//   warp 0      TMA: A tile 128 x 64 and B tile 256 x 64 (bf16, 128B swizzle) per
//               k-block through a 4-stage ring (48 KB per stage)
//   warp 1      MMA: D[128 x 256] += A . B^T, 4 MMAs (K=16) per k-block, into one
//               of two TMEM accumulators (256 columns each) so the epilogue of
//               tile j overlaps the MMAs of tile j+1
//   warps 2-5   epilogue: one thread per output row (TMEM lane), f32 -> bf16,
//               64-byte row segments to global
#include <cuda.h>

#include "tc.h"
#include "tc_ptx.cuh"
#include "tma_util.cuh"

namespace gsa_sm100 {
namespace {

using namespace ptx;

constexpr int GM = 128, GN = 256, GK = 64;  // tile
constexpr int G_NS = 4;                      // ring stages
constexpr int G_ATILE = GM * GK * 2;         // 16 KB
constexpr int G_BTILE = GN * GK * 2;         // 32 KB
constexpr int G_THREADS = 192;

struct __align__(1024) GemmSmem {
    uint8_t a[G_NS][G_ATILE];
    uint8_t b[G_NS][G_BTILE];
    uint64_t full[G_NS], empty[G_NS];
    uint64_t acc_full[2], acc_empty[2];
    uint32_t tmem_base;
};

struct GemmParams {
    int M, N, K;
    int tiles_m, tiles_n;
    __nv_bfloat16* c;
    int64_t ldc;
};

__global__ void __launch_bounds__(G_THREADS, 1)
    gemm_bf16_tc_kernel(const __grid_constant__ CUtensorMap tm_a, const __grid_constant__ CUtensorMap tm_b,
                        const GemmParams p) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    GemmSmem& sm = *reinterpret_cast<GemmSmem*>(smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u));
    const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
    const int ntiles = p.tiles_m * p.tiles_n, kblocks = p.K / GK;
    if (threadIdx.x == 0) {
        for (int i = 0; i < G_NS; ++i) {
            mbar_init(&sm.full[i], 1);
            mbar_init(&sm.empty[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&sm.acc_full[i], 1);
            mbar_init(&sm.acc_empty[i], 128);
        }
        fence_barrier_init();
        prefetch_tmap(&tm_a);
        prefetch_tmap(&tm_b);
    }
    if (warp == 1) tmem_alloc(&sm.tmem_base, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = sm.tmem_base;

    if (warp == 0) {
        // ================================ TMA ================================
        int it = 0;
        for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
            const int m = t / p.tiles_n, n = t - m * p.tiles_n;
            for (int kb = 0; kb < kblocks; ++kb, ++it) {
                const int s = it % G_NS;
                mbar_wait(&sm.empty[s], (uint32_t)(((it / G_NS) & 1) ^ 1));
                if (elect_one()) {
                    mbar_arrive_expect_tx(&sm.full[s], G_ATILE + G_BTILE);
                    tma_load_2d(&sm.a[s][0], &tm_a, &sm.full[s], kb * GK, m * GM);
                    tma_load_2d(&sm.b[s][0], &tm_b, &sm.full[s], kb * GK, n * GN);
                }
                __syncwarp();
            }
        }
    } else if (warp == 1) {
        // ================================ MMA ================================
        const uint32_t idesc = idesc_bf16(GM, GN, 0, 0);
        int it = 0, j = 0;
        for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++j) {
            const int acc = j & 1;
            mbar_wait(&sm.acc_empty[acc], (uint32_t)(((j >> 1) & 1) ^ 1));
            tc_fence_after();
            const uint32_t d = tmem + GN * acc;
            for (int kb = 0; kb < kblocks; ++kb, ++it) {
                const int s = it % G_NS;
                mbar_wait(&sm.full[s], (uint32_t)((it / G_NS) & 1));
                tc_fence_after();
                const uint64_t ad = umma_desc(smem_u32(&sm.a[s][0]), 16, 1024, 2);
                const uint64_t bd = umma_desc(smem_u32(&sm.b[s][0]), 16, 1024, 2);
                if (elect_one()) {
#pragma unroll
                    for (int ks = 0; ks < GK / 16; ++ks) mma_bf16(d, ad + 2 * ks, bd + 2 * ks, idesc, (kb | ks) != 0);
                    mma_commit(&sm.empty[s]);  // the stage is free once these MMAs have read it
                    if (kb == kblocks - 1) mma_commit(&sm.acc_full[acc]);
                }
                __syncwarp();
            }
        }
    } else {
        // ============================== epilogue ==============================
        const int quad = warp & 3;  // TMEM lane quadrant this warp may access
        const int row = 32 * quad + lane;
        int j = 0;
        for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++j) {
            const int m = t / p.tiles_n, n = t - m * p.tiles_n;
            const int acc = j & 1;
            mbar_wait(&sm.acc_full[acc], (uint32_t)((j >> 1) & 1));
            __syncwarp();
            tc_fence_after();
            const int grow = m * GM + row;
            __nv_bfloat16* dst = p.c + (int64_t)grow * p.ldc + (int64_t)n * GN;
            const uint32_t base = tmem + ((uint32_t)(32 * quad) << 16) + GN * acc;
#pragma unroll 2
            for (int c = 0; c < GN / 32; ++c) {
                uint32_t v[32];
                tmem_ld_32x32b_x32(base + 32 * c, v);
                tmem_wait_ld();
                uint32_t pk[16];
#pragma unroll
                for (int e = 0; e < 16; ++e) pk[e] = pack_bf16(__uint_as_float(v[2 * e]), __uint_as_float(v[2 * e + 1]));
                if (grow < p.M && n * GN + 32 * c < p.N) {  // ragged last N tile: its columns past N are zeros
                    uint4* o = reinterpret_cast<uint4*>(dst + 32 * c);
#pragma unroll
                    for (int q = 0; q < 4; ++q) o[q] = make_uint4(pk[4 * q], pk[4 * q + 1], pk[4 * q + 2], pk[4 * q + 3]);
                }
            }
            tc_fence_before();
            mbar_arrive(&sm.acc_empty[acc]);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
}

// [rows][cols] bf16 row-major, row stride ld elements -> boxes of box_rows x 64, 128B swizzle
bool make_2d_tmap(CUtensorMap* m, const void* base, int64_t rows, int64_t cols, int64_t ld, int box_rows) {
    TmapEncodeFn enc = tmap_encode_fn();
    if (!enc) return false;
    cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)ld * 2};
    cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
    cuuint32_t es[2] = {1, 1};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, es,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// X_{l+1} = bf16(X_l + O): x [M][C] bf16, o [M][C] f32 (heads concatenated), 8 per thread
__global__ void residual_bf16_kernel(const __nv_bfloat16* __restrict__ x, const float* __restrict__ o,
                                     __nv_bfloat16* __restrict__ y, int64_t n8) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n8) return;
    const uint4 xv = reinterpret_cast<const uint4*>(x)[i];
    const float4 a = reinterpret_cast<const float4*>(o)[2 * i], b = reinterpret_cast<const float4*>(o)[2 * i + 1];
    const __nv_bfloat162* xp = reinterpret_cast<const __nv_bfloat162*>(&xv);
    const float2 x0 = __bfloat1622float2(xp[0]), x1 = __bfloat1622float2(xp[1]), x2 = __bfloat1622float2(xp[2]),
                 x3 = __bfloat1622float2(xp[3]);
    uint4 r;
    r.x = pack_bf16(x0.x + a.x, x0.y + a.y);
    r.y = pack_bf16(x1.x + a.z, x1.y + a.w);
    r.z = pack_bf16(x2.x + b.x, x2.y + b.y);
    r.w = pack_bf16(x3.x + b.z, x3.y + b.w);
    reinterpret_cast<uint4*>(y)[i] = r;
}

}  // namespace

bool tc_gemm_supported(int M, int N, int K) { return M > 0 && N > 0 && N % 32 == 0 && K % GK == 0 && tmap_encode_fn(); }

cudaError_t tc_gemm_bf16(const __nv_bfloat16* a, int64_t lda, const __nv_bfloat16* bt, int64_t ldb, __nv_bfloat16* c,
                         int64_t ldc, int M, int N, int K, cudaStream_t st) {
    if (!tc_gemm_supported(M, N, K)) return cudaErrorNotSupported;
    CUtensorMap ta, tb;
    if (!make_2d_tmap(&ta, a, M, K, lda, GM) || !make_2d_tmap(&tb, bt, N, K, ldb, GN)) return cudaErrorNotSupported;
    GemmParams p{M, N, K, (M + GM - 1) / GM, (N + GN - 1) / GN, c, ldc};
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const size_t smem = sizeof(GemmSmem) + 1024;
    cudaError_t e = cudaFuncSetAttribute(gemm_bf16_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    const int ntiles = p.tiles_m * p.tiles_n;
    gemm_bf16_tc_kernel<<<ntiles < sms ? ntiles : sms, G_THREADS, smem, st>>>(ta, tb, p);
    note_launch();
    return cudaGetLastError();
}

cudaError_t launch_residual_bf16(const __nv_bfloat16* x, const float* o, __nv_bfloat16* y, int64_t n, cudaStream_t st) {
    if (n % 8) return cudaErrorNotSupported;
    const int64_t n8 = n / 8;
    if (n8 == 0) return cudaSuccess;
    residual_bf16_kernel<<<(unsigned)((n8 + 255) / 256), 256, 0, st>>>(x, o, y, n8);
    note_launch();
    return cudaGetLastError();
}

}  // namespace gsa_sm100
