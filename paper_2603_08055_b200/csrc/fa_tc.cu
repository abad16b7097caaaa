// fa_tc.cu — K5: dense attention on tcgen05 tensor cores (sm_100a): the
// special-token path (special_token_attention / tiled_attention,
// layer.hpp:80-96, compression.hpp:99-165) and the dense baseline.
//
// CTA = 128 query rows x one head x one key split. Warp roles:
//   warp 0  TMA: Q tile once, then K(t+1), V(t) tiles of 128 keys (16 KB each,
//           128B-swizzled) through a 6-stage ring.
//   warp 1  MMA: S(t) = Q.K(t)^T  (M=128, N=128, K=64, both K-major, into TMEM,
//           3 rotating S buffers), O += P(t).V(t) with P read from TMEM
//           (A-from-TMEM form, P as bf16 hi + lo: 2 MMAs per 16-key step).
//   warps 2-5  softmax, one thread per query row = one TMEM lane: row max,
//           lazy rescale (only when the max grows by > 2^8; O is then rescaled
//           in TMEM), P = exp2 via MUFU, written back over S in TMEM as
//           bf16 hi/lo pairs; epilogue O/l and lse.
// Split-KV (few query tiles, e.g. 5 specials/view) writes normalised partials
// + lse that gsa_fa_combine merges.
#include <cuda.h>

#include "tc.h"
#include "tc_ptx.cuh"

namespace gsa_sm100 {
namespace {

using namespace ptx;

constexpr int NS = 6;
constexpr int TILE = 16384;  // 128 rows x 64 bf16
constexpr int NTHREADS = 192;
constexpr uint32_t TMEM_COLS = 512;
constexpr uint32_t O_COL = 384;
constexpr float RESCALE_LOG2 = 8.0f;

struct __align__(1024) FaSmem {
    uint8_t q[TILE];
    uint8_t ring[NS][TILE];
    uint64_t full[NS], empty[NS];
    uint64_t q_full;
    uint64_t s_full[3], s_free[3];
    // by tile parity: the softmax runs up to a tile ahead of the MMA, and parity waits are
    // only unambiguous within one phase of their target
    uint64_t p_full[2], o_done[2];
    uint32_t tmem_base;
};

struct FaParams {
    int heads, mq, mk;
    float scale, c2;
    int kv_tiles, splits, tiles_per_split;
    float* out;
    int64_t out_hs, out_rs;
    float* lse;       // [H][mq] (splits == 1)
    float* part_o;    // [splits][H][mq][64]
    float* part_lse;  // [splits][H][mq]
};

__device__ __forceinline__ uint32_t s_col(int b) { return (uint32_t)(128 * b); }

__global__ void __launch_bounds__(NTHREADS, 1)
    fa_tc_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                 const __grid_constant__ CUtensorMap tm_v, const FaParams p) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    FaSmem& sm = *reinterpret_cast<FaSmem*>(smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u));
    const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
    const int qt = blockIdx.x, split = blockIdx.y, h = blockIdx.z;
    const int t_begin = split * p.tiles_per_split;
    const int t_end = min(p.kv_tiles, t_begin + p.tiles_per_split);
    const int T = t_end - t_begin;

    if (threadIdx.x == 0) {
        for (int i = 0; i < NS; ++i) {
            mbar_init(&sm.full[i], 1);
            mbar_init(&sm.empty[i], 1);
        }
        for (int i = 0; i < 3; ++i) {
            mbar_init(&sm.s_full[i], 1);
            mbar_init(&sm.s_free[i], 1);
        }
        mbar_init(&sm.q_full, 1);
        mbar_init(&sm.p_full[0], 128);
        mbar_init(&sm.p_full[1], 128);
        mbar_init(&sm.o_done[0], 1);
        mbar_init(&sm.o_done[1], 1);
        fence_barrier_init();
        prefetch_tmap(&tm_q);
        prefetch_tmap(&tm_k);
        prefetch_tmap(&tm_v);
    }
    if (warp == 1) tmem_alloc(&sm.tmem_base, TMEM_COLS);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = sm.tmem_base;

    if (warp == 0) {
        if (lane == 0 && T > 0) {
            // ================================ TMA ================================
            mbar_arrive_expect_tx(&sm.q_full, TILE);
            tma_load_3d(&sm.q[0], &tm_q, &sm.q_full, 0, qt * 128, h);
            int st = 0;
            uint32_t eph = 1;
            auto load = [&](const CUtensorMap* tm, int t) {
                mbar_wait(&sm.empty[st], eph);
                mbar_arrive_expect_tx(&sm.full[st], TILE);
                tma_load_3d(&sm.ring[st][0], tm, &sm.full[st], 0, (t_begin + t) * 128, h);
                if (++st == NS) {
                    st = 0;
                    eph ^= 1;
                }
            };
            load(&tm_k, 0);
            for (int t = 0; t < T; ++t) {
                if (t + 1 < T) load(&tm_k, t + 1);
                load(&tm_v, t);
            }
        }
    } else if (warp == 1) {
        if (lane == 0 && T > 0) {
            // ================================ MMA ================================
            const uint32_t id_s = idesc_bf16(128, 128, 0, 0);
            const uint32_t id_o = idesc_bf16(128, 64, 0, 1);
            int st = 0;
            uint32_t fph = 0;
            uint32_t freeph[3] = {1, 1, 1};
            uint32_t pph[2] = {0, 0};
            mbar_wait(&sm.q_full, 0);
            const uint64_t qdesc = umma_desc(smem_u32(&sm.q[0]), 16, 1024, 2);
            auto issue_S = [&](int t) {
                const int b = t % 3;
                mbar_wait(&sm.s_free[b], freeph[b]);
                freeph[b] ^= 1;
                mbar_wait(&sm.full[st], fph);
                tc_fence_after();
                const uint64_t kdesc = umma_desc(smem_u32(&sm.ring[st][0]), 16, 1024, 2);
                for (int ks = 0; ks < 4; ++ks)
                    mma_bf16(tmem + s_col(b), qdesc + (uint64_t)(2 * ks), kdesc + (uint64_t)(2 * ks), id_s, ks != 0);
                mma_commit(&sm.empty[st]);
                mma_commit(&sm.s_full[b]);
                if (++st == NS) {
                    st = 0;
                    fph ^= 1;
                }
            };
            auto issue_PV = [&](int t) {
                const int b = t % 3;
                mbar_wait(&sm.p_full[t & 1], pph[t & 1]);
                pph[t & 1] ^= 1;
                mbar_wait(&sm.full[st], fph);
                tc_fence_after();
                const uint64_t vdesc = umma_desc(smem_u32(&sm.ring[st][0]), 16, 1024, 2);
                for (int ks = 0; ks < 8; ++ks) {
                    // P hi of keys 16ks..16ks+15: TMEM cols 32*(ks/2) + 8*(ks%2); lo 16 columns later
                    const uint32_t a_hi = tmem + s_col(b) + 32 * (ks >> 1) + 8 * (ks & 1);
                    const uint64_t vb = vdesc + (uint64_t)(128 * ks);
                    mma_bf16_ts(tmem + O_COL, a_hi, vb, id_o, (t | ks) != 0);
                    mma_bf16_ts(tmem + O_COL, a_hi + 16, vb, id_o, 1);
                }
                mma_commit(&sm.empty[st]);
                mma_commit(&sm.s_free[b]);
                mma_commit(&sm.o_done[t & 1]);
                if (++st == NS) {
                    st = 0;
                    fph ^= 1;
                }
            };
            issue_S(0);
            for (int t = 0; t < T; ++t) {
                if (t + 1 < T) issue_S(t + 1);
                issue_PV(t);
            }
        }
    } else if (T > 0) {
        // ============================ softmax (warps 2..5) ============================
        const int qd = warp & 3;
        const int row = 32 * qd + lane;
        const uint32_t lane_base = tmem + ((uint32_t)(32 * qd) << 16);
        float m_used = -INFINITY, l = 0.0f;
        uint32_t sph[3] = {0, 0, 0};
        for (int t = 0; t < T; ++t) {
            const int b = t % 3;
            mbar_wait(&sm.s_full[b], sph[b]);
            sph[b] ^= 1;
            __syncwarp();  // .sync.aligned tcgen05 ops below need a converged warp
            tc_fence_after();
            uint32_t sr[4][32];
#pragma unroll
            for (int c = 0; c < 4; ++c) tmem_ld_32x32b_x32(lane_base + s_col(b) + 32 * c, sr[c]);
            tmem_wait_ld();
            const int valid = p.mk - (t_begin + t) * 128;  // keys of this tile that exist
            float mt = -INFINITY;
#pragma unroll
            for (int c = 0; c < 4; ++c)
#pragma unroll
                for (int e = 0; e < 32; ++e) {
                    if (32 * c + e >= valid) sr[c][e] = __float_as_uint(-INFINITY);
                    mt = fmaxf(mt, __uint_as_float(sr[c][e]));
                }
            if (t == 0) {
                m_used = mt;
            } else {
                const bool need = (mt - m_used) * p.c2 > RESCALE_LOG2;
                if (__any_sync(0xffffffffu, need)) {
                    // rescale O (TMEM) and l once PV(t-1) has landed.
                    // PV(t-1) done: completion #((t-1)>>1) of o_done[(t-1)&1]; PV(t-3) is already
                    // implied by s_full(t) and PV(t+1) cannot have run, so this parity is exact
                    mbar_wait(&sm.o_done[(t - 1) & 1], (uint32_t)(((t - 1) >> 1) & 1));
                    __syncwarp();
                    tc_fence_after();
                    const float mnew = need ? mt : m_used;
                    const float f = ex2_approx((m_used - mnew) * p.c2);
                    uint32_t o[32];
#pragma unroll
                    for (int half = 0; half < 2; ++half) {
                        tmem_ld_32x32b_x32(lane_base + O_COL + 32 * half, o);
                        tmem_wait_ld();
#pragma unroll
                        for (int e = 0; e < 32; ++e) o[e] = __float_as_uint(__uint_as_float(o[e]) * f);
                        tmem_st_32x32b_x32(lane_base + O_COL + 32 * half, o);
                    }
                    tmem_wait_st();
                    l *= f;
                    m_used = mnew;
                }
            }
            const float mc = m_used * p.c2;
            float ls = 0.0f;
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                uint32_t hi[16], lo[16];
#pragma unroll
                for (int e2 = 0; e2 < 16; ++e2) {
                    const float x0 = __uint_as_float(sr[c][2 * e2]), x1 = __uint_as_float(sr[c][2 * e2 + 1]);
                    const float p0 = ex2_approx(fmaf(x0, p.c2, -mc));
                    const float p1 = ex2_approx(fmaf(x1, p.c2, -mc));
                    ls += p0 + p1;
                    hi[e2] = pack_bf16(p0, p1);
                    const __nv_bfloat162 hb = *reinterpret_cast<const __nv_bfloat162*>(&hi[e2]);
                    lo[e2] = pack_bf16(p0 - __low2float(hb), p1 - __high2float(hb));
                }
                tmem_st_32x32b_x16(lane_base + s_col(b) + 32 * c, hi);
                tmem_st_32x32b_x16(lane_base + s_col(b) + 32 * c + 16, lo);
            }
            l += ls;
            tmem_wait_st();
            tc_fence_before();
            mbar_arrive(&sm.p_full[t & 1]);
        }
        // ------------------------------- epilogue -------------------------------
        // the commit after PV(T-1) covers every earlier MMA
        mbar_wait(&sm.o_done[(T - 1) & 1], (uint32_t)(((T - 1) >> 1) & 1));
        __syncwarp();
        tc_fence_after();
        uint32_t o[2][32];
        tmem_ld_32x32b_x32(lane_base + O_COL, o[0]);
        tmem_ld_32x32b_x32(lane_base + O_COL + 32, o[1]);
        tmem_wait_ld();
        const int qrow = qt * 128 + row;
        if (qrow < p.mq) {
            const float inv = 1.0f / l;
            const float lse = m_used * p.scale + logf(l);
            float* dst;
            if (p.splits == 1) {
                dst = p.out + (int64_t)h * p.out_hs + (int64_t)qrow * p.out_rs;
                if (p.lse) p.lse[(int64_t)h * p.mq + qrow] = lse;
            } else {
                const int64_t r = ((int64_t)split * p.heads + h) * p.mq + qrow;
                dst = p.part_o + r * 64;
                p.part_lse[r] = lse;
            }
#pragma unroll
            for (int half = 0; half < 2; ++half)
#pragma unroll
                for (int e = 0; e < 32; e += 4)
                    *reinterpret_cast<float4*>(dst + 32 * half + e) =
                        make_float4(__uint_as_float(o[half][e]) * inv, __uint_as_float(o[half][e + 1]) * inv,
                                    __uint_as_float(o[half][e + 2]) * inv, __uint_as_float(o[half][e + 3]) * inv);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc(tmem, TMEM_COLS);
    }
}

// merge split-KV partials: out = sum_s w_s O_s / sum_s w_s, w_s = exp(lse_s - max)
__global__ void fa_combine_kernel(const float* __restrict__ part_o, const float* __restrict__ part_lse, int splits,
                                  int heads, int mq, float* out, int64_t out_hs, int64_t out_rs, float* lse) {
    const int64_t row = (int64_t)blockIdx.x * (blockDim.x / 16) + threadIdx.x / 16;  // (h, q)
    const int sub = threadIdx.x & 15;                                               // 4 features each
    if (row >= (int64_t)heads * mq) return;
    const int h = (int)(row / mq), q = (int)(row % mq);
    float mx = -INFINITY;
    for (int s = 0; s < splits; ++s) mx = fmaxf(mx, part_lse[((int64_t)s * heads + h) * mq + q]);
    float den = 0.0f;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int s = 0; s < splits; ++s) {
        const int64_t r = ((int64_t)s * heads + h) * mq + q;
        const float w = __expf(part_lse[r] - mx);
        den += w;
        const float4 v = reinterpret_cast<const float4*>(part_o + r * 64)[sub];
        acc.x += w * v.x;
        acc.y += w * v.y;
        acc.z += w * v.z;
        acc.w += w * v.w;
    }
    const float inv = 1.0f / den;
    float* dst = out + (int64_t)h * out_hs + (int64_t)q * out_rs + 4 * sub;
    dst[0] = acc.x * inv;
    dst[1] = acc.y * inv;
    dst[2] = acc.z * inv;
    dst[3] = acc.w * inv;
    if (lse && sub == 0) lse[(int64_t)h * mq + q] = mx + logf(den);
}

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn encode_fn() {
    static EncodeFn fn = nullptr;
    if (!fn) {
        void* ptr = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeFn>(ptr);
    }
    return fn;
}

// [H][rows][64] bf16 rows -> 128-row tiles
bool make_rows_map(CUtensorMap* m, const void* base, int heads, int rows, int64_t hs, int64_t rs) {
    EncodeFn enc = encode_fn();
    if (!enc) return false;
    cuuint64_t dims[3] = {64, (cuuint64_t)rows, (cuuint64_t)heads};
    cuuint64_t strides[2] = {(cuuint64_t)rs * 2, (cuuint64_t)hs * 2};
    cuuint32_t box[3] = {64, 128, 1};
    cuuint32_t es[3] = {1, 1, 1};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, es,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

bool rows_ok(const gsa_tensor& t) {
    return t.dtype == GSA_DTYPE_BF16 && t.dim == 64 && t.row_stride % 8 == 0 && t.head_stride % 8 == 0 &&
           (reinterpret_cast<uintptr_t>(t.data) & 15) == 0;
}

}  // namespace

bool tc_dense_supported(const gsa_tensor& q, const gsa_tensor& k, const gsa_tensor& v) {
    return rows_ok(q) && rows_ok(k) && rows_ok(v) && encode_fn() != nullptr;
}

size_t tc_dense_workspace_bytes(int heads, int mq, int mk) {
    const int qtiles = (mq + 127) / 128, kv_tiles = (mk + 127) / 128;
    int splits = 1;
    while (qtiles * heads * splits < 2 * 148 && kv_tiles / (splits * 2) >= 4) splits *= 2;
    if (splits == 1) return 0;
    return (size_t)splits * heads * mq * 65 * sizeof(float) + 256;
}

cudaError_t tc_dense_attention(const gsa_tensor& q, const gsa_tensor& k, const gsa_tensor& v, float scale,
                               int q_row_offset, int mq, float* out, int64_t out_hs, int64_t out_rs,
                               int out_row_offset, float* lse, void* ws, size_t ws_bytes, cudaStream_t st) {
    if (mq == 0) return cudaSuccess;
    CUtensorMap tq, tk, tv;
    const char* qbase = static_cast<const char*>(q.data) + (size_t)q_row_offset * q.row_stride * 2;
    if (!make_rows_map(&tq, qbase, q.heads, mq, q.head_stride, q.row_stride) ||
        !make_rows_map(&tk, k.data, k.heads, k.rows, k.head_stride, k.row_stride) ||
        !make_rows_map(&tv, v.data, v.heads, v.rows, v.head_stride, v.row_stride))
        return cudaErrorNotSupported;
    FaParams p{};
    p.heads = q.heads;
    p.mq = mq;
    p.mk = k.rows;
    p.scale = scale;
    p.c2 = scale * 1.4426950408889634f;
    p.kv_tiles = (k.rows + 127) / 128;
    const int qtiles = (mq + 127) / 128;
    int splits = 1;
    while (qtiles * q.heads * splits < 2 * 148 && p.kv_tiles / (splits * 2) >= 4) splits *= 2;
    // split-KV needs caller workspace for the partials; without it run unsplit
    if (splits > 1 && (!ws || ws_bytes < (size_t)splits * q.heads * mq * 65 * sizeof(float))) splits = 1;
    p.tiles_per_split = (p.kv_tiles + splits - 1) / splits;
    p.splits = (p.kv_tiles + p.tiles_per_split - 1) / p.tiles_per_split;
    p.out = out + (size_t)out_row_offset * out_rs;
    p.out_hs = out_hs;
    p.out_rs = out_rs;
    p.lse = lse;
    if (p.splits > 1) {
        p.part_o = static_cast<float*>(ws);
        p.part_lse = p.part_o + (size_t)p.splits * q.heads * mq * 64;
    }
    const size_t smem = sizeof(FaSmem) + 1024;
    cudaError_t e = cudaFuncSetAttribute(fa_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    dim3 grid(qtiles, p.splits, q.heads);
    fa_tc_kernel<<<grid, NTHREADS, smem, st>>>(tq, tk, tv, p);
    note_launch();
    if (p.splits > 1) {
        const int64_t rows = (int64_t)q.heads * mq;
        fa_combine_kernel<<<(unsigned)((rows + 15) / 16), 256, 0, st>>>(p.part_o, p.part_lse, p.splits, q.heads, mq,
                                                                        p.out, out_hs, out_rs, lse);
        note_launch();
    }
    return cudaGetLastError();
}

}  // namespace gsa_sm100
