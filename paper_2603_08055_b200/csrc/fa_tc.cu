// fa_tc.cu — K5: dense attention on tcgen05 tensor cores (sm_100a): the
// special-token path (special_token_attention / tiled_attention,
// layer.hpp:80-96, compression.hpp:99-165) and the dense baseline.
//
// CTA = two 128-query tiles x one head x one key split. Warp roles:
//   warp 8  TMA: both Q tiles once, then K / V tiles of 128 keys (16 KB each,
//           128B-swizzled) through a 12-stage ring in the MMA's first-use order,
//           plus L2 prefetches FA_PF tiles ahead.
//   warp 9  MMA: S(n) = Q_w.K(t)^T  (M=128, N=128, K=64, into TMEM, 3 rotating
//           S/P buffers, n = 2t + w), O_w += P(n).V16(t) with P read from TMEM
//           (A-from-TMEM form, P and V in fp16: one MMA per 16-key step).
//   warps 0-7  softmax, one warpgroup per query tile, one thread per query row =
//           one TMEM lane: two passes per tile (row max over the loaded scores,
//           then P chunk by chunk from a TMEM re-read), lazy rescale (only when
//           the max grows by > 2^8; O is then rescaled in TMEM), P = exp2 via
//           MUFU (every third pair by a polynomial on the FMA pipe, FA_POLY)
//           written back over S as packed fp16 pairs; epilogue O/l and lse.
// P.V in fp16: V (bf16) is converted once per call to fp16(v * 2^-e_h) with a per-head
// power of two e_h from max |v| -- exact (bf16's 8-bit significands fit fp16's 11 and
// the scale keeps them in range) -- so the only rounding is P's (2^-12 relative), one
// MMA term instead of the two a bf16 hi + lo P needs (kind::f16 takes no mixed A/B
// formats: an fp16 P against bf16 V is an illegal instruction, measured).
// Split-KV (few query tiles, e.g. 5 specials/view) writes normalised partials
// + lse that gsa_fa_combine merges.
#include <cuda.h>

#include "tc.h"
#include <cstdlib>

#include "tc_ptx.cuh"

namespace gsa_sm100 {
namespace {

using namespace ptx;


#ifndef FA_NS
#define FA_NS 12  // 12 x 16 KB: measured special 39.6 -> 39.1 ms at V=1000 (8 stages)
#endif
constexpr int NS = FA_NS;            // K / V ring stages (16 KB each)
constexpr int TILE = 16384;          // 128 rows x 64 bf16
constexpr int NTHREADS = 384;        // warps 0-3 / 4-7: softmax WG0 / WG1, 8: TMA, 9: MMA, 10-11 idle
constexpr int NWG = 2;               // query tiles (softmax warpgroups) per CTA
constexpr int NSB = 3;               // S/P buffers in TMEM, rotating over the S(n) sequence
constexpr uint32_t TMEM_COLS = 512;
constexpr uint32_t O_COL0 = 384;     // O of WG w: [384 + 64 w, +64); S/P buffer b: [128 b, +128)
constexpr float RESCALE_LOG2 = 8.0f;
#ifndef FA_MIN_WAVES
#define FA_MIN_WAVES 32  // key splits: enough CTAs for this many waves of 148 SMs (8 -> 32: special 39.7 -> 38.8 ms, smaller tail)
#endif
#ifndef FA_SM_REGS
#define FA_SM_REGS 224
#define FA_PROD_REGS 56
#endif
#ifndef FA_TWO_PASS
#define FA_TWO_PASS 1
#endif
#ifndef FA_PB_UNROLL
#define FA_PB_UNROLL 4  // measured (special, V=1000): single pass 41.0 ms; two-pass x1 44.5, x2 41.8, x4 39.1-39.7
#endif
constexpr int PB_UNROLL = FA_PB_UNROLL;
#ifndef FA_POLY
#define FA_POLY 3  // exp2 of every FA_POLY-th pair by polynomial on the FMA pipe (measured at V=1000: special 35.3 -> 32.5 ms with 3; 0: all on MUFU)
#endif

#ifndef FA_PF
#define FA_PF 24  // measured: special 41.3 -> 40.8 ms at V=1000
#endif

struct __align__(1024) FaSmem {
    uint8_t q[NWG][TILE];
    uint8_t ring[NS][TILE];
    uint64_t full[NS], empty[NS];
    uint64_t q_full;
    uint64_t s_full[NSB];
    uint64_t p_full[NWG][2];  // by tile parity: a WG may run one tile ahead of the MMA's P wait
    uint64_t o_done[NWG];     // every PV of the WG (lazy O rescale waits on it)
    uint64_t o_final[NWG];
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
    const unsigned* vmax;  // [H] max |v| (float bits): V16 = fp16(v * 2^-vexp(vmax))
};

// per-head power-of-two exponent that brings |v| <= vmax below 2^14 in fp16 (exact scaling)
__device__ __forceinline__ int vexp(float vmax) { return vmax > 0.0f ? ilogbf(vmax) - 13 : 0; }

__device__ __forceinline__ void setmaxnreg_inc() { asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(FA_SM_REGS) : "memory"); }
__device__ __forceinline__ void setmaxnreg_dec() { asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(FA_PROD_REGS) : "memory"); }

// load order = the MMA issuer's first-use order: K0 K1 V0 K2 V1 ... K(T-1) V(T-2) V(T-1)
__device__ __forceinline__ int seq_k(int t) { return t == 0 ? 0 : 2 * t - 1; }
__device__ __forceinline__ int seq_v(int t, int T) { return t == T - 1 ? 2 * T - 1 : 2 * t + 2; }

// Dense flash attention, two 128-query tiles per CTA (one softmax warpgroup
// each) sharing every K/V tile of the CTA's key split:
//   S(n) = Q_w K(t)^T (bf16, 1 term)             -> TMEM S/P buffer n % 3, n = 2t + w
//   O_w += P(n) V(t) (P = hi + lo bf16, from TMEM) -> TMEM O_w
// S(n+3) is issued right after PV(n), ahead of the next P waits, so a warpgroup
// always has its next scores computing while it runs a softmax.
__global__ void __launch_bounds__(NTHREADS, 1)
    fa_tc_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                 const __grid_constant__ CUtensorMap tm_v, const FaParams p) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    FaSmem& sm = *reinterpret_cast<FaSmem*>(smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u));
    const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
    const int qp = blockIdx.x, split = blockIdx.y, h = blockIdx.z;
    const int t_begin = split * p.tiles_per_split;
    const int t_end = min(p.kv_tiles, t_begin + p.tiles_per_split);
    const int T = t_end - t_begin;
    const int N = NWG * T;

    if (threadIdx.x == 0) {
        for (int i = 0; i < NS; ++i) {
            mbar_init(&sm.full[i], 1);
            mbar_init(&sm.empty[i], 1);
        }
        mbar_init(&sm.q_full, 1);
        for (int b = 0; b < NSB; ++b) mbar_init(&sm.s_full[b], 1);
        for (int w = 0; w < NWG; ++w) {
            mbar_init(&sm.p_full[w][0], 128);
            mbar_init(&sm.p_full[w][1], 128);
            mbar_init(&sm.o_done[w], 1);
            mbar_init(&sm.o_final[w], 1);
        }
        fence_barrier_init();
        prefetch_tmap(&tm_q);
        prefetch_tmap(&tm_k);
        prefetch_tmap(&tm_v);
    }
    if (warp == 9) tmem_alloc(&sm.tmem_base, TMEM_COLS);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = sm.tmem_base;

    if (warp >= 8) {
        setmaxnreg_dec();
        if (warp == 8 && T > 0) {
            // ================================ TMA ================================
            if (elect_one()) {
                mbar_arrive_expect_tx(&sm.q_full, NWG * TILE);
                for (int w = 0; w < NWG; ++w) tma_load_3d(&sm.q[w][0], &tm_q, &sm.q_full, 0, (qp * NWG + w) * 128, h);
            }
            __syncwarp();
            int seq = 0;
            auto load = [&](const CUtensorMap* tm, int t) {
                const int st = seq % NS;
                mbar_wait(&sm.empty[st], (uint32_t)(((seq / NS) & 1) ^ 1));
                if (elect_one()) {
                    mbar_arrive_expect_tx(&sm.full[st], TILE);
                    tma_load_3d(&sm.ring[st][0], tm, &sm.full[st], 0, (t_begin + t) * 128, h);
                }
                __syncwarp();
                ++seq;
            };
            load(&tm_k, 0);
            if (T > 1) load(&tm_k, 1);
            for (int t = 0; t < T; ++t) {
                load(&tm_v, t);
                if (t + 2 < T) load(&tm_k, t + 2);
                // warm L2 FA_PF tiles ahead of the ring: the CTA that first touches a K/V tile
                // of its (head, split) group otherwise waits on DRAM (followers hit L2)
                if (FA_PF > 0 && t + 2 + FA_PF < T && elect_one()) {
                    tma_prefetch_3d(&tm_k, 0, (t_begin + t + 2 + FA_PF) * 128, h);
                    tma_prefetch_3d(&tm_v, 0, (t_begin + t + 2 + FA_PF) * 128, h);
                }
                __syncwarp();
            }
        } else if (warp == 9 && T > 0) {
            // ================================ MMA ================================
            const uint32_t id_s = idesc_bf16(128, 128, 0, 0);
            const uint32_t id_o = idesc_f16(128, 64, 0, 1);  // P (TMEM) and V (SMEM) in fp16
            auto wait_tile = [&](int s) {
                mbar_wait(&sm.full[s % NS], (uint32_t)((s / NS) & 1));
                tc_fence_after();
            };
            auto issue_S = [&](int n) {
                const int w = n & 1, t = n >> 1;
                const int s = seq_k(t);
                if (w == 0) wait_tile(s);
                const uint64_t kd = umma_desc(smem_u32(&sm.ring[s % NS][0]), 16, 1024, 2);
                const uint64_t qd = umma_desc(smem_u32(&sm.q[w][0]), 16, 1024, 2);
                const uint32_t d = tmem + 128 * (n % NSB);
                if (elect_one()) {
                    for (int ks = 0; ks < 4; ++ks) mma_bf16(d, qd + 2 * ks, kd + 2 * ks, id_s, ks != 0);
                    mma_commit(&sm.s_full[n % NSB]);
                    if (w == 1) mma_commit(&sm.empty[s % NS]);
                }
                __syncwarp();
            };
            auto issue_PV = [&](int n) {
                const int w = n & 1, t = n >> 1;
                const int s = seq_v(t, T);
                if (w == 0) wait_tile(s);
                mbar_wait(&sm.p_full[w][t & 1], (uint32_t)((t >> 1) & 1));
                tc_fence_after();
                const uint64_t vd = umma_desc(smem_u32(&sm.ring[s % NS][0]), 16, 1024, 2);
                const uint32_t o = tmem + O_COL0 + 64 * w, pb = tmem + 128 * (n % NSB);
                if (elect_one()) {
                    for (int ks = 0; ks < 8; ++ks) {
                        // P fp16 of keys 16ks..16ks+15: columns 32*(ks/2) + 8*(ks%2)
                        mma_bf16_ts(o, pb + 32 * (ks >> 1) + 8 * (ks & 1), vd + 128 * ks, id_o, (t | ks) != 0);
                    }
                    mma_commit(&sm.o_done[w]);
                    if (t == T - 1) mma_commit(&sm.o_final[w]);
                    if (w == 1) mma_commit(&sm.empty[s % NS]);
                }
                __syncwarp();
            };
            mbar_wait(&sm.q_full, 0);
            tc_fence_after();
            for (int n = 0; n < min(NSB, N); ++n) issue_S(n);
            for (int n = 0; n < N; ++n) {
                issue_PV(n);
                if (n + NSB < N) issue_S(n + NSB);
            }
        }
    } else if (T > 0) {
        // ============================ softmax (warps 0..7) ============================
        setmaxnreg_inc();
        const int w = warp >> 2, qd = warp & 3;
        const int row = 32 * qd + lane;
        const uint32_t lane_base = tmem + ((uint32_t)(32 * qd) << 16);
        const uint32_t o_base = lane_base + O_COL0 + 64 * w;
        float m_used = -INFINITY, l = 0.0f;
        for (int t = 0; t < T; ++t) {
            const int n = 2 * t + w, b = n % NSB;
            const uint32_t s_base = lane_base + 128 * b;
            mbar_wait(&sm.s_full[b], (uint32_t)((n / NSB) & 1));
            __syncwarp();  // .sync.aligned tcgen05 ops below need a converged warp
            tc_fence_after();
            uint32_t sr[4][32];
#pragma unroll
            for (int c = 0; c < 4; ++c) tmem_ld_32x32b_x32(s_base + 32 * c, sr[c]);
            tmem_wait_ld();
            const int valid = p.mk - (t_begin + t) * 128;  // keys of this tile that exist
            if (valid < 128) {
#pragma unroll
                for (int c = 0; c < 4; ++c) {
#pragma unroll
                    for (int e = 0; e < 32; ++e)
                        if (32 * c + e >= valid) sr[c][e] = __float_as_uint(-INFINITY);
                    if (FA_TWO_PASS) tmem_st_32x32b_x32(s_base + 32 * c, sr[c]);  // pass B re-reads TMEM
                }
                if (FA_TWO_PASS) tmem_wait_st();
            }
            float a0 = __uint_as_float(sr[0][0]), a1 = __uint_as_float(sr[1][0]);
            float a2 = __uint_as_float(sr[2][0]), a3 = __uint_as_float(sr[3][0]);
#pragma unroll
            for (int e = 1; e < 32; ++e) {
                a0 = fmaxf(a0, __uint_as_float(sr[0][e]));
                a1 = fmaxf(a1, __uint_as_float(sr[1][e]));
                a2 = fmaxf(a2, __uint_as_float(sr[2][e]));
                a3 = fmaxf(a3, __uint_as_float(sr[3][e]));
            }
            const float mt = fmaxf(fmaxf(a0, a1), fmaxf(a2, a3));
            if (t == 0) {
                m_used = mt;
            } else {
                const bool need = (mt - m_used) * p.c2 > RESCALE_LOG2;
                if (__any_sync(0xffffffffu, need)) {
                    // O must hold every tile < t: PV_w(t-1) done = o_done[w] phase t-1
                    mbar_wait(&sm.o_done[w], (uint32_t)((t - 1) & 1));
                    __syncwarp();
                    tc_fence_after();
                    const float mnew = need ? mt : m_used;
                    const float f = ex2_approx((m_used - mnew) * p.c2);
                    uint32_t o[32];
#pragma unroll
                    for (int half = 0; half < 2; ++half) {
                        tmem_ld_32x32b_x32(o_base + 32 * half, o);
                        tmem_wait_ld();
#pragma unroll
                        for (int e = 0; e < 32; ++e) o[e] = __float_as_uint(__uint_as_float(o[e]) * f);
                        tmem_st_32x32b_x32(o_base + 32 * half, o);
                    }
                    tmem_wait_st();
                    l *= f;
                    m_used = mnew;
                }
            }
            const float mc = m_used * p.c2;
            // P packed as fp16 pairs over the first 16 columns of each 32-key chunk
            const float2 c2v = make_float2(p.c2, p.c2), nmc = make_float2(-mc, -mc);
            float2 lsum2[2] = {make_float2(0.0f, 0.0f), make_float2(0.0f, 0.0f)};
            // FA_TWO_PASS: the 128 scores are live only through the max; the P pass re-reads
            // one 32-key chunk at a time from TMEM (fewer live registers, a chunk loop
            // unrolled by PB_UNROLL instead of a fully unrolled tile)
#pragma unroll PB_UNROLL
            for (int c = 0; c < 4; ++c) {
                uint32_t p16[16];
                uint32_t vv[32];
                if (FA_TWO_PASS) {
                    tmem_ld_32x32b_x32(s_base + 32 * c, vv);
                    tmem_wait_ld();
                }
#pragma unroll
                for (int e2 = 0; e2 < 16; ++e2) {
                    const uint32_t s0 = FA_TWO_PASS ? vv[2 * e2] : sr[c & 3][2 * e2];
                    const uint32_t s1 = FA_TWO_PASS ? vv[2 * e2 + 1] : sr[c & 3][2 * e2 + 1];
                    const float2 x = make_float2(__uint_as_float(s0), __uint_as_float(s1));
                    const float2 a = __ffma2_rn(x, c2v, nmc);
                    // FA_POLY: every FA_POLY-th pair on the FMA pipe instead of MUFU
                    const float2 pv = (FA_POLY > 0 && e2 % (FA_POLY > 0 ? FA_POLY : 1) == FA_POLY - 1)
                                          ? exp2_poly2(a)
                                          : make_float2(ex2_approx(a.x), ex2_approx(a.y));
                    lsum2[e2 & 1] = __fadd2_rn(lsum2[e2 & 1], pv);  // the denominator sums the f32 P
                    p16[e2] = pack_f16(pv.x, pv.y);
                }
                tmem_st_32x32b_x16(s_base + 32 * c, p16);
            }
            const float2 ls = __fadd2_rn(lsum2[0], lsum2[1]);
            l += ls.x + ls.y;
            tmem_wait_st();
            tc_fence_before();
            mbar_arrive(&sm.p_full[w][t & 1]);
        }
        // ------------------------------- epilogue -------------------------------
        mbar_wait(&sm.o_final[w], 0);
        __syncwarp();
        tc_fence_after();
        uint32_t o[2][32];
        tmem_ld_32x32b_x32(o_base, o[0]);
        tmem_ld_32x32b_x32(o_base + 32, o[1]);
        tmem_wait_ld();
        const int qrow = (qp * NWG + w) * 128 + row;
        if (qrow < p.mq) {
            const float inv = ldexpf(1.0f / l, vexp(__uint_as_float(p.vmax[h])));  // undo the V16 scaling exactly
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
    if (warp == 9) {
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

// key splits: enough CTAs for ~8 waves of 148 SMs while each split keeps >= 16 key tiles
int fa_splits(int qpairs, int heads, int kv_tiles) {
    int splits = 1;
    while (qpairs * heads * splits < FA_MIN_WAVES * 148 && kv_tiles / (splits * 2) >= 16) splits *= 2;
    return splits;
}

// workspace: [V16 fp16 H*mk*64][vmax H u32, padded to 256 B][split partials, when split]
static size_t v16_bytes(int heads, int mk) { return ((size_t)heads * mk * 64 * 2 + 255) / 256 * 256; }
static size_t vmax_bytes(int heads) { return ((size_t)heads * 4 + 255) / 256 * 256; }

size_t tc_dense_workspace_bytes(int heads, int mq, int mk, bool with_v16) {
    if (mq == 0) return 0;
    const int qpairs = (mq + 255) / 256, kv_tiles = (mk + 127) / 128;
    const int splits = fa_splits(qpairs, heads, kv_tiles);
    const size_t base = with_v16 ? v16_bytes(heads, mk) + vmax_bytes(heads) : 0;
    if (splits == 1) return base;
    return base + (size_t)splits * heads * mq * 65 * sizeof(float) + 256;
}

cudaError_t tc_dense_attention(const gsa_tensor& q, const gsa_tensor& k, const gsa_tensor& v, float scale,
                               int q_row_offset, int mq, float* out, int64_t out_hs, int64_t out_rs,
                               int out_row_offset, float* lse, void* ws, size_t ws_bytes, cudaStream_t st,
                               const __half* v16_pre, const unsigned* vmax_pre) {
    if (mq == 0) return cudaSuccess;
    // V as the fp16 P.V operand: the caller's V16 planes, else converted here (carved from
    // the workspace, else allocated stream-ordered)
    const int H = q.heads, mk = k.rows;
    const size_t vb = v16_bytes(H, mk) + vmax_bytes(H);
    void* vmem = nullptr;
    bool owned = false;
    char* wsb = static_cast<char*>(ws);
    const __half* v16 = v16_pre;
    const unsigned* vmax = vmax_pre;
    if (!v16) {
        if (ws && ws_bytes >= vb) {
            vmem = ws;
            wsb += vb;
            ws_bytes -= vb;
        } else {
            cudaError_t ea = cudaMallocAsync(&vmem, vb, st);
            if (ea != cudaSuccess) return ea;
            owned = true;
            wsb = nullptr;
            ws_bytes = 0;
        }
        __half* v16w = static_cast<__half*>(vmem);
        unsigned* vmaxw = reinterpret_cast<unsigned*>(static_cast<char*>(vmem) + v16_bytes(H, mk));
        cudaError_t ec = launch_v16(TensorRef{v.data, v.dtype, v.head_stride, v.row_stride}, H, mk, vmaxw, v16w, nullptr, st);
        if (ec != cudaSuccess) {
            if (owned) cudaFreeAsync(vmem, st);
            return ec;
        }
        v16 = v16w;
        vmax = vmaxw;
    }
    CUtensorMap tq, tk, tv;
    const char* qbase = static_cast<const char*>(q.data) + (size_t)q_row_offset * q.row_stride * 2;
    if (!make_rows_map(&tq, qbase, q.heads, mq, q.head_stride, q.row_stride) ||
        !make_rows_map(&tk, k.data, k.heads, k.rows, k.head_stride, k.row_stride) ||
        !make_rows_map(&tv, v16, H, mk, (int64_t)mk * 64, 64)) {
        if (owned) cudaFreeAsync(vmem, st);
        return cudaErrorNotSupported;
    }
    ws = wsb;
    FaParams p{};
    p.heads = q.heads;
    p.mq = mq;
    p.mk = k.rows;
    p.scale = scale;
    p.c2 = scale * 1.4426950408889634f;
    p.kv_tiles = (k.rows + 127) / 128;
    const int qpairs = (mq + 255) / 256;
    int splits = fa_splits(qpairs, q.heads, p.kv_tiles);
    // split-KV needs caller workspace for the partials; without it run unsplit
    if (splits > 1 && (!ws || ws_bytes < (size_t)splits * q.heads * mq * 65 * sizeof(float))) splits = 1;
    p.tiles_per_split = (p.kv_tiles + splits - 1) / splits;
    p.splits = (p.kv_tiles + p.tiles_per_split - 1) / p.tiles_per_split;
    p.out = out + (size_t)out_row_offset * out_rs;
    p.out_hs = out_hs;
    p.out_rs = out_rs;
    p.lse = lse;
    p.vmax = vmax;
    if (p.splits > 1) {
        p.part_o = static_cast<float*>(ws);
        p.part_lse = p.part_o + (size_t)p.splits * q.heads * mq * 64;
    }
    const size_t smem = sizeof(FaSmem) + 1024;
    cudaError_t e = cudaFuncSetAttribute(fa_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) {
        if (owned) cudaFreeAsync(vmem, st);
        return e;
    }
    dim3 grid(qpairs, p.splits, q.heads);
    fa_tc_kernel<<<grid, NTHREADS, smem, st>>>(tq, tk, tv, p);
    note_launch();
    if (p.splits > 1) {
        const int64_t rows = (int64_t)q.heads * mq;
        fa_combine_kernel<<<(unsigned)((rows + 15) / 16), 256, 0, st>>>(p.part_o, p.part_lse, p.splits, q.heads, mq,
                                                                        p.out, out_hs, out_rs, lse);
        note_launch();
    }
    if (owned) cudaFreeAsync(vmem, st);
    return cudaGetLastError();
}

}  // namespace gsa_sm100
