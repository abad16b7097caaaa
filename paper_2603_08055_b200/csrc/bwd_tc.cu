// bwd_tc.cu — the dense passes of the layer backward (gradients.hpp:130-155 compressed
// branch, :197-222 special rows) on tcgen05 tensor cores, head dim 64.
//
// One kernel, two roles (FlashAttention-2 split, probabilities rebuilt from the saved
// LSE rows). A CTA owns 128 FIXED rows (TMEM lanes) and streams the other side in tiles
// of 128:
//   key side   (KEYSIDE): fixed = keys, stream = queries
//       S^T = K Q^T, dP^T = V dO^T  -> P^T = exp(scale S^T - lse[q]), dS^T = P^T (dP^T - D[q]) scale
//       dV += P^T dO, dK += dS^T Q
//   query side: fixed = queries, stream = keys (optionally split over key ranges)
//       S = Q K^T, dP = dO V^T      -> P = exp(scale S - lse[q]), dS = P (dP - D[q]) scale
//       dQ += dS K
// Precision: every f32 operand enters as bf16 hi + lo planes (|x - hi - lo| <= 2^-16 |x|)
// and products take the hi.hi + hi.lo + lo.hi terms, terms with an all-zero lo plane
// (bf16 inputs) skipped; P and dS are written back into TMEM as bf16 hi + lo pairs over
// the S / dP columns they replace and feed the output MMAs as A-from-TMEM operands. The
// result is f32-accurate (the CUDA-core kernels' tolerance), deterministic (each output
// row has one CTA) and accumulated in TMEM.
//
// Warp roles (192 threads): warps 0-3 one thread per fixed row (TMEM lane): the
// exponentials, the hi/lo splits, the epilogue; warp 4 TMA (fixed tiles once, streamed
// tiles through a 2-stage ring); warp 5 MMA issue (one elected lane).
// TMEM columns: S 0-127, dP 128-255, out1 256-319, out2 320-383 (512 allocated).
#include <cuda.h>

#include "tc.h"
#include "tc_ptx.cuh"
#include "tma_util.cuh"

namespace gsa_sm100 {
namespace {

using namespace ptx;

constexpr int BT_THREADS = 192;
constexpr int TILE = 16384;  // 128 rows x 64 bf16, 128B-swizzled (fixed side)
constexpr int STILE = 8192;  // 64 rows x 64 bf16 (streamed side)
constexpr int SROWS = 64;    // streamed rows per step
constexpr int NSTAGE = 4;
// TMEM: [step parity] S (64 columns) and dP (64 columns); the output accumulators
constexpr uint32_t T_S = 0, T_DP = 64, T_BUF = 128, T_O1 = 256, T_O2 = 320, T_COLS = 512;

struct __align__(1024) BwdSmem {
    uint8_t fixed[4][TILE];           // A1 hi, A1 lo, A2 hi, A2 lo
    uint8_t ring[NSTAGE][4][STILE];   // B1 hi, B1 lo, B2 hi, B2 lo
    float st_lse[2][SROWS], st_D[2][SROWS];
    uint64_t fixed_full, full[NSTAGE], empty[NSTAGE], s_full[2], p_full[2], done;
    uint32_t tmem_base;
};

struct BwdTcParams {
    int64_t n_fixed, n_stream;  // rows of the fixed / streamed side
    int64_t s_chunk;            // streamed rows per split (multiple of 128)
    int heads;
    float scale, c2;            // c2 = scale * log2(e)
    bool a1_lo, a2_lo, b1_lo, b2_lo;
    const float *lse, *D;       // by query: [H][n_q]
    // outputs: KEYSIDE out1 = dV, out2 = dK; query side out1 = dQ (or the split's partial)
    float *o1, *o2;
    int64_t o1_hs, o1_rs, o2_hs, o2_rs;
    float* part;                // query side, splits > 1: [split][H][n_fixed][64]
    int splits;
    bool accumulate;
};

// Streamed steps of 64 rows; S / dP of step j+1 are issued (into the other TMEM buffer)
// before the output MMAs of step j, so the row threads' exponentials of one step overlap
// the tensor work of the next.
template <bool KEYSIDE>
__global__ void __launch_bounds__(BT_THREADS, 1)
    bwd_tc_kernel(const __grid_constant__ CUtensorMap tm_a1h, const __grid_constant__ CUtensorMap tm_a1l,
                  const __grid_constant__ CUtensorMap tm_a2h, const __grid_constant__ CUtensorMap tm_a2l,
                  const __grid_constant__ CUtensorMap tm_b1h, const __grid_constant__ CUtensorMap tm_b1l,
                  const __grid_constant__ CUtensorMap tm_b2h, const __grid_constant__ CUtensorMap tm_b2l,
                  const BwdTcParams p) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    BwdSmem& sm = *reinterpret_cast<BwdSmem*>(smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u));
    const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
    const int fixed_tile = blockIdx.x, split = blockIdx.y, h = blockIdx.z;
    const int64_t s_begin = (int64_t)split * p.s_chunk;
    const int64_t s_end = min(p.n_stream, s_begin + p.s_chunk);
    const int T = (int)((s_end - s_begin + SROWS - 1) / SROWS);

    if (threadIdx.x == 0) {
        mbar_init(&sm.fixed_full, 1);
        for (int i = 0; i < NSTAGE; ++i) {
            mbar_init(&sm.full[i], 1);
            mbar_init(&sm.empty[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&sm.s_full[i], 1);
            mbar_init(&sm.p_full[i], 128);
        }
        mbar_init(&sm.done, 1);
        fence_barrier_init();
    }
    if (warp == 5) tmem_alloc(&sm.tmem_base, T_COLS);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = sm.tmem_base;

    if (warp == 4) {
        // ================================ TMA ================================
        if (T > 0 && elect_one()) {
            const uint32_t fb = TILE * (2 + (p.a1_lo ? 1 : 0) + (p.a2_lo ? 1 : 0));
            mbar_arrive_expect_tx(&sm.fixed_full, fb);
            const int r0 = fixed_tile * 128;
            tma_load_3d(&sm.fixed[0][0], &tm_a1h, &sm.fixed_full, 0, r0, h);
            if (p.a1_lo) tma_load_3d(&sm.fixed[1][0], &tm_a1l, &sm.fixed_full, 0, r0, h);
            tma_load_3d(&sm.fixed[2][0], &tm_a2h, &sm.fixed_full, 0, r0, h);
            if (p.a2_lo) tma_load_3d(&sm.fixed[3][0], &tm_a2l, &sm.fixed_full, 0, r0, h);
            const uint32_t sb = STILE * (2 + (p.b1_lo ? 1 : 0) + (p.b2_lo ? 1 : 0));
            for (int j = 0; j < T; ++j) {
                const int st = j % NSTAGE;
                mbar_wait(&sm.empty[st], (uint32_t)(((j / NSTAGE) & 1) ^ 1));
                mbar_arrive_expect_tx(&sm.full[st], sb);
                const int c1 = (int)(s_begin + (int64_t)j * SROWS);
                tma_load_3d(&sm.ring[st][0][0], &tm_b1h, &sm.full[st], 0, c1, h);
                if (p.b1_lo) tma_load_3d(&sm.ring[st][1][0], &tm_b1l, &sm.full[st], 0, c1, h);
                tma_load_3d(&sm.ring[st][2][0], &tm_b2h, &sm.full[st], 0, c1, h);
                if (p.b2_lo) tma_load_3d(&sm.ring[st][3][0], &tm_b2l, &sm.full[st], 0, c1, h);
            }
        }
        __syncwarp();
    } else if (warp == 5) {
        // ================================ MMA ================================
        const uint32_t id_s = idesc_bf16(128, SROWS, 0, 0);
        const uint32_t id_o = idesc_bf16(128, 64, 0, 1);  // A (P / dS) from TMEM, B MN-major
        auto kdesc = [](const uint8_t* t) { return umma_desc(smem_u32(t), 16, 1024, 2); };
        if (T > 0) {
            mbar_wait(&sm.fixed_full, 0);
            tc_fence_after();
        }
        const uint64_t a1h = kdesc(sm.fixed[0]), a1l = kdesc(sm.fixed[1]);
        const uint64_t a2h = kdesc(sm.fixed[2]), a2l = kdesc(sm.fixed[3]);
        auto issue_S = [&](int j) {
            const int st = j % NSTAGE;
            mbar_wait(&sm.full[st], (uint32_t)((j / NSTAGE) & 1));
            tc_fence_after();
            const uint64_t b1h = kdesc(sm.ring[st][0]), b1l = kdesc(sm.ring[st][1]);
            const uint64_t b2h = kdesc(sm.ring[st][2]), b2l = kdesc(sm.ring[st][3]);
            const uint32_t ts = tmem + T_S + T_BUF * (j & 1), td = tmem + T_DP + T_BUF * (j & 1);
            if (elect_one()) {
                // S = A1 B1^T and dP = A2 B2^T over d = 64 (4 k-steps of 16)
                for (int ks = 0; ks < 4; ++ks) {
                    const uint32_t acc = ks != 0;
                    mma_bf16(ts, a1h + 2 * ks, b1h + 2 * ks, id_s, acc);
                    if (p.b1_lo) mma_bf16(ts, a1h + 2 * ks, b1l + 2 * ks, id_s, 1);
                    if (p.a1_lo) mma_bf16(ts, a1l + 2 * ks, b1h + 2 * ks, id_s, 1);
                    mma_bf16(td, a2h + 2 * ks, b2h + 2 * ks, id_s, acc);
                    if (p.b2_lo) mma_bf16(td, a2h + 2 * ks, b2l + 2 * ks, id_s, 1);
                    if (p.a2_lo) mma_bf16(td, a2l + 2 * ks, b2h + 2 * ks, id_s, 1);
                }
                mma_commit(&sm.s_full[j & 1]);
            }
            __syncwarp();
        };
        if (T > 0) issue_S(0);
        for (int j = 0; j < T; ++j) {
            if (j + 1 < T) issue_S(j + 1);
            const int st = j % NSTAGE, pb = j & 1;
            mbar_wait(&sm.p_full[pb], (uint32_t)((j >> 1) & 1));
            tc_fence_after();
            const uint64_t b1h = kdesc(sm.ring[st][0]), b1l = kdesc(sm.ring[st][1]);
            const uint64_t b2h = kdesc(sm.ring[st][2]), b2l = kdesc(sm.ring[st][3]);
            const uint32_t ts = tmem + T_S + T_BUF * pb, td = tmem + T_DP + T_BUF * pb;
            if (elect_one()) {
                // outputs over the 64 streamed rows (4 k-steps of 16): the A chunk of k-step ks
                // holds hi pairs at columns 32 (ks/2) + 8 (ks%2), lo pairs 16 columns further
                for (int ks = 0; ks < 4; ++ks) {
                    const uint32_t col = 32 * (ks >> 1) + 8 * (ks & 1);
                    const uint32_t acc0 = (j | ks) != 0;
                    if (KEYSIDE) {
                        // dV += P^T dO (B2), dK += dS^T Q (B1)
                        const uint64_t vh = b2h + 128 * ks, vl = b2l + 128 * ks;
                        mma_bf16_ts(tmem + T_O1, ts + col, vh, id_o, acc0);
                        if (p.b2_lo) mma_bf16_ts(tmem + T_O1, ts + col, vl, id_o, 1);
                        mma_bf16_ts(tmem + T_O1, ts + col + 16, vh, id_o, 1);
                        const uint64_t qh = b1h + 128 * ks, ql = b1l + 128 * ks;
                        mma_bf16_ts(tmem + T_O2, td + col, qh, id_o, acc0);
                        if (p.b1_lo) mma_bf16_ts(tmem + T_O2, td + col, ql, id_o, 1);
                        mma_bf16_ts(tmem + T_O2, td + col + 16, qh, id_o, 1);
                    } else {
                        // dQ += dS K (B1)
                        const uint64_t kh = b1h + 128 * ks, kl = b1l + 128 * ks;
                        mma_bf16_ts(tmem + T_O1, td + col, kh, id_o, acc0);
                        if (p.b1_lo) mma_bf16_ts(tmem + T_O1, td + col, kl, id_o, 1);
                        mma_bf16_ts(tmem + T_O1, td + col + 16, kh, id_o, 1);
                    }
                }
                mma_commit(&sm.empty[st]);
                if (j == T - 1) mma_commit(&sm.done);
            }
            __syncwarp();
        }
    } else {
        // ===================== rows: exponentials, splits, epilogue =====================
        const int row = 32 * warp + lane;
        const uint32_t lane_base = tmem + ((uint32_t)(32 * warp) << 16);
        const int64_t grow = (int64_t)fixed_tile * 128 + row;
        float nl2_r = 0.0f, nD_r = 0.0f;  // -lse * log2(e), -D of this (query) row
        if (!KEYSIDE) {
            const bool ok = grow < p.n_fixed;
            nl2_r = ok ? -p.lse[(int64_t)h * p.n_fixed + grow] * 1.4426950408889634f : 0.0f;
            nD_r = ok ? -p.D[(int64_t)h * p.n_fixed + grow] : 0.0f;
        }
        const float2 c2v = make_float2(p.c2, p.c2), scv = make_float2(p.scale, p.scale), m1 = make_float2(-1.0f, -1.0f);
        // KEYSIDE: streamed queries' (-lse log2 e, -D) for the next step, in registers
        float nxt_l = -INFINITY, nxt_d = 0.0f;
        auto load_stats = [&](int jj) {
            const int64_t q = s_begin + (int64_t)jj * SROWS + row;
            const bool ok = jj < T && q < s_end;
            nxt_l = ok ? -p.lse[(int64_t)h * p.n_stream + q] * 1.4426950408889634f : -INFINITY;
            nxt_d = ok ? -p.D[(int64_t)h * p.n_stream + q] : 0.0f;
        };
        if (KEYSIDE && row < SROWS) load_stats(0);
        for (int j = 0; j < T; ++j) {
            const int pb = j & 1;
            if (KEYSIDE) {
                // the 64 streamed queries' lse / D, shared by every key row: loaded one step
                // ahead (the global-load latency overlaps the previous step), published here
                if (row < SROWS) {
                    sm.st_lse[pb][row] = nxt_l;
                    sm.st_D[pb][row] = nxt_d;
                }
                named_bar_sync(1, 128);
                if (row < SROWS) load_stats(j + 1);
            }
            mbar_wait(&sm.s_full[pb], (uint32_t)((j >> 1) & 1));
            __syncwarp();
            tc_fence_after();
            const uint32_t ts = lane_base + T_S + T_BUF * pb, td = lane_base + T_DP + T_BUF * pb;
#pragma unroll 1
            for (int c = 0; c < SROWS / 32; ++c) {
                uint32_t sv[32], dv[32];
                tmem_ld_32x32b_x32(ts + 32 * c, sv);
                tmem_ld_32x32b_x32(td + 32 * c, dv);
                tmem_wait_ld();
                uint32_t ph[16], pl[16], dh[16], dl[16];
#pragma unroll
                for (int e2 = 0; e2 < 16; ++e2) {
                    // pairs on the packed f32x2 pipe; the statistics are stored negated
                    const float2 nl = KEYSIDE ? *reinterpret_cast<const float2*>(&sm.st_lse[pb][32 * c + 2 * e2])
                                              : make_float2(nl2_r, nl2_r);
                    const float2 nd = KEYSIDE ? *reinterpret_cast<const float2*>(&sm.st_D[pb][32 * c + 2 * e2])
                                              : make_float2(nD_r, nD_r);
                    const float2 a2 = __ffma2_rn(make_float2(__uint_as_float(sv[2 * e2]), __uint_as_float(sv[2 * e2 + 1])),
                                                 c2v, nl);
                    const float2 pv = make_float2(ex2_approx(a2.x), ex2_approx(a2.y));
                    const float2 t2 = __fadd2_rn(make_float2(__uint_as_float(dv[2 * e2]), __uint_as_float(dv[2 * e2 + 1])), nd);
                    const float2 dsv = __fmul2_rn(__fmul2_rn(pv, t2), scv);
                    const __nv_bfloat162 phb = __float22bfloat162_rn(pv);
                    const __nv_bfloat162 dhb = __float22bfloat162_rn(dsv);
                    const float2 plo = __ffma2_rn(__bfloat1622float2(phb), m1, pv);
                    const float2 dlo = __ffma2_rn(__bfloat1622float2(dhb), m1, dsv);
                    ph[e2] = *reinterpret_cast<const uint32_t*>(&phb);
                    dh[e2] = *reinterpret_cast<const uint32_t*>(&dhb);
                    const __nv_bfloat162 plb = __float22bfloat162_rn(plo), dlb = __float22bfloat162_rn(dlo);
                    pl[e2] = *reinterpret_cast<const uint32_t*>(&plb);
                    dl[e2] = *reinterpret_cast<const uint32_t*>(&dlb);
                }
                if (KEYSIDE) {
                    tmem_st_32x32b_x16(ts + 32 * c, ph);
                    tmem_st_32x32b_x16(ts + 32 * c + 16, pl);
                }
                tmem_st_32x32b_x16(td + 32 * c, dh);
                tmem_st_32x32b_x16(td + 32 * c + 16, dl);
            }
            tmem_wait_st();
            tc_fence_before();
            mbar_arrive(&sm.p_full[pb]);
        }
        // ------------------------------- epilogue -------------------------------
        if (T > 0) {
            mbar_wait(&sm.done, 0);
            __syncwarp();
            tc_fence_after();
            for (int o = 0; o < (KEYSIDE ? 2 : 1); ++o) {
                uint32_t v[2][32];
                const uint32_t col = o == 0 ? T_O1 : T_O2;
                tmem_ld_32x32b_x32(lane_base + col, v[0]);
                tmem_ld_32x32b_x32(lane_base + col + 32, v[1]);
                tmem_wait_ld();
                if (grow < p.n_fixed) {
                    float* dst;
                    bool acc = p.accumulate;
                    if (!KEYSIDE && p.splits > 1) {
                        dst = p.part + (((int64_t)split * p.heads + h) * p.n_fixed + grow) * 64;
                        acc = false;
                    } else if (o == 0) {
                        dst = p.o1 + (int64_t)h * p.o1_hs + grow * p.o1_rs;
                    } else {
                        dst = p.o2 + (int64_t)h * p.o2_hs + grow * p.o2_rs;
                    }
                    float4* d4 = reinterpret_cast<float4*>(dst);
                    float4 y[16];
                    if (acc) {  // every load before the first store: the 16 loads overlap
#pragma unroll
                        for (int e = 0; e < 16; ++e) y[e] = d4[e];
                    }
#pragma unroll
                    for (int e = 0; e < 16; ++e) {
                        const uint32_t* u = &v[e >> 3][4 * (e & 7)];
                        float4 x = make_float4(__uint_as_float(u[0]), __uint_as_float(u[1]), __uint_as_float(u[2]),
                                               __uint_as_float(u[3]));
                        if (acc) {
                            x.x += y[e].x;
                            x.y += y[e].y;
                            x.z += y[e].z;
                            x.w += y[e].w;
                        }
                        d4[e] = x;
                    }
                }
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 5) {
        tc_fence_after();
        tmem_dealloc(tmem, T_COLS);
    }
}

// dQ from the key-split partials, summed in split order
__global__ void bwd_tc_reduce_kernel(const float* part, int splits, int heads, int64_t rows, float* out, int64_t hs,
                                     int64_t rs, bool accumulate) {
    const int64_t n = (int64_t)heads * rows * 64;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
        const int j = (int)(e & 63);
        const int64_t r = (e >> 6) % rows, h = (e >> 6) / rows;
        float acc = 0.0f;
        for (int s = 0; s < splits; ++s) acc += part[(int64_t)s * n + e];
        float* o = out + h * hs + r * rs + j;
        *o = accumulate ? *o + acc : acc;
    }
}

bool make_plane_map(CUtensorMap* m, const __nv_bfloat16* plane, int heads, int64_t rows, int64_t hs, int box_rows) {
    // [H][rows][64] bf16 planes (head stride hs, or rows * 64), boxes of box_rows x 64 (128B
    // swizzle); an absent plane maps the hi plane (never loaded)
    TmapEncodeFn enc = tmap_encode_fn();
    if (!enc || rows <= 0) return false;
    cuuint64_t dims[3] = {64, (cuuint64_t)rows, (cuuint64_t)heads};
    cuuint64_t strides[2] = {128, (cuuint64_t)(hs ? hs : rows * 64) * 2};
    cuuint32_t box[3] = {64, (cuuint32_t)box_rows, 1};
    cuuint32_t es[3] = {1, 1, 1};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<__nv_bfloat16*>(plane), dims, strides, box, es,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace

bool tc_bwd_supported(int dim) { return dim == 64 && tmap_encode_fn() != nullptr; }

int tc_bwd_dq_splits(int heads, int64_t n_q, int64_t n_k) {
    // key splits of the query-side pass (few query tiles: the special rows): the count that
    // minimises waves / split (the last wave's idle SMs), each split >= 8 key tiles
    const int64_t ctas = (int64_t)heads * ((n_q + 127) / 128);
    const int64_t cap = std::max<int64_t>(1, std::min<int64_t>(16, ((n_k + 127) / 128) / 8));
    int best = 1;
    double best_cost = 1e30;
    for (int64_t s = 1; s <= cap; ++s) {
        const double cost = (double)((ctas * s + 147) / 148) / (double)s;
        if (cost < best_cost * 0.98) {
            best_cost = cost;
            best = (int)s;
        }
    }
    return best;
}

cudaError_t launch_bwd_tc(const BwdTcArgs& a, cudaStream_t st) {
    if (a.heads == 0 || a.n_q == 0 || a.n_k == 0) return cudaSuccess;
    // [0..7]: Q hi/lo, dO hi/lo, K hi/lo, V hi/lo as FIXED operands (128-row boxes);
    // [8..15]: the same as STREAMED operands (64-row boxes)
    CUtensorMap m[16];
    bool ok = true;
    for (int f = 0; f < 2; ++f) {
        const int br = f == 0 ? 128 : SROWS;
        CUtensorMap* mm = m + 8 * f;
        ok = ok && make_plane_map(&mm[0], a.q_hi, a.heads, a.n_q, a.q_hs, br) &&
             make_plane_map(&mm[1], a.q_lo ? a.q_lo : a.q_hi, a.heads, a.n_q, a.q_hs, br) &&
             make_plane_map(&mm[2], a.do_hi, a.heads, a.n_q, a.do_hs, br) &&
             make_plane_map(&mm[3], a.do_lo ? a.do_lo : a.do_hi, a.heads, a.n_q, a.do_hs, br) &&
             make_plane_map(&mm[4], a.k_hi, a.heads, a.n_k, a.k_hs, br) &&
             make_plane_map(&mm[5], a.k_lo ? a.k_lo : a.k_hi, a.heads, a.n_k, a.k_hs, br) &&
             make_plane_map(&mm[6], a.v_hi, a.heads, a.n_k, a.v_hs, br) &&
             make_plane_map(&mm[7], a.v_lo ? a.v_lo : a.v_hi, a.heads, a.n_k, a.v_hs, br);
    }
    const size_t smem = sizeof(BwdSmem) + 1024;
    cudaError_t e = cudaFuncSetAttribute(bwd_tc_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(bwd_tc_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    const float LOG2E = 1.4426950408889634f;
    if (a.dk) {
        // key side: fixed = K (A1) / V (A2), stream = Q (B1) / dO (B2)
        BwdTcParams p{};
        p.n_fixed = a.n_k;
        p.n_stream = a.n_q;
        p.s_chunk = (a.n_q + 127) / 128 * 128;
        p.heads = a.heads;
        p.scale = a.scale;
        p.c2 = a.scale * LOG2E;
        p.a1_lo = a.k_lo != nullptr;
        p.a2_lo = a.v_lo != nullptr;
        p.b1_lo = a.q_lo != nullptr;
        p.b2_lo = a.do_lo != nullptr;
        p.lse = a.lse;
        p.D = a.D;
        p.o1 = a.dv;
        p.o1_hs = a.dv_hs;
        p.o1_rs = a.dv_rs;
        p.o2 = a.dk;
        p.o2_hs = a.dk_hs;
        p.o2_rs = a.dk_rs;
        p.splits = 1;
        p.accumulate = a.accumulate_kv;
        bwd_tc_kernel<true><<<dim3((unsigned)((a.n_k + 127) / 128), 1, a.heads), BT_THREADS, smem, st>>>(
            m[4], m[5], m[6], m[7], m[8], m[9], m[10], m[11], p);
        note_launch();
    }
    if (a.dq) {
        // query side: fixed = Q (A1) / dO (A2), stream = K (B1) / V (B2)
        BwdTcParams p{};
        p.n_fixed = a.n_q;
        p.n_stream = a.n_k;
        const int splits = a.dq_part ? a.dq_splits : 1;
        const int64_t ktiles = (a.n_k + 127) / 128;
        p.s_chunk = (ktiles + splits - 1) / splits * 128;
        p.splits = (int)((a.n_k + p.s_chunk - 1) / p.s_chunk);
        p.heads = a.heads;
        p.scale = a.scale;
        p.c2 = a.scale * LOG2E;
        p.a1_lo = a.q_lo != nullptr;
        p.a2_lo = a.do_lo != nullptr;
        p.b1_lo = a.k_lo != nullptr;
        p.b2_lo = a.v_lo != nullptr;
        p.lse = a.lse;
        p.D = a.D;
        p.o1 = a.dq;
        p.o1_hs = a.dq_hs;
        p.o1_rs = a.dq_rs;
        p.part = a.dq_part;
        p.accumulate = a.accumulate_q;
        bwd_tc_kernel<false><<<dim3((unsigned)((a.n_q + 127) / 128), p.splits, a.heads), BT_THREADS, smem, st>>>(
            m[0], m[1], m[2], m[3], m[12], m[13], m[14], m[15], p);
        note_launch();
        if (p.splits > 1) {
            const int64_t n = (int64_t)a.heads * a.n_q * 64;
            const unsigned blocks = (unsigned)std::min<int64_t>((n + 255) / 256, 148 * 16);
            bwd_tc_reduce_kernel<<<blocks, 256, 0, st>>>(a.dq_part, p.splits, a.heads, a.n_q, a.dq, a.dq_hs, a.dq_rs,
                                                          a.accumulate_q);
            note_launch();
        }
    }
    return cudaGetLastError();
}

}  // namespace gsa_sm100
