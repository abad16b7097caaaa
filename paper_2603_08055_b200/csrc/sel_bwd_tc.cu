// sel_bwd_tc.cu — the selection-branch backward (gradients.hpp:171-195) on tcgen05
// tensor cores, head dim 64, window side 4 (16 tokens per window).
//
// Same tiling as the forward's select_tc: the gathered side is the MMA's M = 128 (8
// windows gathered by TMA with the 4-D window map, 2 KB each), the 16 rows of the
// CTA's own window are N = 16. One CTA per (head, window), 192 threads: warps 0-3 one
// thread per gathered row (TMEM lane), warp 4 TMA, warp 5 MMA.
//
// dQ pass (window = a query window, gathered = the keys of its plan row):
//   S^T = K_g Q^T, dP^T = V_g dS_sel^T              (M = 128 keys, N = 16 queries)
//   P^T = exp(scale S^T - lse[q]), dS^T = P^T (dP^T - D[q]) scale  -> smem, K-major
//   dQ^T += K_g^T dS^T                               (M = 64 features, N = 16, K = 128 keys;
//                                                     K_g read as an MN-major A operand)
// dK/dV pass (window = a key window, gathered = the query windows of its inverse-plan row):
//   S = Q_g K^T, dP = dS_g V^T                       (M = 128 queries, N = 16 keys)
//   P = exp(scale S - lse[q]), dS = P (dP - D[q]) scale
//   dK^T += Q_g^T dS, dV^T += dS_g^T P               (M = 64, N = 16, K = 128 queries)
// f32 operands as bf16 hi + lo planes, hi.hi + hi.lo + lo.hi products; P and dS as hi + lo
// bf16 planes in shared memory (no-swizzle core-matrix layout: [row group of 8][16-byte
// column chunk][8 rows][16 B]). Outputs accumulate in TMEM and are added to dq / dk / dv
// by the one CTA that owns those rows.
#include <cuda.h>

#include "tc.h"
#include "tc_ptx.cuh"
#include "tma_util.cuh"

namespace gsa_sm100 {
namespace {

using namespace ptx;

constexpr int SB_THREADS = 192;
constexpr int WIN_B = 2048;           // one window: 16 rows x 64 bf16
constexpr int CHUNK = 16384;          // 8 windows
constexpr int SB_RING = 160 * 1024;   // gather ring: as many stages of the pass's planes as fit
constexpr int SB_MAXNS = 6;
constexpr int BQ_STRIDE = 16 * 128;   // bytes per 8-row group of a [16][128] bf16 operand
constexpr int BQ_BYTES = 2 * BQ_STRIDE;
// TMEM: [chunk parity] S, dP (16 columns each) and the two output accumulators
constexpr uint32_t C_S = 0, C_DP = 16, C_BUF = 32, C_O1 = 64, C_O2 = 80, SB_COLS = 128;

struct __align__(1024) SbSmem {
    uint8_t ring[SB_RING];            // stages of the gathered planes present: A1 hi, A2 hi[, A1 lo][, A2 lo]
    uint8_t own[2][4][WIN_B];         // [item parity] the item's window: B1 hi, B1 lo, B2 hi, B2 lo
    uint8_t bx[2][4][BQ_BYTES];       // [chunk parity] X hi, X lo, Y hi, Y lo ([16 own rows][128 gathered])
    float own_lse[2][16], own_D[2][16];
    uint64_t own_full[2], own_empty[2], full[SB_MAXNS], empty[SB_MAXNS], s_full[2], p_full[2], o_done[2], acc_free;
    uint32_t tmem_base;
};

struct SbParams {
    DevLayout L;
    int heads;
    int64_t rows;               // items: heads x windows
    float scale, c2;
    bool a1_lo, a2_lo, b1_lo, b2_lo;  // which operands carry lo planes (f32 values)
    const int64_t *offsets;     // the rows to walk: plan CSR (dQ pass) or inverse plan (dK/dV pass)
    const int32_t* ids;
    const float *lse, *D;       // [H][Mi] by image token
    float* o1;                  // dQ (dQ pass) / dK (dK/dV pass), rows of image token t at row Ms + t
    float* o2;                  // dV (dK/dV pass)
    int64_t o1_hs, o1_rs, o2_hs, o2_rs;
};

__device__ __forceinline__ void win_coords(const DevLayout& L, int wid, int& c1, int& c2) {
    const int f = wid / L.wins_per_frame, r = wid - f * L.wins_per_frame;
    const int wr = r / L.wins_w, wc = r - wr * L.wins_w;
    c1 = wc * 4;
    c2 = f * L.grid_h + wr * 4;
}

// element (row n, column k) of a [16][128] bf16 K-major operand in the no-swizzle layout
__device__ __forceinline__ uint32_t bx_off(int n, int k) {
    return (uint32_t)((n >> 3) * BQ_STRIDE + (k >> 3) * 128 + (n & 7) * 16 + (k & 7) * 2);
}

// Persistent: CTA b walks items b, b + grid, ... (items with an empty row are skipped by
// every role alike). The TMA warp runs ahead through the ring across items; the own
// window's tiles are double-buffered by item parity; the output accumulators are reused
// per item once the previous item's epilogue has read them (acc_free).
// KEYSIDE = false: dQ pass (A1 = K_g, A2 = V_g, B1 = Q, B2 = dS_sel; outputs dQ^T)
// KEYSIDE = true:  dK/dV pass (A1 = Q_g, A2 = dS_g, B1 = K, B2 = V; outputs dK^T, dV^T)
template <bool KEYSIDE>
__global__ void __launch_bounds__(SB_THREADS, 1)
    sel_bwd_tc_kernel(const __grid_constant__ CUtensorMap ta1h, const __grid_constant__ CUtensorMap ta1l,
                      const __grid_constant__ CUtensorMap ta2h, const __grid_constant__ CUtensorMap ta2l,
                      const __grid_constant__ CUtensorMap tb1h, const __grid_constant__ CUtensorMap tb1l,
                      const __grid_constant__ CUtensorMap tb2h, const __grid_constant__ CUtensorMap tb2l,
                      const SbParams p) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    SbSmem& sm = *reinterpret_cast<SbSmem*>(smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u));
    const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
    const DevLayout& L = p.L;
    if (threadIdx.x == 0) {
        for (int i = 0; i < 2; ++i) {
            mbar_init(&sm.own_full[i], 1);
            mbar_init(&sm.own_empty[i], 1);
        }
        for (int i = 0; i < SB_MAXNS; ++i) {
            mbar_init(&sm.full[i], 1);
            mbar_init(&sm.empty[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&sm.s_full[i], 1);
            mbar_init(&sm.p_full[i], 128);
            mbar_init(&sm.o_done[i], 1);
        }
        mbar_init(&sm.acc_free, 128);
        fence_barrier_init();
    }
    if (warp == 5) tmem_alloc(&sm.tmem_base, SB_COLS);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = sm.tmem_base;
    // ring geometry of this pass: planes per stage and stages
    const int np = 2 + p.a1_lo + p.a2_lo, NS = min(SB_MAXNS, SB_RING / (np * CHUNK));
    // CSR row bounds, fetched one or two items ahead of their use (their load latency would
    // otherwise sit on every item's critical path)
    struct Off {
        int64_t b, e;
    };
    auto offs = [&](int64_t it) {
        Off o{0, 0};
        if (it < p.rows) {
            o.b = p.offsets[it];
            o.e = p.offsets[it + 1];
        }
        return o;
    };
    const int64_t G = gridDim.x;
    auto plane = [&](int st, int pl) -> uint8_t* {  // pl: 0 A1 hi, 1 A1 lo, 2 A2 hi, 3 A2 lo
        const int slot = pl == 0 ? 0 : pl == 2 ? 1 : pl == 1 ? 2 : 2 + p.a1_lo;
        return sm.ring + (st * np + slot) * CHUNK;
    };

    if (warp == 4) {
        // ================================ TMA ================================
        int gc = 0, ic = 0;
        // window ids come one lane per window, 32 at a time; the next item's first 32 are
        // fetched while this item streams
        auto ids32 = [&](const Off& o, int64_t base) {
            const int64_t j = o.b + base + lane;
            return j < o.e ? p.ids[j] : 0;
        };
        Off o0 = offs(blockIdx.x), o1 = offs(blockIdx.x + G);
        int id0 = ids32(o0, 0);
        for (int64_t item = blockIdx.x; item < p.rows; item += G) {
            const Off o2 = offs(item + 2 * G);
            const int id1 = ids32(o1, 0);
            const int h = (int)(item / L.windows), w = (int)(item - (int64_t)h * L.windows);
            const int nwin = (int)(o0.e - o0.b);
            const int nch = (nwin + 7) / 8;
            if (nch > 0) {
                const int ob = ic & 1;
                mbar_wait(&sm.own_empty[ob], (uint32_t)(((ic >> 1) & 1) ^ 1));
                if (lane == 0) {
                    int c1, c2;
                    win_coords(L, w, c1, c2);
                    mbar_arrive_expect_tx(&sm.own_full[ob], (2 + p.b1_lo + p.b2_lo) * WIN_B);
                    tma_load_4d(sm.own[ob][0], &tb1h, &sm.own_full[ob], 0, c1, c2, h);
                    tma_load_4d(sm.own[ob][2], &tb2h, &sm.own_full[ob], 0, c1, c2, h);
                    if (p.b1_lo) tma_load_4d(sm.own[ob][1], &tb1l, &sm.own_full[ob], 0, c1, c2, h);
                    if (p.b2_lo) tma_load_4d(sm.own[ob][3], &tb2l, &sm.own_full[ob], 0, c1, c2, h);
                }
                __syncwarp();
                int idg = id0;  // ids of windows 32 * (c / 4) + lane
                for (int c = 0; c < nch; ++c, ++gc) {
                    if (c > 0 && (c & 3) == 0) idg = ids32(o0, 8 * c);
                    const int my_id = __shfl_sync(0xffffffffu, idg, (8 * c + (lane & 7)) & 31);
                    const int st = gc % NS;
                    const int nc = min(8, nwin - 8 * c);
                    mbar_wait(&sm.empty[st], (uint32_t)(((gc / NS) & 1) ^ 1));
                    if (nc < 8) {
                        // slots past a short chunk must hold finite values (they meet zero P / dS):
                        // zero them through the generic proxy before the stage is published
                        for (int pl = 0; pl < 4; ++pl) {
                            if ((pl == 1 && !p.a1_lo) || (pl == 3 && !p.a2_lo)) continue;
                            uint4* z = reinterpret_cast<uint4*>(plane(st, pl) + nc * WIN_B);
                            for (int i = lane; i < (8 - nc) * WIN_B / 16; i += 32) z[i] = make_uint4(0, 0, 0, 0);
                        }
                        fence_proxy_async_smem();
                        __syncwarp();
                    }
                    if (lane == 0) mbar_arrive_expect_tx(&sm.full[st], (2 + p.a1_lo + p.a2_lo) * nc * WIN_B);
                    __syncwarp();
                    if (lane < nc) {
                        int c1, c2;
                        win_coords(L, my_id, c1, c2);
                        tma_load_4d(plane(st, 0) + lane * WIN_B, &ta1h, &sm.full[st], 0, c1, c2, h);
                        tma_load_4d(plane(st, 2) + lane * WIN_B, &ta2h, &sm.full[st], 0, c1, c2, h);
                        if (p.a1_lo) tma_load_4d(plane(st, 1) + lane * WIN_B, &ta1l, &sm.full[st], 0, c1, c2, h);
                        if (p.a2_lo) tma_load_4d(plane(st, 3) + lane * WIN_B, &ta2l, &sm.full[st], 0, c1, c2, h);
                    }
                    __syncwarp();
                }
                ++ic;
            }
            o0 = o1;
            o1 = o2;
            id0 = id1;
        }
    } else if (warp == 5) {
        // ================================ MMA ================================
        // S / dP of chunk c+1 are issued before the outputs of chunk c (two TMEM buffers),
        // so the row warps' exponentials of one chunk overlap the MMAs of the next
        const uint32_t id_s = idesc_bf16(128, 16, 0, 0);  // gathered (K-major) x own window (K-major)
        const uint32_t id_o = idesc_bf16(64, 16, 1, 0);   // gathered as MN-major A x P / dS (K-major)
        auto kd = [](const uint8_t* t) { return umma_desc(smem_u32(t), 16, 1024, 2); };
        auto nd = [](const uint8_t* t) { return umma_desc(smem_u32(t), 128, BQ_STRIDE, 0); };
        int gc = 0, ic = 0;
        Off on = offs(blockIdx.x);
        for (int64_t item = blockIdx.x; item < p.rows; item += G) {
            const Off oc = on;
            on = offs(item + G);
            const int nch = (int)((oc.e - oc.b + 7) / 8);
            if (nch == 0) continue;
            const int ob = ic & 1;
            mbar_wait(&sm.own_full[ob], (uint32_t)((ic >> 1) & 1));
            tc_fence_after();
            const uint64_t b1h = kd(sm.own[ob][0]), b1l = kd(sm.own[ob][1]), b2h = kd(sm.own[ob][2]), b2l = kd(sm.own[ob][3]);
            auto issue_S = [&](int g, bool last) {
                const int st = g % NS;
                mbar_wait(&sm.full[st], (uint32_t)((g / NS) & 1));
                tc_fence_after();
                const uint64_t a1h = kd(plane(st, 0)), a1l = kd(plane(st, 1));
                const uint64_t a2h = kd(plane(st, 2)), a2l = kd(plane(st, 3));
                const uint32_t cs = tmem + C_S + C_BUF * (g & 1), cd = tmem + C_DP + C_BUF * (g & 1);
                if (elect_one()) {
                    for (int ks = 0; ks < 4; ++ks) {
                        mma_bf16(cs, a1h + 2 * ks, b1h + 2 * ks, id_s, ks != 0);
                        mma_bf16(cd, a2h + 2 * ks, b2h + 2 * ks, id_s, ks != 0);
                        if (p.b1_lo) mma_bf16(cs, a1h + 2 * ks, b1l + 2 * ks, id_s, 1);
                        if (p.a1_lo) mma_bf16(cs, a1l + 2 * ks, b1h + 2 * ks, id_s, 1);
                        if (p.b2_lo) mma_bf16(cd, a2h + 2 * ks, b2l + 2 * ks, id_s, 1);
                        if (p.a2_lo) mma_bf16(cd, a2l + 2 * ks, b2h + 2 * ks, id_s, 1);
                    }
                    mma_commit(&sm.s_full[g & 1]);
                    if (last) mma_commit(&sm.own_empty[ob]);
                }
                __syncwarp();
            };
            issue_S(gc, nch == 1);
            for (int c = 0; c < nch; ++c, ++gc) {
                if (c + 1 < nch) issue_S(gc + 1, c + 1 == nch - 1);
                const int st = gc % NS, xb = gc & 1;
                mbar_wait(&sm.p_full[xb], (uint32_t)((gc >> 1) & 1));
                // the first chunk of an item overwrites the accumulators the previous item's
                // epilogue reads
                if (c == 0 && ic > 0) mbar_wait(&sm.acc_free, (uint32_t)((ic - 1) & 1));
                tc_fence_after();
                const uint64_t a1h = kd(plane(st, 0)), a1l = kd(plane(st, 1));
                const uint64_t a2h = kd(plane(st, 2)), a2l = kd(plane(st, 3));
                const uint64_t xh = nd(sm.bx[xb][0]), xl = nd(sm.bx[xb][1]), yh = nd(sm.bx[xb][2]), yl = nd(sm.bx[xb][3]);
                if (elect_one()) {
                    for (int ks = 0; ks < 8; ++ks) {
                        const uint32_t acc = (c | ks) != 0;
                        const uint64_t ko = 128 * ks, bo = 16 * ks;
                        // dQ^T (or dK^T) += A1^T X, X = dS^T (or dS arranged [key][query])
                        mma_bf16(tmem + C_O1, a1h + ko, xh + bo, id_o, acc);
                        mma_bf16(tmem + C_O1, a1h + ko, xl + bo, id_o, 1);
                        if (p.a1_lo) mma_bf16(tmem + C_O1, a1l + ko, xh + bo, id_o, 1);
                        if (KEYSIDE) {
                            // dV^T += A2^T Y, Y = P arranged [key][query]
                            mma_bf16(tmem + C_O2, a2h + ko, yh + bo, id_o, acc);
                            mma_bf16(tmem + C_O2, a2h + ko, yl + bo, id_o, 1);
                            if (p.a2_lo) mma_bf16(tmem + C_O2, a2l + ko, yh + bo, id_o, 1);
                        }
                    }
                    mma_commit(&sm.empty[st]);
                    mma_commit(&sm.o_done[xb]);
                }
                __syncwarp();
            }
            ++ic;
        }
    } else {
        // ===================== gathered rows: P, dS, epilogue =====================
        const int r = 32 * warp + lane;  // gathered row of the chunk = TMEM lane
        const uint32_t lb = tmem + ((uint32_t)(32 * warp) << 16);
        const float2 c2v = make_float2(p.c2, p.c2), scv = make_float2(p.scale, p.scale), m1 = make_float2(-1.0f, -1.0f);
        int gc = 0, ic = 0;
        Off on = offs(blockIdx.x);
        for (int64_t item = blockIdx.x; item < p.rows; item += G) {
            const Off oc = on;
            on = offs(item + G);
            const int h = (int)(item / L.windows), w = (int)(item - (int64_t)h * L.windows);
            const int64_t beg = oc.b;
            const int nwin = (int)(oc.e - oc.b);
            const int nch = (nwin + 7) / 8;
            if (nch == 0) continue;
            const int sb = ic & 1;
            if (!KEYSIDE) {
                if (r < 16) {
                    const int t = L.member(w, r);
                    sm.own_lse[sb][r] = -p.lse[(int64_t)h * L.image_tokens + t] * 1.4426950408889634f;
                    sm.own_D[sb][r] = -p.D[(int64_t)h * L.image_tokens + t];
                }
                named_bar_sync(1, 128);
            }
            // gathered rows' statistics (dK/dV pass), one chunk ahead
            auto gstats = [&](int c, float& l2, float& dg) {
                l2 = 0.0f;
                dg = 0.0f;
                if (c < nch && r < min(8, nwin - 8 * c) * 16) {
                    const int t = L.member(p.ids[beg + 8 * c + (r >> 4)], r & 15);
                    l2 = p.lse[(int64_t)h * L.image_tokens + t] * 1.4426950408889634f;
                    dg = p.D[(int64_t)h * L.image_tokens + t];
                }
            };
            float nl2 = 0.0f, nD = 0.0f;
            if (KEYSIDE) gstats(0, nl2, nD);
            for (int c = 0; c < nch; ++c, ++gc) {
                const int nc = min(8, nwin - 8 * c);
                const bool valid = r < nc * 16;
                const float lse2 = nl2, Dg = nD;
                if (KEYSIDE) gstats(c + 1, nl2, nD);
                const int xb = gc & 1;
                mbar_wait(&sm.s_full[xb], (uint32_t)((gc >> 1) & 1));
                __syncwarp();
                tc_fence_after();
                uint32_t sv[16], dv[16];
                tmem_ld_32x32b_x16(lb + C_S + C_BUF * xb, sv);
                tmem_ld_32x32b_x16(lb + C_DP + C_BUF * xb, dv);
                tmem_wait_ld();
                // the output MMAs of chunk gc - 2 read this X / Y buffer: wait before overwriting
                if (gc >= 2) mbar_wait(&sm.o_done[xb], (uint32_t)(((gc - 2) >> 1) & 1));
#pragma unroll
                for (int n2 = 0; n2 < 8; ++n2) {
                    // pairs of own rows on the packed f32x2 pipe (the statistics stored negated)
                    const float2 nl = KEYSIDE ? make_float2(-lse2, -lse2)
                                              : *reinterpret_cast<const float2*>(&sm.own_lse[sb][2 * n2]);
                    const float2 nd = KEYSIDE ? make_float2(-Dg, -Dg)
                                              : *reinterpret_cast<const float2*>(&sm.own_D[sb][2 * n2]);
                    float2 pv = make_float2(0.0f, 0.0f), dsv = pv;
                    if (valid) {
                        const float2 a2 = __ffma2_rn(make_float2(__uint_as_float(sv[2 * n2]), __uint_as_float(sv[2 * n2 + 1])),
                                                     c2v, nl);
                        pv = make_float2(ex2_approx(a2.x), ex2_approx(a2.y));
                        const float2 t2 =
                            __fadd2_rn(make_float2(__uint_as_float(dv[2 * n2]), __uint_as_float(dv[2 * n2 + 1])), nd);
                        dsv = __fmul2_rn(__fmul2_rn(pv, t2), scv);
                    }
                    const __nv_bfloat162 dh = __float22bfloat162_rn(dsv);
                    const __nv_bfloat162 dl = __float22bfloat162_rn(__ffma2_rn(__bfloat1622float2(dh), m1, dsv));
                    const uint32_t o0 = bx_off(2 * n2, r), o1 = bx_off(2 * n2 + 1, r);
                    *reinterpret_cast<__nv_bfloat16*>(sm.bx[xb][0] + o0) = dh.x;
                    *reinterpret_cast<__nv_bfloat16*>(sm.bx[xb][0] + o1) = dh.y;
                    *reinterpret_cast<__nv_bfloat16*>(sm.bx[xb][1] + o0) = dl.x;
                    *reinterpret_cast<__nv_bfloat16*>(sm.bx[xb][1] + o1) = dl.y;
                    if (KEYSIDE) {
                        const __nv_bfloat162 ph = __float22bfloat162_rn(pv);
                        const __nv_bfloat162 pl = __float22bfloat162_rn(__ffma2_rn(__bfloat1622float2(ph), m1, pv));
                        *reinterpret_cast<__nv_bfloat16*>(sm.bx[xb][2] + o0) = ph.x;
                        *reinterpret_cast<__nv_bfloat16*>(sm.bx[xb][2] + o1) = ph.y;
                        *reinterpret_cast<__nv_bfloat16*>(sm.bx[xb][3] + o0) = pl.x;
                        *reinterpret_cast<__nv_bfloat16*>(sm.bx[xb][3] + o1) = pl.y;
                    }
                }
                fence_proxy_async_smem();
                tc_fence_before();
                mbar_arrive(&sm.p_full[xb]);
            }
            // ------------------------------- epilogue -------------------------------
            mbar_wait(&sm.o_done[(gc - 1) & 1], (uint32_t)(((gc - 1) >> 1) & 1));
            __syncwarp();
            tc_fence_after();
            uint32_t o1[16], o2[16];
            tmem_ld_32x32b_x16(lb + C_O1, o1);
            if (KEYSIDE) tmem_ld_32x32b_x16(lb + C_O2, o2);
            tmem_wait_ld();
            tc_fence_before();
            mbar_arrive(&sm.acc_free);
            if (lane < 16) {  // M = 64: feature 16 warp + lane lives in lane `lane` of warp `warp`
                // the window's 16 rows: all loads first, then the stores (no load waits on a
                // store to a row the compiler cannot prove distinct)
                const int f = 16 * warp + lane;
                const int64_t t0 = L.num_special + L.member(w, 0);
                float* b1 = p.o1 + (int64_t)h * p.o1_hs + f;
                float* b2 = KEYSIDE ? p.o2 + (int64_t)h * p.o2_hs + f : nullptr;
                float x1[16], x2[16];
#pragma unroll
                for (int n = 0; n < 16; ++n) {
                    const int64_t t = t0 + (n >> 2) * L.grid_w + (n & 3);  // member n of the window
                    x1[n] = b1[t * p.o1_rs];
                    if (KEYSIDE) x2[n] = b2[t * p.o2_rs];
                }
#pragma unroll
                for (int n = 0; n < 16; ++n) {
                    const int64_t t = t0 + (n >> 2) * L.grid_w + (n & 3);
                    b1[t * p.o1_rs] = x1[n] + __uint_as_float(o1[n]);
                    if (KEYSIDE) b2[t * p.o2_rs] = x2[n] + __uint_as_float(o2[n]);
                }
            }
            ++ic;
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 5) {
        tc_fence_after();
        tmem_dealloc(tmem, SB_COLS);
    }
}

// [H][rows][64] bf16 image rows (strides in elements) as windows: box 64 x 4 x 4 (one window)
bool make_win_map(CUtensorMap* m, const void* base, int64_t hs, int64_t rs, int heads, const DevLayout& L) {
    TmapEncodeFn enc = tmap_encode_fn();
    if (!enc) return false;
    cuuint64_t dims[4] = {64, (cuuint64_t)L.grid_w, (cuuint64_t)L.grid_h * L.num_frames, (cuuint64_t)heads};
    cuuint64_t strides[3] = {(cuuint64_t)rs * 2, (cuuint64_t)L.grid_w * rs * 2, (cuuint64_t)hs * 2};
    cuuint32_t box[4] = {64, 4, 4, 1};
    cuuint32_t es[4] = {1, 1, 1, 1};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(base), dims, strides, box, es,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace

bool tc_sel_bwd_supported(int dim, int s) { return dim == 64 && s == 4 && tmap_encode_fn() != nullptr; }

cudaError_t launch_sel_bwd_tc(const SelBwdTcArgs& a, cudaStream_t st) {
    const DevLayout& L = a.L;
    const int64_t rows = (int64_t)a.heads * L.windows;
    if (rows == 0) return cudaSuccess;
    CUtensorMap q_h, q_l, k_h, k_l, v_h, v_l, d_h, d_l;
    auto mk = [&](CUtensorMap* m, const BwdPlane& pl) {
        return make_win_map(m, pl.p ? pl.p : a.q_hi.p, pl.p ? pl.hs : a.q_hi.hs, pl.p ? pl.rs : a.q_hi.rs, a.heads, L);
    };
    if (!mk(&q_h, a.q_hi) || !mk(&q_l, a.q_lo) || !mk(&k_h, a.k_hi) || !mk(&k_l, a.k_lo) || !mk(&v_h, a.v_hi) ||
        !mk(&v_l, a.v_lo) || !mk(&d_h, a.ds_hi) || !mk(&d_l, a.ds_lo))
        return cudaErrorNotSupported;
    const size_t smem = sizeof(SbSmem) + 1024;
    cudaError_t e = cudaFuncSetAttribute(sel_bwd_tc_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(sel_bwd_tc_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    const bool qkv_lo = a.k_lo.p != nullptr;  // f32 Q / K / V carry lo planes (dS always does)
    SbParams p{};
    p.L = L;
    p.heads = a.heads;
    p.rows = rows;
    p.scale = a.scale;
    p.c2 = a.scale * 1.4426950408889634f;
    p.lse = a.lse;
    p.D = a.D;
    // dQ pass: gathered K / V (plan rows), own Q / dS_sel
    p.a1_lo = p.a2_lo = p.b1_lo = qkv_lo;
    p.b2_lo = true;
    p.offsets = a.offsets;
    p.ids = a.ids;
    p.o1 = a.dq;
    p.o1_hs = a.dq_hs;
    p.o1_rs = a.dq_rs;
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const unsigned grid = (unsigned)std::min<int64_t>(rows, sms);  // persistent: one CTA per SM
    sel_bwd_tc_kernel<false><<<grid, SB_THREADS, smem, st>>>(k_h, k_l, v_h, v_l, q_h, q_l, d_h, d_l, p);
    note_launch();
    // dK / dV pass: gathered Q / dS_sel (inverse plan rows), own K / V
    p.a1_lo = p.b1_lo = p.b2_lo = qkv_lo;
    p.a2_lo = true;
    p.offsets = a.inv_offsets;
    p.ids = a.inv_q;
    p.o1 = a.dk;
    p.o1_hs = a.dk_hs;
    p.o1_rs = a.dk_rs;
    p.o2 = a.dv;
    p.o2_hs = a.dv_hs;
    p.o2_rs = a.dv_rs;
    sel_bwd_tc_kernel<true><<<grid, SB_THREADS, smem, st>>>(q_h, q_l, d_h, d_l, k_h, k_l, v_h, v_l, p);
    note_launch();
    return cudaGetLastError();
}

}  // namespace gsa_sm100
