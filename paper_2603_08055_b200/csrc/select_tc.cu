// select_tc.cu — K4: block-sparse selection attention fused with the gate and
// the gated merge, on tcgen05 tensor cores with TMA gathers (sm_100a).
//
// Reference: block_sparse_attention (selection.hpp:63-136), gate
// (layer.hpp:99-119), assemble_image_output (layer.hpp:154-170).
//
// One work item = (head h, query window w): its 16 queries attend the 16 keys
// of every window in the plan row (forced ++ top-k). Persistent CTAs (two per
// SM) walk the items head-major; inside a CTA the items' key windows form one
// global stream of "groups" (<= GROUP_WIN = 16 windows = 256 keys each):
//
//   warp 0 (TMA)   : gathers each selected window of K (bf16, straight from the
//                    head-major [H][M][64] tensor) and of V (the layer's fp16 V16
//                    planes: v * 2^-e_h per head, exact for bf16) with a 4-D tensor
//                    map (box 64 x 4 x 4 = one 2 KB window, 128B-swizzled), 8
//                    windows per 16 KB stage of a 4-stage ring; Q tile per item;
//                    W_g (hi/lo bf16 split, pre-swizzled) per head.
//   warp 1 (MMA)   : S^T[128 keys x 16 q] = K_chunk . Q^T   (M=128, N=16, K=64)
//                    G^T[64 x 16]        = W_g^T . Q^T       (hi + lo, M=64)
//                    O^T[64 x 16]       += V16_chunk^T . P16^T (fp16, M=64, K=16/step)
//                    accumulators in TMEM; S double-buffered across groups so
//                    S(j+1) overlaps the softmax of group j.
//   warps 2-5      : exact two-phase softmax over the whole group (keys are the
//                    TMEM lanes: reductions = in-thread + 3 shuffles + 4-warp
//                    smem), P written as fp16 with stmatrix.trans straight into
//                    the K-major B-operand layout; online rescale across groups
//                    (long or hybrid rows); epilogue g = sigmoid(z),
//                    out = g*O_comp[w] + (1-g)*2^e_h*O_sel in f32.
// Modes: without W_g the plain block_sparse_attention operator (out = O_sel, any CSR
// plan); `split`: f32 inputs as bf16 hi/lo Q, K and fp16 hi/lo V planes (3-term S and
// G, 2-term P.V), each window gathered into two consecutive ring stages.
//
// HBM/L2-gather bound on iid inputs: 4 KB of K+V per selected window for
// 65536 MACs (16 flop/B), see DESIGN.md.
#include <cuda.h>

#include <cstdio>
#include <cstdlib>

#include "tc.h"
#include "tc_ptx.cuh"

namespace gsa_sm100 {
namespace {

using namespace ptx;


// Two CTAs per SM (SEL_CTAS): the per-item chain (gather -> S -> softmax -> PV ->
// epilogue) is latency-bound with one consumer warpgroup, so a second CTA hides it.
// That caps shared memory at ~113 KB per CTA: 256-key groups (SEL_GROUP_WIN 16, so
// P^T buffers are 32 KB) and a 3-stage ring. Measured at V=1000 (select stage):
// 1 CTA, 512-key groups, 8 stages 53 ms; 2 CTAs, 16-window groups, 3 stages 33 ms;
// 2 CTAs with 8-window groups 42 ms.
#ifndef SEL_NS
#define SEL_NS 4
#endif
#ifndef SEL_CTAS
#define SEL_CTAS 2
#endif
#ifndef SEL_GROUP_WIN
#define SEL_GROUP_WIN 16
#endif
constexpr int NS = SEL_NS;               // ring stages
constexpr int STAGE = 16384;             // 8 windows x 2 KB
constexpr int WIN = 2048;                // 16 tokens x 64 bf16
constexpr int NTHREADS = 192;
constexpr int NGB = 3;  // G^T buffers: item j+1's G MMA must not wait for item j-1's epilogue
constexpr int GROUP_WIN = SEL_GROUP_WIN;  // windows per softmax group (<= 32, 16 keys each)
constexpr int P_QSTRIDE = GROUP_WIN * 256; // bytes per 8-query half of a P^T buffer
// TMEM: two S^T buffers (16 columns per 8-window chunk of the group), two O^T, NGB G^T
constexpr uint32_t S_COLS = (GROUP_WIN / 8) * 16;
constexpr uint32_t S_COL0 = 0, S_COL1 = S_COLS, O_COL0 = 2 * S_COLS, O_COL1 = O_COL0 + 16, G_COL0 = O_COL1 + 16;
constexpr uint32_t TMEM_COLS = (G_COL0 + 16 * NGB <= 128) ? 128 : 256;  // power of two >= the layout
#ifndef SEL_L2HINT
#define SEL_L2HINT 0  // 1: K/V gathers evict_last, query tiles evict_first, outputs st.cs (measured neutral at V=1000)
#endif
#ifndef SEL_PF
#define SEL_PF 0
#endif
constexpr int PREFETCH_AHEAD = SEL_PF;  // items of L2 prefetch ahead of the gathers (measured slower: 1 CTA/SM 54 -> 71 ms; 2 CTAs/SM 34 -> 47 ms)

struct __align__(1024) SelSmem {
    uint8_t ring[NS][STAGE];
    uint8_t q[2][WIN];
    uint8_t ql[2][WIN];       // split mode: the query tile's bf16 lo plane
    uint8_t wg[2][8192];      // W_g hi / lo, [a][j] 128B-swizzled
    uint8_t p[2][2 * P_QSTRIDE];  // [group parity] P^T fp16: [q-group 2][key-chunk][8 rows][16 B]
    float red[2][4][16];      // cross-warp max / sum partials
    float run_m[2][16];       // [group parity] running row max (raw score units)
    float run_l[2][16];       // [group parity] running denominator
    float alpha[2][16];       // [group parity] rescale of the previous groups' accumulator
    uint64_t full[NS], empty[NS];
    uint64_t q_full[2], q_empty[2];
    uint64_t wg_full, wg_empty;
    uint64_t s_full[2], s_empty[2];
    uint64_t p_full[2], o_full[2];
    uint64_t g_empty[NGB];
    uint32_t tmem_base;
};

// n / d for n, d < 2^31 by a multiply-high (Granlund-Montgomery): the per-window and
// per-item index math runs on every gathered window, where a hardware-less integer
// division costs ~20 instructions
struct FastDiv {
    uint32_t d, m, s;
    void init(uint32_t dd) {
        d = dd;
        s = 0;
        while ((1u << s) < d) ++s;
        m = (uint32_t)(((uint64_t(1) << 32) * ((uint64_t(1) << s) - d)) / d + 1);
    }
    __device__ __forceinline__ uint32_t div(uint32_t n) const { return (__umulhi(n, m) + n) >> s; }
};

struct SelTcParams {
    int heads;
    FastDiv fd_windows, fd_wpf, fd_ww;  // L.windows (item -> head), L.wins_per_frame, L.wins_w
    DevLayout L;
    RowSource rows;
    float scale, c2;  // c2 = scale * log2(e)
    int64_t items;
    const float* o_comp;
    float* out;
    int64_t out_hs, out_rs;
    float* lse;
    float* o_sel_ctx;
    float* gate_ctx;
    const float* prior_o;     // hybrid fast path: reference-frame softmax, merged by LSE (or null)
    const float* prior_lse;
    const uint8_t* wg_prep;  // [H][2][8192] bytes
    const unsigned* vmax;    // [H] max |v| (float bits): the V operand is fp16(v * 2^-vexp(vmax))
    // split: f32 Q/K as bf16 hi + lo planes and V as fp16 hi + lo planes (every window
    // gathered twice, into two consecutive ring stages); S = Kh.Qh + Kl.Qh + Kh.Ql,
    // O += Vh.P + Vl.P,
    // G = Wgh.Qh + Wgl.Qh + Wgh.Ql. gate: fused gate + merge (else out = o_sel)
    bool split, gate;
};

__device__ __forceinline__ int vexp(float vmax) { return vmax > 0.0f ? ilogbf(vmax) - 13 : 0; }

// Iterates this CTA's (item, group) sequence.
struct GroupIt {
    int64_t item;
    int g, ng, nwin;
    __device__ void start(const SelTcParams& p) {
        item = blockIdx.x;
        g = 0;
        load(p);
    }
    __device__ void load(const SelTcParams& p) {
        if (item < p.items) {
            nwin = (int)p.rows.size(item);
            ng = (nwin + GROUP_WIN - 1) / GROUP_WIN;
        } else {
            nwin = ng = 0;
        }
    }
    __device__ bool valid(const SelTcParams& p) const { return item < p.items; }
    __device__ void next(const SelTcParams& p) {
        if (++g >= ng) {
            g = 0;
            item += gridDim.x;
            load(p);
        }
    }
    __device__ int group_windows() const { return min(GROUP_WIN, nwin - g * GROUP_WIN); }
};

__device__ __forceinline__ void window_coords(const DevLayout& L, const SelTcParams& p, int wid, int& c1, int& c2) {
    const int f = (int)p.fd_wpf.div((uint32_t)wid), r = wid - f * L.wins_per_frame;
    const int wr = (int)p.fd_ww.div((uint32_t)r), wc = r - wr * L.wins_w;
    c1 = wc * 4;
    c2 = f * L.grid_h + wr * 4;
}

__global__ void __launch_bounds__(NTHREADS, SEL_CTAS)
    select_tc_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                     const __grid_constant__ CUtensorMap tm_v, const __grid_constant__ CUtensorMap tm_ql,
                     const __grid_constant__ CUtensorMap tm_kl, const __grid_constant__ CUtensorMap tm_vl,
                     const SelTcParams p) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    // keep the shared address space visible to the compiler (LDS/STS, not generic LD/ST)
    SelSmem& sm = *reinterpret_cast<SelSmem*>(smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u));
    const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;

    // ---- setup: zero the operand buffers (slots past a short row stay finite)
    {
        uint4* z0 = reinterpret_cast<uint4*>(&sm.ring[0][0]);
        for (int i = threadIdx.x; i < (int)(sizeof(sm.ring) / 16); i += NTHREADS) z0[i] = make_uint4(0, 0, 0, 0);
        uint4* z1 = reinterpret_cast<uint4*>(&sm.p[0][0]);
        for (int i = threadIdx.x; i < (int)(sizeof(sm.p) / 16); i += NTHREADS) z1[i] = make_uint4(0, 0, 0, 0);
    }
    if (threadIdx.x == 0) {
        for (int i = 0; i < NS; ++i) {
            mbar_init(&sm.full[i], 1);
            mbar_init(&sm.empty[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&sm.q_full[i], 1);
            mbar_init(&sm.q_empty[i], 1);
            mbar_init(&sm.s_full[i], 1);
            mbar_init(&sm.s_empty[i], 128);
            mbar_init(&sm.p_full[i], 128);
            mbar_init(&sm.o_full[i], 1);
        }
        mbar_init(&sm.wg_full, 1);
        mbar_init(&sm.wg_empty, 1);
        for (int i = 0; i < NGB; ++i) mbar_init(&sm.g_empty[i], 128);
        fence_barrier_init();
        prefetch_tmap(&tm_q);
        prefetch_tmap(&tm_k);
        prefetch_tmap(&tm_v);
        if (p.split) {
            prefetch_tmap(&tm_ql);
            prefetch_tmap(&tm_kl);
            prefetch_tmap(&tm_vl);
        }
    }
    if (warp == 1) tmem_alloc(&sm.tmem_base, TMEM_COLS);
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = sm.tmem_base;
    const DevLayout& L = p.L;

    if (warp == 0) {
        // ============================== TMA producer ==============================
        // The whole warp walks the stream: each lane fetches one window id of the
        // group (one coalesced load instead of a serial id chain) and issues that
        // window's TMA; lane 0 arms the stage barrier first.
        int st = 0;
        uint32_t eph = 1;  // empty barriers: first pass succeeds
        const uint64_t pol_last = policy_evict_last(), pol_first = policy_evict_first();
        uint32_t qph[2] = {1, 1};
        int cur_head = -1;
        int n_heads = 0;      // W_g loads issued
        int64_t n_items = 0;  // items whose Q/Wg prelude has been issued
        auto load_chunks = [&](const GroupIt& it, const CUtensorMap* tm, bool with_prelude, int my_wid) {
            const int h = (int)p.fd_windows.div((uint32_t)it.item), w = (int)(it.item - (int64_t)h * L.windows);
            if (with_prelude) {
                if (p.gate && h != cur_head) {
                    // W_g of the new head: wait until every G MMA of the old head completed.
                    // wg_empty completes once per head (after its last item's G MMA), so
                    // this wait and that commit advance in lockstep: a parity wait is exact
                    if (n_heads > 0) mbar_wait(&sm.wg_empty, (uint32_t)((n_heads - 1) & 1));
                    ++n_heads;
                    if (lane == 0) {
                        mbar_arrive_expect_tx(&sm.wg_full, 16384);
                        bulk_load(&sm.wg[0][0], p.wg_prep + (size_t)h * 16384, 16384, &sm.wg_full);
                    }
                    cur_head = h;
                }
                const int qb = (int)(n_items & 1);
                mbar_wait(&sm.q_empty[qb], qph[qb]);
                qph[qb] ^= 1;
                if (lane == 0) {
                    mbar_arrive_expect_tx(&sm.q_full[qb], p.split ? 2 * WIN : WIN);
                    int c1, c2;
                    window_coords(L, p, w, c1, c2);
                    if (SEL_L2HINT) {
                        tma_load_4d_hint(&sm.q[qb][0], &tm_q, &sm.q_full[qb], 0, c1, c2, h, pol_first);
                        if (p.split) tma_load_4d_hint(&sm.ql[qb][0], &tm_ql, &sm.q_full[qb], 0, c1, c2, h, pol_first);
                    } else {
                        tma_load_4d(&sm.q[qb][0], &tm_q, &sm.q_full[qb], 0, c1, c2, h);
                        if (p.split) tma_load_4d(&sm.ql[qb][0], &tm_ql, &sm.q_full[qb], 0, c1, c2, h);
                    }
                }
                ++n_items;
            }
            const int nw = it.group_windows();
            int c1, c2;
            window_coords(L, p, my_wid, c1, c2);
            if (PREFETCH_AHEAD > 0 && tm == &tm_k && it.g == 0) {
                // warm L2 with the K and V windows of the item PREFETCH_AHEAD items ahead: the
                // ring holds about one item, so without this every item pays a DRAM round trip
                const int64_t pi = it.item + (int64_t)PREFETCH_AHEAD * gridDim.x;
                if (pi < p.items) {
                    const int ph = (int)p.fd_windows.div((uint32_t)pi);
                    const int64_t pn = p.rows.size(pi);
                    for (int64_t j = lane; j < pn; j += 32) {
                        int d1, d2;
                        window_coords(L, p, p.rows.window(pi, j), d1, d2);
                        tma_prefetch_4d(&tm_k, 0, d1, d2, ph);
                        tma_prefetch_4d(&tm_v, 0, d1, d2, ph);
                    }
                }
            }
            const CUtensorMap* tml = tm == &tm_k ? &tm_kl : &tm_vl;
            for (int c0 = 0; c0 < nw; c0 += 8) {
                const int nc = min(8, nw - c0);
                for (int part = 0; part < (p.split ? 2 : 1); ++part) {  // split: hi stage, then lo stage
                    mbar_wait(&sm.empty[st], eph);
                    if (lane == 0) mbar_arrive_expect_tx(&sm.full[st], nc * WIN);
                    __syncwarp();
                    if (lane >= c0 && lane < c0 + nc) {
                        if (SEL_L2HINT)
                            tma_load_4d_hint(&sm.ring[st][(lane - c0) * WIN], part ? tml : tm, &sm.full[st], 0, c1, c2, h,
                                             pol_last);
                        else
                            tma_load_4d(&sm.ring[st][(lane - c0) * WIN], part ? tml : tm, &sm.full[st], 0, c1, c2, h);
                    }
                    if (++st == NS) {
                        st = 0;
                        eph ^= 1;
                    }
                }
            }
        };
        // window ids run two groups ahead of the K loads (one lane per window of the
        // group): the index loads' round trip overlaps the gathers instead of preceding them
        GroupIt kit, vit, pit;
        kit.start(p);
        vit.start(p);
        pit.start(p);
        auto ids_of = [&](const GroupIt& g) {
            return (g.valid(p) && lane < g.group_windows()) ? p.rows.window(g.item, (int64_t)g.g * GROUP_WIN + lane) : 0;
        };
        int wid_k = ids_of(pit);  // ids of kit's group
        if (pit.valid(p)) pit.next(p);
        int wid_n = ids_of(pit);  // ids of the group after kit's
        if (pit.valid(p)) pit.next(p);
        auto advance_k = [&]() {
            wid_k = wid_n;
            wid_n = ids_of(pit);
            if (pit.valid(p)) pit.next(p);
        };
        int wid_vq = wid_k;  // ids of vit's current group
        if (kit.valid(p)) {
            load_chunks(kit, &tm_k, true, wid_k);
            kit.next(p);
            wid_vq = wid_k;
            advance_k();
        }
        while (vit.valid(p)) {
            const int wv = wid_vq;
            if (kit.valid(p)) {
                load_chunks(kit, &tm_k, kit.g == 0, wid_k);
                kit.next(p);
                wid_vq = wid_k;
                advance_k();
            }
            load_chunks(vit, &tm_v, false, wv);
            vit.next(p);
        }
    } else if (warp == 1) {
        // ================================ MMA issuer ===============================
        // Stream order: S(0); then per group j: S(j+1) (look-ahead), PV(j). The whole
        // (must match the TMA producer's load order K0, K1, V0, K2, V1, ...).
        // warp walks the stream (uniform descriptors); one elected lane issues.
        {
            const uint32_t id_s = idesc_bf16(128, 16, 0, 0);
            const uint32_t id_o = idesc_bf16(64, 16, 1, 0);   // G^T = Wg^T . Q^T (bf16)
            const uint32_t id_pv = idesc_f16(64, 16, 1, 0);  // O^T += V16^T . P16^T (fp16)
            int st = 0;
            uint32_t fph = 0;
            uint32_t qph[2] = {0, 0}, sph[2] = {1, 1}, pph[2] = {0, 0};
            uint32_t gphase = (1u << NGB) - 1u;  // bit b: parity to wait on g_empty[b] (first use passes)
            uint32_t wgph = 0;
            int cur_head = -1;
            int64_t n_items = 0;
            int64_t jS = 0, jP = 0;  // global group indices of the next S / PV
            auto issue_S = [&](const GroupIt& it) {
                const int h = (int)p.fd_windows.div((uint32_t)it.item);
                const int qb = (int)((n_items - (it.g == 0 ? 0 : 1)) & 1);
                if (it.g == 0) {
                    mbar_wait(&sm.q_full[qb], qph[qb]);
                    qph[qb] ^= 1;
                    if (p.gate && h != cur_head) {
                        mbar_wait(&sm.wg_full, wgph);
                        wgph ^= 1;
                        cur_head = h;
                    }
                    // G^T = Wg^T . Q^T (hi + lo), into the item's G buffer
                    const int gb = (int)(n_items % NGB);
                    if (p.gate) {
                        mbar_wait(&sm.g_empty[gb], (gphase >> gb) & 1u);
                        gphase ^= 1u << gb;
                        tc_fence_after();

                        const uint32_t gcol = tmem + G_COL0 + 16u * (uint32_t)gb;
                        // the last item of this head on this CTA releases W_g
                        const int64_t nxt = it.item + gridDim.x;
                        const bool last_of_head = nxt >= p.items || (int)p.fd_windows.div((uint32_t)nxt) != h;
                        if (elect_one()) {
                            for (int part = 0; part < (p.split ? 3 : 2); ++part)  // Wgh.Qh, Wgl.Qh (, Wgh.Ql)
                                for (int ks = 0; ks < 4; ++ks)
                                    mma_bf16(gcol, umma_desc(smem_u32(&sm.wg[part & 1][0]) + ks * 2048, 16, 1024, 2),
                                             umma_desc(smem_u32(part == 2 ? &sm.ql[qb][0] : &sm.q[qb][0]) + ks * 32, 16,
                                                       1024, 2),
                                             id_o, (part | ks) != 0);
                            if (last_of_head) mma_commit(&sm.wg_empty);
                        }
                        __syncwarp();
                    }
                    ++n_items;
                }
                const int sb = (int)(jS & 1);
                mbar_wait(&sm.s_empty[sb], sph[sb]);
                sph[sb] ^= 1;
                tc_fence_after();
                const int nw = it.group_windows();
                const uint32_t scol = tmem + (sb ? S_COL1 : S_COL0);
                const uint64_t qdesc = umma_desc(smem_u32(&sm.q[qb][0]), 16, 1024, 2);
                const uint64_t qldesc = umma_desc(smem_u32(&sm.ql[qb][0]), 16, 1024, 2);
                for (int c0 = 0, c = 0; c0 < nw; c0 += 8, ++c) {
                    mbar_wait(&sm.full[st], fph);
                    const int st0 = st;
                    if (++st == NS) {
                        st = 0;
                        fph ^= 1;
                    }
                    int st1 = st0;
                    if (p.split) {  // the chunk's lo plane sits in the next stage
                        mbar_wait(&sm.full[st], fph);
                        st1 = st;
                        if (++st == NS) {
                            st = 0;
                            fph ^= 1;
                        }
                    }
                    tc_fence_after();
                    const uint64_t kdesc = umma_desc(smem_u32(&sm.ring[st0][0]), 16, 1024, 2);
                    const uint64_t kldesc = umma_desc(smem_u32(&sm.ring[st1][0]), 16, 1024, 2);
                    if (elect_one()) {
                        for (int ks = 0; ks < 4; ++ks) {
                            mma_bf16(scol + 16 * c, kdesc + (uint64_t)(ks * 2), qdesc + (uint64_t)(ks * 2), id_s,
                                     ks != 0);
                            if (p.split) {
                                mma_bf16(scol + 16 * c, kldesc + (uint64_t)(ks * 2), qdesc + (uint64_t)(ks * 2), id_s, 1);
                                mma_bf16(scol + 16 * c, kdesc + (uint64_t)(ks * 2), qldesc + (uint64_t)(ks * 2), id_s, 1);
                            }
                        }
                        mma_commit(&sm.empty[st0]);
                        if (p.split) mma_commit(&sm.empty[st1]);
                    }
                    __syncwarp();
                }
                if (elect_one()) {
                    mma_commit(&sm.s_full[sb]);
                    if (it.g == it.ng - 1) mma_commit(&sm.q_empty[qb]);
                }
                __syncwarp();
                ++jS;
            };
            auto issue_PV = [&](const GroupIt& it) {
                const int pb = (int)(jP & 1);
                mbar_wait(&sm.p_full[pb], pph[pb]);
                pph[pb] ^= 1;
                tc_fence_after();
                const int nw = it.group_windows();
                const uint32_t ocol = tmem + (pb ? O_COL1 : O_COL0);
                const uint64_t pdesc = umma_desc(smem_u32(&sm.p[pb][0]), 128, P_QSTRIDE, 0);
                for (int c0 = 0, c = 0; c0 < nw; c0 += 8, ++c) {
                    mbar_wait(&sm.full[st], fph);
                    const int st0 = st;
                    if (++st == NS) {
                        st = 0;
                        fph ^= 1;
                    }
                    int st1 = st0;
                    if (p.split) {
                        mbar_wait(&sm.full[st], fph);
                        st1 = st;
                        if (++st == NS) {
                            st = 0;
                            fph ^= 1;
                        }
                    }
                    tc_fence_after();
                    const uint64_t vdesc = umma_desc(smem_u32(&sm.ring[st0][0]), 16, 1024, 2);
                    const uint64_t vldesc = umma_desc(smem_u32(&sm.ring[st1][0]), 16, 1024, 2);
                    // descriptor start addresses are in 16-byte units
                    if (elect_one()) {
                        for (int ks = 0; ks < 8; ++ks) {
                            const uint64_t va = vdesc + (uint64_t)(ks * 128);
                            const uint64_t po = (uint64_t)(c * 128 + ks * 16);
                            mma_bf16(ocol, va, pdesc + po, id_pv, (c | ks) != 0);
                            if (p.split) mma_bf16(ocol, vldesc + (uint64_t)(ks * 128), pdesc + po, id_pv, 1);
                        }
                        mma_commit(&sm.empty[st0]);
                        if (p.split) mma_commit(&sm.empty[st1]);
                    }
                    __syncwarp();
                }
                if (elect_one()) mma_commit(&sm.o_full[pb]);
                __syncwarp();
                ++jP;
            };
            GroupIt kit, vit;
            kit.start(p);
            vit.start(p);
            if (kit.valid(p)) {
                issue_S(kit);
                kit.next(p);
            }
            while (vit.valid(p)) {
                if (kit.valid(p)) {
                    issue_S(kit);
                    kit.next(p);
                }
                issue_PV(vit);
                vit.next(p);
            }
        }
    } else {
        // ======================= softmax + epilogue (warps 2..5) ====================
        // Software-pipelined by one group: softmax(j) runs while the tensor core
        // computes PV(j-1); then finish(j-1) folds O(j-1) into the accumulator
        // and, at the end of an item, writes the gated output.
        const int ws = warp - 2;        // 0..3 (reduction slot)
        const int qd = warp & 3;        // TMEM lane quadrant this warp may access
        const int t0 = lane & 3, t1 = lane >> 2;
        const bool stat_owner = (ws == 0 && t1 == 0);  // 4 threads x 4 query slots = 16 queries
        float acc[16];
        uint32_t sph[2] = {0, 0}, oph[2] = {0, 0};
        int64_t j = 0, n_fin_items = 0, n_started = 0;
        float comp_pf0 = 0.0f, comp_pf1 = 0.0f;  // o_comp rows of the items in flight, loaded when an item starts
        GroupIt it, fin;
        it.start(p);
        fin.start(p);

#ifdef SELECT_PROF
        const bool prof_on = blockIdx.x == 0 && threadIdx.x == 64;
        unsigned long long pt[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0}, c0 = clock64(), c1;
#endif
        auto finish = [&](const GroupIt& f, int64_t jf) {
            const int fb = (int)(jf & 1);
            // the compressed-branch row this item merges with: issued before the PV wait
            // so its global-load latency overlaps it
            mbar_wait(&sm.o_full[fb], oph[fb]);
            oph[fb] ^= 1;
#ifdef SELECT_PROF
            if (prof_on) { c1 = clock64(); pt[9] += c1 - c0; c0 = c1; }
#endif
            __syncwarp();
            tc_fence_after();
            uint32_t orr[16];
            tmem_ld_32x32b_x16(tmem + ((uint32_t)(32 * qd) << 16) + (fb ? O_COL1 : O_COL0), orr);
            tmem_wait_ld();
            if (f.g == 0) {
#pragma unroll
                for (int q = 0; q < 16; ++q) acc[q] = __uint_as_float(orr[q]);
            } else {
#pragma unroll
                for (int q = 0; q < 16; ++q) acc[q] = fmaf(acc[q], sm.alpha[fb][q], __uint_as_float(orr[q]));
            }
            if (f.g != f.ng - 1) return;
            // ------------------------------- epilogue -------------------------------
            const int gb = (int)(n_fin_items % NGB);
            uint32_t grr[16];
            if (p.gate) {
                tmem_ld_32x32b_x16(tmem + ((uint32_t)(32 * qd) << 16) + G_COL0 + 16u * (uint32_t)gb, grr);
                tmem_wait_ld();
                tc_fence_before();
                mbar_arrive(&sm.g_empty[gb]);
            } else {
#pragma unroll
                for (int q = 0; q < 16; ++q) grr[q] = 0u;
            }
            ++n_fin_items;
            // lanes 0-15 hold feature 16*qd+lane for all 16 queries; lanes 16-31 take
            // queries 8..15 of lane-16 so every lane writes 8 outputs
            const int hi_half = lane >> 4;
            float a8[8], z8[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const float a_hi = __shfl_sync(0xffffffffu, acc[i + 8], lane & 15);
                const float z_hi = __shfl_sync(0xffffffffu, __uint_as_float(grr[i + 8]), lane & 15);
                a8[i] = hi_half ? a_hi : acc[i];
                z8[i] = hi_half ? z_hi : __uint_as_float(grr[i]);
            }
            const int h = (int)p.fd_windows.div((uint32_t)f.item), w = (int)(f.item - (int64_t)h * L.windows);
            const int jf_feat = 16 * qd + (lane & 15);
            const float comp = ((n_fin_items - 1) & 1) ? comp_pf1 : comp_pf0;
            const float vscale = ldexpf(1.0f, vexp(__uint_as_float(p.vmax[h])));  // undo the V16 scaling
            const int fr = (int)p.fd_wpf.div((uint32_t)w), rr = w - fr * L.wins_per_frame;
            const int wr = (int)p.fd_ww.div((uint32_t)rr), wc = rr - wr * L.wins_w;
            const int tok0 = fr * L.tokens_per_frame + wr * 4 * L.grid_w + wc * 4;
            float* outh = p.out + (int64_t)h * p.out_hs;
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const int q = i + 8 * hi_half;
                const int tok = tok0 + (q >> 2) * L.grid_w + (q & 3);
                float sel = a8[i] * __fdividef(vscale, sm.run_l[fb][q]);
                if (p.prior_o) {  // merge with the reference-frame partial softmax (LSE weights)
                    const int64_t ti = (int64_t)h * L.image_tokens + tok;
                    const float l1 = p.prior_lse[ti];
                    const float l2 = sm.run_m[fb][q] * p.scale + logf(sm.run_l[fb][q]);
                    const float mm = fmaxf(l1, l2);
                    const float w1 = __expf(l1 - mm), w2 = __expf(l2 - mm);
                    sel = (w1 * p.prior_o[ti * 64 + jf_feat] + w2 * sel) / (w1 + w2);
                }
                const float g = __fdividef(1.0f, 1.0f + __expf(-z8[i]));
                const float ov = p.gate ? g * comp + (1.0f - g) * sel : sel;
                if (SEL_L2HINT)
                    __stcs(outh + (int64_t)tok * p.out_rs + jf_feat, ov);  // streamed: keep L2 for the K/V gathers
                else
                    outh[(int64_t)tok * p.out_rs + jf_feat] = ov;
                if (p.o_sel_ctx || p.gate_ctx) {
                    const int64_t ti = (int64_t)h * L.image_tokens + tok;
                    if (p.o_sel_ctx) p.o_sel_ctx[ti * 64 + jf_feat] = sel;
                    if (p.gate_ctx) p.gate_ctx[ti * 64 + jf_feat] = g;
                }
            }
            if (p.lse && ws == 0 && lane < 16) {
                const int tok = tok0 + (lane >> 2) * L.grid_w + (lane & 3);
                float lse = sm.run_m[fb][lane] * p.scale + logf(sm.run_l[fb][lane]);
                if (p.prior_o) {
                    const float l1 = p.prior_lse[(int64_t)h * L.image_tokens + tok], mm = fmaxf(l1, lse);
                    lse = mm + logf(__expf(l1 - mm) + __expf(lse - mm));
                }
                p.lse[(int64_t)h * L.image_tokens + tok] = lse;
            }
        };

        while (it.valid(p)) {
            const int sb = (int)(j & 1);
            const int nkeys = it.group_windows() * 16;
            if (it.g == 0 && p.gate) {  // the compressed-branch row this item merges with, a full item ahead
                // o_comp is [H][W][64] with W = L.windows: row = item
                const float cv = __ldg(p.o_comp + it.item * 64 + 16 * qd + (lane & 15));
                if (n_started & 1) comp_pf1 = cv;
                else comp_pf0 = cv;
                ++n_started;
            }
            mbar_wait(&sm.s_full[sb], sph[sb]);
#ifdef SELECT_PROF
            if (prof_on) { c1 = clock64(); pt[0] += c1 - c0; c0 = c1; }
#endif
            sph[sb] ^= 1;
            __syncwarp();
            tc_fence_after();
            float s[4][2][8];
            const uint32_t scol = tmem + (sb ? S_COL1 : S_COL0);
#pragma unroll
            for (int c = 0; c < 4; ++c)
#pragma unroll
                for (int hf = 0; hf < 2; ++hf) {
                    uint32_t r[8];
                    if (c * 128 < nkeys) {
                        tmem_ld_16x256b_x2(scol + ((uint32_t)(32 * qd + 16 * hf) << 16) + 16 * c, r);
                    } else {
#pragma unroll
                        for (int e = 0; e < 8; ++e) r[e] = 0u;
                    }
#pragma unroll
                    for (int e = 0; e < 8; ++e) s[c][hf][e] = __uint_as_float(r[e]);
                }
            tmem_wait_ld();
#ifdef SELECT_PROF
            if (prof_on) { c1 = clock64(); pt[1] += c1 - c0; c0 = c1; }
#endif
            tc_fence_before();
            mbar_arrive(&sm.s_empty[sb]);
            // mask keys past the row end; key of s[c][hf][e] = 128c + 32qd + 16hf + t1 + 8*((e>>1)&1)
            float mx[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
            for (int c = 0; c < 4; ++c)
#pragma unroll
                for (int hf = 0; hf < 2; ++hf)
#pragma unroll
                    for (int e = 0; e < 8; ++e) {
                        const int key = 128 * c + 32 * qd + 16 * hf + t1 + 8 * ((e >> 1) & 1);
                        if (nkeys < GROUP_WIN * 16 && key >= nkeys) s[c][hf][e] = -INFINITY;
                        const int slot = (e & 1) | ((e >> 2) << 1);  // query 2*t0 + (e&1) + 8*(e>>2)
                        mx[slot] = fmaxf(mx[slot], s[c][hf][e]);
                    }
#pragma unroll
            for (int sl = 0; sl < 4; ++sl) {
                mx[sl] = fmaxf(mx[sl], __shfl_xor_sync(0xffffffffu, mx[sl], 4));
                mx[sl] = fmaxf(mx[sl], __shfl_xor_sync(0xffffffffu, mx[sl], 8));
                mx[sl] = fmaxf(mx[sl], __shfl_xor_sync(0xffffffffu, mx[sl], 16));
            }
            if (t1 == 0) {
#pragma unroll
                for (int sl = 0; sl < 4; ++sl) sm.red[0][ws][2 * t0 + (sl & 1) + 8 * (sl >> 1)] = mx[sl];
            }
            named_bar_sync(1, 128);
#ifdef SELECT_PROF
            if (prof_on) { c1 = clock64(); pt[2] += c1 - c0; c0 = c1; }
#endif
            const int pb = sb;           // this group's statistics / P buffers
            const int ob = sb ^ 1;       // previous group's
            float mq[4], al[4];
#pragma unroll
            for (int sl = 0; sl < 4; ++sl) {
                const int q = 2 * t0 + (sl & 1) + 8 * (sl >> 1);
                const float gm = fmaxf(fmaxf(sm.red[0][0][q], sm.red[0][1][q]), fmaxf(sm.red[0][2][q], sm.red[0][3][q]));
                const float mold = it.g == 0 ? -INFINITY : sm.run_m[ob][q];
                const float mnew = fmaxf(mold, gm);
                al[sl] = mold == -INFINITY ? 0.0f : ex2_approx((mold - mnew) * p.c2);
                mq[sl] = mnew * p.c2;
                if (stat_owner) {
                    sm.run_m[pb][q] = mnew;
                    sm.alpha[pb][q] = al[sl];
                }
            }
            float sum[4] = {0.f, 0.f, 0.f, 0.f};
            // P = exp(scale*(s - m)); stored as fp16 through stmatrix.trans
            const uint32_t pbase = smem_u32(&sm.p[pb][0]);
            const int mi = lane >> 3, rr = lane & 7;
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                if (c * 128 >= nkeys) continue;  // (continue keeps the unroll static)
#pragma unroll
                for (int hf = 0; hf < 2; ++hf) {
                    float pv[8];
#pragma unroll
                    for (int e = 0; e < 8; ++e) {
                        const int slot = (e & 1) | ((e >> 2) << 1);
                        // masked keys are -inf: ex2(-inf) = +0
                        pv[e] = ex2_approx(fmaf(s[c][hf][e], p.c2, -mq[slot]));
                        sum[slot] += pv[e];
                    }
                    uint32_t p16[4];
#pragma unroll
                    for (int e2 = 0; e2 < 4; ++e2) p16[e2] = pack_f16(pv[2 * e2], pv[2 * e2 + 1]);
                    // matrix mi: keys +8*(mi&1), queries 8*(mi>>1); memory row rr = query
                    const int kc = (128 * c + 32 * qd + 16 * hf) / 8 + (mi & 1);
                    const uint32_t off = (uint32_t)((mi >> 1) * P_QSTRIDE + kc * 128 + rr * 16);
                    stmatrix_x4_trans(pbase + off, p16[0], p16[1], p16[2], p16[3]);
                }
            }
#ifdef SELECT_PROF
            if (prof_on) { c1 = clock64(); pt[3] += c1 - c0; c0 = c1; }
#endif
            fence_proxy_async_smem();
            mbar_arrive(&sm.p_full[pb]);
#ifdef SELECT_PROF
            if (prof_on) { c1 = clock64(); pt[4] += c1 - c0; c0 = c1; }
#endif
#pragma unroll
            for (int sl = 0; sl < 4; ++sl) {
                sum[sl] += __shfl_xor_sync(0xffffffffu, sum[sl], 4);
                sum[sl] += __shfl_xor_sync(0xffffffffu, sum[sl], 8);
                sum[sl] += __shfl_xor_sync(0xffffffffu, sum[sl], 16);
            }
            if (t1 == 0) {
#pragma unroll
                for (int sl = 0; sl < 4; ++sl) sm.red[1][ws][2 * t0 + (sl & 1) + 8 * (sl >> 1)] = sum[sl];
            }
            named_bar_sync(1, 128);
#ifdef SELECT_PROF
            if (prof_on) { c1 = clock64(); pt[5] += c1 - c0; c0 = c1; }
#endif
            if (stat_owner) {
#pragma unroll
                for (int sl = 0; sl < 4; ++sl) {
                    const int q = 2 * t0 + (sl & 1) + 8 * (sl >> 1);
                    const float gs = (sm.red[1][0][q] + sm.red[1][1][q]) + (sm.red[1][2][q] + sm.red[1][3][q]);
                    const float lold = it.g == 0 ? 0.0f : sm.run_l[ob][q];
                    sm.run_l[pb][q] = lold * al[sl] + gs;
                }
            }
            // fold in the previous group's PV (computed while this softmax ran)
            if (j > 0) {
                finish(fin, j - 1);
#ifdef SELECT_PROF
            if (prof_on) { c1 = clock64(); pt[6] += c1 - c0; c0 = c1; }
#endif
                fin.next(p);
            }
            ++j;
            it.next(p);
#ifdef SELECT_PROF
            if (prof_on) { c1 = clock64(); pt[7] += c1 - c0; c0 = c1; }
#endif
#ifdef SELECT_PROF
            if (prof_on) pt[8] += 1;
#endif
        }
        if (j > 0) {
            named_bar_sync(1, 128);  // run_l of the last group visible to every finishing thread
            finish(fin, j - 1);
        }
#ifdef SELECT_PROF
        if (prof_on)
            printf("select prof CTA0 warp2 per item (%llu items): wait_S %llu ldS %llu max+bar %llu exp+P %llu fence+arrive %llu sum+bar %llu finish %llu (o_wait %llu) tail %llu\n",
                   pt[8], pt[0] / pt[8], pt[1] / pt[8], pt[2] / pt[8], pt[3] / pt[8], pt[4] / pt[8], pt[5] / pt[8],
                   pt[6] / pt[8], pt[9] / pt[8], pt[7] / pt[8]);
#endif
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc(tmem, TMEM_COLS);
    }
}

// W_g f32 [H][64][64] -> bf16 hi / lo, [a][j] rows of 128 B with the 128B swizzle
// pre-applied (chunk j/8 stored at chunk (j/8) ^ (a%8)), so one bulk copy lands
// the MN-major UMMA A-operand of G^T = W_g^T . Q^T.
__global__ void wg_prep_kernel(const float* __restrict__ wg, int heads, uint8_t* out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;  // over heads*64*64
    if (i >= heads * 4096) return;
    const int h = i / 4096, a = (i / 64) % 64, jj = i % 64;
    const float x = wg[i];
    const __nv_bfloat16 hi = __float2bfloat16_rn(x);
    const __nv_bfloat16 lo = __float2bfloat16_rn(x - __bfloat162float(hi));
    const int byte = a * 128 + ((((jj * 2) >> 4) ^ (a & 7)) << 4) + ((jj * 2) & 15);
    *reinterpret_cast<__nv_bfloat16*>(out + (size_t)h * 16384 + byte) = hi;
    *reinterpret_cast<__nv_bfloat16*>(out + (size_t)h * 16384 + 8192 + byte) = lo;
}

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn get_encode() {
    static EncodeFn fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeFn>(p);
    }
    return fn;
}

// window gather map over the image rows of a head-major [H][M][64] bf16 tensor
bool make_window_map(CUtensorMap* m, const TensorRef& t, int heads, const DevLayout& L) {
    EncodeFn enc = get_encode();
    if (!enc) return false;
    cuuint64_t dims[4] = {64, (cuuint64_t)L.grid_w, (cuuint64_t)L.grid_h * L.num_frames, (cuuint64_t)heads};
    // rows of rs elements: head-major [H][M][64] (rs = 64) or strided views such as the
    // token-major [M][3][H][64] output of a fused QKV projection (rs = 3 * H * 64)
    cuuint64_t strides[3] = {(cuuint64_t)t.rs * 2, (cuuint64_t)L.grid_w * t.rs * 2, (cuuint64_t)t.hs * 2};
    cuuint32_t box[4] = {64, 4, 4, 1};
    cuuint32_t es[4] = {1, 1, 1, 1};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(t.data), dims, strides, box, es,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

bool tensor_ok(const TensorRef& t, int dtype = GSA_DTYPE_BF16) {
    return t.dtype == dtype && t.rs >= 64 && t.rs % 8 == 0 && t.hs % 8 == 0 &&
           (reinterpret_cast<uintptr_t>(t.data) & 15) == 0;
}

}  // namespace

bool tc_select_supported(const SelectArgs& a) {
    // every precondition of tc_select (TMA window maps: bf16 rows, 16-byte aligned strides
    // and base), so a supported call never fails on shape grounds. f32 inputs reach it as
    // bf16 hi/lo planes (pack_select_inputs in abi.cu)
    const bool split = a.ql.data != nullptr;
    return a.dim == 64 && a.L.s == 4 && a.Lkv.s == 4 && tensor_ok(a.q) && tensor_ok(a.k) &&
           tensor_ok(a.v16, kDtypeF16) && a.vmax &&
           (!split || (tensor_ok(a.ql) && tensor_ok(a.kl) && tensor_ok(a.v16l, kDtypeF16))) &&
           (!a.w_g || (a.o_comp && a.wg_prep)) && get_encode() != nullptr;
}

size_t tc_select_workspace_bytes(int heads) { return (size_t)heads * 16384; }

cudaError_t tc_select(const SelectArgs& a, cudaStream_t st) {
    if (!tc_select_supported(a)) return cudaErrorNotSupported;
    const bool split = a.ql.data != nullptr, gate = a.w_g != nullptr;
    CUtensorMap tq, tk, tv, tql, tkl, tvl;
    // (the fp16 V planes move through the 2-byte bf16 map type bit for bit)
    if (!make_window_map(&tq, a.q, a.heads, a.L) || !make_window_map(&tk, a.k, a.heads, a.Lkv) ||
        !make_window_map(&tv, a.v16, a.heads, a.Lkv))
        return cudaErrorNotSupported;
    if (split) {
        if (!make_window_map(&tql, a.ql, a.heads, a.L) || !make_window_map(&tkl, a.kl, a.heads, a.Lkv) ||
            !make_window_map(&tvl, a.v16l, a.heads, a.Lkv))
            return cudaErrorNotSupported;
    } else {
        tql = tq;
        tkl = tk;
        tvl = tv;
    }
    if (gate) {
        wg_prep_kernel<<<(a.heads * 4096 + 255) / 256, 256, 0, st>>>(a.w_g, a.heads, a.wg_prep);
        note_launch();
    }
    SelTcParams p;
    p.heads = a.heads;
    p.L = a.L;
    p.rows = a.rows;
    p.scale = a.scale;
    p.c2 = a.scale * 1.4426950408889634f;
    p.items = (int64_t)a.heads * a.L.windows;
    p.fd_windows.init((uint32_t)a.L.windows);
    p.fd_wpf.init((uint32_t)a.L.wins_per_frame);
    p.fd_ww.init((uint32_t)a.L.wins_w);
    p.o_comp = a.o_comp;
    p.out = a.out;
    p.out_hs = a.out_hs;
    p.out_rs = a.out_rs;
    p.lse = a.lse;
    p.o_sel_ctx = a.o_sel_ctx;
    p.prior_o = a.prior_o;
    p.prior_lse = a.prior_lse;
    p.gate_ctx = gate ? a.gate_ctx : nullptr;
    p.wg_prep = a.wg_prep;
    p.split = split;
    p.gate = gate;
    p.vmax = a.vmax;
    int dev = 0, nsm = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    const size_t smem = sizeof(SelSmem) + 1024;
    cudaError_t e = cudaFuncSetAttribute(select_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    const int grid = (int)std::min<int64_t>((int64_t)nsm * SEL_CTAS, p.items);
    select_tc_kernel<<<grid, NTHREADS, smem, st>>>(tq, tk, tv, tql, tkl, tvl, p);
    note_launch();
    return cudaGetLastError();
}

}  // namespace gsa_sm100
