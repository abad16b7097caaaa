// compress_tc.cu — K2: compressed attention with streaming top-k on tcgen05
// tensor cores (fused_compressed_attention_topk, compression.hpp:180-297),
// indices bit-exact with the reference by construction.
//
// Pooled Qc/Kc/Vc are f32 means (not bf16-representable), so every operand is
// split x = hi + lo (bf16 each, |x - hi - lo| <= 2^-16 |x|) for the scores, which set
// the softmax AND the ranking, and
//   S  = Qh.Kh^T + Qh.Kl^T + Ql.Kh^T            (12 MMAs, M=N=128, per key tile)
//   O += P16.V16                                 (8 MMAs, P fp16 from TMEM)
// where P and V go through fp16 (11-bit significands, V scaled per head by a power of
// two into fp16 range): relative error <= ~2^-11 in O'_comp (measured ~3e-4 rel L2),
// far inside the 1e-3 layer tolerance, for one PV MMA term instead of three. The scores run on centred keys
// kc - kbar (kbar = per-head mean key: a per-row shift, invisible to the softmax and
// the ranking, added back to the lse). S is only an APPROXIMATION of the reference
// guide score (scaled_dot: 4 stride-4 f32 lane sums, no FMA), so the top-k runs in
// two steps:
//   1. here, per query row (one thread = one TMEM lane): a lower bound LB of the
//      row's k-th best approximate score (seeded from key tile 0, raised by an
//      8-bin histogram of the streamed candidates) and a candidate list in global
//      memory of every selectable score >= LB - margin, margin = 2 eps + 2^-20 |LB|,
//      eps = 2^-11 ||qc|| max ||kc - kbar|| + 2^-17 ||qc|| max ||kc|| >= |S' - exact'|.
//      Every true top-k member satisfies S >= tau - 2 eps (tau: k-th largest S),
//      so the candidate set is a guaranteed superset;
//   2. rescore_kernel: the k-th best approximate score by radix select, the
//      survivors within the margin, exact scaled_dot for each, a warp bitonic sort
//      by (score desc, index asc) = topk_better (compression.hpp:67-73).
// Rows whose list overflows (mass near-ties, clumps of near-equal keys) are
// re-selected exactly by largek_topk_kernel in row-list mode; k_eff > 128 (budget
// sweep) runs the softmax here and the whole selection in largek_topk_kernel.
#include <cuda.h>

#include <cstdio>
#include <cstdlib>
#include <cub/block/block_radix_sort.cuh>
#include <cub/block/block_scan.cuh>
#include <vector>

#include "tc.h"
#include "tc_ptx.cuh"
#include "tma_util.cuh"

namespace gsa_sm100 {
namespace {

using namespace ptx;

// bring-up switches, compile-time only (-DGSA_DEBUG_COMPRESS=<bits>; 0 in every shipped build)
#ifndef GSA_DEBUG_COMPRESS
#define GSA_DEBUG_COMPRESS 0
#endif
constexpr int kDebug = GSA_DEBUG_COMPRESS;

#ifndef COMP_NS
#define COMP_NS 4
#endif
constexpr int NS = COMP_NS;             // K/V ring stages
constexpr int TILE = 16384;             // 128 rows x 64 bf16
constexpr int STAGE = 2 * TILE;         // hi + lo
constexpr int NTHREADS = 384;           // warps 0-3 / 4-7: softmax WG0 / WG1, 8: TMA, 9: MMA, 10-11 idle
// (registers are split per SM sub-partition: 3 warps each; setmaxnreg moves 2 x 224 + 56 per SMSP)
constexpr int NWG = 2;                  // query tiles (softmax warpgroups) per CTA
constexpr int NSB = 3;                  // S/P buffers in TMEM, rotating over the S(n) sequence
constexpr uint32_t TMEM_COLS = 512;
constexpr uint32_t O_COL0 = 384;        // O of WG w: [384 + 64 w, +64); S/P buffer b: [128 b, +128)
constexpr float RESCALE_LOG2 = 8.0f;
#ifndef COMP_SM_REGS
#define COMP_SM_REGS 224
#define COMP_PROD_REGS 56
#endif
#ifndef COMP_SMALL_K_BIN_DIV
#define COMP_SMALL_K_BIN_DIV 8  // histogram bin width std/div for k <= 32
#endif
#ifndef COMP_LARGE_K_BIN_DIV
#define COMP_LARGE_K_BIN_DIV 4  // histogram bin width std/div for k > 32 (k=128 @500 views: 8 -> 49.4 ms, 4 -> 45.6 ms)
#endif
#ifndef COMP_MASK_VOTE
#define COMP_MASK_VOTE 1
#endif
#ifndef COMP_PB_UNROLL
#define COMP_PB_UNROLL 2
#endif
constexpr int SM_REGS = COMP_SM_REGS, PROD_REGS = COMP_PROD_REGS;  // 8 x 32 x SM + 4 x 32 x PROD <= 384 x 168
constexpr int PB_UNROLL = COMP_PB_UNROLL;
constexpr int KCAP = 128;               // max k_eff on this path
// candidates a row may stream out (more: exact per-row fallback) and survivors
// of the approximate radix select handed to the exact re-score: sized by k
// (the streamed count grows like k (1 + ln(W / k)))
// hybrid rows (excluded reference windows) start from a weaker first-tile bound: more candidates
#ifndef COMP_PLAIN_CCAP
#define COMP_PLAIN_CCAP 1024
#endif
__host__ __device__ constexpr int ccap_for(int k, bool excl = false) {
    return k <= 32 ? (excl ? 1024 : COMP_PLAIN_CCAP) : 2048;
}
// (a row's candidate count is typically ~k(1 + ln(W/k)), ~330 at k = 32, W = 81000; the
// larger list absorbs clumps of near-equal keys -- clustered activations -- and the
// re-score splits rows by count so the common case keeps the 512-entry register tile)
__host__ __device__ constexpr int surv_for(int k) { return k <= 32 ? 64 : 256; }
constexpr int NBIN = 8;                 // threshold histogram bins (8-bit saturating counters)
constexpr float EPS_REL = 0.00048828125f;          // 2^-11: split + accumulation error, x |q| max|kc - kbar|
constexpr float EPS_REF = 7.62939453125e-06f;      // 2^-17: the reference's own f32 rounding, x |q| max|kc|
constexpr float DELTA_REL = 9.5367431640625e-07f;  // 2^-20: collapse of distinct sums under *scale

struct __align__(1024) CompSmem {
    uint8_t q[NWG][2][TILE];  // the CTA's two query tiles, bf16 hi / lo
    uint8_t ring[NS][STAGE];  // K / V tiles, bf16 hi / lo
    // per softmax thread: the scores of the 32-key chunk it is extracting candidates from,
    // so a candidate's score is one indexed shared load instead of a register select tree
    // (16-byte groups XOR-swizzled by lane so a warp's row writes spread over the banks)
    float cstage[256][32];
    uint64_t full[NS], empty[NS];
    uint64_t q_full;
    uint64_t s_full[NSB];
    uint64_t p_full[NWG][2];  // by tile parity: a WG may run one tile ahead of the MMA's P wait
    uint64_t o_done[NWG];     // every PV of the WG (lazy O rescale waits on it)
    uint64_t o_final[NWG];    // the WG's last PV
    uint32_t tmem_base;
};

struct CompParams {
    int heads, Wq, Wk, k_eff;  // query rows (windows of this shard) / key rows (all windows)
    float scale, c2;
    int kv_tiles;
    const float* qnorm;       // [H][Wq]
    const float* kmax;        // [H] max |kc|
    const float* cmax;        // [H] max |kc - kbar| (the scores are computed on centred keys)
    const float* kbar;        // [H][64] per-head mean key: S' = q.(kc - kbar) = S - q.kbar
    const float* qc;          // [H][Wq][64] f32 (lse correction q.kbar)
    int64_t qc_hs, qc_rs;
    const float* vmax;        // [H] max |vc|: V is fed to the MMA as fp16(vc * 2^-e_h), e_h = vexp(vmax[h])
    const uint32_t* exbits;   // [ceil(Wk/32)] or null
    float* out;
    int64_t out_hs, out_rs;
    float* lse;               // [H][Wq]
    float2* cand;             // [H*Wq][ccap] (approx score, window id)
    int ccap;
    int* cand_n;              // [H*Wq]
    uint8_t* flag;            // [H*Wq]
    unsigned long long* prof; // COMPRESS_PROF builds: per-phase cycles of one softmax warp
};

// order-preserving map float -> uint32 (finite and +-inf); 0 is below every real key
__device__ __forceinline__ uint32_t fkey(float x) {
    const uint32_t b = __float_as_uint(x);
    return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
__device__ __forceinline__ float fkey_inv(uint32_t k) {
    return __uint_as_float((k & 0x80000000u) ? (k & 0x7fffffffu) : ~k);
}

// per-head power-of-two exponent that brings |vc| <= vmax below 2^14 in fp16 (exact scaling)
__device__ __forceinline__ int vexp(float vmax) { return vmax > 0.0f ? ilogbf(vmax) - 13 : 0; }

__device__ __forceinline__ float topk_threshold(float tau, float eps) {
    return tau - (2.0f * eps + DELTA_REL * fabsf(tau));
}

__device__ __forceinline__ void setmaxnreg_inc() { asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(SM_REGS) : "memory"); }
__device__ __forceinline__ void setmaxnreg_dec() { asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(PROD_REGS) : "memory"); }

#ifndef COMP_POLY
#define COMP_POLY 0  // exp2 of every COMP_POLY-th pair by polynomial on the FMA pipe (measured: 3, 4, 6 all slower -- K2 is not MUFU-bound)
#endif
#ifndef COMP_STAGE
#define COMP_STAGE 0  // 1: candidates read back from a shared staging row (measured: 71.0 vs 68.7 ms compress at V=1000 for the register select tree)
#endif
// The lowest set bit of m (m != 0): its index e and v[e], by a binary search over m's
// halves fused with a 5-level select tree (COMP_STAGE 0).
__device__ __forceinline__ float lowest_candidate(const uint32_t (&v)[32], uint32_t m, int& e) {
    uint32_t a[16];
    const bool b4 = (m & 0xffffu) == 0u;
#pragma unroll
    for (int i = 0; i < 16; ++i) a[i] = b4 ? v[i + 16] : v[i];
    m = b4 ? m >> 16 : m;
    const bool b3 = (m & 0xffu) == 0u;
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = b3 ? a[i + 8] : a[i];
    m = b3 ? m >> 8 : m;
    const bool b2 = (m & 0xfu) == 0u;
#pragma unroll
    for (int i = 0; i < 4; ++i) a[i] = b2 ? a[i + 4] : a[i];
    m = b2 ? m >> 4 : m;
    const bool b1 = (m & 0x3u) == 0u;
#pragma unroll
    for (int i = 0; i < 2; ++i) a[i] = b1 ? a[i + 2] : a[i];
    m = b1 ? m >> 2 : m;
    const bool b0 = (m & 0x1u) == 0u;
    e = (b4 ? 16 : 0) | (b3 ? 8 : 0) | (b2 ? 4 : 0) | (b1 ? 2 : 0) | (b0 ? 1 : 0);
    return __uint_as_float(b0 ? a[1] : a[0]);
}

// Per-row streaming top-k, run by the thread that owns the row. The row keeps a
// lower bound LB of its K-th best approximate score and streams every
// selectable score >= LB - margin into its global candidate list. LB rises via
// a histogram of the candidates above it (8 bins of width `delta`, saturating
// byte counters): once >= K candidates sit at or above bin j, LB += j*delta is
// still a lower bound. No sorting or shared state on the hot path; the exact
// K-th best and the final candidate set are resolved by the re-score kernel.
struct RowTopk {
    float lb, thr, delta, inv_delta, eps;
    // byte b = candidates in bin b >= 1 relative to lb (bin 7 open-ended). Bin 0 is never
    // counted (raise() only reads bins >= 1), so no byte overflows without saturation: before
    // a tile every suffix from bin 1 up is < K (else raise() had lifted LB), and one tile
    // adds at most 128: a byte stays <= K - 1 + 128 <= 255 for K <= KCAP
    uint64_t hist;
    int cnt;           // candidates streamed; -1 = none (invalid row) / overflow
    int ccap;
    float2* dst;
#ifdef COMPRESS_PROF
    int dbg;
#endif

    // branch-free: predicated store, select-based count and bin updates
    __device__ __forceinline__ void add(float v, int col) {
        const bool ok = (unsigned)cnt < (unsigned)ccap;  // cnt < 0 (no row / overflowed) is huge unsigned
#ifdef COMPRESS_PROF
        if (ok && !(dbg & 512)) dst[cnt] = make_float2(v, __int_as_float(col));
        if (dbg & 1024) { cnt = ok ? cnt + 1 : -1; return; }
#else
        if (ok) dst[cnt] = make_float2(v, __int_as_float(col));
#endif
        cnt = ok ? cnt + 1 : -1;  // reaching ccap overflows the row: exact fallback
        // bin = floor(clamp(rel, 0, 7)) without F2I (XU pipe): a round-down add of 2^23
        // leaves floor(x) in the mantissa bits
        const float rel = fminf(fmaxf((v - lb) * inv_delta, 0.0f), (float)(NBIN - 1));
        const int b = __float_as_int(__fadd_rd(rel, 8388608.0f)) - 0x4B000000;
        hist += (ok && b > 0) ? 1ull << (8 * b) : 0ull;
    }
    // after each tile: raise LB by the largest j with >= K counted at or above bin j
    __device__ __forceinline__ void raise(int K) {
        int suffix = 0, j = 0;
        float jf = 0.0f;  // (float)j without I2F (XU pipe)
#pragma unroll
        for (int b = NBIN - 1; b >= 1; --b) {
            suffix += (int)((hist >> (8 * b)) & 0xffu);
            if (j == 0 && suffix >= K) {
                j = b;
                jf = (float)b;
            }
        }
        if (j == 0) return;
        lb += jf * delta;
        thr = fmaxf(thr, topk_threshold(lb, eps));
        hist >>= 8 * j;
        if (j == NBIN - 1) {
            // LB climbed the whole histogram in one tile: the bins are too fine. Double
            // them; merged counts stay lower bounds (new bin b holds old bins 2b, 2b+1,
            // all >= lb + b * 2 delta; the open-ended old bin 7 lands in new bin 3)
            const uint32_t h0 = (uint32_t)hist, h1 = (uint32_t)(hist >> 32);
            hist = __vaddus4(__byte_perm(h0, h1, 0x6420), __byte_perm(h0, h1, 0x7531));
            delta *= 2.0f;
            inv_delta *= 0.5f;
        }
    }
};

// Position of K(t) / V(t) in the TMA load sequence K0 K1 V0 K2 V1 K3 V2 ...
// K(T-1) V(T-2) V(T-1) (the MMA issuer's first-use order); ring slot = seq % NS,
// fill phase = seq / NS.
__device__ __forceinline__ int seq_k(int t) { return t == 0 ? 0 : 2 * t - 1; }
__device__ __forceinline__ int seq_v(int t, int T) { return t == T - 1 ? 2 * T - 1 : 2 * t + 2; }

__global__ void __launch_bounds__(NTHREADS, 1)
    compress_tc_kernel(const __grid_constant__ CUtensorMap tm_qh, const __grid_constant__ CUtensorMap tm_ql,
                       const __grid_constant__ CUtensorMap tm_kh, const __grid_constant__ CUtensorMap tm_kl,
                       const __grid_constant__ CUtensorMap tm_v16, const CompParams p) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    CompSmem& sm = *reinterpret_cast<CompSmem*>(smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u));
    const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
    const int h = blockIdx.y;
    const int T = p.kv_tiles;
    const int N = NWG * T;  // S(n), n = 2t + w: WG w's scores against key tile t

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
    }
    if (warp == 9) tmem_alloc(&sm.tmem_base, TMEM_COLS);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = sm.tmem_base;

    if (warp >= 8) {
        setmaxnreg_dec();
        if (warp == 8) {
            // ================================ TMA ================================
            if (elect_one()) {
                mbar_arrive_expect_tx(&sm.q_full, NWG * 2 * TILE);
                for (int w = 0; w < NWG; ++w) {
                    tma_load_3d(&sm.q[w][0][0], &tm_qh, &sm.q_full, 0, (blockIdx.x * NWG + w) * 128, h);
                    tma_load_3d(&sm.q[w][1][0], &tm_ql, &sm.q_full, 0, (blockIdx.x * NWG + w) * 128, h);
                }
            }
            __syncwarp();
            int seq = 0;
            auto load = [&](const CUtensorMap* th, const CUtensorMap* tl, int t) {  // tl null: fp16 V tile only
                const int st = seq % NS;
                mbar_wait(&sm.empty[st], (uint32_t)(((seq / NS) & 1) ^ 1));
                if (elect_one()) {
                    mbar_arrive_expect_tx(&sm.full[st], tl ? STAGE : TILE);
                    tma_load_3d(&sm.ring[st][0], th, &sm.full[st], 0, t * 128, h);
                    if (tl) tma_load_3d(&sm.ring[st][TILE], tl, &sm.full[st], 0, t * 128, h);
                }
                __syncwarp();
                ++seq;
            };
            load(&tm_kh, &tm_kl, 0);
            if (T > 1) load(&tm_kh, &tm_kl, 1);
            for (int t = 0; t < T; ++t) {
                load(&tm_v16, nullptr, t);
                if (t + 2 < T) load(&tm_kh, &tm_kl, t + 2);
            }
        } else if (warp == 9) {
            // ================================ MMA ================================
            // S(n) = Q_w . K(t)^T  (Qh.Kh + Qh.Kl + Ql.Kh)          -> S/P buffer n % 3
            // O_w += P(n) . V(t)    (Ph.Vh + Ph.Vl + Pl.Vh; P in TMEM)  n = 2t + w
            // Issue order: S(0) S(1) S(2) | PV(n) S(n+3) | ... S(n+3) reuses PV(n)'s
            // buffer (in-order execution) and is issued BEFORE the P waits of n+1, n+2,
            // so every WG always has its next S computing while it runs a softmax.
            const uint32_t id_s = idesc_bf16(128, 128, 0, 0);
            const uint32_t id_o = idesc_f16(128, 64, 0, 1);  // P (TMEM) and V (SMEM) in fp16
#ifdef COMPRESS_PROF
            const bool mprof = p.prof && blockIdx.x == 0 && blockIdx.y == 0 && lane == 0;
            unsigned long long mw_full = 0, mw_p = 0, m_t0 = clock64(), m_c;
#define MPROF_T(acc) if (mprof) { m_c = clock64(); acc += m_c - m_t0; m_t0 = m_c; }
#define MPROF_MARK() if (mprof) m_t0 = clock64();
#else
#define MPROF_T(acc)
#define MPROF_MARK()
#endif
            auto wait_tile = [&](int s) {
                MPROF_MARK();
                mbar_wait(&sm.full[s % NS], (uint32_t)((s / NS) & 1));
                MPROF_T(mw_full);
                tc_fence_after();
            };
            auto issue_S = [&](int n) {
                const int w = n & 1, t = n >> 1;
                const int s = seq_k(t);
                if (w == 0) wait_tile(s);
                const uint64_t kh = umma_desc(smem_u32(&sm.ring[s % NS][0]), 16, 1024, 2);
                const uint64_t kl = umma_desc(smem_u32(&sm.ring[s % NS][TILE]), 16, 1024, 2);
                const uint64_t qh = umma_desc(smem_u32(&sm.q[w][0][0]), 16, 1024, 2);
                const uint64_t ql = umma_desc(smem_u32(&sm.q[w][1][0]), 16, 1024, 2);
                const uint32_t d = tmem + 128 * (n % NSB);
                if (elect_one()) {
                    for (int ks = 0; ks < 4; ++ks) {
                        mma_bf16(d, qh + 2 * ks, kh + 2 * ks, id_s, ks != 0);
                        mma_bf16(d, qh + 2 * ks, kl + 2 * ks, id_s, 1);
                        mma_bf16(d, ql + 2 * ks, kh + 2 * ks, id_s, 1);
                    }
                    mma_commit(&sm.s_full[n % NSB]);
                    if (w == 1) mma_commit(&sm.empty[s % NS]);  // K(t) fully used
                }
                __syncwarp();
            };
            auto issue_PV = [&](int n) {
                const int w = n & 1, t = n >> 1;
                const int s = seq_v(t, T);
                if (w == 0) wait_tile(s);
                MPROF_MARK();
                mbar_wait(&sm.p_full[w][t & 1], (uint32_t)((t >> 1) & 1));
                MPROF_T(mw_p);
                tc_fence_after();
                const uint64_t v16 = umma_desc(smem_u32(&sm.ring[s % NS][0]), 16, 1024, 2);
                const uint32_t o = tmem + O_COL0 + 64 * w, pb = tmem + 128 * (n % NSB);
                if (elect_one()) {
                    for (int ks = 0; ks < 8; ++ks)  // P fp16 of keys [16 ks, 16 ks + 16): columns 32 (ks/2) + 8 (ks%2)
                        mma_bf16_ts(o, pb + 32 * (ks >> 1) + 8 * (ks & 1), v16 + 128 * ks, id_o, (t | ks) != 0);
                    mma_commit(&sm.o_done[w]);
                    if (t == T - 1) mma_commit(&sm.o_final[w]);
                    if (w == 1) mma_commit(&sm.empty[s % NS]);  // V(t) fully used
                }
                __syncwarp();
            };
            mbar_wait(&sm.q_full, 0);
            tc_fence_after();
            for (int n = 0; n < min(NSB, N); ++n) issue_S(n);
#ifdef COMPRESS_PROF
            const unsigned long long m_start = clock64();
#endif
            for (int n = 0; n < N; ++n) {
                issue_PV(n);
                if (n + NSB < N) issue_S(n + NSB);
            }
#ifdef COMPRESS_PROF
            if (mprof) {
                p.prof[6] = mw_full;
                p.prof[7] = mw_p;
                p.prof[8] = clock64() - m_start;
            }
#endif
#undef MPROF_T
#undef MPROF_MARK
        }
    } else {
        // ===================== softmax + streaming top-k (warps 0..7) =====================
        setmaxnreg_inc();
        const int w = warp >> 2;           // warpgroup = query tile of this CTA
        const int qd = warp & 3;           // TMEM lane quadrant
        const int row = 32 * qd + lane;
        const int grow = (blockIdx.x * NWG + w) * 128 + row;
        const bool row_ok = grow < p.Wq;
        const uint32_t lane_base = tmem + ((uint32_t)(32 * qd) << 16);
        const uint32_t o_base = lane_base + O_COL0 + 64 * w;
        const int K = p.k_eff;
        const int64_t r = (int64_t)h * p.Wq + grow;
        RowTopk tk;
        tk.lb = -INFINITY;
        tk.thr = -INFINITY;
        tk.delta = 1.0f;
        tk.inv_delta = 1.0f;
        tk.eps = row_ok ? EPS_REL * p.qnorm[r] * p.cmax[h] + EPS_REF * p.qnorm[r] * p.kmax[h] : 0.0f;
        tk.hist = 0ull;
        tk.cnt = (row_ok && K > 0) ? 0 : -1;
        tk.ccap = p.ccap;
        tk.dst = p.cand + r * p.ccap;
#ifdef COMPRESS_PROF
        tk.dbg = kDebug;
#endif
        float m_used = -INFINITY, l = 0.0f;

#ifdef COMPRESS_PROF
        const bool prof_on = p.prof && blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0;
        unsigned long long pt[8] = {0, 0, 0, 0, 0, 0, 0, 0}, pb[5] = {0, 0, 0, 0, 0}, c0 = clock64(), c1;
#endif
        const bool do_topk = K > 0 && !(kDebug & 1);
        if (do_topk) {
            // ---- top-k seed from key tile 0 (its own register scope: peeled off the loop)
            // initial LB: the largest 16-bit key prefix P with >= K selectable keys >= P<<16
            // bounds the row's K-th best from below; bins span [LB, max]
            mbar_wait(&sm.s_full[w], 0u);  // S(n = w) lives in buffer w, first fill
            __syncwarp();
            tc_fence_after();
            uint32_t sr[4][32];
#pragma unroll
            for (int c = 0; c < 4; ++c) tmem_ld_32x32b_x32(lane_base + 128 * w + 32 * c, sr[c]);
            tmem_wait_ld();
            uint32_t keep[4];
            {
                uint4 ex = make_uint4(0, 0, 0, 0);
                if (p.exbits) ex = __ldg(reinterpret_cast<const uint4*>(p.exbits));
                const uint32_t exw[4] = {ex.x, ex.y, ex.z, ex.w};
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    const int vc = p.Wk - 32 * c;
                    keep[c] = (vc >= 32 ? 0xffffffffu : (vc <= 0 ? 0u : ((1u << vc) - 1u))) & ~exw[c];
                }
            }
#pragma unroll
            for (int c = 0; c < 4; ++c)
#pragma unroll
                for (int e = 0; e < 32; ++e)
                    sr[c][e] = ((keep[c] >> e) & 1u) ? fkey(__uint_as_float(sr[c][e])) : 0u;
            uint32_t res = 0;
#pragma unroll 1
            for (int bit = 31; bit >= 16; --bit) {
                const uint32_t cand = res | (1u << bit);
                int cnt = 0;
#pragma unroll
                for (int c = 0; c < 4; ++c)
#pragma unroll
                    for (int e = 0; e < 32; ++e) cnt += sr[c][e] >= cand ? 1 : 0;
                if (cnt >= K) res = cand;
            }
            if (res != 0) {
                // bin width = (std of the row's first 128 scores) / 8: fine enough
                // that LB trails the running K-th best by a fraction of the spread
                float s1 = 0.0f, s2 = 0.0f;
#pragma unroll
                for (int c = 0; c < 4; ++c)
#pragma unroll
                    for (int e = 0; e < 32; ++e) {
                        const float x = ((keep[c] >> e) & 1u) ? fkey_inv(sr[c][e]) : 0.0f;
                        s1 += x;
                        s2 = fmaf(x, x, s2);
                    }
                const float nk = (float)(__popc(keep[0]) + __popc(keep[1]) + __popc(keep[2]) + __popc(keep[3]));
                const float mean = s1 / nk, var = fmaxf(s2 / nk - mean * mean, 0.0f);
                tk.lb = fkey_inv(res);
                tk.thr = topk_threshold(tk.lb, tk.eps);
                const float bin_div = K <= 32 ? (float)COMP_SMALL_K_BIN_DIV : (float)COMP_LARGE_K_BIN_DIV;
                tk.delta = var > 0.0f ? sqrtf(var) / bin_div : fmaxf(fabsf(tk.lb) * 0.0009765625f, 1e-30f);
                tk.inv_delta = 1.0f / tk.delta;
            }
        }
        for (int t = 0; t < T; ++t) {
            const int n = 2 * t + w, b = n % NSB;
            const uint32_t s_base = lane_base + 128 * b;
            mbar_wait(&sm.s_full[b], (uint32_t)((n / NSB) & 1));
#ifdef COMPRESS_PROF
            if (prof_on) { c1 = clock64(); pt[0] += c1 - c0; c0 = c1; }
#endif
            __syncwarp();  // .sync.aligned tcgen05 ops below need a converged warp
            tc_fence_after();
            const int valid = p.Wk - t * 128;  // < 128 on the last key tile only
            uint32_t keep[4] = {~0u, ~0u, ~0u, ~0u};  // selectable columns (in range, not excluded)
            if (valid < 128 || (do_topk && p.exbits)) {
                uint4 ex = make_uint4(0, 0, 0, 0);
                if (do_topk && p.exbits) ex = __ldg(reinterpret_cast<const uint4*>(p.exbits) + t);
                const uint32_t exw[4] = {ex.x, ex.y, ex.z, ex.w};
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    const int vc = valid - 32 * c;
                    keep[c] = (vc >= 32 ? 0xffffffffu : (vc <= 0 ? 0u : ((1u << vc) - 1u))) & ~exw[c];
                }
            }
            // ---- pass A: chunk maxima of S and the top-k candidate masks. The
            // 128 scores are live only here; pass B re-reads them from TMEM one chunk at a
            // time, so the softmax and the top-k run with ~100 registers instead of 200+.
            float cmax[4];
            uint32_t cmask[4] = {0u, 0u, 0u, 0u};  // top-k candidate columns per chunk
            {
                uint32_t sr[4][32];
#pragma unroll
                for (int c = 0; c < 4; ++c) tmem_ld_32x32b_x32(s_base + 32 * c, sr[c]);
                tmem_wait_ld();
                if (valid < 128) {
                    // last key tile: columns past Wk do not exist. -inf goes back to TMEM too,
                    // so pass B needs no masking code (P = exp2(-inf) = 0)
#pragma unroll
                    for (int c = 0; c < 4; ++c) {
#pragma unroll
                        for (int e = 0; e < 32; ++e)
                            if (32 * c + e >= valid) sr[c][e] = __float_as_uint(-INFINITY);
                        tmem_st_32x32b_x32(s_base + 32 * c, sr[c]);
                    }
                    tmem_wait_st();
                }
#pragma unroll
                for (int c = 0; c < 4; ++c) {  // 3-input max trees (short dependency chains)
                    float a0 = __uint_as_float(sr[c][0]), a1 = __uint_as_float(sr[c][1]);
                    float a2 = __uint_as_float(sr[c][2]), a3 = __uint_as_float(sr[c][3]);
#pragma unroll
                    for (int e = 4; e < 32; e += 4) {
                        a0 = fmaxf(a0, __uint_as_float(sr[c][e]));
                        a1 = fmaxf(a1, __uint_as_float(sr[c][e + 1]));
                        a2 = fmaxf(a2, __uint_as_float(sr[c][e + 2]));
                        a3 = fmaxf(a3, __uint_as_float(sr[c][e + 3]));
                    }
                    cmax[c] = fmaxf(fmaxf(a0, a1), fmaxf(a2, a3));
                }
                if (do_topk && !(kDebug & 256)) {
                    // candidate masks: bit e = (S[e] >= tq) = NOT sign(S - tq) (FADD2), gathered by
                    // funnel shifts into four independent 8-bit chains per chunk
                    const float tq = tk.cnt < 0 ? INFINITY : tk.thr;
                    const float2 ntq = make_float2(-tq, -tq);
#pragma unroll
                    for (int c = 0; c < 4; ++c) {
                        // most chunks hold no candidate of any of the warp's 32 rows late in the row
                        if (COMP_MASK_VOTE && !__any_sync(0xffffffffu, cmax[c] >= tq)) continue;
                        uint32_t ch[4] = {0u, 0u, 0u, 0u};
#pragma unroll
                        for (int i = 3; i >= 0; --i)  // element pair 2i, 2i+1 of every 8-element group
#pragma unroll
                            for (int j = 0; j < 4; ++j) {
                                const int e = 8 * j + 2 * i;
                                const float2 dd = __fadd2_rn(make_float2(__uint_as_float(sr[c][e]), __uint_as_float(sr[c][e + 1])), ntq);
                                ch[j] = __funnelshift_l(__float_as_uint(dd.y), ch[j], 1);
                                ch[j] = __funnelshift_l(__float_as_uint(dd.x), ch[j], 1);
                            }
                        cmask[c] = ~(ch[0] | (ch[1] << 8) | (ch[2] << 16) | (ch[3] << 24)) & keep[c];
                    }
                    if (kDebug & 128) cmask[0] = cmask[1] = cmask[2] = cmask[3] = 0u;  // bring-up: no extraction
                    // Re-seed on a clump: when >= K selectable scores of THIS tile clear the
                    // threshold (the query's own view arriving in clustered activations: 81
                    // near-equal windows; or the first tiles of any row), this tile's K-th best
                    // approximate score bounds the row's K-th best from below. Raise LB to it
                    // right away (16-bit radix search over the tile's 128 scores, as the tile-0
                    // seed) instead of letting the histogram climb bin by bin while the later
                    // tiles flood the candidate list.
                    const int nc = __popc(cmask[0]) + __popc(cmask[1]) + __popc(cmask[2]) + __popc(cmask[3]);
                    const bool reseed = t > 0 && tk.cnt >= 0 && nc >= K;
                    if (__any_sync(0xffffffffu, reseed)) {
                        if (reseed) {
                            // sr is dead after pass A: turn it into order-preserving keys in
                            // place (0 = not selectable, below every key)
#pragma unroll
                            for (int c = 0; c < 4; ++c)
#pragma unroll
                                for (int e = 0; e < 32; ++e)
                                    sr[c][e] = ((keep[c] >> e) & 1u) ? fkey(__uint_as_float(sr[c][e])) : 0u;
                            uint32_t res = 0;
#pragma unroll 1
                            for (int bit = 31; bit >= 16; --bit) {
                                const uint32_t cand = res | (1u << bit);
                                int cnt = 0;
#pragma unroll
                                for (int c = 0; c < 4; ++c)
#pragma unroll
                                    for (int e = 0; e < 32; ++e) cnt += sr[c][e] >= cand ? 1 : 0;
                                if (cnt >= K) res = cand;
                            }
                            const float lbt = fkey_inv(res);
                            if (res != 0u && lbt > tk.lb) {
                                tk.lb = lbt;
                                tk.thr = fmaxf(tk.thr, topk_threshold(lbt, tk.eps));
                                tk.hist = 0ull;  // counts were relative to the old LB
                                const uint32_t kthr = fkey(tk.thr);
#pragma unroll
                                for (int c = 0; c < 4; ++c) {
                                    uint32_t m = 0u;
#pragma unroll
                                    for (int e = 0; e < 32; ++e) m |= (sr[c][e] >= kthr ? 1u : 0u) << e;
                                    cmask[c] &= m;
                                }
                            }
                        }
                        __syncwarp();
                    }
                }
            }
            const float mt = fmaxf(fmaxf(cmax[0], cmax[1]), fmaxf(cmax[2], cmax[3]));
#ifdef COMPRESS_PROF
            if (prof_on) { c1 = clock64(); pt[1] += c1 - c0; c0 = c1; }
#endif
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
            // ---- pass B, per 32-key chunk: P = exp2(S*c2 - m*c2) as packed fp16 pairs written
            // over the first 16 columns of the chunk's S (one cvt per pair); then the chunk's
            // top-k candidates. The P barrier is released after the last chunk's stores,
            // before its top-k.
            const float mc = m_used * p.c2;
            const float2 c2v = make_float2(p.c2, p.c2), nmc = make_float2(-mc, -mc);
            float2 lsum2[2] = {make_float2(0.0f, 0.0f), make_float2(0.0f, 0.0f)};
            // unrolled by 2 only: the fully unrolled loop did not fit the instruction cache
            // (20-50 % no_instruction stalls); measured at V=1000: x1 82.2 ms, x2 76-78 ms, x4 85 ms
            uint32_t mrot = cmask[0], mq1 = cmask[1], mq2 = cmask[2], mq3 = cmask[3];
#pragma unroll PB_UNROLL
            for (int c = 0; c < 4; ++c) {
                uint32_t v[32];
#ifdef COMPRESS_PROF
                if (prof_on) { c1 = clock64(); pt[3] += c1 - c0; c0 = c1; }
#endif
                const uint32_t cb = s_base + 32 * c;
                tmem_ld_32x32b_x32(cb, v);
                tmem_wait_ld();
#ifdef COMPRESS_PROF
                if (prof_on) { c1 = clock64(); pb[0] += c1 - c0; c0 = c1; }
#endif
                {
                    uint32_t p16[16];
#pragma unroll
                    for (int e2 = 0; e2 < 16; ++e2) {
                        const float2 x = make_float2(__uint_as_float(v[2 * e2]), __uint_as_float(v[2 * e2 + 1]));
                        const float2 a = __ffma2_rn(x, c2v, nmc);
                        const float2 pv = (COMP_POLY > 0 && e2 % (COMP_POLY > 0 ? COMP_POLY : 1) == COMP_POLY - 1)
                                              ? exp2_poly2(a)
                                              : make_float2(ex2_approx(a.x), ex2_approx(a.y));
                        lsum2[e2 & 1] = __fadd2_rn(lsum2[e2 & 1], pv);  // the denominator sums the exact f32 P
                        p16[e2] = pack_f16(pv.x, pv.y);
                    }
                    tmem_st_32x32b_x16(cb, p16);
                }
#ifdef COMPRESS_PROF
                if (prof_on) { c1 = clock64(); pb[1] += c1 - c0; c0 = c1; }
#endif
                if (c == 3) {
                    tmem_wait_st();
                    tc_fence_before();
                    mbar_arrive(&sm.p_full[w][t & 1]);
#ifdef COMPRESS_PROF
                    if (prof_on) { c1 = clock64(); pb[2] += c1 - c0; c0 = c1; }
#endif
                }
                // this chunk's candidates (overlaps the MMAs)
                uint32_t m = mrot;
                mrot = mq1;
                mq1 = mq2;
                mq2 = mq3;
#ifdef COMPRESS_PROF
                {
                    const unsigned mx = __reduce_max_sync(0xffffffffu, (unsigned)__popc(m));
                    const unsigned sm_ = __reduce_add_sync(0xffffffffu, (unsigned)__popc(m));
                    if (prof_on) { pt[2] += mx; pt[6] += sm_; pt[7] += mx ? 1 : 0; }
                }
#endif
                const int col0 = t * 128 + 32 * c;
#ifdef COMPRESS_PROF
                if (prof_on) { c1 = clock64(); pb[3] += c1 - c0; c0 = c1; }
#endif
#if COMP_STAGE
                if (__any_sync(0xffffffffu, m != 0u)) {
                    float4* srow = reinterpret_cast<float4*>(&sm.cstage[threadIdx.x][0]);
#pragma unroll
                    for (int j = 0; j < 8; ++j)
                        srow[j ^ (lane & 7)] = make_float4(__uint_as_float(v[4 * j]), __uint_as_float(v[4 * j + 1]),
                                                           __uint_as_float(v[4 * j + 2]), __uint_as_float(v[4 * j + 3]));
                    const float* sf = &sm.cstage[threadIdx.x][0];  // the thread's own row: no barrier
                    while (m) {
                        const int e = __ffs(m) - 1;
                        m &= m - 1;
                        tk.add(sf[(((e >> 2) ^ (lane & 7)) << 2) | (e & 3)], col0 + e);
                    }
                }
#else
                while (m) {
                    int e;
                    const float x = lowest_candidate(v, m, e);
                    m &= m - 1;
                    tk.add(x, col0 + e);
                }
#endif
#ifdef COMPRESS_PROF
                if (prof_on) { c1 = clock64(); pb[4] += c1 - c0; c0 = c1; }
#endif
            }
            {
                const float2 ls = __fadd2_rn(lsum2[0], lsum2[1]);
                l += ls.x + ls.y;
            }
#ifdef COMPRESS_PROF
            if (prof_on) { c1 = clock64(); pt[3] += c1 - c0; c0 = c1; }
#endif
            if (do_topk && tk.cnt > 0) tk.raise(K);
#ifdef COMPRESS_PROF
            if (prof_on) { c1 = clock64(); pt[4] += c1 - c0; c0 = c1; pt[5] += 1; }
#endif
            __syncwarp();
        }
#ifdef COMPRESS_PROF
        if (prof_on) {
            for (int i = 0; i < 6; ++i) p.prof[i] = pt[i];
            p.prof[9] = pt[2];   // warp extraction iterations (max over lanes, summed over chunks)
            p.prof[10] = pt[6];  // candidates of the warp's 32 rows
            p.prof[11] = pt[7];  // chunks with a mask pass
            p.prof[12] = pb[0];  // pass B: TMEM load + wait
            p.prof[13] = pb[1];  // pass B: exp2 + P split + TMEM stores
            p.prof[14] = pb[2];  // pass B: wait_st + arrive
            p.prof[15] = pb[3];  // pass B: before the extraction loops
            p.prof[16] = pb[4];  // pass B: extraction loops
        }
#endif
        // ------------------------------- epilogue -------------------------------
        mbar_wait(&sm.o_final[w], 0);
        __syncwarp();
        tc_fence_after();
        uint32_t o[2][32];
        tmem_ld_32x32b_x32(o_base, o[0]);
        tmem_ld_32x32b_x32(o_base + 32, o[1]);
        tmem_wait_ld();
        if (row_ok) {
            const float inv = ldexpf(1.0f / l, vexp(p.vmax[h]));  // undo the fp16 V scaling exactly
            float* dst = p.out + (int64_t)h * p.out_hs + (int64_t)grow * p.out_rs;
#pragma unroll
            for (int half = 0; half < 2; ++half)
#pragma unroll
                for (int e = 0; e < 32; e += 4)
                    *reinterpret_cast<float4*>(dst + 32 * half + e) =
                        make_float4(__uint_as_float(o[half][e]) * inv, __uint_as_float(o[half][e + 1]) * inv,
                                    __uint_as_float(o[half][e + 2]) * inv, __uint_as_float(o[half][e + 3]) * inv);
            if (p.lse) {
                // the softmax ran on S' = S - q.kbar (a per-row shift): add it back to the lse
                const float* qrow = p.qc + (int64_t)h * p.qc_hs + (int64_t)grow * p.qc_rs;
                const float* kb = p.kbar + h * 64;
                float qk = 0.0f;
#pragma unroll 8
                for (int j = 0; j < 64; ++j) qk = fmaf(__ldg(qrow + j), __ldg(kb + j), qk);
                p.lse[r] = m_used * p.scale + logf(l) + qk * p.scale;
            }
            if (K > 0) {
                p.cand_n[r] = tk.cnt < 0 ? 0 : tk.cnt;
                p.flag[r] = (tk.cnt < 0 || (kDebug & 16)) ? 1 : 0;
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 9) {
        tc_fence_after();
        tmem_dealloc(tmem, TMEM_COLS);
    }
}

// Exact top-k of one row from its streamed candidates. One warp per row:
//  1. the K-th best APPROXIMATE score tau_a by a 32-step radix select over the
//     candidates' order-preserving keys (<= CCAP, 16 per lane);
//  2. the candidates within the error margin of tau_a (a superset of the true
//     top-k: |approx - exact| <= eps) — at most CAND, else the row is flagged
//     for the exact CUDA-core recompute;
//  3. exact scaled_dot (dot.hpp:11-23 order, no FMA) for those, rank by
//     (score desc, index asc) = topk_better (compression.hpp:67-73).
// Query rows index [H][Wq], key windows [H][Wk] (Wq < Wk for a view shard).
template <int PER, int SLOTS>
__global__ void __launch_bounds__(256) rescore_kernel(const float* __restrict__ qc, int64_t q_hs,
                                                      const float* __restrict__ kc, int heads, int Wq, int Wk,
                                                      float scale, int k_eff, const float* __restrict__ qnorm,
                                                      const float* __restrict__ kmax, const float* __restrict__ cmax,
                                                      const float2* __restrict__ cand, int cstride, int n_lo, int n_hi,
                                                      const int* __restrict__ cand_n, uint8_t* flag, int32_t* topk,
                                                      float* guide) {
    constexpr int CC = PER * 32, SV = SLOTS * 32;  // candidate capacity / survivor capacity
    extern __shared__ float2 surv_all[];           // [8 warps][SV]
    const int64_t r = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
    const int lane = threadIdx.x & 31;
    if (r >= (int64_t)heads * Wq || flag[r]) return;
    // this instance takes the rows with n_lo < candidates <= n_hi (register capacity CC)
    if (cand_n[r] <= n_lo || cand_n[r] > n_hi) return;
    const int h = (int)(r / Wq);
    const int n = min(cand_n[r], CC);
    const float2* cr = cand + r * cstride;
    float2 cv[PER];
    uint32_t key[PER];
#pragma unroll
    for (int i = 0; i < PER; ++i) {
        const int j = lane + 32 * i;
        cv[i] = j < n ? cr[j] : make_float2(-INFINITY, __int_as_float(-1));
        key[i] = j < n ? fkey(cv[i].x) : 0u;
    }
    uint32_t res = 0;
#pragma unroll 1
    for (int bit = 31; bit >= 0; --bit) {
        const uint32_t c = res | (1u << bit);
        int cnt = 0;
#pragma unroll
        for (int i = 0; i < PER; ++i) cnt += key[i] >= c ? 1 : 0;
        if ((int)__reduce_add_sync(0xffffffffu, (unsigned)cnt) >= k_eff) res = c;
    }
    const float eps = EPS_REL * qnorm[r] * cmax[h] + EPS_REF * qnorm[r] * kmax[h];  // as in the main kernel
    const float thr = topk_threshold(fkey_inv(res), eps);
    // compact the survivors (through shared memory) into SLOTS slots per lane
    float2* sv = surv_all + (threadIdx.x / 32) * SV;
    int total = 0;
#pragma unroll
    for (int i = 0; i < PER; ++i) {
        const bool keep = key[i] != 0u && cv[i].x >= thr;
        const unsigned b = __ballot_sync(0xffffffffu, keep);
        const int pos = total + __popc(b & ((1u << lane) - 1u));
        if (keep && pos < SV) sv[pos] = cv[i];
        total += __popc(b);
    }
    __syncwarp();
    if (total > SV) {
        if (lane == 0) flag[r] = 2;  // near-tie flood: the exact per-row kernel redoes this row
        return;
    }
    float e[SLOTS];
    int idx[SLOTS];
    const float* q = qc + (int64_t)h * q_hs + (r - (int64_t)h * Wq) * 64;
#pragma unroll
    for (int s = 0; s < SLOTS; ++s) {
        const int j = lane + 32 * s;
        e[s] = -INFINITY;
        idx[s] = j < total ? __float_as_int(sv[j].y) : -1;
        if (idx[s] >= 0) {  // exact scaled_dot (dot.hpp:11-23 order)
            const float* k = kc + ((int64_t)h * Wk + idx[s]) * 64;
            ExactDot4 d;
            d.zero();
#pragma unroll 4
            for (int x = 0; x < 64; x += 4) {
                const float4 qv = __ldg(reinterpret_cast<const float4*>(q + x));
                const float4 kv = __ldg(reinterpret_cast<const float4*>(k + x));
                d.step(qv.x, qv.y, qv.z, qv.w, kv.x, kv.y, kv.z, kv.w);
            }
            e[s] = d.finish(scale);
        }
    }
    // order by topk_better (compression.hpp:67-73) = descending 64-bit keys
    // (fkey(score) << 32 | ~index): a warp bitonic sort over SLOTS x 32 entries, element
    // i = 32 s + lane; position p of the sorted sequence is rank p. (Exact scores are never
    // -0: the lane sums start at +0, so +0 + x never yields -0 -- fkey orders them as floats.)
    unsigned long long skey[SLOTS];
#pragma unroll
    for (int s = 0; s < SLOTS; ++s)
        skey[s] = idx[s] >= 0 ? ((unsigned long long)fkey(e[s]) << 32) | (0xffffffffu - (uint32_t)idx[s]) : 0ull;
#pragma unroll
    for (int size = 2; size <= SLOTS * 32; size <<= 1) {
#pragma unroll
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            if (stride >= 32) {  // partner in another slot of the same lane
#pragma unroll
                for (int s = 0; s < SLOTS; ++s) {
                    const int so = s ^ (stride >> 5);
                    if (so > s) {
                        const int i = 32 * s + lane;
                        const bool desc = (i & size) == 0;  // keep the larger at the lower index
                        const unsigned long long a = skey[s], b = skey[so];
                        const bool sw = desc ? (a < b) : (a > b);
                        skey[s] = sw ? b : a;
                        skey[so] = sw ? a : b;
                    }
                }
            } else {
#pragma unroll
                for (int s = 0; s < SLOTS; ++s) {
                    const int i = 32 * s + lane;
                    const unsigned long long o = __shfl_xor_sync(0xffffffffu, skey[s], stride);
                    const bool lower = (lane & stride) == 0;
                    const bool desc = (i & size) == 0;
                    // lower index keeps max when desc, min otherwise; the upper the opposite
                    const bool take_max = lower == desc;
                    skey[s] = take_max ? (skey[s] > o ? skey[s] : o) : (skey[s] < o ? skey[s] : o);
                }
            }
        }
    }
#pragma unroll
    for (int s = 0; s < SLOTS; ++s) {
        const int p = 32 * s + lane;
        if (p < k_eff && skey[s] != 0ull) {
            topk[r * k_eff + p] = (int32_t)(0xffffffffu - (uint32_t)(skey[s] & 0xffffffffu));
            if (guide) guide[r * k_eff + p] = fkey_inv((uint32_t)(skey[s] >> 32));
        }
    }
}

// f32 [H][W][64] (strided) -> bf16 hi, lo contiguous + row norms
__global__ void split_kernel(const float* __restrict__ x, int64_t hs, int64_t rs, int heads, int W,
                             __nv_bfloat16* hi, __nv_bfloat16* lo, float* norm) {
    const int64_t row = (int64_t)blockIdx.x * (blockDim.x / 8) + threadIdx.x / 8;
    const int c = threadIdx.x & 7;
    float sq = 0.0f;
    if (row < (int64_t)heads * W) {
        const int h = (int)(row / W), w = (int)(row % W);
        const float* src = x + (int64_t)h * hs + (int64_t)w * rs + 8 * c;
        __nv_bfloat16 H8[8], L8[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const float v = src[i];
            H8[i] = __float2bfloat16_rn(v);
            L8[i] = __float2bfloat16_rn(v - __bfloat162float(H8[i]));
            sq = fmaf(v, v, sq);
        }
        *reinterpret_cast<uint4*>(hi + row * 64 + 8 * c) = *reinterpret_cast<uint4*>(H8);
        *reinterpret_cast<uint4*>(lo + row * 64 + 8 * c) = *reinterpret_cast<uint4*>(L8);
    }
    sq += __shfl_xor_sync(0xffffffffu, sq, 1);
    sq += __shfl_xor_sync(0xffffffffu, sq, 2);
    sq += __shfl_xor_sync(0xffffffffu, sq, 4);
    if (norm && c == 0 && row < (int64_t)heads * W) norm[row] = sqrtf(sq);
}

// per-head max |x| of an f32 [H][W][64] tensor (strided rows). grid (chunks, H); out[h]
// zeroed beforehand; |x| >= 0, so the f32 bit patterns order like the values and an
// integer atomicMax merges the chunks (order-free, deterministic)
__global__ void absmax_kernel(const float* __restrict__ x, int64_t hs, int64_t rs, int W, float* out) {
    const int h = blockIdx.y;
    const int64_t n = (int64_t)W * 64;
    const int64_t i0 = n * blockIdx.x / gridDim.x, i1 = n * (blockIdx.x + 1) / gridDim.x;
    float m = 0.0f;
    for (int64_t i = i0 + threadIdx.x; i < i1; i += blockDim.x)
        m = fmaxf(m, fabsf(x[(int64_t)h * hs + (i >> 6) * rs + (i & 63)]));
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    __shared__ float red[32];
    if ((threadIdx.x & 31) == 0) red[threadIdx.x / 32] = m;
    __syncthreads();
    if (threadIdx.x < 32) {
        m = threadIdx.x < blockDim.x / 32 ? red[threadIdx.x] : 0.0f;
        for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
        if (threadIdx.x == 0) atomicMax(reinterpret_cast<int*>(out) + h, __float_as_int(m));
    }
}

// vc f32 [H][W][64] (strided) -> fp16(vc * 2^-e_h) contiguous, e_h = vexp(vmax[h]) (the PV
// MMA operand; the epilogue multiplies O by 2^e_h)
__global__ void v16_kernel(const float* __restrict__ x, int64_t hs, int64_t rs, int heads, int W,
                           const float* __restrict__ vmax, __half* out) {
    const int64_t row = (int64_t)blockIdx.x * (blockDim.x / 8) + threadIdx.x / 8;
    const int c = threadIdx.x & 7;
    if (row >= (int64_t)heads * W) return;
    const int h = (int)(row / W), w = (int)(row % W);
    const int e = vexp(vmax[h]);
    const float* src = x + (int64_t)h * hs + (int64_t)w * rs + 8 * c;
    __half o8[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) o8[i] = __float2half_rn(ldexpf(src[i], -e));
    *reinterpret_cast<uint4*>(out + row * 64 + 8 * c) = *reinterpret_cast<uint4*>(o8);
}

// per-head mean key kbar[h] = sum_w kc[h][w] / Wk (fixed summation order: deterministic).
// Any fixed vector would do -- the scores are shifted by q.kbar per row, which changes
// neither the softmax nor the ranking -- the mean makes |kc - kbar| small when the
// key windows share a large common component (over-smoothed activations), which is
// what keeps the top-k error margin narrower than the spread of the scores.
constexpr int KMEAN_CHUNKS = 64;  // row chunks per head (grid H x 64): the 20 MB/head read is spread over the GPU
__global__ void kmean_partial_kernel(const float* __restrict__ x, int64_t hs, int64_t rs, int W, float* part_out) {
    const int h = blockIdx.y, ch = blockIdx.x, j = threadIdx.x & 63, part = threadIdx.x >> 6;
    const int w0 = (int)((int64_t)W * ch / KMEAN_CHUNKS), w1 = (int)((int64_t)W * (ch + 1) / KMEAN_CHUNKS);
    float acc = 0.0f;
    for (int w = w0 + part; w < w1; w += 4) acc += x[(int64_t)h * hs + (int64_t)w * rs + j];
    __shared__ float red[4][64];
    red[part][j] = acc;
    __syncthreads();
    if (part == 0) part_out[((int64_t)h * KMEAN_CHUNKS + ch) * 64 + j] = (red[0][j] + red[1][j]) + (red[2][j] + red[3][j]);
}
__global__ void kmean_final_kernel(const float* __restrict__ part_in, int W, float* kbar) {
    const int h = blockIdx.x, j = threadIdx.x;
    float acc = 0.0f;
    for (int ch = 0; ch < KMEAN_CHUNKS; ++ch) acc += part_in[((int64_t)h * KMEAN_CHUNKS + ch) * 64 + j];
    kbar[h * 64 + j] = acc / (float)W;
}

// c = kc - kbar (f32) -> bf16 hi, lo + norms |c| and |kc|
__global__ void center_split_kernel(const float* __restrict__ x, int64_t hs, int64_t rs, int heads, int W,
                                    const float* __restrict__ kbar, __nv_bfloat16* hi, __nv_bfloat16* lo,
                                    float* cnorm, float* knorm) {
    const int64_t row = (int64_t)blockIdx.x * (blockDim.x / 8) + threadIdx.x / 8;
    const int c = threadIdx.x & 7;
    float sq = 0.0f, sk = 0.0f;
    if (row < (int64_t)heads * W) {
        const int h = (int)(row / W), w = (int)(row % W);
        const float* src = x + (int64_t)h * hs + (int64_t)w * rs + 8 * c;
        __nv_bfloat16 H8[8], L8[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const float k = src[i];
            const float v = k - kbar[h * 64 + 8 * c + i];
            H8[i] = __float2bfloat16_rn(v);
            L8[i] = __float2bfloat16_rn(v - __bfloat162float(H8[i]));
            sq = fmaf(v, v, sq);
            sk = fmaf(k, k, sk);
        }
        *reinterpret_cast<uint4*>(hi + row * 64 + 8 * c) = *reinterpret_cast<uint4*>(H8);
        *reinterpret_cast<uint4*>(lo + row * 64 + 8 * c) = *reinterpret_cast<uint4*>(L8);
    }
#pragma unroll
    for (int o = 1; o < 8; o <<= 1) {
        sq += __shfl_xor_sync(0xffffffffu, sq, o);
        sk += __shfl_xor_sync(0xffffffffu, sk, o);
    }
    if (c == 0 && row < (int64_t)heads * W) {
        // 1 ulp of headroom: the norms bound error terms, they must not round low
        cnorm[row] = sqrtf(sq) * 1.0000002f;
        knorm[row] = sqrtf(sk) * 1.0000002f;
    }
}

// per-head max of the key-window norms (order-free, deterministic)
// grid (chunks, H); out[h] zeroed beforehand; norms are >= 0, so the f32 bit patterns
// order like the values and an integer atomicMax merges the chunks (order-free)
__global__ void rowmax_kernel(const float* __restrict__ norm, int W, float* out) {
    const int h = blockIdx.y;
    const int i0 = (int)((int64_t)W * blockIdx.x / gridDim.x), i1 = (int)((int64_t)W * (blockIdx.x + 1) / gridDim.x);
    float m = 0.0f;
    for (int i = i0 + threadIdx.x; i < i1; i += blockDim.x) m = fmaxf(m, norm[(int64_t)h * W + i]);
    __shared__ float red[32];
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x / 32] = m;
    __syncthreads();
    if (threadIdx.x < 32) {
        m = threadIdx.x < blockDim.x / 32 ? red[threadIdx.x] : 0.0f;
        for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
        if (threadIdx.x == 0) atomicMax(reinterpret_cast<int*>(out) + h, __float_as_int(m));
    }
}

__global__ void exbits_kernel(const uint8_t* __restrict__ ex, int W, int words, uint32_t* bits) {
    const int wd = blockIdx.x * blockDim.x + threadIdx.x;
    if (wd >= words) return;
    uint32_t v = 0;
    for (int b = 0; b < 32; ++b) {
        const int i = wd * 32 + b;
        if (i < W && ex[i]) v |= 1u << b;
    }
    bits[wd] = v;
}

// flagged rows (candidate list overflow / near-tie flood) -> list for the exact per-row path

// Ordered compaction of the flagged rows (ascending row ids: the fallback's blocks of 32
// then share a head). Three tiny passes: per-block counts, one-block scan, scatter.
constexpr int FL_BLOCK = 1024;
__global__ void flag_count_kernel(const uint8_t* __restrict__ flag, int64_t rows, int* block_counts) {
    const int64_t i = (int64_t)blockIdx.x * FL_BLOCK + threadIdx.x;
    const int f = (i < rows && flag[i]) ? 1 : 0;
    const int c = __syncthreads_count(f);
    if (threadIdx.x == 0) block_counts[blockIdx.x] = c;
}
__global__ void flag_scan_kernel(int* block_counts, int nb, int* total) {
    // single block, sequential chunks of blockDim.x with a shared running offset
    __shared__ int carry;
    __shared__ int wsum[32];
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (int base = 0; base < nb; base += blockDim.x) {
        const int i = base + threadIdx.x;
        const int v = i < nb ? block_counts[i] : 0;
        int x = v;  // inclusive warp scan
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, x, o);
            if ((threadIdx.x & 31) >= o) x += y;
        }
        if ((threadIdx.x & 31) == 31) wsum[threadIdx.x >> 5] = x;
        __syncthreads();
        int woff = 0;
        for (int w = 0; w < (int)(threadIdx.x >> 5); ++w) woff += wsum[w];
        if (i < nb) block_counts[i] = carry + woff + x - v;  // exclusive offset
        __syncthreads();
        if (threadIdx.x == blockDim.x - 1) carry += woff + x;
        __syncthreads();
    }
    if (threadIdx.x == 0) *total = carry;
}
__global__ void flag_scatter_kernel(const uint8_t* __restrict__ flag, int64_t rows, const int* __restrict__ offsets,
                                    int* list) {
    __shared__ int wcnt[FL_BLOCK / 32];
    const int64_t i = (int64_t)blockIdx.x * FL_BLOCK + threadIdx.x;
    const bool f = i < rows && flag[i];
    const unsigned b = __ballot_sync(0xffffffffu, f);
    if ((threadIdx.x & 31) == 0) wcnt[threadIdx.x >> 5] = __popc(b);
    __syncthreads();
    int off = offsets[blockIdx.x];
    for (int w = 0; w < (int)(threadIdx.x >> 5); ++w) off += wcnt[w];
    if (f) list[off + __popc(b & ((1u << (threadIdx.x & 31)) - 1u))] = (int)i;
}

// ---------------------------------------------------------------------------------------
// Large budgets (KCAP < k_eff <= HK_KMAX; the 2-25 % points of the budget sweep, SURVEY
// §8(f) #2). The streaming candidate lists of the main kernel would need ~k(1+ln(W/k))
// entries per row, so the softmax kernel runs without top-k and this kernel selects
// from EXACT scores: a CTA takes LK_ROWS query rows of one head, streams Kc tiles
// through shared memory (each tile serves all LK_ROWS rows), writes the rows'
// order-preserving score keys to its scratch, then per row (all 256 threads): a 4-pass
// 8-bit radix select for the k-th key T, the keys > T plus the lowest-index keys == T,
// a bitonic sort by (score desc, index asc) = topk_better (compression.hpp:67-73).
// ---------------------------------------------------------------------------------------
#ifndef LK_CTAS_N
#define LK_CTAS_N 296
#endif
constexpr int LK_ROWS = 32, LK_THREADS = 256, LK_KT = 64, LK_CTAS = LK_CTAS_N;
constexpr int LK_KMAX = 2048;
constexpr int LK_QS = 68;  // padded row strides (floats) of the shared q / k tiles: no bank conflicts
constexpr int LK_CL = 2048;  // keys sharing the k-th key's top 16 bits, kept in shared memory (fast path)
constexpr size_t LK_SMEM = (size_t)(LK_ROWS + 2 * LK_KT) * LK_QS * 4 + (size_t)LK_KMAX * 8 + (size_t)LK_ROWS * 256 * 4 +
                           (size_t)LK_CL * 8;  // ~107 KB: two CTAs per SM

// 16-byte global -> shared copies that bypass registers (LDGSTS); src_bytes 0 zero-fills
__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gmem_src, int src_bytes) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_u32(smem_dst)), "l"(gmem_src),
                 "r"(src_bytes)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

// Radix digit search by warp 0 over a 256-bin histogram: the largest digit d with
// (count of digits >= d) >= need; writes d and the count strictly above it.
__device__ __forceinline__ void lk_find_digit(const int* hist, int need, int lane, int* out_digit, int* out_above) {
    int c[8], tot = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        c[i] = hist[8 * lane + i];
        tot += c[i];
    }
    int incl = tot;  // suffix scan over lanes: bins of lanes >= this one
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_down_sync(0xffffffffu, incl, o);
        if (lane + o < 32) incl += v;
    }
    int suf = incl - tot, found = -1, above_d = 0;
#pragma unroll
    for (int i = 7; i >= 0; --i) {
        if (found < 0 && suf + c[i] >= need) {
            found = 8 * lane + i;
            above_d = suf;
        }
        suf += c[i];
    }
    const unsigned b = __ballot_sync(0xffffffffu, found >= 0);
    const int src = 31 - __clz(b);
    const int d = __shfl_sync(0xffffffffu, found, src);
    const int ab = __shfl_sync(0xffffffffu, above_d, src);
    if (lane == 0) {
        *out_digit = d;
        *out_above = ab;
    }
}

// Budgets beyond the shared sort buffer (LK_KMAX < k_eff <= HK_KMAX: the 10 % and 25 %
// points of the budget sweep, k = 4050 / 10125 at 500 views). Per row, from the row's
// exact keys in the scratch: an 8-bit radix select of the k-th key T (4 passes; the
// first histogram was accumulated while the keys were written), the winners (every key
// > T, then the lowest-index keys == T) collected in index order by block scans, and a
// block radix sort of their unique 64-bit keys (fkey(score) << 32 | ~index) descending
// = topk_better order (compression.hpp:67-73). Shared memory: HK_SMEM past LK_SMEM.
constexpr int HK_IPT = 40;                      // keys per thread of the block radix sort
constexpr int HK_KMAX = LK_THREADS * HK_IPT;    // 10240
static_assert(HK_KMAX == kMaxTopK, "tc.h kMaxTopK is the huge-k capacity");
using HkSort = cub::BlockRadixSort<unsigned long long, LK_THREADS, HK_IPT>;
using HkScan = cub::BlockScan<int, LK_THREADS>;
constexpr size_t HK_WIN_BYTES = (size_t)HK_KMAX * 8;  // collected winners (64-bit keys)
constexpr size_t HK_SMEM = (HK_WIN_BYTES > sizeof(typename HkSort::TempStorage) ? HK_WIN_BYTES
                                                                                  : sizeof(typename HkSort::TempStorage)) +
                           sizeof(typename HkScan::TempStorage) + 256;

__device__ void hugek_row(const uint32_t* __restrict__ rk, int Wk, int k_eff, const int* row_hist, int64_t row,
                          int32_t* topk, float* guide, uint8_t* hk, int* hist, int* sh) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    unsigned long long* win = reinterpret_cast<unsigned long long*>(hk);
    typename HkSort::TempStorage& sort_tmp = *reinterpret_cast<typename HkSort::TempStorage*>(hk);  // aliases win
    typename HkScan::TempStorage& scan_tmp =
        *reinterpret_cast<typename HkScan::TempStorage*>(hk + (HK_SMEM - 256 - sizeof(typename HkScan::TempStorage)));
    // 1. radix select of the k-th largest key
    uint32_t prefix = 0;
    int need = k_eff;
    for (int pass = 0; pass < 4; ++pass) {
        const int shift = 24 - 8 * pass;
        __syncthreads();
        if (pass == 0) {
            for (int i = tid; i < 256; i += LK_THREADS) hist[i] = row_hist[i];
        } else {
            for (int i = tid; i < 256; i += LK_THREADS) hist[i] = 0;
            __syncthreads();
            for (int j = tid; j < Wk; j += LK_THREADS) {
                const uint32_t key = rk[j];
                if ((key >> (shift + 8)) == prefix) atomicAdd(&hist[(key >> shift) & 255u], 1);
            }
        }
        __syncthreads();
        if (warp == 0) lk_find_digit(hist, need, lane, &sh[0], &sh[1]);
        __syncthreads();
        prefix = (prefix << 8) | (uint32_t)sh[0];
        need -= sh[1];
    }
    const uint32_t T = prefix;  // need = how many keys == T to take (lowest indices first)
    // 2. winners in index order
    int base = 0, eq_base = 0;
    for (int j0 = 0; j0 < Wk; j0 += LK_THREADS) {
        const int j = j0 + tid;
        const uint32_t key = j < Wk ? rk[j] : 0u;
        const int eq = (j < Wk && key == T) ? 1 : 0;
        int eq_rank, eq_tot;
        HkScan(scan_tmp).ExclusiveSum(eq, eq_rank, eq_tot);
        __syncthreads();
        const int take = (j < Wk && (key > T || (eq && eq_base + eq_rank < need))) ? 1 : 0;
        int pos, tot;
        HkScan(scan_tmp).ExclusiveSum(take, pos, tot);
        __syncthreads();
        if (take) win[base + pos] = ((unsigned long long)key << 32) | (0xffffffffu - (uint32_t)j);
        base += tot;
        eq_base += eq_tot;
    }
    __syncthreads();
    // 3. sort descending (unique keys: no stability needed), write in rank order
    unsigned long long keys[HK_IPT];
#pragma unroll
    for (int i = 0; i < HK_IPT; ++i) {
        const int q = tid * HK_IPT + i;
        keys[i] = q < k_eff ? win[q] : 0ull;
    }
    __syncthreads();  // the sort's temp storage aliases win
    HkSort(sort_tmp).SortDescending(keys);
#pragma unroll
    for (int i = 0; i < HK_IPT; ++i) {
        const int q = tid * HK_IPT + i;
        if (q < k_eff) {
            topk[row * k_eff + q] = (int32_t)(0xffffffffu - (uint32_t)(keys[i] & 0xffffffffu));
            if (guide) guide[row * k_eff + q] = fkey_inv((uint32_t)(keys[i] >> 32));
        }
    }
    __syncthreads();
}

#pragma nv_diag_suppress 128  // the HUGE instance leaves the k <= LK_KMAX row body unreachable
template <bool HUGE>  // HUGE: k_eff > LK_KMAX (hugek_row); a separate instance keeps the common one's registers low
__global__ void __launch_bounds__(LK_THREADS) largek_topk_kernel(
    const float* __restrict__ qc, int64_t q_hs, const float* __restrict__ kc, int heads, int Wq, int Wk, float scale,
    int k_eff, const uint32_t* __restrict__ exbits, uint32_t* scratch, int32_t* topk, float* guide,
    const int* __restrict__ row_list = nullptr, const int* __restrict__ row_count = nullptr) {
    // row_list mode (the exact fallback of the main path): the rows are the listed ones
    // (ascending, so mostly one head per block of 32); otherwise every row of every head
    extern __shared__ __align__(16) uint8_t lk_smem[];
    float* qs = reinterpret_cast<float*>(lk_smem);                           // [LK_ROWS][LK_QS]
    float* ks2 = qs + LK_ROWS * LK_QS;                                       // [2][LK_KT][LK_QS] (double buffer)
    unsigned long long* sb = reinterpret_cast<unsigned long long*>(ks2 + 2 * LK_KT * LK_QS);  // [LK_KMAX] sort buffer
    int* rhist = reinterpret_cast<int*>(sb + LK_KMAX);                       // [LK_ROWS][256] pass-0 histograms
    unsigned long long* cl = reinterpret_cast<unsigned long long*>(rhist + LK_ROWS * 256);  // [LK_CL] bin list
    __shared__ int hist[256];
    __shared__ int sh_digit, sh_above, sh_cnt_gt, sh_eq_taken, sh_cl, sh_fast;
    __shared__ int warp_cnt[LK_THREADS / 32];
    __shared__ int row_id[LK_ROWS], row_h[LK_ROWS];
    __shared__ int hk_sh[2];
    uint32_t* sk = scratch + (size_t)blockIdx.x * LK_ROWS * Wk;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int blocks_per_head = (Wq + LK_ROWS - 1) / LK_ROWS;
    const int n_list = row_list ? *row_count : 0;
    const int nblocks = row_list ? (n_list + LK_ROWS - 1) / LK_ROWS : heads * blocks_per_head;
    for (int blk = blockIdx.x; blk < nblocks; blk += gridDim.x) {
        int nr;
        __syncthreads();
        if (row_list) {
            nr = min(LK_ROWS, n_list - blk * LK_ROWS);
            if (tid < nr) {
                row_id[tid] = row_list[blk * LK_ROWS + tid];
                row_h[tid] = row_id[tid] / Wq;
            }
        } else {
            const int hb = blk / blocks_per_head, w0 = (blk - hb * blocks_per_head) * LK_ROWS;
            nr = min(LK_ROWS, Wq - w0);
            if (tid < nr) {
                row_id[tid] = hb * Wq + w0 + tid;
                row_h[tid] = hb;
            }
        }
        for (int i = tid; i < LK_ROWS * 256; i += LK_THREADS) rhist[i] = 0;
        __syncthreads();
        // one pass over the keys per distinct head among the block's rows
        for (int done = 0; done < nr;) {
        const int h = row_h[done];
        int span = done;
        while (span < nr && row_h[span] == h) ++span;  // rows [done, span) share head h (list ascending)
        for (int i = tid; i < LK_ROWS * 64; i += LK_THREADS) {
            const int rr = i / 64;
            qs[rr * LK_QS + (i & 63)] =
                (rr >= done && rr < span) ? qc[(int64_t)h * q_hs + (int64_t)(row_id[rr] - h * Wq) * 64 + (i & 63)] : 0.0f;
        }
        // ---- exact scores of the block's rows against every key window; the next Kc
        // tile streams into the other buffer (cp.async) while this one is scored
        auto load_tile = [&](int kt0, float* dst) {
            for (int i = tid; i < LK_KT * 16; i += LK_THREADS) {
                const int j = kt0 + i / 16;
                const float* src = kc + ((int64_t)h * Wk + (j < Wk ? j : 0)) * 64 + 4 * (i & 15);
                cp_async16(dst + (i / 16) * LK_QS + 4 * (i & 15), src, j < Wk ? 16 : 0);
            }
            cp_async_commit();
        };
        __syncthreads();
        load_tile(0, ks2);
        for (int kt0 = 0, tb = 0; kt0 < Wk; kt0 += LK_KT, tb ^= 1) {
            float* ks = ks2 + tb * LK_KT * LK_QS;
            if (kt0 + LK_KT < Wk) {
                load_tile(kt0 + LK_KT, ks2 + (tb ^ 1) * LK_KT * LK_QS);
                cp_async_wait<1>();
            } else {
                cp_async_wait<0>();
            }
            __syncthreads();
            const int r = tid >> 3;  // row of this thread; 8 threads per row, keys jj0 + 8 i
            const int jj0 = tid & 7;
            if (r >= done && r < span) {
                // 8 independent dots per thread (32 add chains in flight), dot.hpp:11-23 order
                ExactDot4 d[LK_KT / 8];
#pragma unroll
                for (int i = 0; i < LK_KT / 8; ++i) d[i].zero();
                const float4* a = reinterpret_cast<const float4*>(qs + r * LK_QS);
#pragma unroll 4
                for (int x = 0; x < 16; ++x) {
                    const float4 av = a[x];
#pragma unroll
                    for (int i = 0; i < LK_KT / 8; ++i) {
                        const float4 bv = reinterpret_cast<const float4*>(ks + (jj0 + 8 * i) * LK_QS)[x];
                        d[i].step(av.x, av.y, av.z, av.w, bv.x, bv.y, bv.z, bv.w);
                    }
                }
#pragma unroll
                for (int i = 0; i < LK_KT / 8; ++i) {
                    const int j = kt0 + jj0 + 8 * i;
                    if (j < Wk) {
                        const bool ex = exbits && ((exbits[j >> 5] >> (j & 31)) & 1u);
                        // +0.0f folds -0 into +0: the keys order like topk_better's float compare
                        const uint32_t key = ex ? 0u : fkey(d[i].finish(scale) + 0.0f);
                        sk[(size_t)r * Wk + j] = key;
                        atomicAdd(&rhist[r * 256 + (key >> 24)], 1);  // radix pass 0, fused
                    }
                }
            }
            __syncthreads();  // this buffer is refilled by the prefetch of the next iteration
        }
        __syncthreads();
        done = span;
        }
        // ---- per row: radix select, collect, sort, write
#ifdef LK_SKIP_SELECT
        continue;
#endif
        for (int r = 0; r < nr; ++r) {
            const uint32_t* rk = sk + (size_t)r * Wk;
            if constexpr (HUGE) {  // budgets past the shared sort buffer (the rest is the k <= LK_KMAX body)
                hugek_row(rk, Wk, k_eff, rhist + r * 256, row_id[r], topk, guide, lk_smem + LK_SMEM, hist, hk_sh);
                continue;
            }
            // ---- fast path: digits 0 (fused histogram) and 1 (one scan); then ONE scan sends
            // the keys above the 16-bit prefix bin straight to the sort buffer and the bin's
            // keys to a shared list, where digits 2 and 3 are resolved
            {
                for (int i = tid; i < 256; i += LK_THREADS) hist[i] = rhist[r * 256 + i];
                __syncthreads();
                if (warp == 0) lk_find_digit(hist, k_eff, lane, &sh_digit, &sh_above);
                __syncthreads();
                const uint32_t d0 = (uint32_t)sh_digit;
                int need = k_eff - sh_above;
                for (int i = tid; i < 256; i += LK_THREADS) hist[i] = 0;
                __syncthreads();
                for (int j = tid; j < Wk; j += LK_THREADS) {
                    const uint32_t key = rk[j];
                    if ((key >> 24) == d0) atomicAdd(&hist[(key >> 16) & 255u], 1);
                }
                __syncthreads();
                if (warp == 0) lk_find_digit(hist, need, lane, &sh_digit, &sh_above);
                __syncthreads();
                const uint32_t p16 = (d0 << 8) | (uint32_t)sh_digit;
                const int bin_n = hist[sh_digit];
                need -= sh_above;
                __syncthreads();
                if (tid == 0) {
                    sh_cnt_gt = 0;
                    sh_cl = 0;
                    sh_fast = bin_n <= LK_CL;
                }
                __syncthreads();
                if (sh_fast) {
                    for (int j = tid; j < Wk; j += LK_THREADS) {
                        const uint32_t key = rk[j];
                        const uint32_t t16 = key >> 16;
                        const unsigned long long e = ((unsigned long long)key << 32) | (0xffffffffu - (uint32_t)j);
                        if (t16 > p16) sb[atomicAdd(&sh_cnt_gt, 1)] = e;
                        else if (t16 == p16) cl[atomicAdd(&sh_cl, 1)] = e;
                    }
                    __syncthreads();
                    const int m = sh_cl;
                    uint32_t prefix = p16;
                    int cnt_eq = 0;
                    for (int pass = 2; pass < 4; ++pass) {
                        const int shift = 24 - 8 * pass;
                        for (int i = tid; i < 256; i += LK_THREADS) hist[i] = 0;
                        __syncthreads();
                        for (int i = tid; i < m; i += LK_THREADS) {
                            const uint32_t key = (uint32_t)(cl[i] >> 32);
                            if ((key >> (shift + 8)) == prefix) atomicAdd(&hist[(key >> shift) & 255u], 1);
                        }
                        __syncthreads();
                        if (warp == 0) lk_find_digit(hist, need, lane, &sh_digit, &sh_above);
                        __syncthreads();
                        prefix = (prefix << 8) | (uint32_t)sh_digit;
                        need -= sh_above;
                        cnt_eq = hist[sh_digit];
                        __syncthreads();
                    }
                    const uint32_t T = prefix;
                    if (cnt_eq == need) {  // every key equal to T is taken: no tie ordering needed
                        for (int i = tid; i < m; i += LK_THREADS) {
                            const unsigned long long e = cl[i];
                            if ((uint32_t)(e >> 32) >= T) sb[atomicAdd(&sh_cnt_gt, 1)] = e;
                        }
                        __syncthreads();
                    } else {
                        if (tid == 0) sh_fast = 0;  // ties straddle the k-th place: ordered path
                        __syncthreads();
                    }
                }
            }
            if (!sh_fast) {
            uint32_t prefix = 0;
            int need = k_eff;  // still to take at or below the current prefix
            for (int pass = 0; pass < 4; ++pass) {
                const int shift = 24 - 8 * pass;
                if (pass == 0) {  // accumulated while the scores were written
                    for (int i = tid; i < 256; i += LK_THREADS) hist[i] = rhist[r * 256 + i];
                    __syncthreads();
                } else {
                    for (int i = tid; i < 256; i += LK_THREADS) hist[i] = 0;
                    __syncthreads();
                    for (int j = tid; j < Wk; j += LK_THREADS) {
                        const uint32_t key = rk[j];
                        if ((key >> (shift + 8)) == prefix) atomicAdd(&hist[(key >> shift) & 255u], 1);
                    }
                    __syncthreads();
                }
                if (warp == 0) {
                    // suffix sums over 256 bins: lane l owns bins 8l..8l+7
                    int c[8], tot = 0;
#pragma unroll
                    for (int i = 0; i < 8; ++i) {
                        c[i] = hist[8 * lane + i];
                        tot += c[i];
                    }
                    int incl = tot;  // suffix scan over lanes: bins of lanes >= this one
#pragma unroll
                    for (int o = 1; o < 32; o <<= 1) {
                        const int v = __shfl_down_sync(0xffffffffu, incl, o);
                        if (lane + o < 32) incl += v;
                    }
                    const int above = incl - tot;  // count in the bins of higher lanes
                    // digit d: suffix(d+1) < need <= suffix(d)
                    int suf = above, found = -1, above_d = 0;
#pragma unroll
                    for (int i = 7; i >= 0; --i) {
                        if (found < 0 && suf + c[i] >= need) {
                            found = 8 * lane + i;
                            above_d = suf;
                        }
                        suf += c[i];
                    }
                    const unsigned b = __ballot_sync(0xffffffffu, found >= 0);
                    const int src = 31 - __clz(b);  // the highest lane holding the digit
                    const int d = __shfl_sync(0xffffffffu, found, src);
                    const int ab = __shfl_sync(0xffffffffu, above_d, src);
                    if (lane == 0) {
                        sh_digit = d;
                        sh_above = ab;
                    }
                }
                __syncthreads();
                prefix = (prefix << 8) | (uint32_t)sh_digit;
                need -= sh_above;
            }
            const uint32_t T = prefix;  // the k-th largest key; `need` keys equal to T are taken
            // collect: keys > T (their count is k_eff - need) in any order, then the `need`
            // lowest-index keys == T, in index order
            if (tid == 0) {
                sh_cnt_gt = 0;
                sh_eq_taken = 0;
            }
            __syncthreads();
            for (int j0 = 0; j0 < Wk; j0 += LK_THREADS) {
                const int j = j0 + tid;
                const uint32_t key = j < Wk ? rk[j] : 0u;
                const bool gt = j < Wk && key > T;
                const bool eq = j < Wk && key == T;
                if (gt) {
                    const int slot = atomicAdd(&sh_cnt_gt, 1);
                    sb[slot] = ((unsigned long long)key << 32) | (0xffffffffu - (uint32_t)j);
                }
                // ties in index order: block-wide exclusive prefix of eq
                const unsigned be = __ballot_sync(0xffffffffu, eq);
                if (lane == 0) warp_cnt[warp] = __popc(be);
                __syncthreads();
                int before = 0, tot = 0;
                for (int i = 0; i < LK_THREADS / 32; ++i) {
                    before += i < warp ? warp_cnt[i] : 0;
                    tot += warp_cnt[i];
                }
                const int rank = sh_eq_taken + before + __popc(be & ((1u << lane) - 1u));
                if (eq && rank < need)
                    sb[(k_eff - need) + rank] = ((unsigned long long)key << 32) | (0xffffffffu - (uint32_t)j);
                __syncthreads();
                if (tid == 0) sh_eq_taken += tot;
            }
            __syncthreads();
            }  // ordered (slow) path
            __syncthreads();
            // bitonic sort of sb[0..n2) descending (pad with 0 = below every real entry)
#ifdef LK_SKIP_SORT
            continue;
#endif
            int n2 = 1;
            while (n2 < k_eff) n2 <<= 1;
            for (int i = k_eff + tid; i < n2; i += LK_THREADS) sb[i] = 0ull;
            __syncthreads();
            for (int size = 2; size <= n2; size <<= 1) {
                for (int stride = size >> 1; stride > 0; stride >>= 1) {
                    for (int i = tid; i < n2 / 2; i += LK_THREADS) {
                        const int lo = 2 * i - (i & (stride - 1));
                        const int hi = lo + stride;
                        const bool desc = (lo & size) == 0;
                        const unsigned long long a = sb[lo], b = sb[hi];
                        if ((a < b) == desc) {
                            sb[lo] = b;
                            sb[hi] = a;
                        }
                    }
                    __syncthreads();
                }
            }
            const int64_t row = row_id[r];
            for (int i = tid; i < k_eff; i += LK_THREADS) {
                const unsigned long long e = sb[i];
                topk[row * k_eff + i] = (int32_t)(0xffffffffu - (uint32_t)(e & 0xffffffffu));
                if (guide) guide[row * k_eff + i] = fkey_inv((uint32_t)(e >> 32));
            }
            __syncthreads();
        }
    }
}

struct Ws {
    __nv_bfloat16 *qh, *ql, *kh, *kl;
    __half* v16;
    float *qn, *kn, *kmax, *vmax;
    float *cn, *cmax, *kbar, *kpart;
    uint32_t* exbits;
    float2* cand;
    int* cand_n;
    uint8_t* flag;
    int* blocks;
    int* nblocks;
    uint32_t* scratch;
    size_t used;
};

// dense: softmax-only use (tc_dense_f32: no top-k, so no candidate lists / scratch)
Ws carve_ws(void* base, int heads, int Wq, int Wk, int k_eff, bool dry, bool dense = false) {
    Ws w{};
    size_t off = 0;
    auto take = [&](size_t bytes) -> char* {
        off = (off + 255) & ~size_t(255);
        char* p = dry ? nullptr : static_cast<char*>(base) + off;
        off += bytes;
        return p;
    };
    const size_t nq = (size_t)heads * Wq, nk = (size_t)heads * Wk;
    w.qh = reinterpret_cast<__nv_bfloat16*>(take(nq * 128));
    w.ql = reinterpret_cast<__nv_bfloat16*>(take(nq * 128));
    w.kh = reinterpret_cast<__nv_bfloat16*>(take(nk * 128));
    w.kl = reinterpret_cast<__nv_bfloat16*>(take(nk * 128));
    w.v16 = reinterpret_cast<__half*>(take(nk * 128));
    w.vmax = reinterpret_cast<float*>(take((size_t)heads * 4));
    w.qn = reinterpret_cast<float*>(take(nq * 4));
    w.kn = reinterpret_cast<float*>(take(nk * 4));
    w.kmax = reinterpret_cast<float*>(take((size_t)heads * 4));
    w.cn = reinterpret_cast<float*>(take(nk * 4));
    w.cmax = reinterpret_cast<float*>(take((size_t)heads * 4));
    w.kbar = reinterpret_cast<float*>(take((size_t)heads * 64 * 4));
    w.kpart = reinterpret_cast<float*>(take((size_t)heads * KMEAN_CHUNKS * 64 * 4));
    w.exbits = reinterpret_cast<uint32_t*>(take((size_t)((Wk + 127) / 128) * 16));
    const bool large_k = k_eff > KCAP;  // exact large-budget selection: no candidate lists
    const size_t nl = dense ? 1 : nq;
    w.cand = reinterpret_cast<float2*>(take(large_k || dense ? 8 : nq * (size_t)ccap_for(k_eff, true) * 8));
    w.cand_n = reinterpret_cast<int*>(take(nl * 4));
    w.flag = reinterpret_cast<uint8_t*>(take(nl));
    w.blocks = reinterpret_cast<int*>(take(nl * 4 + ((nl + 1023) / 1024 + 1) * 4));  // flagged rows + block counts
    w.nblocks = reinterpret_cast<int*>(take(4));
    w.scratch = reinterpret_cast<uint32_t*>(take(dense ? 4 : (size_t)LK_CTAS * LK_ROWS * Wk * 4));  // large-k / fallback scores
    w.used = off + 256;
    return w;
}

bool contiguous_f32(const gsa_tensor& t) {
    return t.dtype == GSA_DTYPE_F32 && t.dim == 64 && (reinterpret_cast<uintptr_t>(t.data) & 15) == 0 &&
           t.row_stride == 64 && t.head_stride == (int64_t)t.rows * 64;
}

}  // namespace

size_t tc_compress_workspace_bytes(int heads, int windows, int dim, int k_eff) {
    return tc_compress_workspace_bytes_qk(heads, windows, windows, dim, k_eff);
}

size_t tc_compress_workspace_bytes_qk(int heads, int wq, int wk, int dim, int k_eff) {
    if (dim != 64 || k_eff > HK_KMAX) return 0;
    return carve_ws(nullptr, heads, wq, wk, k_eff, true).used;
}

bool tc_compress_split_buffers(void* ws, size_t ws_bytes, int heads, int windows, int dim, int k_eff,
                               CompressSplits* out) {
    if (dim != 64 || k_eff > HK_KMAX || !ws || ws_bytes < carve_ws(nullptr, heads, windows, windows, k_eff, true).used)
        return false;
    Ws w = carve_ws(ws, heads, windows, windows, k_eff, false);
    *out = CompressSplits{w.qh, w.ql, w.qn};
    return true;
}

cudaError_t tc_compress_topk(const gsa_tensor& qc, const gsa_tensor& kc, const gsa_tensor& vc, int k_eff, float scale,
                             const uint8_t* excluded, float* out, int64_t out_hs, int64_t out_rs, float* lse,
                             int32_t* topk, float* guide, void* ws, size_t ws_bytes, cudaStream_t st) {
    return tc_compress_topk_splits(nullptr, qc, kc, vc, k_eff, scale, excluded, out, out_hs, out_rs, lse, topk, guide,
                                   ws, ws_bytes, st);
}

cudaError_t tc_compress_topk_splits(const CompressSplits* pre, const gsa_tensor& qc, const gsa_tensor& kc,
                                    const gsa_tensor& vc, int k_eff, float scale, const uint8_t* excluded,
                                    float* out, int64_t out_hs, int64_t out_rs, float* lse, int32_t* topk,
                                    float* guide, void* ws, size_t ws_bytes, cudaStream_t st) {
    const int H = qc.heads, Wq = qc.rows, Wk = kc.rows;
    AttnArgs ex{};  // exact CUDA-core kernel (phase-1 path and fallback)
    ex.q = TensorRef{qc.data, qc.dtype, qc.head_stride, qc.row_stride};
    ex.k = TensorRef{kc.data, kc.dtype, kc.head_stride, kc.row_stride};
    ex.v = TensorRef{vc.data, vc.dtype, vc.head_stride, vc.row_stride};
    ex.heads = H;
    ex.mq = Wq;
    ex.mk = Wk;
    ex.dim = qc.dim;
    ex.scale = scale;
    ex.out = out;
    ex.out_hs = out_hs;
    ex.out_rs = out_rs;
    ex.lse = lse;
    ex.topk = k_eff > 0 ? topk : nullptr;
    ex.guide = guide;
    ex.k_eff = k_eff;
    ex.excluded = excluded;
    const bool tc_ok = qc.dim == 64 && k_eff <= HK_KMAX && contiguous_f32(qc) && contiguous_f32(kc) &&
                       contiguous_f32(vc) && tmap_encode_fn() != nullptr && ws &&
                       ws_bytes >= carve_ws(nullptr, H, Wq, Wk, k_eff, true).used && Wq > 0 && Wk > 0;
    if (!tc_ok) return launch_attn_f32(ex, st);

    Ws w = carve_ws(ws, H, Wq, Wk, k_eff, false);
    const __nv_bfloat16 *qh = w.qh, *ql = w.ql, *kh = w.kh, *kl = w.kl;
    const float* qn = w.qn;
    if (pre) {  // Q splits + norms written by the pooling pass
        qh = pre->qh;
        ql = pre->ql;
        qn = pre->qnorm;
    } else {
        const unsigned qb = (unsigned)(((int64_t)H * Wq + 31) / 32);
        split_kernel<<<qb, 256, 0, st>>>(static_cast<const float*>(qc.data), qc.head_stride, qc.row_stride, H, Wq,
                                          w.qh, w.ql, w.qn);
        note_launch();
    }
    // V as the fp16 PV operand, scaled per head by a power of two into fp16 range
    cudaMemsetAsync(w.vmax, 0, (size_t)H * 4, st);
    absmax_kernel<<<dim3(32, H), 256, 0, st>>>(static_cast<const float*>(vc.data), vc.head_stride, vc.row_stride,
                                               Wk, w.vmax);
    v16_kernel<<<(unsigned)(((int64_t)H * Wk + 31) / 32), 256, 0, st>>>(
        static_cast<const float*>(vc.data), vc.head_stride, vc.row_stride, H, Wk, w.vmax, w.v16);
    note_launch(2);
    // centred keys for the scores (kc - kbar), written over the K splits
    kmean_partial_kernel<<<dim3(KMEAN_CHUNKS, H), 256, 0, st>>>(static_cast<const float*>(kc.data), kc.head_stride,
                                                                 kc.row_stride, Wk, w.kpart);
    kmean_final_kernel<<<H, 64, 0, st>>>(w.kpart, Wk, w.kbar);
    center_split_kernel<<<(unsigned)(((int64_t)H * Wk + 31) / 32), 256, 0, st>>>(
        static_cast<const float*>(kc.data), kc.head_stride, kc.row_stride, H, Wk, w.kbar, w.kh, w.kl, w.cn, w.kn);
    const float* kn = w.kn;
    cudaMemsetAsync(w.kmax, 0, (size_t)H * 4, st);
    cudaMemsetAsync(w.cmax, 0, (size_t)H * 4, st);
    rowmax_kernel<<<dim3(32, H), 256, 0, st>>>(kn, Wk, w.kmax);
    rowmax_kernel<<<dim3(32, H), 256, 0, st>>>(w.cn, Wk, w.cmax);
    note_launch(5);
    const int tiles = (Wk + 127) / 128;
    if (excluded) {
        exbits_kernel<<<(tiles * 4 + 127) / 128, 128, 0, st>>>(excluded, Wk, tiles * 4, w.exbits);
        note_launch();
    }
    CUtensorMap tqh, tql, tkh, tkl, tv16;
    const int64_t qhs = (int64_t)Wq * 64, khs = (int64_t)Wk * 64;
    // (2-byte elements: the bf16 tensor-map type moves the fp16 V tile bit for bit)
    if (!make_rows_tmap(&tqh, qh, H, Wq, qhs, 64) || !make_rows_tmap(&tql, ql, H, Wq, qhs, 64) ||
        !make_rows_tmap(&tkh, kh, H, Wk, khs, 64) || !make_rows_tmap(&tkl, kl, H, Wk, khs, 64) ||
        !make_rows_tmap(&tv16, reinterpret_cast<const __nv_bfloat16*>(w.v16), H, Wk, khs, 64))
        return launch_attn_f32(ex, st);
    CompParams p{};
    p.heads = H;
    p.Wq = Wq;
    p.Wk = Wk;
    p.k_eff = k_eff > KCAP ? 0 : k_eff;  // large budgets: softmax only here, exact selection below
    p.scale = scale;
    p.c2 = scale * 1.4426950408889634f;
    p.kv_tiles = tiles;
    p.qnorm = qn;
    p.kmax = w.kmax;
    p.cmax = w.cmax;
    p.kbar = w.kbar;
    p.qc = static_cast<const float*>(qc.data);
    p.qc_hs = qc.head_stride;
    p.qc_rs = qc.row_stride;
    p.vmax = w.vmax;
    p.exbits = excluded ? w.exbits : nullptr;
    p.out = out;
    p.out_hs = out_hs;
    p.out_rs = out_rs;
    p.lse = lse;
    p.cand = w.cand;
#ifdef COMPRESS_PROF
    static unsigned long long* prof_buf = nullptr;
    if (!prof_buf) cudaMalloc(&prof_buf, 256);
    p.prof = prof_buf;
#endif
    p.ccap = ccap_for(k_eff, excluded != nullptr);
    p.cand_n = w.cand_n;
    p.flag = w.flag;
    const size_t smem = sizeof(CompSmem) + 1024;
    cudaError_t e = cudaFuncSetAttribute(compress_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    stage_mark(5, st);  // (instrumentation: the kernel's own duration)
    compress_tc_kernel<<<dim3((Wq + 128 * NWG - 1) / (128 * NWG), H), NTHREADS, smem, st>>>(tqh, tql, tkh, tkl, tv16, p);
    stage_mark(6, st);
    note_launch();
#ifdef COMPRESS_PROF
    {
        unsigned long long hp[17];
        cudaMemcpyAsync(hp, p.prof, sizeof(hp), cudaMemcpyDeviceToHost, st);
        cudaStreamSynchronize(st);
        fprintf(stderr, "compress prof (CTA0 warp0): tiles %llu  wait_S %.0f  pass A %.0f  pass B (softmax+P+topk) %.0f  raise %.0f cyc/tile\n", hp[5],
                (double)hp[0] / hp[5], (double)hp[1] / hp[5], (double)hp[3] / hp[5], (double)hp[4] / hp[5]);
        fprintf(stderr, "compress prof (CTA0 MMA warp): per key tile  wait TMA %.0f  wait P %.0f  total %.0f cyc\n",
                (double)hp[6] / hp[5], (double)hp[7] / hp[5], (double)hp[8] / hp[5]);
        fprintf(stderr, "compress prof (CTA0 warp0): extraction iterations %llu  candidates/row %.1f  masked chunks %llu of %llu\n",
                hp[9], (double)hp[10] / 32.0, hp[11], 4 * hp[5]);
        fprintf(stderr, "compress prof (CTA0 warp0): pass B per tile: ld %.0f  softmax %.0f  wait_st+arrive %.0f  (rest = top-k)\n",
                (double)hp[12] / hp[5], (double)hp[13] / hp[5], (double)hp[14] / hp[5]);
        fprintf(stderr, "compress prof (CTA0 warp0): pass B per tile: pre-extraction %.0f  extraction %.0f\n",
                (double)hp[15] / hp[5], (double)hp[16] / hp[5]);
    }
#endif
    if (k_eff > KCAP) {
        const bool huge = k_eff > LK_KMAX;
        const size_t lk_smem = LK_SMEM + (huge ? HK_SMEM : 0);
        auto kern = huge ? largek_topk_kernel<true> : largek_topk_kernel<false>;
        cudaError_t e2 = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)lk_smem);
        if (e2 != cudaSuccess) return e2;
        kern<<<LK_CTAS, LK_THREADS, lk_smem, st>>>(static_cast<const float*>(qc.data), qc.head_stride,
                                                    static_cast<const float*>(kc.data), H, Wq, Wk, scale, k_eff,
                                                    excluded ? w.exbits : nullptr, w.scratch, topk, guide, nullptr,
                                                    nullptr);
        note_launch();
        return cudaGetLastError();
    }
    if (k_eff > 0) {
        const int64_t rows = (int64_t)H * Wq;
        const float* qcp = static_cast<const float*>(qc.data);
        const float* kcp = static_cast<const float*>(kc.data);
        const unsigned rb = (unsigned)((rows + 7) / 8);
        const int cs = ccap_for(k_eff, excluded != nullptr);
        if (k_eff <= 32) {
            static_assert(ccap_for(32) <= 1024 && ccap_for(32, true) <= 1024 && surv_for(32) == 2 * 32, "rescore instances");
            rescore_kernel<16, 2><<<rb, 256, 8 * 64 * sizeof(float2), st>>>(
                qcp, qc.head_stride, kcp, H, Wq, Wk, scale, k_eff, qn, w.kmax, w.cmax, w.cand, cs, -1, 512, w.cand_n,
                w.flag, topk, guide);
            rescore_kernel<32, 2><<<rb, 256, 8 * 64 * sizeof(float2), st>>>(
                qcp, qc.head_stride, kcp, H, Wq, Wk, scale, k_eff, qn, w.kmax, w.cmax, w.cand, cs, 512, 1024, w.cand_n,
                w.flag, topk, guide);
            note_launch();
        } else {
            static_assert(ccap_for(128) == 64 * 32 && ccap_for(128, true) == 64 * 32 && surv_for(128) == 8 * 32, "rescore instance");
            rescore_kernel<64, 8><<<rb, 256, 8 * 256 * sizeof(float2), st>>>(
                qcp, qc.head_stride, kcp, H, Wq, Wk, scale, k_eff, qn, w.kmax, w.cmax, w.cand, cs, -1, 2048, w.cand_n,
                w.flag, topk, guide);
        }
        note_launch();
        // rows whose candidate list overflowed (near-tie floods, clumps of near-equal keys):
        // exact recompute of just those rows by the large-k kernel in row-list mode (exact
        // scores tiled over blocks of 32 listed rows, radix select, lowest-index ties, sort)
        const unsigned nfb = (unsigned)((rows + FL_BLOCK - 1) / FL_BLOCK);
        int* fl_counts = w.blocks + rows;  // carve_ws reserves rows + nfb ints
        flag_count_kernel<<<nfb, FL_BLOCK, 0, st>>>(w.flag, rows, fl_counts);
        flag_scan_kernel<<<1, 1024, 0, st>>>(fl_counts, (int)nfb, w.nblocks);
        flag_scatter_kernel<<<nfb, FL_BLOCK, 0, st>>>(w.flag, rows, fl_counts, w.blocks);
        const size_t lk_smem = LK_SMEM;
        cudaError_t e3 = cudaFuncSetAttribute(largek_topk_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)lk_smem);
        if (e3 != cudaSuccess) return e3;
        largek_topk_kernel<false><<<LK_CTAS, LK_THREADS, lk_smem, st>>>(static_cast<const float*>(qc.data), qc.head_stride,
                                                                  static_cast<const float*>(kc.data), H, Wq, Wk, scale,
                                                                  k_eff, excluded ? w.exbits : nullptr, w.scratch, topk,
                                                                  guide, w.blocks, w.nblocks);
        note_launch(4);
#ifdef GSA_DEBUG_STATS
        {  // bring-up builds only: candidate statistics (synchronises)
            const int64_t rows = (int64_t)H * Wq;
            std::vector<int> cn(rows);
            std::vector<uint8_t> fl(rows);
            int nblk = 0;
            cudaMemcpyAsync(cn.data(), w.cand_n, rows * 4, cudaMemcpyDeviceToHost, st);
            cudaMemcpyAsync(fl.data(), w.flag, rows, cudaMemcpyDeviceToHost, st);
            cudaMemcpyAsync(&nblk, w.nblocks, 4, cudaMemcpyDeviceToHost, st);
            cudaStreamSynchronize(st);
            int64_t sum = 0, mx = 0, nfl = 0, nzero = 0, nover = 0, nflood = 0;
            for (int64_t i = 0; i < rows; ++i) {
                sum += cn[i];
                mx = cn[i] > mx ? cn[i] : mx;
                nfl += fl[i] ? 1 : 0;
                nover += fl[i] == 1 ? 1 : 0;
                nflood += fl[i] == 2 ? 1 : 0;
                nzero += cn[i] == 0 ? 1 : 0;
            }
            fprintf(stderr, "compress stats: rows %lld mean cand %.1f max %lld flagged %lld (list overflow %lld, "
                    "survivor flood %lld) zero %lld blocks %d\n",
                    (long long)rows, (double)sum / rows, (long long)mx, (long long)nfl, (long long)nover,
                    (long long)nflood, (long long)nzero, nblk);
            int shown = 0;
            for (int64_t i = 0; i < rows && shown < 8; ++i)
                if (fl[i]) {
                    fprintf(stderr, "  flagged row %lld (h %lld, w %lld)\n", (long long)i, (long long)(i / Wq), (long long)(i % Wq));
                    ++shown;
                }
        }
#endif
    }
    return cudaGetLastError();
}

size_t tc_dense_f32_workspace_bytes(int heads, int mq, int mk) {
    return carve_ws(nullptr, heads, mq, mk, 0, true, true).used;
}

// Dense attention of f32 Q/K/V on the tensor cores: the compressed-branch kernel in
// softmax-only mode (no top-k). Scores from the bf16 hi/lo split of Q and of the
// centred keys (S = Qh.Kh + Qh.Kl + Ql.Kh, ~2^-16 relative), P.V in fp16 with V
// scaled per head (~2^-11 relative in O), lse exact to the split. q rows
// [q_row_offset, + mq) of q; out rows written at out + h*out_hs + r*out_rs.
cudaError_t tc_dense_f32(const gsa_tensor& q, int q_row_offset, int mq, const gsa_tensor& k, const gsa_tensor& v,
                         float scale, float* out, int64_t out_hs, int64_t out_rs, float* lse, void* ws,
                         size_t ws_bytes, cudaStream_t st) {
    const int H = q.heads, Wk = k.rows;
    if (mq == 0) return cudaSuccess;
    if (q.dtype != GSA_DTYPE_F32 || k.dtype != GSA_DTYPE_F32 || v.dtype != GSA_DTYPE_F32 || q.dim != 64 || Wk == 0 ||
        !tmap_encode_fn())
        return cudaErrorNotSupported;
    void* own = nullptr;
    const size_t need = tc_dense_f32_workspace_bytes(H, mq, Wk);
    if (!ws || ws_bytes < need) {  // operator entry points without a workspace argument
        cudaError_t e = cudaMallocAsync(&own, need, st);
        if (e != cudaSuccess) return e;
        ws = own;
    }
    Ws w = carve_ws(ws, H, mq, Wk, 0, false, true);
    const float* qb = static_cast<const float*>(q.data) + (int64_t)q_row_offset * q.row_stride;
    split_kernel<<<(unsigned)(((int64_t)H * mq + 31) / 32), 256, 0, st>>>(qb, q.head_stride, q.row_stride, H, mq,
                                                                          w.qh, w.ql, w.qn);
    cudaMemsetAsync(w.vmax, 0, (size_t)H * 4, st);
    cudaMemsetAsync(w.kmax, 0, (size_t)H * 4, st);  // (top-k margins: unused without a top-k)
    cudaMemsetAsync(w.cmax, 0, (size_t)H * 4, st);
    absmax_kernel<<<dim3(32, H), 256, 0, st>>>(static_cast<const float*>(v.data), v.head_stride, v.row_stride, Wk,
                                               w.vmax);
    v16_kernel<<<(unsigned)(((int64_t)H * Wk + 31) / 32), 256, 0, st>>>(
        static_cast<const float*>(v.data), v.head_stride, v.row_stride, H, Wk, w.vmax, w.v16);
    kmean_partial_kernel<<<dim3(KMEAN_CHUNKS, H), 256, 0, st>>>(static_cast<const float*>(k.data), k.head_stride,
                                                                 k.row_stride, Wk, w.kpart);
    kmean_final_kernel<<<H, 64, 0, st>>>(w.kpart, Wk, w.kbar);
    center_split_kernel<<<(unsigned)(((int64_t)H * Wk + 31) / 32), 256, 0, st>>>(
        static_cast<const float*>(k.data), k.head_stride, k.row_stride, H, Wk, w.kbar, w.kh, w.kl, w.cn, w.kn);
    note_launch(6);
    CUtensorMap tqh, tql, tkh, tkl, tv16;
    const int64_t qhs = (int64_t)mq * 64, khs = (int64_t)Wk * 64;
    cudaError_t e = cudaSuccess;
    if (!make_rows_tmap(&tqh, w.qh, H, mq, qhs, 64) || !make_rows_tmap(&tql, w.ql, H, mq, qhs, 64) ||
        !make_rows_tmap(&tkh, w.kh, H, Wk, khs, 64) || !make_rows_tmap(&tkl, w.kl, H, Wk, khs, 64) ||
        !make_rows_tmap(&tv16, reinterpret_cast<const __nv_bfloat16*>(w.v16), H, Wk, khs, 64))
        e = cudaErrorNotSupported;
    if (e == cudaSuccess) {
        CompParams p{};
        p.heads = H;
        p.Wq = mq;
        p.Wk = Wk;
        p.k_eff = 0;
        p.scale = scale;
        p.c2 = scale * 1.4426950408889634f;
        p.kv_tiles = (Wk + 127) / 128;
        p.qnorm = w.qn;
        p.kmax = w.kmax;
        p.cmax = w.cmax;
        p.kbar = w.kbar;
        p.qc = qb;
        p.qc_hs = q.head_stride;
        p.qc_rs = q.row_stride;
        p.vmax = w.vmax;
        p.out = out;
        p.out_hs = out_hs;
        p.out_rs = out_rs;
        p.lse = lse;
        p.cand = w.cand;
        p.ccap = 1;
        p.cand_n = w.cand_n;
        p.flag = w.flag;
        const size_t smem = sizeof(CompSmem) + 1024;
        e = cudaFuncSetAttribute(compress_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e == cudaSuccess) {
            compress_tc_kernel<<<dim3((mq + 128 * NWG - 1) / (128 * NWG), H), NTHREADS, smem, st>>>(tqh, tql, tkh, tkl,
                                                                                                 tv16, p);
            note_launch();
            e = cudaGetLastError();
        }
    }
    if (own) cudaFreeAsync(own, st);
    return e;
}

}  // namespace gsa_sm100
