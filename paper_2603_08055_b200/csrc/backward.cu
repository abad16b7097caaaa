// backward.cu — the CUDA-core side of the layer backward (gsa_backward, gradients.hpp:
// 54-265): the elementwise steps every call runs, and the attention / projection passes for
// the shapes the tensor-core kernels do not take (head dim != 64, window side != 4). At
// d = 64, s = 4 the dense passes run in bwd_tc.cu, the selection passes in sel_bwd_tc.cu and
// the projection backward in proj_bwd_tc.cu.
//
// The backward of each branch is the flash-style recomputation the reference
// uses: probabilities are rebuilt from the saved log-sum-exp rows,
// p = exp(scale * q.k - lse), dS = p * (dO.v - D) * scale with D = dO.o, and the
// top-k selection is a constant (gradients.hpp:52-54). Every gradient is
// produced by exactly one owner thread per element and kernels touching the same
// output run in a fixed stream order, so the result is deterministic without
// floating-point atomics.
//
// Every call:
//   gate_bwd         gate fuse (gradients.hpp:96-119): dS_sel = (1-g) dO, dz =
//                    g(1-g)(O_comp - O_sel) dO, dq_img = W_g dz (written), the
//                    window sums of g dO (upsample backward, :122-128) and the D
//                    rows of both branches (8 windows per CTA, W_g staged once)
//   pool_bwd         pooled-gradient scatter (avg-pool adjoint, :158-169)
//   inverse plan     (head, key window, query window) keys radix-sorted: each key
//                    window's query windows, ascending (the selection key-side passes)
//   atb / atb_reduce dW = A^T B split over rows with a fixed-order reduction of the
//                    partials (dW_g = Q_img^T dz)
//   hybrid helpers   the plan without its forced windows, forced-frame row gathers and
//                    the scatter-add of their dK / dV
// Other shapes:
//   dense_bwd_dkdv   FlashAttention-2 key-side pass (one CTA per 64 keys, loop over
//   dense_bwd_dq     every query tile) and query-side pass: the compressed branch
//                    (:131-155, windows x windows) and the special rows (:197-222)
//   sel16_bwd / sel_bwd_dq / sel_bwd_dkdv  selection branch (:172-194) over the plan
//                    and its inverse
//   atb, dx_gemm     projection backward (:245-263)
//
// The dense tiles use one register blocking: 256 threads as a 16 x 16 grid, thread
// (ty, tx) owning rows ty + 16 i and columns tx + 16 j, so every shared-memory read is
// either a broadcast or 16 distinct padded rows (conflict-free).
#include <cub/device/device_radix_sort.cuh>

#include "kernels.h"

namespace gsa_sm100 {
namespace {

constexpr int BT = 256;  // threads per CTA
constexpr int TB = 64;   // dense tiles: 64 queries x 64 keys
constexpr int GATE_WPC = 8;  // windows per CTA in the gate-fuse backward

// ------------------------------------------------------------------ gate fuse
template <int DP>
__global__ void __launch_bounds__(BT) gate_bwd_kernel(GateBwdArgs a) {
    extern __shared__ __align__(16) float sm[];
    const DevLayout& L = a.L;
    const int dim = a.dim, s2 = L.s * L.s, W = L.windows, Mi = L.image_tokens, Ms = L.num_special;
    float* wg = sm;                   // [DP][DP+4]: W_g^T (wg[j][c] = W_g[c][j])
    float* dz = wg + DP * (DP + 4);   // [s2][DP]
    float* dcf = dz + s2 * DP;        // [s2][DP]  g * dO (upsample-backward terms)
    float* pr = dcf + s2 * DP;        // [s2][DP]  dS_sel * O_sel (D_sel terms)
    float* red = pr + s2 * DP;        // [DP]      dO_comp * O_comp (D_comp terms)
    // a CTA takes GATE_WPC consecutive windows of one head: W_g is staged once for all of them
    const int nblk = (W + GATE_WPC - 1) / GATE_WPC;
    const int h = blockIdx.x / nblk, w0 = (blockIdx.x - h * nblk) * GATE_WPC;
    const int tid = threadIdx.x;

    const float* wgh = a.w_g + (int64_t)h * dim * dim;
    // W_g^T, zero-padded to DP x DP (rows of DP + 1 floats would break float4 alignment:
    // use DP + 4 like the dense tiles)
    for (int e = tid; e < DP * DP; e += BT) {
        const int j = e / DP, c = e - j * DP;
        wg[j * (DP + 4) + c] = (j < dim && c < dim) ? wgh[c * dim + j] : 0.0f;
    }
    for (int w = w0; w < min(W, w0 + GATE_WPC); ++w) {
        __syncthreads();  // W_g staged; the previous window's smem rows consumed
        if (dim < DP)
            for (int e = tid; e < s2 * DP; e += BT)
                if (e % DP >= dim) dz[e] = 0.0f;
        const float* comp = a.o_comp + ((int64_t)h * W + w) * dim;
        for (int e = tid; e < s2 * dim; e += BT) {
            const int m = e / dim, j = e - m * dim;
            const int i = L.member(w, m);
            const int64_t r = ((int64_t)h * Mi + i) * dim + j;
            const float go = a.dout.p[(int64_t)h * a.dout.hs + (int64_t)(Ms + i) * a.dout.rs + j];
            const float g = a.gate[r], sel = a.o_sel[r];
            const float ds = (1.0f - g) * go;
            const float dzv = g * (1.0f - g) * ((comp[j] - sel) * go);
            a.ds[r] = ds;
            a.dz[r] = dzv;
            dz[m * DP + j] = dzv;
            dcf[m * DP + j] = g * go;
            pr[m * DP + j] = ds * sel;
        }
        __syncthreads();
        // upsample backward: window sum of g * dO in ascending member order
        for (int j = tid; j < dim; j += BT) {
            float acc = 0.0f;
            for (int m = 0; m < s2; ++m) acc += dcf[m * DP + j];
            a.d_oc[((int64_t)h * W + w) * dim + j] = acc;
            red[j] = acc * comp[j];
        }
        // D_sel rows: one warp per member row
        const int warp = tid >> 5, lane = tid & 31;
        for (int m = warp; m < s2; m += BT / 32) {
            float acc = 0.0f;
            for (int j = lane; j < dim; j += 32) acc += pr[m * DP + j];
            for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
            if (lane == 0) a.d_sel[(int64_t)h * Mi + L.member(w, m)] = acc;
        }
        // dq_img = W_g dz (gradients.hpp:108-117), written: the first contribution to dQ.
        // Thread: one member row x 4 consecutive features; float4 reads of dz and W_g^T rows
        for (int e = tid; e < s2 * (DP / 4); e += BT) {
            const int m = e / (DP / 4), c0 = 4 * (e - m * (DP / 4));
            float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 4
            for (int j = 0; j < DP; j += 4) {
                const float4 z = *reinterpret_cast<const float4*>(dz + m * DP + j);
                const float zz[4] = {z.x, z.y, z.z, z.w};
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const float4 wv = *reinterpret_cast<const float4*>(wg + (j + u) * (DP + 4) + c0);
                    acc.x = fmaf(wv.x, zz[u], acc.x);
                    acc.y = fmaf(wv.y, zz[u], acc.y);
                    acc.z = fmaf(wv.z, zz[u], acc.z);
                    acc.w = fmaf(wv.w, zz[u], acc.w);
                }
            }
            float* dst = a.dq.p + (int64_t)h * a.dq.hs + (int64_t)(Ms + L.member(w, m)) * a.dq.rs + c0;
            const float av[4] = {acc.x, acc.y, acc.z, acc.w};
#pragma unroll
            for (int u = 0; u < 4; ++u)
                if (c0 + u < dim) dst[u] = av[u];
        }
        __syncthreads();
        if (warp == 0) {
            float acc = 0.0f;
            for (int j = lane; j < dim; j += 32) acc += red[j];
            for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
            if (lane == 0) a.d_comp[(int64_t)h * W + w] = acc;
        }
    }
}

// ---------------------------------------------------------- dense attention
// Tiles of 64 rows padded to DP + 4 floats (16-byte aligned rows: float4 reads, and 16
// consecutive rows start 4 banks apart, so a float4 read of 16 rows takes the minimum
// two wavefronts). P / dS tiles are 64 x 68.
constexpr int PT = TB + 4;

template <int DP>
__device__ __forceinline__ void load_tile(float* dst, const FMat& m, int h, int64_t r0, int64_t rows, int dim) {
    constexpr int RP = DP + 4;
    for (int e = threadIdx.x; e < TB * DP; e += BT) {
        const int r = e / DP, j = e - r * DP;
        float x = 0.0f;
        if (r0 + r < rows && j < dim) x = m.p[(int64_t)h * m.hs + (r0 + r) * m.rs + j];
        dst[r * RP + j] = x;
    }
}

__device__ __forceinline__ float4 ld4(const float* p) { return *reinterpret_cast<const float4*>(p); }
__device__ __forceinline__ float dot4(float4 a, float4 b, float c) {
    return fmaf(a.w, b.w, fmaf(a.z, b.z, fmaf(a.y, b.y, fmaf(a.x, b.x, c))));
}

// S and dP of the 64 x 64 tile (thread: query rows ty + 16 i, keys tx + 16 j), then
// P = exp(scale S - lse) and dS = P (dP - D) scale into Ps / dSs, either [q][k]
// (TRANS = false) or [k][q]; keys >= kn get P = dS = 0.
template <int DP, bool TRANS>
__device__ __forceinline__ void score_tile(const float* Qs, const float* dOs, const float* Ks, const float* Vs,
                                           const float* lse, const float* D, int kn, float scale, float* Ps,
                                           float* dSs) {
    constexpr int RP = DP + 4;
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    float s[4][4], dp[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) s[i][j] = dp[i][j] = 0.0f;
#pragma unroll 2
    for (int d = 0; d < DP; d += 4) {
        float4 qv[4], ov[4], kv[4], vv[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            qv[i] = ld4(Qs + (ty + 16 * i) * RP + d);
            ov[i] = ld4(dOs + (ty + 16 * i) * RP + d);
            kv[i] = ld4(Ks + (tx + 16 * i) * RP + d);
            vv[i] = ld4(Vs + (tx + 16 * i) * RP + d);
        }
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                s[i][j] = dot4(qv[i], kv[j], s[i][j]);
                dp[i][j] = dot4(ov[i], vv[j], dp[i][j]);
            }
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int q = ty + 16 * i;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int k = tx + 16 * j;
            const float p = k < kn ? expf(s[i][j] * scale - lse[q]) : 0.0f;
            const int at = TRANS ? k * PT + q : q * PT + k;
            Ps[at] = p;
            dSs[at] = p * (dp[i][j] - D[q]) * scale;
        }
    }
}

__device__ __forceinline__ void load_stats(float* lse_s, float* D_s, const DenseBwdArgs& a, int h, int64_t q0) {
    for (int r = threadIdx.x; r < TB; r += BT) {
        const int64_t q = q0 + r;
        const bool ok = q < a.nq;
        lse_s[r] = ok ? a.lse[(int64_t)h * a.lse_hs + q] : INFINITY;  // exp(-inf) = 0 for padding rows
        D_s[r] = ok ? a.D[(int64_t)h * a.D_hs + q] : 0.0f;
    }
}

// rows 4 ty + i (i < 4) x features 4 tx + 64 c (c < DP / 64, 4 each) of an accumulator tile
template <int DP>
__device__ __forceinline__ void store_rows(float (*acc)[DP / 16], const FOut& o, int h, int64_t r0, int64_t rows,
                                           int dim, bool accumulate) {
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int64_t r = r0 + 4 * ty + i;
        if (r >= rows) continue;
        float* row = o.p + (int64_t)h * o.hs + r * o.rs;
#pragma unroll
        for (int c = 0; c < DP / 64; ++c)
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int j = 64 * c + 4 * tx + e;
                if (j < dim) row[j] = accumulate ? row[j] + acc[i][4 * c + e] : acc[i][4 * c + e];
            }
    }
}

// key side: one CTA per (64 keys, head); dK, dV accumulated over every query tile.
// Accumulators: keys 4 ty + i, features 4 tx + 64 c + e.
template <int DP>
__global__ void __launch_bounds__(BT) dense_bwd_dkdv_kernel(DenseBwdArgs a) {
    extern __shared__ __align__(16) float sm[];
    constexpr int RP = DP + 4, RS = TB * RP, NC = DP / 64, NA = DP / 16;
    float* Ks = sm;
    float* Vs = Ks + RS;
    float* Qs = Vs + RS;
    float* dOs = Qs + RS;
    float* Ps = dOs + RS;  // [q][k]
    float* dSs = Ps + TB * PT;
    float* lse_s = dSs + TB * PT;
    float* D_s = lse_s + TB;
    const int h = blockIdx.y;
    const int64_t k0 = (int64_t)blockIdx.x * TB;
    const int kn = (int)min((int64_t)TB, a.nk - k0);
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    load_tile<DP>(Ks, a.k, h, k0, a.nk, a.dim);
    load_tile<DP>(Vs, a.v, h, k0, a.nk, a.dim);
    float adk[4][NA], adv[4][NA];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < NA; ++j) adk[i][j] = adv[i][j] = 0.0f;

    for (int64_t q0 = 0; q0 < a.nq; q0 += TB) {
        __syncthreads();
        load_tile<DP>(Qs, a.q, h, q0, a.nq, a.dim);
        load_tile<DP>(dOs, a.dout, h, q0, a.nq, a.dim);
        load_stats(lse_s, D_s, a, h, q0);
        __syncthreads();
        score_tile<DP, false>(Qs, dOs, Ks, Vs, lse_s, D_s, kn, a.scale, Ps, dSs);
        __syncthreads();
#pragma unroll 2
        for (int q = 0; q < TB; ++q) {
            const float4 p = ld4(Ps + q * PT + 4 * ty), ds = ld4(dSs + q * PT + 4 * ty);
            const float pv[4] = {p.x, p.y, p.z, p.w}, dv[4] = {ds.x, ds.y, ds.z, ds.w};
#pragma unroll
            for (int c = 0; c < NC; ++c) {
                const float4 o = ld4(dOs + q * RP + 64 * c + 4 * tx), x = ld4(Qs + q * RP + 64 * c + 4 * tx);
                const float ov[4] = {o.x, o.y, o.z, o.w}, xv[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        adv[i][4 * c + e] = fmaf(pv[i], ov[e], adv[i][4 * c + e]);
                        adk[i][4 * c + e] = fmaf(dv[i], xv[e], adk[i][4 * c + e]);
                    }
            }
        }
    }
    if (a.dk.p) store_rows<DP>(adk, a.dk, h, k0, a.nk, a.dim, a.accumulate);
    if (a.dv.p) store_rows<DP>(adv, a.dv, h, k0, a.nk, a.dim, a.accumulate);
}

// query side: one CTA per (64 queries, head, key split); dQ accumulated over the split's
// key tiles, written (or, with splits, stored as a partial the reduction sums in order)
template <int DP>
__global__ void __launch_bounds__(BT) dense_bwd_dq_kernel(DenseBwdArgs a) {
    extern __shared__ __align__(16) float sm[];
    constexpr int RP = DP + 4, RS = TB * RP, NC = DP / 64, NA = DP / 16;
    float* Qs = sm;
    float* dOs = Qs + RS;
    float* Ks = dOs + RS;
    float* Vs = Ks + RS;
    float* Ps = Vs + RS;
    float* dSs = Ps + TB * PT;  // [k][q]
    float* lse_s = dSs + TB * PT;
    float* D_s = lse_s + TB;
    const int h = blockIdx.z, split = blockIdx.y;
    const int64_t q0 = (int64_t)blockIdx.x * TB;
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    load_tile<DP>(Qs, a.q, h, q0, a.nq, a.dim);
    load_tile<DP>(dOs, a.dout, h, q0, a.nq, a.dim);
    load_stats(lse_s, D_s, a, h, q0);
    float adq[4][NA];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < NA; ++j) adq[i][j] = 0.0f;

    const int64_t kb = (int64_t)split * a.k_chunk, ke = min(a.nk, kb + a.k_chunk);
    for (int64_t k0 = kb; k0 < ke; k0 += TB) {
        const int kn = (int)min((int64_t)TB, ke - k0);
        __syncthreads();
        load_tile<DP>(Ks, a.k, h, k0, ke, a.dim);
        load_tile<DP>(Vs, a.v, h, k0, ke, a.dim);
        __syncthreads();
        score_tile<DP, true>(Qs, dOs, Ks, Vs, lse_s, D_s, kn, a.scale, Ps, dSs);
        __syncthreads();
#pragma unroll 2
        for (int k = 0; k < TB; ++k) {
            const float4 ds = ld4(dSs + k * PT + 4 * ty);
            const float dv[4] = {ds.x, ds.y, ds.z, ds.w};
#pragma unroll
            for (int c = 0; c < NC; ++c) {
                const float4 x = ld4(Ks + k * RP + 64 * c + 4 * tx);
                const float xv[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int e = 0; e < 4; ++e) adq[i][4 * c + e] = fmaf(dv[i], xv[e], adq[i][4 * c + e]);
            }
        }
    }
    if (a.k_splits > 1) {
        const FOut part{a.dq_part + (int64_t)split * a.heads * a.nq * a.dim, a.nq * a.dim, a.dim};
        store_rows<DP>(adq, part, h, q0, a.nq, a.dim, false);
    } else {
        store_rows<DP>(adq, a.dq, h, q0, a.nq, a.dim, a.accumulate);
    }
}

// dQ from the key-split partials, summed in split order
__global__ void dq_reduce_kernel(DenseBwdArgs a) {
    const int64_t n = (int64_t)a.heads * a.nq * a.dim, stride = n;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
        const int j = (int)(e % a.dim);
        const int64_t q = (e / a.dim) % a.nq, h = e / ((int64_t)a.dim * a.nq);
        float acc = 0.0f;
        for (int s = 0; s < a.k_splits; ++s) acc += a.dq_part[s * stride + e];
        float* o = a.dq.p + h * a.dq.hs + q * a.dq.rs + j;
        *o = a.accumulate ? *o + acc : acc;
    }
}

// ------------------------------------------------------------ pool adjoint
// dq_img += dQc[w] / s^2; dk_img = dKc[w] / s^2; dv_img = dVc[w] / s^2; special rows of
// dk / dv zeroed (the special pass accumulates into every row afterwards)
__global__ void pool_bwd_kernel(PoolBwdArgs a) {
    const int64_t n = (int64_t)a.heads * a.rows * a.dim;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
        const int j = (int)(e % a.dim);
        const int64_t t = (e / a.dim) % a.rows;
        const int h = (int)(e / ((int64_t)a.dim * a.rows));
        const int64_t ok = (int64_t)h * a.dk.hs + t * a.dk.rs + j, ov = (int64_t)h * a.dv.hs + t * a.dv.rs + j;
        if (t < a.L.num_special) {
            a.dk.p[ok] = 0.0f;
            a.dv.p[ov] = 0.0f;
            continue;
        }
        const int w = a.L.window_of_token((int)(t - a.L.num_special));
        const int64_t c = ((int64_t)h * a.L.windows + w) * a.dim + j;
        float* pq = a.dq.p + (int64_t)h * a.dq.hs + t * a.dq.rs + j;
        *pq += a.dqc[c] * a.inv;
        a.dk.p[ok] = a.dkc[c] * a.inv;
        a.dv.p[ov] = a.dvc[c] * a.inv;
    }
}

// -------------------------------------------------------- selection branch
template <int DP>
__device__ __forceinline__ float dot_rows(const float* a, const float* b) {
    float acc = 0.0f;
#pragma unroll 8
    for (int d = 0; d < DP; ++d) acc = fmaf(a[d], b[d], acc);
    return acc;
}

constexpr int CK = 64;  // keys (or queries) staged per chunk

// query side: CTA per (head, query window); the s^2 queries share the plan row
template <int DP>
__global__ void __launch_bounds__(BT) sel_bwd_dq_kernel(SelBwdArgs a) {
    extern __shared__ __align__(16) float sm[];
    const DevLayout& L = a.L;
    const int dim = a.dim, s2 = L.s * L.s, W = L.windows, Mi = L.image_tokens, Ms = L.num_special;
    constexpr int RP = DP + 1;
    float* Qs = sm;               // [s2][RP]
    float* dOs = Qs + s2 * RP;    // [s2][RP]  dS_sel rows
    float* Ks = dOs + s2 * RP;    // [CK][RP]
    float* Vs = Ks + CK * RP;     // [CK][RP]
    float* dSs = Vs + CK * RP;    // [s2][CK+1]
    float* lse_s = dSs + s2 * (CK + 1);
    float* D_s = lse_s + s2;
    __shared__ int ktok[CK];
    const int64_t row = blockIdx.x;
    const int h = (int)(row / W), w = (int)(row - (int64_t)h * W);
    const int tid = threadIdx.x;
    for (int e = tid; e < s2 * DP; e += BT) {
        const int m = e / DP, j = e - m * DP;
        const int i = L.member(w, m);
        Qs[m * RP + j] = j < dim ? a.q.p[(int64_t)h * a.q.hs + (int64_t)(Ms + i) * a.q.rs + j] : 0.0f;
        dOs[m * RP + j] = j < dim ? a.ds[((int64_t)h * Mi + i) * dim + j] : 0.0f;
    }
    for (int m = tid; m < s2; m += BT) {
        const int i = L.member(w, m);
        lse_s[m] = a.lse[(int64_t)h * Mi + i];
        D_s[m] = a.D[(int64_t)h * Mi + i];
    }
    constexpr int R = CK * DP / BT;  // accumulator slots per thread (covers s2 <= 64)
    float acc[R];
#pragma unroll
    for (int r = 0; r < R; ++r) acc[r] = 0.0f;

    const int64_t nkeys = (a.offsets[row + 1] - a.offsets[row]) * s2;
    const int32_t* ids = a.ids + a.offsets[row];
    for (int64_t k0 = 0; k0 < nkeys; k0 += CK) {
        const int kn = (int)min((int64_t)CK, nkeys - k0);
        __syncthreads();
        if (tid < CK) {
            const int64_t kk = k0 + tid;
            ktok[tid] = tid < kn ? L.member(ids[kk / s2], (int)(kk % s2)) : 0;
        }
        __syncthreads();
        for (int e = tid; e < CK * DP; e += BT) {
            const int r = e / DP, j = e - r * DP;
            float kx = 0.0f, vx = 0.0f;
            if (r < kn && j < dim) {
                const int64_t t = Ms + ktok[r];
                kx = a.k.p[(int64_t)h * a.k.hs + t * a.k.rs + j];
                vx = a.v.p[(int64_t)h * a.v.hs + t * a.v.rs + j];
            }
            Ks[r * RP + j] = kx;
            Vs[r * RP + j] = vx;
        }
        __syncthreads();
        for (int e = tid; e < s2 * CK; e += BT) {
            const int m = e / CK, c = e - m * CK;
            float ds = 0.0f;
            if (c < kn) {
                const float p = expf(dot_rows<DP>(Qs + m * RP, Ks + c * RP) * a.scale - lse_s[m]);
                ds = p * (dot_rows<DP>(dOs + m * RP, Vs + c * RP) - D_s[m]) * a.scale;
            }
            dSs[m * (CK + 1) + c] = ds;
        }
        __syncthreads();
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const int e = tid + r * BT;
            const int m = e / DP, j = e - m * DP;
            if (m < s2) {
                float x = acc[r];
                for (int c = 0; c < kn; ++c) x = fmaf(dSs[m * (CK + 1) + c], Ks[c * RP + j], x);
                acc[r] = x;
            }
        }
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int e = tid + r * BT;
        const int m = e / DP, j = e - m * DP;
        if (m < s2 && j < dim) a.dq.p[(int64_t)h * a.dq.hs + (int64_t)(Ms + L.member(w, m)) * a.dq.rs + j] += acc[r];
    }
}

// key side: CTA per (head, key window); the query windows come from the inverse plan
template <int DP>
__global__ void __launch_bounds__(BT) sel_bwd_dkdv_kernel(SelBwdArgs a) {
    extern __shared__ __align__(16) float sm[];
    const DevLayout& L = a.L;
    const int dim = a.dim, s2 = L.s * L.s, W = L.windows, Mi = L.image_tokens, Ms = L.num_special;
    constexpr int RP = DP + 1;
    float* Ks = sm;               // [s2][RP]
    float* Vs = Ks + s2 * RP;     // [s2][RP]
    float* Qs = Vs + s2 * RP;     // [CK][RP]
    float* dOs = Qs + CK * RP;    // [CK][RP]
    float* Ps = dOs + CK * RP;    // [CK][s2+1]
    float* dSs = Ps + CK * (s2 + 1);
    float* lse_s = dSs + CK * (s2 + 1);
    float* D_s = lse_s + CK;
    __shared__ int qtok[CK];
    const int64_t row = blockIdx.x;
    const int h = (int)(row / W), w = (int)(row - (int64_t)h * W);
    const int tid = threadIdx.x;
    for (int e = tid; e < s2 * DP; e += BT) {
        const int m = e / DP, j = e - m * DP;
        const int64_t t = Ms + L.member(w, m);
        Ks[m * RP + j] = j < dim ? a.k.p[(int64_t)h * a.k.hs + t * a.k.rs + j] : 0.0f;
        Vs[m * RP + j] = j < dim ? a.v.p[(int64_t)h * a.v.hs + t * a.v.rs + j] : 0.0f;
    }
    constexpr int R = CK * DP / BT;
    float acck[R], accv[R];
#pragma unroll
    for (int r = 0; r < R; ++r) acck[r] = accv[r] = 0.0f;

    const int64_t nq = (a.inv_offsets[row + 1] - a.inv_offsets[row]) * s2;
    const int32_t* qwins = a.inv_q + a.inv_offsets[row];
    for (int64_t q0 = 0; q0 < nq; q0 += CK) {
        const int qn = (int)min((int64_t)CK, nq - q0);
        __syncthreads();
        if (tid < CK) {
            const int64_t qq = q0 + tid;
            const int i = tid < qn ? L.member(qwins[qq / s2], (int)(qq % s2)) : 0;
            qtok[tid] = i;
            lse_s[tid] = tid < qn ? a.lse[(int64_t)h * Mi + i] : INFINITY;
            D_s[tid] = tid < qn ? a.D[(int64_t)h * Mi + i] : 0.0f;
        }
        __syncthreads();
        for (int e = tid; e < CK * DP; e += BT) {
            const int r = e / DP, j = e - r * DP;
            float qx = 0.0f, ox = 0.0f;
            if (r < qn && j < dim) {
                const int i = qtok[r];
                qx = a.q.p[(int64_t)h * a.q.hs + (int64_t)(Ms + i) * a.q.rs + j];
                ox = a.ds[((int64_t)h * Mi + i) * dim + j];
            }
            Qs[r * RP + j] = qx;
            dOs[r * RP + j] = ox;
        }
        __syncthreads();
        for (int e = tid; e < CK * s2; e += BT) {
            const int r = e / s2, c = e - r * s2;
            float p = 0.0f, ds = 0.0f;
            if (r < qn) {
                p = expf(dot_rows<DP>(Qs + r * RP, Ks + c * RP) * a.scale - lse_s[r]);
                ds = p * (dot_rows<DP>(dOs + r * RP, Vs + c * RP) - D_s[r]) * a.scale;
            }
            Ps[r * (s2 + 1) + c] = p;
            dSs[r * (s2 + 1) + c] = ds;
        }
        __syncthreads();
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const int e = tid + r * BT;
            const int c = e / DP, j = e - c * DP;
            if (c < s2) {
                float xk = acck[r], xv = accv[r];
                for (int q = 0; q < qn; ++q) {
                    xv = fmaf(Ps[q * (s2 + 1) + c], dOs[q * RP + j], xv);
                    xk = fmaf(dSs[q * (s2 + 1) + c], Qs[q * RP + j], xk);
                }
                acck[r] = xk;
                accv[r] = xv;
            }
        }
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int e = tid + r * BT;
        const int c = e / DP, j = e - c * DP;
        if (c < s2 && j < dim) {
            const int64_t t = Ms + L.member(w, c);
            a.dk.p[(int64_t)h * a.dk.hs + t * a.dk.rs + j] += acck[r];
            a.dv.p[(int64_t)h * a.dv.hs + t * a.dv.rs + j] += accv[r];
        }
    }
}

// s = 4 fast path of both selection passes, register-tiled: a CTA (128 threads) owns the
// 16 rows of one window (the FIXED side: its queries, or with KEYSIDE its keys) and streams
// the GATHERED side in chunks of 64 rows (4 windows of the plan row, or of the inverse plan
// row). Per chunk:
//   S = A1 . B1^T and T = A2 . B2^T (16 x 64; thread: fixed rows la + 4 i, gathered rows
//   16 warp + lb + 8 j), P = exp(scale S - lse), dS = P (T - D) scale -> X (and P -> Y)
//   stored [gathered][fixed];
//   out1 += X^T B1 (and out2 += Y^T B2) (thread: fixed rows 4 la + i, features
//   warp DP/4 + lb DP/32 + e).
// dq pass:   A1 = Q, A2 = dS_sel rows, B1 = K, B2 = V; stats by fixed row; out1 = dQ.
// dkdv pass: A1 = K, A2 = V, B1 = Q, B2 = dS_sel rows; stats by gathered row; out1 = dK,
//            out2 = dV.
// Every shared read is a broadcast or 4 / 8 consecutive padded rows (one wavefront).
constexpr int SF = 16, SG = 64, ST = 128, XP = SF + 4;

__device__ __forceinline__ float4 ldg4(const float* p) { return __ldg(reinterpret_cast<const float4*>(p)); }

template <int DP, bool KEYSIDE>
__global__ void __launch_bounds__(ST) sel16_bwd_kernel(SelBwdArgs a) {
    extern __shared__ __align__(16) float sm[];
    constexpr int RP = DP + 4, ND = DP / 32, C4 = DP / 4;
    float* A1 = sm;
    float* A2 = A1 + SF * RP;
    float* B1 = A2 + SF * RP;
    float* B2 = B1 + SG * RP;
    float* X = B2 + SG * RP;
    float* Y = X + SG * XP;
    __shared__ int gtok[SG];
    __shared__ float st_lse[SG], st_D[SG];
    const DevLayout& L = a.L;
    const int dim = a.dim, W = L.windows, Mi = L.image_tokens, Ms = L.num_special;
    const int64_t row = blockIdx.x;
    const int h = (int)(row / W), w = (int)(row - (int64_t)h * W);
    const int tid = threadIdx.x, warp = tid >> 5, la = (tid & 31) >> 3, lb = tid & 7;
    const float* dsb = a.ds + (int64_t)h * Mi * dim;

    for (int e = tid; e < SF * C4; e += ST) {
        const int r = e / C4, c = (e - r * C4) * 4;
        const int i = L.member(w, r);
        float4 v1 = make_float4(0.f, 0.f, 0.f, 0.f), v2 = v1;
        if (c < dim) {
            const int64_t t = Ms + i;
            if (KEYSIDE) {
                v1 = ldg4(a.k.p + (int64_t)h * a.k.hs + t * a.k.rs + c);
                v2 = ldg4(a.v.p + (int64_t)h * a.v.hs + t * a.v.rs + c);
            } else {
                v1 = ldg4(a.q.p + (int64_t)h * a.q.hs + t * a.q.rs + c);
                v2 = ldg4(dsb + (int64_t)i * dim + c);
            }
        }
        *reinterpret_cast<float4*>(A1 + r * RP + c) = v1;
        *reinterpret_cast<float4*>(A2 + r * RP + c) = v2;
    }
    __shared__ float f_lse[SF], f_D[SF];
    if (!KEYSIDE && tid < SF) {
        const int i = L.member(w, tid);
        f_lse[tid] = a.lse[(int64_t)h * Mi + i];
        f_D[tid] = a.D[(int64_t)h * Mi + i];
    }
    float o1[4][ND], o2[4][ND];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int e = 0; e < ND; ++e) o1[i][e] = o2[i][e] = 0.0f;

    const int64_t beg = KEYSIDE ? a.inv_offsets[row] : a.offsets[row];
    const int64_t n = ((KEYSIDE ? a.inv_offsets[row + 1] : a.offsets[row + 1]) - beg) * SF;
    const int32_t* list = (KEYSIDE ? a.inv_q : a.ids) + beg;
    for (int64_t g0 = 0; g0 < n; g0 += SG) {
        const int gn = (int)min((int64_t)SG, n - g0);
        __syncthreads();
        if (tid < SG) {
            int t = 0;
            if (tid < gn) {
                const int64_t gg = g0 + tid;
                t = L.member(list[gg / SF], (int)(gg % SF));
            }
            gtok[tid] = t;
            if (KEYSIDE) {
                st_lse[tid] = tid < gn ? a.lse[(int64_t)h * Mi + t] : INFINITY;
                st_D[tid] = tid < gn ? a.D[(int64_t)h * Mi + t] : 0.0f;
            }
        }
        __syncthreads();
        for (int e = tid; e < SG * C4; e += ST) {
            const int r = e / C4, c = (e - r * C4) * 4;
            float4 v1 = make_float4(0.f, 0.f, 0.f, 0.f), v2 = v1;
            if (r < gn && c < dim) {
                const int i = gtok[r];
                const int64_t t = Ms + i;
                if (KEYSIDE) {
                    v1 = ldg4(a.q.p + (int64_t)h * a.q.hs + t * a.q.rs + c);
                    v2 = ldg4(dsb + (int64_t)i * dim + c);
                } else {
                    v1 = ldg4(a.k.p + (int64_t)h * a.k.hs + t * a.k.rs + c);
                    v2 = ldg4(a.v.p + (int64_t)h * a.v.hs + t * a.v.rs + c);
                }
            }
            *reinterpret_cast<float4*>(B1 + r * RP + c) = v1;
            *reinterpret_cast<float4*>(B2 + r * RP + c) = v2;
        }
        __syncthreads();
        float sv[4][2], tv[4][2];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 2; ++j) sv[i][j] = tv[i][j] = 0.0f;
#pragma unroll 4
        for (int d = 0; d < DP; d += 4) {
            float4 a1[4], a2[4], b1[2], b2[2];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                a1[i] = ld4(A1 + (la + 4 * i) * RP + d);
                a2[i] = ld4(A2 + (la + 4 * i) * RP + d);
            }
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                b1[j] = ld4(B1 + (16 * warp + lb + 8 * j) * RP + d);
                b2[j] = ld4(B2 + (16 * warp + lb + 8 * j) * RP + d);
            }
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 2; ++j) {
                    sv[i][j] = dot4(a1[i], b1[j], sv[i][j]);
                    tv[i][j] = dot4(a2[i], b2[j], tv[i][j]);
                }
        }
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                const int f = la + 4 * i, g = 16 * warp + lb + 8 * j;
                const float lse = KEYSIDE ? st_lse[g] : f_lse[f];
                const float Dv = KEYSIDE ? st_D[g] : f_D[f];
                const float p = g < gn ? expf(sv[i][j] * a.scale - lse) : 0.0f;
                X[g * XP + f] = p * (tv[i][j] - Dv) * a.scale;
                if (KEYSIDE) Y[g * XP + f] = p;
            }
        __syncthreads();
        const int d0 = warp * (DP / 4) + lb * ND;
        for (int g = 0; g < gn; ++g) {
            const float4 x = ld4(X + g * XP + 4 * la);
            const float xv[4] = {x.x, x.y, x.z, x.w};
            float c1[ND];
#pragma unroll
            for (int e = 0; e < ND; ++e) c1[e] = B1[g * RP + d0 + e];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int e = 0; e < ND; ++e) o1[i][e] = fmaf(xv[i], c1[e], o1[i][e]);
            if (KEYSIDE) {
                const float4 y = ld4(Y + g * XP + 4 * la);
                const float yv[4] = {y.x, y.y, y.z, y.w};
                float c2[ND];
#pragma unroll
                for (int e = 0; e < ND; ++e) c2[e] = B2[g * RP + d0 + e];
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int e = 0; e < ND; ++e) o2[i][e] = fmaf(yv[i], c2[e], o2[i][e]);
            }
        }
    }
    const int d0 = warp * (DP / 4) + lb * ND;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int64_t t = Ms + L.member(w, 4 * la + i);
#pragma unroll
        for (int e = 0; e < ND; ++e) {
            const int j = d0 + e;
            if (j >= dim) continue;
            if (KEYSIDE) {
                a.dk.p[(int64_t)h * a.dk.hs + t * a.dk.rs + j] += o1[i][e];
                a.dv.p[(int64_t)h * a.dv.hs + t * a.dv.rs + j] += o2[i][e];
            } else {
                a.dq.p[(int64_t)h * a.dq.hs + t * a.dq.rs + j] += o1[i][e];
            }
        }
    }
}

// inverse plan: one sort key (head * W + key window) << 32 | query window per plan entry
__global__ void inv_keys_kernel(const int64_t* offsets, const int32_t* ids, int64_t rows, int W,
                                unsigned long long* keys, unsigned long long* counts) {
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= rows) return;
    const int64_t h = r / W, qw = r - h * W;
    for (int64_t e = offsets[r]; e < offsets[r + 1]; ++e) {
        const unsigned long long hk = (unsigned long long)(h * W + ids[e]);
        keys[e] = (hk << 32) | (unsigned long long)qw;
        atomicAdd(counts + hk, 1ull);  // integer counts: order-independent
    }
}

__global__ void inv_extract_kernel(const unsigned long long* keys, int64_t n, int32_t* q) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e < n) q[e] = (int32_t)(keys[e] & 0xffffffffull);
}

// ------------------------------------------------------------- small GEMMs
// part[h][split] (R x N) = A[h][rows of split]^T B[h][rows of split]
__global__ void __launch_bounds__(BT) atb_kernel(AtbArgs a) {
    __shared__ float As[16][TB + 1], Bs[16][TB + 1];
    const int tilesN = (a.N + TB - 1) / TB;
    const int r0 = (blockIdx.x / tilesN) * TB, n0 = (blockIdx.x % tilesN) * TB;
    const int split = blockIdx.y, h = blockIdx.z;
    const int64_t m_begin = (int64_t)split * a.chunk, m_end = min(a.rows, m_begin + a.chunk);
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    const float* A = a.A + (int64_t)h * a.a_hs;
    const float* B = a.B + (int64_t)h * a.b_hs;
    float acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = 0.0f;
    for (int64_t m0 = m_begin; m0 < m_end; m0 += 16) {
        __syncthreads();
        for (int e = threadIdx.x; e < 16 * TB; e += BT) {
            const int kk = e / TB, c = e - kk * TB;
            const int64_t m = m0 + kk;
            As[kk][c] = (m < m_end && r0 + c < a.R) ? A[m * a.a_rs + r0 + c] : 0.0f;
            Bs[kk][c] = (m < m_end && n0 + c < a.N) ? B[m * a.b_rs + n0 + c] : 0.0f;
        }
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < 16; ++kk) {
            float av[4], bv[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                av[i] = As[kk][ty + 16 * i];
                bv[i] = Bs[kk][tx + 16 * i];
            }
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
        }
    }
    float* P = a.part + ((int64_t)h * a.splits + split) * a.R * a.N;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int r = r0 + ty + 16 * i;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int n = n0 + tx + 16 * j;
            if (r < a.R && n < a.N) P[(int64_t)r * a.N + n] = acc[i][j];
        }
    }
}

__global__ void atb_reduce_kernel(const float* part, int splits, int64_t per_head, int64_t total, float* out) {
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t h = e / per_head, r = e - h * per_head;
        const float* p = part + h * splits * per_head + r;
        float acc = 0.0f;
        for (int s = 0; s < splits; ++s) acc += p[(int64_t)s * per_head];
        out[e] = acc;
    }
}

// dX[m][c] = sum over (matrix, head, j) of G[mat][h][m][j] * W[mat][h][c][j]
__global__ void __launch_bounds__(BT) dx_gemm_kernel(DxArgs a) {
    __shared__ float As[16][TB + 1], Bs[16][TB + 1];
    const int tilesC = (a.C + TB - 1) / TB;
    const int64_t m0 = (int64_t)(blockIdx.x / tilesC) * TB;
    const int c0 = (blockIdx.x % tilesC) * TB;
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    float acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = 0.0f;
    for (int mat = 0; mat < 3; ++mat)
        for (int h = 0; h < a.heads; ++h) {
            const float* G = a.g[mat] + (int64_t)h * a.tokens * a.dim;
            const float* Wm = a.w[mat] + (int64_t)h * a.C * a.dim;
            for (int j0 = 0; j0 < a.dim; j0 += 16) {
                __syncthreads();
                for (int e = threadIdx.x; e < 16 * TB; e += BT) {
                    const int r = e / 16, kk = e - r * 16;
                    const int j = j0 + kk;
                    As[kk][r] = (m0 + r < a.tokens && j < a.dim) ? G[(m0 + r) * a.dim + j] : 0.0f;
                    Bs[kk][r] = (c0 + r < a.C && j < a.dim) ? Wm[(int64_t)(c0 + r) * a.dim + j] : 0.0f;
                }
                __syncthreads();
#pragma unroll
                for (int kk = 0; kk < 16; ++kk) {
                    float av[4], bv[4];
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        av[i] = As[kk][ty + 16 * i];
                        bv[i] = Bs[kk][tx + 16 * i];
                    }
#pragma unroll
                    for (int i = 0; i < 4; ++i)
#pragma unroll
                        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
                }
            }
        }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int64_t m = m0 + ty + 16 * i;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int c = c0 + tx + 16 * j;
            if (m < a.tokens && c < a.C) a.dx[m * a.C + c] = acc[i][j];
        }
    }
}

// strided f32 / bf16 rows -> contiguous f32 [H][rows][dim]
template <typename T>
__global__ void to_f32_kernel(TensorRef in, int heads, int64_t rows, int dim, float* out) {
    const int64_t n = (int64_t)heads * rows * dim;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
        const int j = (int)(e % dim);
        const int64_t r = (e / dim) % rows;
        const int64_t h = e / ((int64_t)dim * rows);
        out[e] = to_f32(reinterpret_cast<const T*>(in.data)[h * in.hs + r * in.rs + j]);
    }
}

// f32 [H][Ms][d] . [H][Ms][d] row dots (D of the special rows)
__global__ void rowdot_kernel(FMat a, FMat b, int heads, int rows, int dim, float* out) {
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (warp >= (int64_t)heads * rows) return;
    const int h = (int)(warp / rows), r = (int)(warp % rows);
    const float* x = a.p + (int64_t)h * a.hs + (int64_t)r * a.rs;
    const float* y = b.p + (int64_t)h * b.hs + (int64_t)r * b.rs;
    float acc = 0.0f;
    for (int j = lane; j < dim; j += 32) acc += x[j] * y[j];
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) out[warp] = acc;
}

// avg_pool_backward (gradients.hpp:21-34): out[h][t] = in[h][window_of(t)] * (1/s^2)
__global__ void pool_adjoint_kernel(FMat in, int heads, int dim, DevLayout L, float inv, FOut out) {
    const int64_t n = (int64_t)heads * L.image_tokens * dim;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
        const int j = (int)(e % dim);
        const int t = (int)((e / dim) % L.image_tokens);
        const int64_t h = e / ((int64_t)dim * L.image_tokens);
        out.p[h * out.hs + (int64_t)t * out.rs + j] =
            __fmul_rn(in.p[h * in.hs + (int64_t)L.window_of_token(t) * in.rs + j], inv);
    }
}

// upsample_backward (gradients.hpp:37-49): member rows summed in ascending token order
__global__ void window_sum_kernel(FMat in, int heads, int dim, DevLayout L, FOut out) {
    const int64_t n = (int64_t)heads * L.windows * dim;
    const int s2 = L.s * L.s;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
        const int j = (int)(e % dim);
        const int w = (int)((e / dim) % L.windows);
        const int64_t h = e / ((int64_t)dim * L.windows);
        float acc = 0.0f;
        for (int m = 0; m < s2; ++m) acc = __fadd_rn(acc, in.p[h * in.hs + (int64_t)L.member(w, m) * in.rs + j]);
        out.p[h * out.hs + (int64_t)w * out.rs + j] = acc;
    }
}

// ------------------------------------------------ hybrid fast path (forced windows)
// the plan without its forced windows: per-row counts, then the kept ids in row order
// (ids outside [0, W) are kept: the caller's plan check reports them before anything reads them)
__device__ __forceinline__ bool dropped(const uint8_t* mask, int W, int32_t id) {
    return id >= 0 && id < W && mask[id];
}
__global__ void plan_drop_count_kernel(const int64_t* offsets, const int32_t* ids, int64_t rows, const uint8_t* mask,
                                       int W, int64_t* sizes) {
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= rows) return;
    int64_t n = 0;
    for (int64_t e = offsets[r]; e < offsets[r + 1]; ++e) n += dropped(mask, W, ids[e]) ? 0 : 1;
    sizes[r] = n;
}
__global__ void plan_drop_fill_kernel(const int64_t* offsets, const int32_t* ids, int64_t rows, const uint8_t* mask,
                                      int W, const int64_t* out_offsets, int32_t* out_ids) {
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= rows) return;
    int64_t o = out_offsets[r];
    for (int64_t e = offsets[r]; e < offsets[r + 1]; ++e)
        if (!dropped(mask, W, ids[e])) out_ids[o++] = ids[e];
}

// rows of the forced frames (every ref_stride-th frame, all its tokens) of [H][M][64] bf16
// planes -> contiguous [H][n_ff * tokens_per_frame][64]; 16 bytes per thread
__global__ void forced_gather_kernel(const __nv_bfloat16* src, int64_t src_hs, int heads, DevLayout L, int ref_stride,
                                     int64_t rows, __nv_bfloat16* dst) {
    const int64_t n = (int64_t)heads * rows * 8;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
        const int c = (int)(e & 7);
        const int64_t i = (e >> 3) % rows, h = (e >> 3) / rows;
        const int64_t f = (i / L.tokens_per_frame) * ref_stride, t = i % L.tokens_per_frame;
        const int64_t sr = L.num_special + f * L.tokens_per_frame + t;
        reinterpret_cast<uint4*>(dst + (h * rows + i) * 64)[c] = reinterpret_cast<const uint4*>(src + h * src_hs + sr * 64)[c];
    }
}

// dK / dV of the forced rows (contiguous [H][rows][64] f32) added to their rows of dk / dv
__global__ void forced_scatter_add_kernel(const float* gk, const float* gv, int heads, DevLayout L, int ref_stride,
                                          int64_t rows, FOut dk, FOut dv) {
    const int64_t n = (int64_t)heads * rows * 64;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
        const int j = (int)(e & 63);
        const int64_t i = (e >> 6) % rows, h = (e >> 6) / rows;
        const int64_t f = (i / L.tokens_per_frame) * ref_stride, t = i % L.tokens_per_frame;
        const int64_t r = L.num_special + f * L.tokens_per_frame + t;
        dk.p[h * dk.hs + r * dk.rs + j] += gk[e];
        dv.p[h * dv.hs + r * dv.rs + j] += gv[e];
    }
}

unsigned grid_for(int64_t n, int threads = 256) {
    const int64_t b = (n + threads - 1) / threads;
    return (unsigned)(b < 148 * 64 ? (b > 0 ? b : 1) : 148 * 64);
}

template <int DP>
size_t dense_smem() {
    return (size_t)(4 * TB * (DP + 4) + 2 * TB * PT + 2 * TB) * sizeof(float);
}

template <int DP>
cudaError_t dense_bwd_dp(DenseBwdArgs a, int heads, cudaStream_t st) {
    const size_t smem = dense_smem<DP>();
    cudaError_t e = cudaFuncSetAttribute(dense_bwd_dkdv_kernel<DP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(dense_bwd_dq_kernel<DP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    a.heads = heads;
    if (a.dk.p || a.dv.p) {
        dense_bwd_dkdv_kernel<DP><<<dim3((unsigned)((a.nk + TB - 1) / TB), heads), BT, smem, st>>>(a);
        note_launch();
    }
    if (a.dq.p) {
        const int64_t qtiles = (a.nq + TB - 1) / TB, ktiles = (a.nk + TB - 1) / TB;
        if (a.k_splits < 1 || !a.dq_part) a.k_splits = 1;
        a.k_chunk = (ktiles + a.k_splits - 1) / a.k_splits * TB;
        a.k_splits = (int)((a.nk + a.k_chunk - 1) / a.k_chunk);
        dense_bwd_dq_kernel<DP><<<dim3((unsigned)qtiles, a.k_splits, heads), BT, smem, st>>>(a);
        note_launch();
        if (a.k_splits > 1) {
            dq_reduce_kernel<<<grid_for((int64_t)heads * a.nq * a.dim), 256, 0, st>>>(a);
            note_launch();
        }
    }
    return cudaGetLastError();
}

template <int DP>
cudaError_t gate_bwd_dp(const GateBwdArgs& a, int heads, cudaStream_t st) {
    const int s2 = a.L.s * a.L.s;
    const size_t smem = (size_t)(DP * (DP + 4) + 3 * s2 * DP + DP) * sizeof(float);
    cudaError_t e = cudaFuncSetAttribute(gate_bwd_kernel<DP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    gate_bwd_kernel<DP><<<(unsigned)((int64_t)heads * ((a.L.windows + GATE_WPC - 1) / GATE_WPC)), BT, smem, st>>>(a);
    note_launch();
    return cudaGetLastError();
}

template <int DP>
cudaError_t sel_bwd_dp(const SelBwdArgs& a, int heads, cudaStream_t st) {
    const int s2 = a.L.s * a.L.s;
    const int64_t rows = (int64_t)heads * a.L.windows;
    const size_t smem_q = (size_t)(2 * s2 * (DP + 1) + 2 * CK * (DP + 1) + s2 * (CK + 1) + 2 * s2) * sizeof(float);
    const size_t smem_k = (size_t)(2 * s2 * (DP + 1) + 2 * CK * (DP + 1) + 2 * CK * (s2 + 1) + 2 * CK) * sizeof(float);
    cudaError_t e = cudaFuncSetAttribute(sel_bwd_dq_kernel<DP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_q);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(sel_bwd_dkdv_kernel<DP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_k);
    if (e != cudaSuccess) return e;
    sel_bwd_dq_kernel<DP><<<(unsigned)rows, BT, smem_q, st>>>(a);
    sel_bwd_dkdv_kernel<DP><<<(unsigned)rows, BT, smem_k, st>>>(a);
    note_launch(2);
    return cudaGetLastError();
}

int dp_of(int dim) { return dim <= 32 ? 32 : dim <= 64 ? 64 : 128; }

}  // namespace

cudaError_t launch_gate_bwd(const GateBwdArgs& a, int heads, cudaStream_t st) {
    if ((int64_t)heads * a.L.windows == 0) return cudaSuccess;
    switch (dp_of(a.dim)) {
        case 32: return gate_bwd_dp<32>(a, heads, st);
        case 64: return gate_bwd_dp<64>(a, heads, st);
        default: return gate_bwd_dp<128>(a, heads, st);
    }
}

// key splits for the query-side pass when there are too few query tiles to fill the GPU
// (the special rows: Ms / 64 tiles per head), each split at least 16 key tiles
int dense_dq_splits(int heads, int64_t nq, int64_t nk) {
    const int64_t ctas = (int64_t)heads * ((nq + TB - 1) / TB);
    const int64_t want = (4 * 148 + ctas - 1) / ctas;
    const int64_t cap = ((nk + TB - 1) / TB) / 16;
    int64_t s = want < cap ? want : cap;
    return (int)(s < 1 ? 1 : s > 64 ? 64 : s);
}

cudaError_t launch_dense_bwd(const DenseBwdArgs& a, int heads, cudaStream_t st) {
    if (heads == 0 || a.nq == 0 || a.nk == 0) return cudaSuccess;
    // feature tiling 4 tx + 64 c needs DP >= 64 (padding columns are zero)
    return a.dim <= 64 ? dense_bwd_dp<64>(a, heads, st) : dense_bwd_dp<128>(a, heads, st);
}

cudaError_t launch_pool_bwd(const PoolBwdArgs& a, cudaStream_t st) {
    const int64_t n = (int64_t)a.heads * a.rows * a.dim;
    if (n == 0) return cudaSuccess;
    pool_bwd_kernel<<<grid_for(n), 256, 0, st>>>(a);
    note_launch();
    return cudaGetLastError();
}

namespace {

template <int DP>
cudaError_t sel16_bwd_dp(const SelBwdArgs& a, int heads, cudaStream_t st) {
    const int64_t rows = (int64_t)heads * a.L.windows;
    const size_t smem = (size_t)((2 * SF + 2 * SG) * (DP + 4) + 2 * SG * XP) * sizeof(float);
    cudaError_t e = cudaFuncSetAttribute(sel16_bwd_kernel<DP, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(sel16_bwd_kernel<DP, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    sel16_bwd_kernel<DP, false><<<(unsigned)rows, ST, smem, st>>>(a);
    sel16_bwd_kernel<DP, true><<<(unsigned)rows, ST, smem, st>>>(a);
    note_launch(2);
    return cudaGetLastError();
}

bool aligned4(const FMat& m) {
    return (reinterpret_cast<uintptr_t>(m.p) & 15) == 0 && m.hs % 4 == 0 && m.rs % 4 == 0;
}

}  // namespace

cudaError_t launch_sel_bwd(const SelBwdArgs& a, int heads, cudaStream_t st) {
    if ((int64_t)heads * a.L.windows == 0) return cudaSuccess;
    if (a.L.s == 4 && a.dim % 4 == 0 && aligned4(a.q) && aligned4(a.k) && aligned4(a.v)) {
        switch (dp_of(a.dim)) {
            case 32: return sel16_bwd_dp<32>(a, heads, st);
            case 64: return sel16_bwd_dp<64>(a, heads, st);
            default: return sel16_bwd_dp<128>(a, heads, st);
        }
    }
    switch (dp_of(a.dim)) {
        case 32: return sel_bwd_dp<32>(a, heads, st);
        case 64: return sel_bwd_dp<64>(a, heads, st);
        default: return sel_bwd_dp<128>(a, heads, st);
    }
}

size_t inverse_plan_tmp_bytes(int64_t rows, int64_t entries) {
    size_t sort_bytes = 0;
    cub::DeviceRadixSort::SortKeys(nullptr, sort_bytes, (const unsigned long long*)nullptr,
                                   (unsigned long long*)nullptr, (int64_t)entries, 0, 64);
    const size_t scan = scan_offsets_tmp_bytes(rows);
    return (sort_bytes > scan ? sort_bytes : scan) + 256;
}

cudaError_t launch_inverse_plan(const int64_t* offsets, const int32_t* ids, int64_t rows, int W, int64_t entries,
                                unsigned long long* keys, unsigned long long* keys_sorted, int64_t* counts,
                                int64_t* inv_offsets, int32_t* inv_q, void* tmp, size_t tmp_bytes,
                                cudaStream_t st) {
    cudaError_t e = cudaMemsetAsync(counts, 0, (size_t)rows * sizeof(int64_t), st);
    if (e != cudaSuccess) return e;
    if (rows == 0) return cudaSuccess;
    inv_keys_kernel<<<(unsigned)((rows + 255) / 256), 256, 0, st>>>(offsets, ids, rows, W, keys,
                                                                  reinterpret_cast<unsigned long long*>(counts));
    note_launch();
    int hi_bits = 1;
    while ((int64_t(1) << hi_bits) < rows) ++hi_bits;
    size_t tb = tmp_bytes;
    e = cub::DeviceRadixSort::SortKeys(tmp, tb, keys, keys_sorted, entries, 0, 32 + hi_bits, st);
    if (e != cudaSuccess) return e;
    e = launch_scan_offsets(counts, rows, inv_offsets, tmp, tmp_bytes, st);
    if (e != cudaSuccess) return e;
    if (entries) {
        inv_extract_kernel<<<(unsigned)((entries + 255) / 256), 256, 0, st>>>(keys_sorted, entries, inv_q);
        note_launch();
    }
    return cudaGetLastError();
}

int atb_splits(int heads, int R, int N, int64_t rows) {
    const int64_t tiles = (int64_t)heads * ((R + TB - 1) / TB) * ((N + TB - 1) / TB);
    int64_t s = (2 * 148 + tiles - 1) / tiles;
    const int64_t max_s = (rows + 511) / 512;
    if (s > max_s) s = max_s;
    if (s > 64) s = 64;
    return (int)(s < 1 ? 1 : s);
}

cudaError_t launch_atb(AtbArgs a, int heads, float* out, cudaStream_t st) {
    if (heads == 0 || a.R == 0 || a.N == 0) return cudaSuccess;
    a.chunk = (a.rows + a.splits - 1) / a.splits;
    a.chunk = (a.chunk + 15) / 16 * 16;
    const unsigned tiles = (unsigned)(((a.R + TB - 1) / TB) * ((a.N + TB - 1) / TB));
    atb_kernel<<<dim3(tiles, a.splits, heads), BT, 0, st>>>(a);
    const int64_t per_head = (int64_t)a.R * a.N, total = per_head * heads;
    atb_reduce_kernel<<<grid_for(total), 256, 0, st>>>(a.part, a.splits, per_head, total, out);
    note_launch(2);
    return cudaGetLastError();
}

cudaError_t launch_dx_gemm(const DxArgs& a, cudaStream_t st) {
    if (a.tokens == 0 || a.C == 0) return cudaSuccess;
    const int64_t tiles = ((a.tokens + TB - 1) / TB) * (int64_t)((a.C + TB - 1) / TB);
    dx_gemm_kernel<<<(unsigned)tiles, BT, 0, st>>>(a);
    note_launch();
    return cudaGetLastError();
}

cudaError_t launch_to_f32(const TensorRef& in, int heads, int64_t rows, int dim, float* out, cudaStream_t st) {
    const int64_t n = (int64_t)heads * rows * dim;
    if (n == 0) return cudaSuccess;
    if (in.dtype == GSA_DTYPE_BF16) to_f32_kernel<__nv_bfloat16><<<grid_for(n), 256, 0, st>>>(in, heads, rows, dim, out);
    else to_f32_kernel<float><<<grid_for(n), 256, 0, st>>>(in, heads, rows, dim, out);
    note_launch();
    return cudaGetLastError();
}

cudaError_t launch_pool_adjoint(const FMat& in, int heads, int dim, const DevLayout& L, float inv, const FOut& out,
                                cudaStream_t st) {
    const int64_t n = (int64_t)heads * L.image_tokens * dim;
    if (n == 0) return cudaSuccess;
    pool_adjoint_kernel<<<grid_for(n), 256, 0, st>>>(in, heads, dim, L, inv, out);
    note_launch();
    return cudaGetLastError();
}

cudaError_t launch_window_sum(const FMat& in, int heads, int dim, const DevLayout& L, const FOut& out, cudaStream_t st) {
    const int64_t n = (int64_t)heads * L.windows * dim;
    if (n == 0) return cudaSuccess;
    window_sum_kernel<<<grid_for(n), 256, 0, st>>>(in, heads, dim, L, out);
    note_launch();
    return cudaGetLastError();
}

cudaError_t launch_plan_drop(const int64_t* offsets, const int32_t* ids, int64_t rows, const uint8_t* mask, int W,
                             int64_t* sizes, int64_t* out_offsets, int32_t* out_ids, void* tmp, size_t tmp_bytes,
                             cudaStream_t st) {
    if (rows == 0) return cudaSuccess;
    const unsigned b = (unsigned)((rows + 255) / 256);
    plan_drop_count_kernel<<<b, 256, 0, st>>>(offsets, ids, rows, mask, W, sizes);
    note_launch();
    cudaError_t e = launch_scan_offsets(sizes, rows, out_offsets, tmp, tmp_bytes, st);
    if (e != cudaSuccess) return e;
    plan_drop_fill_kernel<<<b, 256, 0, st>>>(offsets, ids, rows, mask, W, out_offsets, out_ids);
    note_launch();
    return cudaGetLastError();
}

cudaError_t launch_forced_gather(const __nv_bfloat16* src, int64_t src_hs, int heads, const DevLayout& L, int ref_stride,
                                 int64_t rows, __nv_bfloat16* dst, cudaStream_t st) {
    const int64_t n = (int64_t)heads * rows * 8;
    if (n == 0) return cudaSuccess;
    forced_gather_kernel<<<grid_for(n), 256, 0, st>>>(src, src_hs, heads, L, ref_stride, rows, dst);
    note_launch();
    return cudaGetLastError();
}

cudaError_t launch_forced_scatter_add(const float* gk, const float* gv, int heads, const DevLayout& L, int ref_stride,
                                      int64_t rows, const FOut& dk, const FOut& dv, cudaStream_t st) {
    const int64_t n = (int64_t)heads * rows * 64;
    if (n == 0) return cudaSuccess;
    forced_scatter_add_kernel<<<grid_for(n), 256, 0, st>>>(gk, gv, heads, L, ref_stride, rows, dk, dv);
    note_launch();
    return cudaGetLastError();
}

cudaError_t launch_rowdot(const FMat& a, const FMat& b, int heads, int rows, int dim, float* out, cudaStream_t st) {
    const int64_t n = (int64_t)heads * rows * 32;
    if (n == 0) return cudaSuccess;
    rowdot_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(a, b, heads, rows, dim, out);
    note_launch();
    return cudaGetLastError();
}

}  // namespace gsa_sm100
