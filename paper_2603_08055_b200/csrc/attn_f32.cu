// attn_f32.cu — flash-style attention on CUDA cores in fp32, with an optional
// fused streaming top-k (fused_compressed_attention_topk, compression.hpp:180-297).
//
// This is the exact (phase-1) compressed-attention kernel and the generic
// dense kernel (tiled_attention / special_token_attention) for shapes and
// dtypes outside the tensor-core fast path. Scores use the reference's
// scaled_dot order with round-to-nearest mul/add (no FMA), so the top-k rows
// are bit-identical to the CPU reference; the softmax/PV half is tolerance-
// checked only.
//
// CTA = 64 query rows of one head, 256 threads; key tiles of 64 rows staged in
// shared memory as f32. Scoring: each thread owns a 4x4 (row, col) block with
// rows/cols interleaved by 16 (conflict-free LDS.128). Softmax/PV: 4 threads
// per query row, each owning a quarter of the output features. Top-k: one thread per
// row scans its row in ascending column order and inserts into a sorted list
// in shared memory (ties keep the lower index: identical to naive_topk).
#include <float.h>

#include "kernels.h"

namespace gsa_sm100 {
namespace {

constexpr int BQ = 64, BK = 64, NT = 256;

template <typename T>
__device__ __forceinline__ void stage_rows(float* dst, int dp, const T* src, int64_t rs, int nrows,
                                           int rows_valid, int dim, bool vec8) {
    // rows [0,nrows) x dim -> dst[r*dp + j] (f32); rows >= rows_valid are zero
    if (vec8) {
        const int cpr = dim / 8;
        for (int idx = threadIdx.x; idx < nrows * cpr; idx += NT) {
            const int r = idx / cpr, c = (idx - r * cpr) * 8;
            float x[8];
            if (r < rows_valid) {
                load8(src + (int64_t)r * rs + c, x);
            } else {
#pragma unroll
                for (int i = 0; i < 8; ++i) x[i] = 0.0f;
            }
            float4* o = reinterpret_cast<float4*>(dst + r * dp + c);
            o[0] = make_float4(x[0], x[1], x[2], x[3]);
            o[1] = make_float4(x[4], x[5], x[6], x[7]);
        }
    } else {
        for (int idx = threadIdx.x; idx < nrows * dim; idx += NT) {
            const int r = idx / dim, c = idx - r * dim;
            dst[r * dp + c] = r < rows_valid ? to_f32(src[(int64_t)r * rs + c]) : 0.0f;
        }
    }
}

template <typename T, int DMAX, bool TOPK>
__global__ void __launch_bounds__(NT) attn_f32_kernel(AttnArgs a, bool vec8) {
    extern __shared__ __align__(16) float smem[];
    const int dim = a.dim, dp = ((dim + 3) & ~3) + 4;
    float* Qs = smem;
    float* Ks = Qs + BQ * dp;
    float* Vs = Ks + BK * dp;
    float* S = Vs + BK * dp;  // [BQ][BK+1]
    float* lst_s = S + BQ * (BK + 1);
    int* lst_i = reinterpret_cast<int*>(lst_s + (TOPK ? BQ * a.k_eff : 0));
    __shared__ int lst_n[BQ];

    int h = blockIdx.y, q0 = blockIdx.x * BQ;
    if (a.block_list) {
        if ((int)blockIdx.x >= *a.block_count) return;
        const int qtiles = (a.mq + BQ - 1) / BQ;
        const int blk = a.block_list[blockIdx.x];
        h = blk / qtiles;
        q0 = (blk - h * qtiles) * BQ;
    }
    if (TOPK && a.glist_s) {  // k_eff too large for shared memory: per-CTA lists in global scratch
        const int64_t cta = (int64_t)h * ((a.mq + BQ - 1) / BQ) + q0 / BQ;
        lst_s = a.glist_s + cta * BQ * a.k_eff;
        lst_i = a.glist_i + cta * BQ * a.k_eff;
    }
    const int tid = threadIdx.x;
    const int qrows = min(BQ, a.mq - q0);
    const T* qb = reinterpret_cast<const T*>(a.q.data) + (int64_t)h * a.q.hs + (int64_t)q0 * a.q.rs;
    const T* kb = reinterpret_cast<const T*>(a.k.data) + (int64_t)h * a.k.hs;
    const T* vb = reinterpret_cast<const T*>(a.v.data) + (int64_t)h * a.v.hs;
    stage_rows(Qs, dp, qb, a.q.rs, BQ, qrows, dim, vec8);
    if (TOPK && tid < BQ) lst_n[tid] = 0;

    // softmax/PV ownership: row r = tid/4, features [p*DMAX/4, (p+1)*DMAX/4)
    const int r = tid >> 2, p = tid & 3;
    float m = -INFINITY, l = 0.0f;
    float acc[DMAX / 4];
#pragma unroll
    for (int e = 0; e < DMAX / 4; ++e) acc[e] = 0.0f;
    // scoring ownership
    const int ty = tid >> 4, tx = tid & 15;
    const int d4 = dim & ~3;

    for (int k0 = 0; k0 < a.mk; k0 += BK) {
        const int kn = min(BK, a.mk - k0);
        __syncthreads();  // previous tile fully consumed (and Q staged on the first pass)
        stage_rows(Ks, dp, kb + (int64_t)k0 * a.k.rs, a.k.rs, BK, kn, dim, vec8);
        stage_rows(Vs, dp, vb + (int64_t)k0 * a.v.rs, a.v.rs, BK, kn, dim, vec8);
        __syncthreads();
        {
            ExactDot4 d[4][4];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) d[i][j].zero();
            for (int x = 0; x < d4; x += 4) {
                float4 qv[4], kv[4];
#pragma unroll
                for (int i = 0; i < 4; ++i) qv[i] = *reinterpret_cast<const float4*>(Qs + (ty + 16 * i) * dp + x);
#pragma unroll
                for (int j = 0; j < 4; ++j) kv[j] = *reinterpret_cast<const float4*>(Ks + (tx + 16 * j) * dp + x);
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int j = 0; j < 4; ++j)
                        d[i][j].step(qv[i].x, qv[i].y, qv[i].z, qv[i].w, kv[j].x, kv[j].y, kv[j].z, kv[j].w);
            }
            for (int x = d4; x < dim; ++x)
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int j = 0; j < 4; ++j) d[i][j].tail(Qs[(ty + 16 * i) * dp + x], Ks[(tx + 16 * j) * dp + x]);
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const int c = tx + 16 * j;
                    S[(ty + 16 * i) * (BK + 1) + c] = c < kn ? d[i][j].finish(a.scale) : -INFINITY;
                }
        }
        __syncthreads();
        float* srow = S + r * (BK + 1);
        if (TOPK && p == 0 && a.k_eff > 0) {
            // streaming top-k: ascending columns, keep entries strictly better than the tail
            int n = lst_n[r];
            float* ls = lst_s + r * a.k_eff;
            int* li = lst_i + r * a.k_eff;
            for (int c = 0; c < kn; ++c) {
                const int col = k0 + c;
                if (a.excluded && a.excluded[col]) continue;
                const float sc = srow[c];
                if (n == a.k_eff && !(sc > ls[n - 1])) continue;
                int pos = n < a.k_eff ? n : n - 1;
                while (pos > 0 && sc > ls[pos - 1]) {
                    ls[pos] = ls[pos - 1];
                    li[pos] = li[pos - 1];
                    --pos;
                }
                ls[pos] = sc;
                li[pos] = col;
                if (n < a.k_eff) ++n;
            }
            lst_n[r] = n;
        }
        __syncwarp();
        // online softmax (rescaled-accumulator form, compression.hpp:242-257)
        float mt = -INFINITY;
        for (int c = p; c < kn; c += 4) mt = fmaxf(mt, srow[c]);
        mt = fmaxf(mt, __shfl_xor_sync(0xffffffffu, mt, 1));
        mt = fmaxf(mt, __shfl_xor_sync(0xffffffffu, mt, 2));
        const float mn = fmaxf(m, mt);
        const float alpha = (m == -INFINITY) ? 0.0f : expf(m - mn);
        float ls = 0.0f;
        for (int c = p; c < kn; c += 4) {
            const float e = expf(srow[c] - mn);
            srow[c] = e;
            ls += e;
        }
        ls += __shfl_xor_sync(0xffffffffu, ls, 1);
        ls += __shfl_xor_sync(0xffffffffu, ls, 2);
        l = l * alpha + ls;
        m = mn;
        __syncwarp();
#pragma unroll
        for (int e = 0; e < DMAX / 4; ++e) acc[e] *= alpha;
        // PV: this thread owns features [p*CH, p*CH+CH); float4 reads of the V row
        // (reads past `dim` stay inside the shared allocation and are discarded)
        for (int c = 0; c < kn; ++c) {
            const float pc = srow[c];
            const float4* vrow = reinterpret_cast<const float4*>(Vs + c * dp + p * (DMAX / 4));
#pragma unroll
            for (int e4 = 0; e4 < DMAX / 16; ++e4) {
                const float4 v4 = vrow[e4];
                acc[4 * e4 + 0] = fmaf(pc, v4.x, acc[4 * e4 + 0]);
                acc[4 * e4 + 1] = fmaf(pc, v4.y, acc[4 * e4 + 1]);
                acc[4 * e4 + 2] = fmaf(pc, v4.z, acc[4 * e4 + 2]);
                acc[4 * e4 + 3] = fmaf(pc, v4.w, acc[4 * e4 + 3]);
            }
        }
    }
    if (r < qrows && !(TOPK && a.topk_only)) {
        const float inv = 1.0f / l;
        float* orow = a.out + (int64_t)h * a.out_hs + (int64_t)(q0 + r) * a.out_rs;
#pragma unroll
        for (int e = 0; e < DMAX / 4; ++e)
            if (p * (DMAX / 4) + e < dim) orow[p * (DMAX / 4) + e] = acc[e] * inv;
        if (p == 0 && a.lse) a.lse[(int64_t)h * a.mq + q0 + r] = m + logf(l);
    }
    if (r < qrows) {
        if (TOPK && p == 0 && a.k_eff > 0) {
            const int64_t base = ((int64_t)h * a.mq + q0 + r) * a.k_eff;
            for (int j = 0; j < a.k_eff; ++j) {
                a.topk[base + j] = lst_i[r * a.k_eff + j];
                if (a.guide) a.guide[base + j] = lst_s[r * a.k_eff + j];
            }
        }
    }
}

template <typename T, int DMAX, bool TOPK>
cudaError_t launch_typed(const AttnArgs& a, bool vec8, cudaStream_t st) {
    const int dp = ((a.dim + 3) & ~3) + 4;
    size_t smem = sizeof(float) * ((size_t)(BQ + 2 * BK) * dp + BQ * (BK + 1));
    const size_t list_bytes = TOPK ? (size_t)BQ * a.k_eff * (sizeof(float) + sizeof(int)) : 0;
    AttnArgs b = a;
    b.glist_s = nullptr;
    b.glist_i = nullptr;
    void* glist = nullptr;
    if (smem + list_bytes <= 200 * 1024) {
        smem += list_bytes;
    } else {
        // large budgets on this generic (head dim != 64) path: the sorted per-row lists
        // go to stream-ordered global scratch instead of shared memory
        const size_t n = (size_t)a.heads * ((a.mq + BQ - 1) / BQ) * list_bytes;
        cudaError_t e = cudaMallocAsync(&glist, n, st);
        if (e != cudaSuccess) return e;
        b.glist_s = static_cast<float*>(glist);
        b.glist_i = reinterpret_cast<int*>(static_cast<char*>(glist) + n / 2);
        // per CTA: [BQ][k] floats in the first half, [BQ][k] ints in the second
    }
    auto kern = attn_f32_kernel<T, DMAX, TOPK>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    dim3 grid((a.mq + BQ - 1) / BQ, a.heads);
    if (a.block_list) grid = dim3(((a.mq + BQ - 1) / BQ) * a.heads, 1);
    { kern<<<grid, NT, smem, st>>>(b, vec8); note_launch(); }
    e = cudaGetLastError();
    if (glist) cudaFreeAsync(glist, st);
    return e;
}

template <typename T>
cudaError_t launch_dt(const AttnArgs& a, bool vec8, cudaStream_t st) {
    const bool topk = a.topk != nullptr;
    if (a.dim <= 64) return topk ? launch_typed<T, 64, true>(a, vec8, st) : launch_typed<T, 64, false>(a, vec8, st);
    return topk ? launch_typed<T, 128, true>(a, vec8, st) : launch_typed<T, 128, false>(a, vec8, st);
}

}  // namespace

cudaError_t launch_attn_f32(const AttnArgs& a, cudaStream_t st) {
    if (a.mq == 0 || a.heads == 0) return cudaSuccess;
    if (a.dim > 128) return cudaErrorInvalidValue;
    const int align = a.q.dtype == GSA_DTYPE_BF16 ? 8 : 4;
    auto ok = [&](const TensorRef& t) {
        return t.rs % align == 0 && t.hs % align == 0 && (reinterpret_cast<uintptr_t>(t.data) & 15) == 0;
    };
    const bool vec8 = a.dim % 8 == 0 && ok(a.q) && ok(a.k) && ok(a.v);
    if (a.q.dtype == GSA_DTYPE_BF16) return launch_dt<__nv_bfloat16>(a, vec8, st);
    return launch_dt<float>(a, vec8, st);
}

}  // namespace gsa_sm100
