// select_f32.cu — selection branch on CUDA cores (block_sparse_attention,
// selection.hpp:63-136), optionally fused with the gate (layer.hpp:99-119) and
// the gated merge (layer.hpp:154-170).
//
// Generic path (any s in {1,2,4,8}, d <= 128, f32 or bf16 inputs); the bf16 /
// d=64 / s=4 fast path is the tcgen05 kernel in select_tc.cu. One CTA per
// (head, query window): the s^2 queries of the window share the plan row, so
// the gathered keys are staged once per chunk of 64 keys and reused by every
// query (selection.hpp:99-105 gathers once per (head, window) too).
#include "kernels.h"

namespace gsa_sm100 {
namespace {

constexpr int NT = 128, CK = 64;

template <typename T, int DMAX>
__global__ void __launch_bounds__(NT) select_f32_kernel(SelectArgs a, bool vec8) {
    extern __shared__ __align__(16) float smem[];
    const int dim = a.dim, dp = ((dim + 3) & ~3) + 4;
    const DevLayout& L = a.L;
    const int s2 = L.s * L.s;
    float* Qs = smem;              // [s2][dp]
    float* Ks = Qs + s2 * dp;      // [CK][dp]
    float* Vs = Ks + CK * dp;      // [CK][dp]
    float* S = Vs + CK * dp;       // [s2][CK+1]
    float* stat = S + s2 * (CK + 1);  // m[s2], alpha[s2], l[s2]
    __shared__ int ktok[CK];

    const int64_t item = blockIdx.x;
    const int h = (int)(item / L.windows), w = (int)(item % L.windows);
    const int tid = threadIdx.x;
    const T* qb = reinterpret_cast<const T*>(a.q.data) + (int64_t)h * a.q.hs;
    const T* kb = reinterpret_cast<const T*>(a.k.data) + (int64_t)h * a.k.hs;
    const T* vb = reinterpret_cast<const T*>(a.v.data) + (int64_t)h * a.v.hs;

    // stage the window's queries
    for (int idx = tid; idx < s2 * dim; idx += NT) {
        const int qi = idx / dim, j = idx - qi * dim;
        Qs[qi * dp + j] = to_f32(qb[(int64_t)L.member(w, qi) * a.q.rs + j]);
    }
    if (tid < s2) {
        stat[tid] = -INFINITY;
        stat[2 * s2 + tid] = 0.0f;
    }
    const int tpq = NT / s2;                       // threads per query
    const int ch = DMAX / tpq > 0 ? DMAX / tpq : 1;  // features per thread (<= DMAX/2)
    const int qi = tid / tpq, t = tid - qi * tpq;
    const int j0 = t * ch;
    float acc[DMAX / 2];  // only the first `ch` are used (ch <= DMAX/2 since s^2 <= 64)
#pragma unroll
    for (int e = 0; e < DMAX / 2; ++e) acc[e] = 0.0f;

    const int64_t nkeys = a.rows.size(item) * s2;
    for (int64_t k0 = 0; k0 < nkeys; k0 += CK) {
        const int kn = (int)(nkeys - k0 < CK ? nkeys - k0 : CK);
        __syncthreads();
        if (tid < CK) {
            const int64_t kk = k0 + tid;
            ktok[tid] = tid < kn ? L.member(a.rows.window(item, kk / s2), (int)(kk % s2)) : 0;
        }
        __syncthreads();
        if (vec8) {
            const int cpr = dim / 8;
            for (int idx = tid; idx < CK * cpr; idx += NT) {
                const int r = idx / cpr, c = (idx - r * cpr) * 8;
                float x[8], y[8];
                if (r < kn) {
                    load8(kb + (int64_t)ktok[r] * a.k.rs + c, x);
                    load8(vb + (int64_t)ktok[r] * a.v.rs + c, y);
                } else {
#pragma unroll
                    for (int i = 0; i < 8; ++i) x[i] = y[i] = 0.0f;
                }
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    Ks[r * dp + c + i] = x[i];
                    Vs[r * dp + c + i] = y[i];
                }
            }
        } else {
            for (int idx = tid; idx < CK * dim; idx += NT) {
                const int r = idx / dim, c = idx - r * dim;
                Ks[r * dp + c] = r < kn ? to_f32(kb[(int64_t)ktok[r] * a.k.rs + c]) : 0.0f;
                Vs[r * dp + c] = r < kn ? to_f32(vb[(int64_t)ktok[r] * a.v.rs + c]) : 0.0f;
            }
        }
        __syncthreads();
        for (int idx = tid; idx < s2 * CK; idx += NT) {
            const int q = idx / CK, c = idx - q * CK;
            S[q * (CK + 1) + c] = c < kn ? exact_scaled_dot(Qs + q * dp, Ks + c * dp, dim, a.scale) : -INFINITY;
        }
        __syncthreads();
        if (tid < s2) {  // per-query online-softmax statistics
            float* srow = S + tid * (CK + 1);
            const float m = stat[tid];
            float mt = -INFINITY;
            for (int c = 0; c < kn; ++c) mt = fmaxf(mt, srow[c]);
            const float mn = fmaxf(m, mt);
            const float alpha = m == -INFINITY ? 0.0f : expf(m - mn);
            float ls = 0.0f;
            for (int c = 0; c < kn; ++c) {
                const float e = expf(srow[c] - mn);
                srow[c] = e;
                ls += e;
            }
            stat[tid] = mn;
            stat[s2 + tid] = alpha;
            stat[2 * s2 + tid] = stat[2 * s2 + tid] * alpha + ls;
        }
        __syncthreads();
        const float alpha = stat[s2 + qi];
        const float* srow = S + qi * (CK + 1);
#pragma unroll
        for (int e = 0; e < DMAX / 2; ++e)
            if (e < ch) acc[e] *= alpha;
        for (int c = 0; c < kn; ++c) {
            const float pc = srow[c];
            const float* vrow = Vs + c * dp + j0;
#pragma unroll
            for (int e = 0; e < DMAX / 2; ++e)
                if (e < ch && j0 + e < dim) acc[e] = fmaf(pc, vrow[e], acc[e]);
        }
    }
    __syncthreads();
    const int tok = L.member(w, qi);
    const float l = stat[2 * s2 + qi];
    const float inv = 1.0f / l;
    const int64_t ti = (int64_t)h * L.image_tokens + tok;
    if (t == 0 && a.lse) a.lse[ti] = stat[qi] + logf(l);
    float* orow = a.out + (int64_t)h * a.out_hs + (int64_t)tok * a.out_rs;
    const float* comp = a.o_comp ? a.o_comp + ((int64_t)h * L.windows + w) * dim : nullptr;
    const float* wg = a.w_g ? a.w_g + (int64_t)h * dim * dim : nullptr;
    for (int e = 0; e < ch; ++e) {
        const int j = j0 + e;
        if (j >= dim) break;
        const float sel = acc[e] * inv;
        if (a.o_sel_ctx) a.o_sel_ctx[ti * dim + j] = sel;
        if (wg) {
            float z = 0.0f;  // layer.hpp:110-115: sum over a ascending
            for (int x = 0; x < dim; ++x) z = fmaf(Qs[qi * dp + x], wg[(int64_t)x * dim + j], z);
            const float g = 1.0f / (1.0f + expf(-z));
            if (a.gate_ctx) a.gate_ctx[ti * dim + j] = g;
            orow[j] = g * comp[j] + (1.0f - g) * sel;
        } else {
            orow[j] = sel;
        }
    }
}

template <typename T, int DMAX>
cudaError_t launch_typed(const SelectArgs& a, bool vec8, cudaStream_t st) {
    const int dp = ((a.dim + 3) & ~3) + 4;
    const int s2 = a.L.s * a.L.s;
    const size_t smem = sizeof(float) * ((size_t)(s2 + 2 * CK) * dp + s2 * (CK + 1) + 3 * s2);
    auto kern = select_f32_kernel<T, DMAX>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    const int64_t items = (int64_t)a.heads * a.L.windows;
    { kern<<<(unsigned)items, NT, smem, st>>>(a, vec8); note_launch(); }
    return cudaGetLastError();
}

}  // namespace

cudaError_t launch_select_f32(const SelectArgs& a, cudaStream_t st) {
    const int s2 = a.L.s * a.L.s;
    if (a.heads == 0 || a.L.windows == 0) return cudaSuccess;
    if (a.dim > 128 || NT % s2 != 0) return cudaErrorInvalidValue;
    const int align = a.q.dtype == GSA_DTYPE_BF16 ? 8 : 4;
    auto ok = [&](const TensorRef& t) {
        return t.rs % align == 0 && t.hs % align == 0 && (reinterpret_cast<uintptr_t>(t.data) & 15) == 0;
    };
    const bool vec8 = a.dim % 8 == 0 && ok(a.k) && ok(a.v);
    if (a.q.dtype == GSA_DTYPE_BF16) {
        return a.dim <= 64 ? launch_typed<__nv_bfloat16, 64>(a, vec8, st) : launch_typed<__nv_bfloat16, 128>(a, vec8, st);
    }
    return a.dim <= 64 ? launch_typed<float, 64>(a, vec8, st) : launch_typed<float, 128>(a, vec8, st);
}

}  // namespace gsa_sm100
