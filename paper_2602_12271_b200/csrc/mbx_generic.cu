// SIMT (CUDA-core, fp32 arithmetic) kernels of the tiled MonarchAttention
// forward.  They implement every plan the reference supports (untiled
// `solve`, tiled `solve_tiled`, permuted aligned / raw orderings, any T,
// rectangular chunked-KV grids) and are the fp32 parity path; the tcgen05
// kernels (mbx_tc.cu) take the hot bf16 shapes.
//
// Kernel-oriented restatement of solver.py:161-204:
//   row stage    per (query tile a, key tile c, row k), queries j, keys i:
//                z = (alpha_R . K) / max(c_R, eps_div)         solver.py:187-188
//                R = softmax_i z                               solver.py:189
//                alpha_L = R K, Y = R V, c_L = sum R log R     solver.py:190-191, factors.py:123
//   column stage per (query tile a, column j), queries l, keys (c, k):
//                S = Q . alpha_L - c_L, L = softmax_(c,k) S    solver.py:192-195
//                O = L Y                                       factors.py:124
//   alpha_R step alpha_R = sum_l L Q, c_R = sum_l L            solver.py:185-186
// Softmaxes are online (running max / sum) so s1, s2 and the key count are
// unbounded; c_L uses sum R log R = sum R z - lse (exact, Σ R = 1).
#include "mbx_internal.h"

#include <math.h>

namespace mbx {
namespace {

constexpr int kWarps = 8;          // warps per CTA; one query (or key) per warp
constexpr int kThreads = kWarps * 32;
constexpr int kChunk = 32;         // keys staged in shared memory per step
constexpr int kMaxVec = 8;         // features per lane: d, dv <= 256

__device__ __forceinline__ float load_el(const float* p) { return __ldg(p); }
__device__ __forceinline__ float load_el(const __nv_bfloat16* p) { return __bfloat162float(*p); }
__device__ __forceinline__ void store_el(float* p, float x) { *p = x; }
__device__ __forceinline__ void store_el(__nv_bfloat16* p, float x) { *p = __float2bfloat16_rn(x); }

__device__ __forceinline__ float warp_max(float x) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x = fmaxf(x, __shfl_xor_sync(0xffffffffu, x, o));
    return x;
}
__device__ __forceinline__ float warp_sum(float x) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    return x;
}

// slot index of (tile, row, col): p = ((l1*s1 + r)*c2 + j1)*s2 + j (solver.py:178)
__device__ __forceinline__ int slot_of(const Geometry& g, int tile, int r, int j) {
    const int l1 = tile / g.c2, j1 = tile - (tile / g.c2) * g.c2;
    return ((l1 * g.s1 + r) * g.c2 + j1) * g.s2 + j;
}
__device__ __forceinline__ int64_t q_row(const Geometry& g, int tile, int r, int j) {
    const int p = slot_of(g, tile, r, j);
    return g.q_order ? (int64_t)g.q_order[p] : (int64_t)p;
}
__device__ __forceinline__ int64_t kv_row(const Geometry& g, int tile, int r, int j) {
    const int p = slot_of(g, tile, r, j);
    return g.kv_order ? (int64_t)g.kv_order[p] : (int64_t)p;
}

// --------------------------------------------------------------------------
// Row stage.  grid = (gq*gk*s1, ceil(s2/8), bh); warp -> query column j.
// --------------------------------------------------------------------------
template <typename T>
__global__ void __launch_bounds__(kThreads)
row_stage(Geometry g, const T* __restrict__ q, const T* __restrict__ k, const T* __restrict__ v,
          Workspace ws, int iter, int last, float* __restrict__ r_factor) {
    extern __shared__ float smem[];
    const int d = g.d, dv = g.dv;
    float* Ks = smem;                          // [kChunk][d+1]
    float* Vs = Ks + kChunk * (d + 1);         // [kChunk][dv+1]
    float* Qs = Vs + kChunk * (dv + 1);        // [kWarps][d]

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int x = blockIdx.x;
    const int kr = x % g.s1;
    const int c = (x / g.s1) % g.gk;
    const int a = x / (g.s1 * g.gk);
    const int bh = blockIdx.z;
    const int b = bh / g.heads, h = bh - (bh / g.heads) * g.heads;
    const int j = blockIdx.y * kWarps + warp;
    const bool jv = j < g.s2;
    const bool need_y = last && dv > 0 && ws.y != nullptr;

    const T* qb = q + b * g.qs[0] + h * g.qs[1];
    const T* kb = k + b * g.ks[0] + h * g.ks[1];
    const T* vb = v + b * g.vs[0] + h * g.vs[1];

    // query row: alpha_R / c_R.  At iter 0, L = I => alpha_R = scale*Q, c_R = 1.
    float div = 1.f;
    if (jv) {
        if (iter == 0) {
            const T* src = qb + q_row(g, a, kr, j) * g.qs[2];
            for (int e = lane; e < d; e += 32) Qs[warp * d + e] = g.scale * load_el(src + e);
        } else {
            const int64_t o = ((((int64_t)bh * g.gq + a) * g.gk + c) * g.s1 + kr) * g.s2 + j;
            const float* src = ws.alpha_r + o * d;
            for (int e = lane; e < d; e += 32) Qs[warp * d + e] = src[e];
            div = fmaxf(ws.c_r[o], g.eps_div);
        }
    }

    float m = -INFINITY, l = 0.f, A = 0.f;
    float acc_k[kMaxVec], acc_v[kMaxVec];
#pragma unroll
    for (int t = 0; t < kMaxVec; ++t) { acc_k[t] = 0.f; acc_v[t] = 0.f; }

    for (int i0 = 0; i0 < g.s2; i0 += kChunk) {
        __syncthreads();
        const int nvalid = min(kChunk, g.s2 - i0);
        for (int idx = threadIdx.x; idx < kChunk * d; idx += kThreads) {
            const int ii = idx / d, e = idx - (idx / d) * d;
            Ks[ii * (d + 1) + e] = ii < nvalid ? load_el(kb + kv_row(g, c, kr, i0 + ii) * g.ks[2] + e) : 0.f;
        }
        if (need_y) {
            for (int idx = threadIdx.x; idx < kChunk * dv; idx += kThreads) {
                const int ii = idx / dv, e = idx - (idx / dv) * dv;
                Vs[ii * (dv + 1) + e] = ii < nvalid ? load_el(vb + kv_row(g, c, kr, i0 + ii) * g.vs[2] + e) : 0.f;
            }
        }
        __syncthreads();
        if (!jv) continue;
        float z = -INFINITY;
        if (lane < nvalid) {
            float dot = 0.f;
            const float* kr_ = Ks + lane * (d + 1);
            const float* qr_ = Qs + warp * d;
            for (int e = 0; e < d; ++e) dot = fmaf(qr_[e], kr_[e], dot);
            z = (iter == 0) ? dot : dot / div;
        }
        const float mn = fmaxf(m, warp_max(z));
        const float corr = (m == -INFINITY) ? 0.f : __expf(m - mn);
        const float p = lane < nvalid ? expf(z - mn) : 0.f;
        l = l * corr + warp_sum(p);
        A = A * corr + warp_sum(lane < nvalid ? p * z : 0.f);
        m = mn;
#pragma unroll
        for (int t = 0; t < kMaxVec; ++t) { acc_k[t] *= corr; acc_v[t] *= corr; }
        for (int ii = 0; ii < nvalid; ++ii) {
            const float pi = __shfl_sync(0xffffffffu, p, ii);
#pragma unroll
            for (int t = 0; t < kMaxVec; ++t) {
                const int e = lane + 32 * t;
                if (e < d) acc_k[t] = fmaf(pi, Ks[ii * (d + 1) + e], acc_k[t]);
                if (need_y && e < dv) acc_v[t] = fmaf(pi, Vs[ii * (dv + 1) + e], acc_v[t]);
            }
        }
    }

    const float lse = m + logf(l);
    if (jv) {
        const float inv_l = 1.f / l;
        const int key = c * g.s1 + kr;
        const int64_t o = (((int64_t)bh * g.gq + a) * g.s2 + j) * g.nkeys + key;
#pragma unroll
        for (int t = 0; t < kMaxVec; ++t) {
            const int e = lane + 32 * t;
            if (e < d) ws.alpha_l[o * d + e] = acc_k[t] * inv_l;
            if (need_y && e < dv) ws.y[o * dv + e] = acc_v[t] * inv_l;
        }
        if (lane == 0) ws.c_l[o] = A * inv_l - lse;   // sum_i R_i z_i - lse = sum R log R
    }

    // Optional export of R' [l1,j1,k1,i1,k2,j2,i2] (factors.py:61-64): the final one, or this
    // refinement's slice when every refinement is exported (MBX_FLAG_ALL_ITERS).
    if (!r_factor) return;
    float* rrow = r_factor + (((((int64_t)bh * g.gq + a) * g.gk + c) * g.s1 + kr) * g.s2 + (jv ? j : 0)) * g.s2;
    for (int i0 = 0; i0 < g.s2; i0 += kChunk) {
        __syncthreads();
        const int nvalid = min(kChunk, g.s2 - i0);
        for (int idx = threadIdx.x; idx < kChunk * d; idx += kThreads) {
            const int ii = idx / d, e = idx - (idx / d) * d;
            Ks[ii * (d + 1) + e] = ii < nvalid ? load_el(kb + kv_row(g, c, kr, i0 + ii) * g.ks[2] + e) : 0.f;
        }
        __syncthreads();
        if (!jv || lane >= nvalid) continue;
        float dot = 0.f;
        const float* kr_ = Ks + lane * (d + 1);
        const float* qr_ = Qs + warp * d;
        for (int e = 0; e < d; ++e) dot = fmaf(qr_[e], kr_[e], dot);
        const float z = (iter == 0) ? dot : dot / div;
        rrow[i0 + lane] = expf(z - lse);
    }
}

// --------------------------------------------------------------------------
// Column stage.  grid = (gq*s2, ceil(s1/8), bh); warp -> query row l.
// Writes lse of each L row; on the last iteration also O = L Y.
// --------------------------------------------------------------------------
template <typename T>
__global__ void __launch_bounds__(kThreads)
column_stage(Geometry g, const T* __restrict__ q, T* __restrict__ out, Workspace ws, int last) {
    extern __shared__ float smem[];
    const int d = g.d, dv = g.dv;
    float* As = smem;                          // [kChunk][d+1]
    float* Ys = As + kChunk * (d + 1);         // [kChunk][dv+1]
    float* Cs = Ys + kChunk * (dv + 1);        // [kChunk]
    float* Qs = Cs + kChunk;                   // [kWarps][d]

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int j = blockIdx.x % g.s2, a = blockIdx.x / g.s2;
    const int bh = blockIdx.z;
    const int b = bh / g.heads, h = bh - (bh / g.heads) * g.heads;
    const int l = blockIdx.y * kWarps + warp;
    const bool lv = l < g.s1;
    const bool emit = last && out != nullptr;

    int64_t tok = 0;
    if (lv) {
        tok = q_row(g, a, l, j);
        const T* src = q + b * g.qs[0] + h * g.qs[1] + tok * g.qs[2];
        for (int e = lane; e < d; e += 32) Qs[warp * d + e] = g.scale * load_el(src + e);
    }
    const int64_t col = ((int64_t)bh * g.gq + a) * g.s2 + j;
    const float* A_col = ws.alpha_l + col * g.nkeys * d;
    const float* Y_col = ws.y ? ws.y + col * g.nkeys * dv : nullptr;
    const float* C_col = ws.c_l + col * g.nkeys;

    float m = -INFINITY, s = 0.f;
    float acc[kMaxVec];
#pragma unroll
    for (int t = 0; t < kMaxVec; ++t) acc[t] = 0.f;

    for (int k0 = 0; k0 < g.nkeys; k0 += kChunk) {
        __syncthreads();
        const int nvalid = min(kChunk, g.nkeys - k0);
        for (int idx = threadIdx.x; idx < kChunk * d; idx += kThreads) {
            const int ii = idx / d, e = idx - (idx / d) * d;
            As[ii * (d + 1) + e] = ii < nvalid ? A_col[(int64_t)(k0 + ii) * d + e] : 0.f;
        }
        if (emit) {
            for (int idx = threadIdx.x; idx < kChunk * dv; idx += kThreads) {
                const int ii = idx / dv, e = idx - (idx / dv) * dv;
                Ys[ii * (dv + 1) + e] = ii < nvalid ? Y_col[(int64_t)(k0 + ii) * dv + e] : 0.f;
            }
        }
        if (threadIdx.x < kChunk) Cs[threadIdx.x] = threadIdx.x < nvalid ? C_col[k0 + threadIdx.x] : 0.f;
        __syncthreads();
        if (!lv) continue;
        float sc = -INFINITY;
        if (lane < nvalid) {
            float dot = 0.f;
            const float* ar = As + lane * (d + 1);
            const float* qr = Qs + warp * d;
            for (int e = 0; e < d; ++e) dot = fmaf(qr[e], ar[e], dot);
            sc = dot - Cs[lane];
        }
        const float mn = fmaxf(m, warp_max(sc));
        const float corr = (m == -INFINITY) ? 0.f : __expf(m - mn);
        const float p = lane < nvalid ? expf(sc - mn) : 0.f;
        s = s * corr + warp_sum(p);
        m = mn;
        if (emit) {
#pragma unroll
            for (int t = 0; t < kMaxVec; ++t) acc[t] *= corr;
            for (int ii = 0; ii < nvalid; ++ii) {
                const float pi = __shfl_sync(0xffffffffu, p, ii);
#pragma unroll
                for (int t = 0; t < kMaxVec; ++t) {
                    const int e = lane + 32 * t;
                    if (e < dv) acc[t] = fmaf(pi, Ys[ii * (dv + 1) + e], acc[t]);
                }
            }
        }
    }
    if (!lv) return;
    if (lane == 0) ws.lse[col * g.s1 + l] = m + logf(s);
    if (emit) {
        const float inv = 1.f / s;
        T* dst = out + b * g.os[0] + h * g.os[1] + tok * g.os[2];
#pragma unroll
        for (int t = 0; t < kMaxVec; ++t) {
            const int e = lane + 32 * t;
            if (e < dv) store_el(dst + e, acc[t] * inv);
        }
    }
}

// --------------------------------------------------------------------------
// alpha_R / L-export step.  grid = (gq*s2, ceil(nkeys/8), bh); warp -> key.
// L[l,(c,k)] = exp(S - lse_l);  alpha_R[a,c,k,j] = sum_l L q_l,  c_R = sum_l L.
// --------------------------------------------------------------------------
template <typename T>
__global__ void __launch_bounds__(kThreads)
alpha_r_stage(Geometry g, const T* __restrict__ q, Workspace ws, int want_alpha,
              float* __restrict__ l_factor) {
    extern __shared__ float smem[];
    const int d = g.d;
    float* Qs = smem;                          // [kChunk][d+1]
    float* Ls = Qs + kChunk * (d + 1);         // [kChunk] lse
    float* Ak = Ls + kChunk;                   // [kWarps][d]

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int j = blockIdx.x % g.s2, a = blockIdx.x / g.s2;
    const int bh = blockIdx.z;
    const int b = bh / g.heads, h = bh - (bh / g.heads) * g.heads;
    const int key = blockIdx.y * kWarps + warp;
    const bool kv = key < g.nkeys;
    const int c = kv ? key / g.s1 : 0, kr = kv ? key - (key / g.s1) * g.s1 : 0;
    const int64_t col = ((int64_t)bh * g.gq + a) * g.s2 + j;
    const T* qb = q + b * g.qs[0] + h * g.qs[1];

    float ck = 0.f;
    if (kv) {
        const float* src = ws.alpha_l + (col * g.nkeys + key) * d;
        for (int e = lane; e < d; e += 32) Ak[warp * d + e] = src[e];
        ck = ws.c_l[col * g.nkeys + key];
    }
    float acc[kMaxVec];
#pragma unroll
    for (int t = 0; t < kMaxVec; ++t) acc[t] = 0.f;
    float mass = 0.f;

    for (int l0 = 0; l0 < g.s1; l0 += kChunk) {
        __syncthreads();
        const int nvalid = min(kChunk, g.s1 - l0);
        for (int idx = threadIdx.x; idx < kChunk * d; idx += kThreads) {
            const int ii = idx / d, e = idx - (idx / d) * d;
            Qs[ii * (d + 1) + e] =
                ii < nvalid ? g.scale * load_el(qb + q_row(g, a, l0 + ii, j) * g.qs[2] + e) : 0.f;
        }
        if (threadIdx.x < kChunk) Ls[threadIdx.x] = threadIdx.x < nvalid ? ws.lse[col * g.s1 + l0 + threadIdx.x] : 0.f;
        __syncthreads();
        if (!kv) continue;
        float p = 0.f;
        if (lane < nvalid) {
            float dot = 0.f;
            const float* qr = Qs + lane * (d + 1);
            const float* ar = Ak + warp * d;
            for (int e = 0; e < d; ++e) dot = fmaf(qr[e], ar[e], dot);
            p = expf(dot - ck - Ls[lane]);
            if (l_factor) {
                // L' [l1,j1,k1,i1,j2,l2,k2] = [a][c][j][l][k]
                const int64_t o = (((((int64_t)bh * g.gq + a) * g.gk + c) * g.s2 + j) * g.s1 + (l0 + lane)) * g.s1 + kr;
                l_factor[o] = p;
            }
        }
        if (!want_alpha) continue;
        mass += warp_sum(p);
        for (int ii = 0; ii < nvalid; ++ii) {
            const float pi = __shfl_sync(0xffffffffu, p, ii);
#pragma unroll
            for (int t = 0; t < kMaxVec; ++t) {
                const int e = lane + 32 * t;
                if (e < d) acc[t] = fmaf(pi, Qs[ii * (d + 1) + e], acc[t]);
            }
        }
    }
    if (!kv || !want_alpha) return;
    const int64_t o = ((((int64_t)bh * g.gq + a) * g.gk + c) * g.s1 + kr) * g.s2 + j;
#pragma unroll
    for (int t = 0; t < kMaxVec; ++t) {
        const int e = lane + 32 * t;
        if (e < d) ws.alpha_r[o * d + e] = acc[t];
    }
    if (lane == 0) ws.c_r[o] = mass;
}

// --------------------------------------------------------------------------
// Block-apply of given factors (factors.py:110-125): Y = R' V then O = L' Y.
// --------------------------------------------------------------------------
template <typename T>
__global__ void __launch_bounds__(kThreads)
apply_y(Geometry g, const float* __restrict__ r_factor, const T* __restrict__ v, Workspace ws) {
    extern __shared__ float smem[];
    const int dv = g.dv;
    float* Vs = smem;                          // [kChunk][dv+1]
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int x = blockIdx.x;
    const int kr = x % g.s1, c = (x / g.s1) % g.gk, a = x / (g.s1 * g.gk);
    const int bh = blockIdx.z;
    const int b = bh / g.heads, h = bh - (bh / g.heads) * g.heads;
    const int j = blockIdx.y * kWarps + warp;
    const bool jv = j < g.s2;
    const T* vb = v + b * g.vs[0] + h * g.vs[1];
    const float* rrow = r_factor + (((((int64_t)bh * g.gq + a) * g.gk + c) * g.s1 + kr) * g.s2 + (jv ? j : 0)) * g.s2;
    float acc[kMaxVec];
#pragma unroll
    for (int t = 0; t < kMaxVec; ++t) acc[t] = 0.f;
    for (int i0 = 0; i0 < g.s2; i0 += kChunk) {
        __syncthreads();
        const int nvalid = min(kChunk, g.s2 - i0);
        for (int idx = threadIdx.x; idx < kChunk * dv; idx += kThreads) {
            const int ii = idx / dv, e = idx - (idx / dv) * dv;
            Vs[ii * (dv + 1) + e] = ii < nvalid ? load_el(vb + kv_row(g, c, kr, i0 + ii) * g.vs[2] + e) : 0.f;
        }
        __syncthreads();
        if (!jv) continue;
        const float p = lane < nvalid ? rrow[i0 + lane] : 0.f;
        for (int ii = 0; ii < nvalid; ++ii) {
            const float pi = __shfl_sync(0xffffffffu, p, ii);
#pragma unroll
            for (int t = 0; t < kMaxVec; ++t) {
                const int e = lane + 32 * t;
                if (e < dv) acc[t] = fmaf(pi, Vs[ii * (dv + 1) + e], acc[t]);
            }
        }
    }
    if (!jv) return;
    const int64_t o = (((int64_t)bh * g.gq + a) * g.s2 + j) * g.nkeys + (c * g.s1 + kr);
#pragma unroll
    for (int t = 0; t < kMaxVec; ++t) {
        const int e = lane + 32 * t;
        if (e < dv) ws.y[o * dv + e] = acc[t];
    }
}

template <typename T>
__global__ void __launch_bounds__(kThreads)
apply_out(Geometry g, const float* __restrict__ l_factor, T* __restrict__ out, Workspace ws) {
    extern __shared__ float smem[];
    const int dv = g.dv;
    float* Ys = smem;                          // [kChunk][dv+1]
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int j = blockIdx.x % g.s2, a = blockIdx.x / g.s2;
    const int bh = blockIdx.z;
    const int b = bh / g.heads, h = bh - (bh / g.heads) * g.heads;
    const int l = blockIdx.y * kWarps + warp;
    const bool lv = l < g.s1;
    const int64_t col = ((int64_t)bh * g.gq + a) * g.s2 + j;
    const float* Y_col = ws.y + col * g.nkeys * dv;
    float acc[kMaxVec];
#pragma unroll
    for (int t = 0; t < kMaxVec; ++t) acc[t] = 0.f;
    for (int k0 = 0; k0 < g.nkeys; k0 += kChunk) {
        __syncthreads();
        const int nvalid = min(kChunk, g.nkeys - k0);
        for (int idx = threadIdx.x; idx < kChunk * dv; idx += kThreads) {
            const int ii = idx / dv, e = idx - (idx / dv) * dv;
            Ys[ii * (dv + 1) + e] = ii < nvalid ? Y_col[(int64_t)(k0 + ii) * dv + e] : 0.f;
        }
        __syncthreads();
        if (!lv) continue;
        float p = 0.f;
        if (lane < nvalid) {
            const int key = k0 + lane, c = key / g.s1, kr = key - (key / g.s1) * g.s1;
            p = l_factor[(((((int64_t)bh * g.gq + a) * g.gk + c) * g.s2 + j) * g.s1 + l) * g.s1 + kr];
        }
        for (int ii = 0; ii < nvalid; ++ii) {
            const float pi = __shfl_sync(0xffffffffu, p, ii);
#pragma unroll
            for (int t = 0; t < kMaxVec; ++t) {
                const int e = lane + 32 * t;
                if (e < dv) acc[t] = fmaf(pi, Ys[ii * (dv + 1) + e], acc[t]);
            }
        }
    }
    if (!lv) return;
    T* dst = out + b * g.os[0] + h * g.os[1] + q_row(g, a, l, j) * g.os[2];
#pragma unroll
    for (int t = 0; t < kMaxVec; ++t) {
        const int e = lane + 32 * t;
        if (e < dv) store_el(dst + e, acc[t]);
    }
}

template <typename K>
cudaError_t set_smem(K kernel, size_t bytes) {
    return cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

inline int cdiv(int a, int b) { return (a + b - 1) / b; }

template <typename T>
cudaError_t forward_t(const Geometry& g, const T* q, const T* k, const T* v, T* out,
                      float* l_factor, float* r_factor, const Workspace& ws, cudaStream_t st, bool all_iters) {
    const size_t sm_row = sizeof(float) * (kChunk * (g.d + 1) + kChunk * (g.dv + 1) + kWarps * g.d);
    const size_t sm_col = sizeof(float) * (kChunk * (g.d + 1) + kChunk * (g.dv + 1) + kChunk + kWarps * g.d);
    const size_t sm_ar = sizeof(float) * (kChunk * (g.d + 1) + kChunk + kWarps * g.d);
    cudaError_t e;
    if ((e = set_smem(row_stage<T>, sm_row)) != cudaSuccess) return e;
    if ((e = set_smem(column_stage<T>, sm_col)) != cudaSuccess) return e;
    if ((e = set_smem(alpha_r_stage<T>, sm_ar)) != cudaSuccess) return e;
    const dim3 grid_row(g.gq * g.gk * g.s1, cdiv(g.s2, kWarps), g.bh);
    const dim3 grid_col(g.gq * g.s2, cdiv(g.s1, kWarps), g.bh);
    const dim3 grid_ar(g.gq * g.s2, cdiv(g.nkeys, kWarps), g.bh);
    const size_t rslice = (size_t)g.bh * g.gq * g.gk * g.s1 * g.s2 * g.s2;
    const size_t lslice = (size_t)g.bh * g.gq * g.gk * g.s2 * g.s1 * g.s1;
    for (int it = 0; it < g.T; ++it) {
        const int last = it == g.T - 1;
        float* rf = !r_factor ? nullptr : all_iters ? r_factor + it * rslice : last ? r_factor : nullptr;
        float* lf = !l_factor ? nullptr : all_iters ? l_factor + it * lslice : last ? l_factor : nullptr;
        {
            ProfScope p("simt_row_stage", st);
            row_stage<T><<<grid_row, kThreads, sm_row, st>>>(g, q, k, v, ws, it, last, rf);
        }
        {
            ProfScope p("simt_column_stage", st);
            column_stage<T><<<grid_col, kThreads, sm_col, st>>>(g, q, last ? out : nullptr, ws, last);
        }
        if (!last || lf) {
            ProfScope p("simt_alpha_r_stage", st);
            alpha_r_stage<T><<<grid_ar, kThreads, sm_ar, st>>>(g, q, ws, last ? 0 : 1, lf);
        }
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
    }
    return cudaSuccess;
}

template <typename T>
cudaError_t apply_t(const Geometry& g, const float* l_factor, const float* r_factor,
                    const T* v, T* out, const Workspace& ws, cudaStream_t st) {
    const size_t sm = sizeof(float) * kChunk * (g.dv + 1);
    cudaError_t e;
    if ((e = set_smem(apply_y<T>, sm)) != cudaSuccess) return e;
    if ((e = set_smem(apply_out<T>, sm)) != cudaSuccess) return e;
    apply_y<T><<<dim3(g.gq * g.gk * g.s1, cdiv(g.s2, kWarps), g.bh), kThreads, sm, st>>>(g, r_factor, v, ws);
    apply_out<T><<<dim3(g.gq * g.s2, cdiv(g.s1, kWarps), g.bh), kThreads, sm, st>>>(g, l_factor, out, ws);
    return cudaGetLastError();
}

}  // namespace

cudaError_t generic_forward(const Geometry& g, int dtype, const void* q, const void* k,
                            const void* v, void* out, float* l_factor, float* r_factor,
                            const Workspace& ws, cudaStream_t stream, bool all_iters) {
    if (dtype == MBX_F32)
        return forward_t<float>(g, (const float*)q, (const float*)k, (const float*)v, (float*)out,
                                l_factor, r_factor, ws, stream, all_iters);
    return forward_t<__nv_bfloat16>(g, (const __nv_bfloat16*)q, (const __nv_bfloat16*)k,
                                    (const __nv_bfloat16*)v, (__nv_bfloat16*)out, l_factor,
                                    r_factor, ws, stream, all_iters);
}

cudaError_t generic_apply(const Geometry& g, int dtype, const float* l_factor,
                          const float* r_factor, const void* v, void* out,
                          const Workspace& ws, cudaStream_t stream) {
    if (dtype == MBX_F32)
        return apply_t<float>(g, l_factor, r_factor, (const float*)v, (float*)out, ws, stream);
    return apply_t<__nv_bfloat16>(g, l_factor, r_factor, (const __nv_bfloat16*)v,
                                  (__nv_bfloat16*)out, ws, stream);
}

}  // namespace mbx
