// Backward pass of the tiled MonarchAttention forward (the
// paper's finetuning backward, PAPER.md:135-136, 644 -- not in the reference
// package, whose SPEC.md:8 leaves it out).  Batched contractions (TF32 mma.sync for
// bf16 I/O, fp32 SIMT for fp32 I/O) and row kernels over the fp32 factors the
// forward exports (R' and L' of every refinement, factors.py:57-79 layout),
// restating the chain rule of solver.py:184-195 / factors.py:123-124:
//
//   forward per refinement t:  z = A_t K^T,  R = softmax_i z,  aL = R K,
//     c_L = sum R z - lse,  S = Q aL - c_L,  L = softmax_(c,k) S,
//     A_{t+1} = (sum_l L Q) / max(sum_l L, eps);  last: Y = R V,  O = L Y.
//   backward (last refinement first):
//     dL = dO . Y,  dS = L (dL - sum L dL),  dQ += dS aL,  daL = dS^T Q,  dc_L = -sum_l dS,
//     dY = L^T dO,  dR = dY V^T + daL K^T,  dz = R (dR - sum R dR) + dc_L R (z - sum R z),
//     dK += dz^T A_t + R^T daL,  dV += R^T dY,  dA_t = dz K;
//     t = 0: dQ += sum_c dA_0;  t > 0: dalpha_R = dA_t / m, dc_R = -(dA_t . A_t) / m
//     (m = max(c_R, eps), zero where clamped), dL_{t-1} = Q dalpha_R^T + dc_R, dQ += L_{t-1} dalpha_R.
//
// Every contraction is one launch of a strided batched GEMM (4 batch levels, a
// two-level reduction index); the softmax backward steps are row kernels.  The
// oracle is torch autograd of oracle/monarch_torch.py (tests/test_backward_gpu.py).
#include "mbx_internal.h"

#include <cublas_v2.h>
#include <dlfcn.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>
#include <mutex>
#include <type_traits>

namespace mbx {
namespace {

__device__ __forceinline__ float ld(const float* p) { return *p; }
__device__ __forceinline__ float ld(const __nv_bfloat16* p) { return __bfloat162float(*p); }
__device__ __forceinline__ void store(float* p, float x) { *p = x; }
__device__ __forceinline__ void store(__nv_bfloat16* p, float x) { *p = __float2bfloat16_rn(x); }

__device__ __forceinline__ float4 ld4(const float* p) { return *reinterpret_cast<const float4*>(p); }
__device__ __forceinline__ float4 ld4(const __nv_bfloat16* p) {
    const uint2 u = *reinterpret_cast<const uint2*>(p);
    const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.x));
    const float2 b = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.y));
    return make_float4(a.x, a.y, b.x, b.y);
}
__device__ __forceinline__ void store4(float* p, float4 x) { *reinterpret_cast<float4*>(p) = x; }
__device__ __forceinline__ void store4(__nv_bfloat16* p, float4 x) {
    __nv_bfloat162 a = __floats2bfloat162_rn(x.x, x.y), b = __floats2bfloat162_rn(x.z, x.w);
    uint2 u;
    u.x = *reinterpret_cast<uint32_t*>(&a);
    u.y = *reinterpret_cast<uint32_t*>(&b);
    *reinterpret_cast<uint2*>(p) = u;
}

// ---------------------------------------------------------------- batched GEMM
// C[b][m][n] = alpha * sum_{k1 < K1, k2 < K2} A[b][m][k1][k2] B[b][k1][k2][n] (+ C if acc),
// b = (b0, b1, b2, b3); every operand addressed by element strides (0 = broadcast).
struct Operand {
    const float* p;
    int64_t s0, s1;        // A: (m, k1) / B: (n, k1) / C: (m, n)
    int64_t s2;            // A, B: k2 stride
    int64_t b[4];          // batch strides
};
struct Gemm {
    int M, N, K1, K2;
    int nb[4];
    Operand A, B, C;
    float alpha;
    int acc;
};

constexpr int kTM = 64, kTN = 64, kTK = 16, kGemmThreads = 256;

__global__ void __launch_bounds__(kGemmThreads) gemm_batched(Gemm G) {
    __shared__ float As[kTK][kTM + 4];
    __shared__ float Bs[kTK][kTN + 4];
    const int tiles_n = (G.N + kTN - 1) / kTN;
    int64_t bx = blockIdx.x;
    const int tn = (int)(bx % tiles_n);
    bx /= tiles_n;
    int bi[4];
    bi[3] = (int)(bx % G.nb[3]); bx /= G.nb[3];
    bi[2] = (int)(bx % G.nb[2]); bx /= G.nb[2];
    bi[1] = (int)(bx % G.nb[1]); bx /= G.nb[1];
    bi[0] = (int)bx;
    const int m0 = blockIdx.y * kTM, n0 = tn * kTN;
    const float* A = G.A.p;
    const float* B = G.B.p;
    float* C = const_cast<float*>(G.C.p);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        A += bi[i] * G.A.b[i];
        B += bi[i] * G.B.b[i];
        C += bi[i] * G.C.b[i];
    }
    const int tid = threadIdx.x;
    const int tx = tid & 15, ty = tid >> 4;   // 16 x 16 threads, 4 x 4 outputs each
    float acc[4][4] = {};
    const int K = G.K1 * G.K2;
    for (int k0 = 0; k0 < K; k0 += kTK) {
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            const int idx = tid + r * kGemmThreads;   // 0 .. 1023
            // A tile: kTK x kTM, consecutive threads walk m (A's m stride is the common small one)
            {
                const int kk = idx / kTM, mm = idx % kTM;
                const int k = k0 + kk, m = m0 + mm;
                float x = 0.f;
                if (k < K && m < G.M) {
                    const int k1 = k / G.K2, k2 = k - (k / G.K2) * G.K2;
                    x = A[m * G.A.s0 + k1 * G.A.s1 + k2 * G.A.s2];
                }
                As[kk][mm] = x;
            }
            {
                const int kk = idx / kTN, nn = idx % kTN;
                const int k = k0 + kk, n = n0 + nn;
                float x = 0.f;
                if (k < K && n < G.N) {
                    const int k1 = k / G.K2, k2 = k - (k / G.K2) * G.K2;
                    x = B[n * G.B.s0 + k1 * G.B.s1 + k2 * G.B.s2];
                }
                Bs[kk][nn] = x;
            }
        }
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < kTK; ++kk) {
            float a[4], b[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                a[i] = As[kk][ty + 16 * i];
                b[i] = Bs[kk][tx + 16 * i];
            }
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int m = m0 + ty + 16 * i;
        if (m >= G.M) continue;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int n = n0 + tx + 16 * j;
            if (n >= G.N) continue;
            float* c = C + m * G.C.s0 + n * G.C.s1;
            const float v = G.alpha * acc[i][j];
            *c = G.acc ? *c + v : v;
        }
    }
}

// ------------------------------------------- batched GEMM on the tensor cores (TF32)
// The same contraction for bf16 I/O: 64 x 64 CTA tiles, four warps of 32 x 32 issuing
// mma.sync m16n8k8 TF32 (fp32 accumulate), K in steps of 32 with the next step's
// global loads in registers while the current one computes.  Each operand is staged
// in the shared layout its global unit stride gives coalesced loads for: [row][k]
// (stride 36) when k is the unit stride, [k][row] (stride 72) when rows are -- both
// bank-conflict free for the stores and for the fragment reads.  The reduction runs
// k1 outer (K1 > 1 only when it does not fold into one stride), k2 inner.  The
// per-batch matrices are tiny (30-128 rows), so one launch holds thousands of CTAs and
// several are resident per SM; cuBLAS's batched TF32 GEMM on these shapes ran at
// ~1/15 of the bandwidth its bytes need (bwd_dl: 183 us for 77 MB at C2).
constexpr int kMT = 64, kMK = 32, kMThreads = 128;


// stage a kMT x kMK tile of rows [r0, r0 + kMT) and k2 [k0, k0 + kMK) of operand P into
// registers.  MODE bit 0 (KC): k is the unit stride, else rows are; bit 1 (VEC): 16-byte
// loads along the unit stride (host-checked alignment, extent a multiple of 4).  Scalar
// KC -- element r of a thread is row tid / 32 + 4 r, k tid % 32 (a warp reads 128 B of one
// row); scalar rows -- row tid % 64, k tid / 64 + 2 r.  Vector KC -- row tid / 8 + 16 r,
// k 4 (tid % 8); vector rows -- rows 4 (tid % 16), k tid / 16 + 8 r.  One index is fixed
// per thread, so the address steps by a constant.
template <int MODE>
__device__ __forceinline__ void mma_load(float (&x)[kMT * kMK / kMThreads], const float* P, int64_t s_row,
                                         int64_t s_k, int r0, int rows, int k0, int K2, int tid) {
    constexpr int kN = kMT * kMK / kMThreads;
    if (MODE == 3) {
        const int row = r0 + tid / 8, kk = k0 + 4 * (tid % 8);
        const float* p = P + (int64_t)row * s_row + kk;
        const bool kin = kk < K2;
#pragma unroll
        for (int r = 0; r < kN / 4; ++r) {
            const float4 v = (kin && row + 16 * r < rows) ? __ldg(reinterpret_cast<const float4*>(p + 16 * r * s_row))
                                                          : make_float4(0.f, 0.f, 0.f, 0.f);
            x[4 * r] = v.x; x[4 * r + 1] = v.y; x[4 * r + 2] = v.z; x[4 * r + 3] = v.w;
        }
    } else if (MODE == 2) {
        const int row = r0 + 4 * (tid % 16), kk = k0 + tid / 16;
        const float* p = P + row + (int64_t)kk * s_k;
        const bool rin = row < rows;
#pragma unroll
        for (int r = 0; r < kN / 4; ++r) {
            const float4 v = (rin && kk + 8 * r < K2) ? __ldg(reinterpret_cast<const float4*>(p + 8 * r * s_k))
                                                      : make_float4(0.f, 0.f, 0.f, 0.f);
            x[4 * r] = v.x; x[4 * r + 1] = v.y; x[4 * r + 2] = v.z; x[4 * r + 3] = v.w;
        }
    } else if (MODE == 1) {
        const int row = r0 + tid / kMK, kk = k0 + tid % kMK;
        const float* p = P + (int64_t)row * s_row + (int64_t)kk * s_k;
        const int64_t step = (int64_t)(kMThreads / kMK) * s_row;
        const bool kin = kk < K2;
#pragma unroll
        for (int r = 0; r < kN; ++r, p += step) x[r] = (kin && row + (kMThreads / kMK) * r < rows) ? __ldg(p) : 0.f;
    } else {
        const int row = r0 + tid % kMT, kk = k0 + tid / kMT;
        const float* p = P + (int64_t)row * s_row + (int64_t)kk * s_k;
        const int64_t step = (int64_t)(kMThreads / kMT) * s_k;
        const bool rin = row < rows;
#pragma unroll
        for (int r = 0; r < kN; ++r, p += step) x[r] = (rin && kk + (kMThreads / kMT) * r < K2) ? __ldg(p) : 0.f;
    }
}
// fp32 -> TF32, round to nearest (ties away): two integer ops instead of the emulated cvt.rna
__device__ __forceinline__ float tf32r(float x) { return __uint_as_float((__float_as_uint(x) + 0x1000u) & 0xffffe000u); }
template <int MODE>
__device__ __forceinline__ void mma_store(float* S, const float (&x)[kMT * kMK / kMThreads], int tid) {
    constexpr int kN = kMT * kMK / kMThreads;
    if (MODE >= 2) {
        float* s = MODE == 3 ? S + (tid / 8) * (kMK + 4) + 4 * (tid % 8) : S + (tid / 16) * (kMT + 8) + 4 * (tid % 16);
#pragma unroll
        for (int r = 0; r < kN / 4; ++r)
            *reinterpret_cast<float4*>(s + (MODE == 3 ? 16 * r * (kMK + 4) : 8 * r * (kMT + 8))) =
                make_float4(tf32r(x[4 * r]), tf32r(x[4 * r + 1]), tf32r(x[4 * r + 2]), tf32r(x[4 * r + 3]));
    } else {
        constexpr bool KC = MODE == 1;
        float* s = KC ? S + (tid / kMK) * (kMK + 4) + tid % kMK : S + (tid / kMT) * (kMT + 8) + tid % kMT;
#pragma unroll
        for (int r = 0; r < kN; ++r)
            s[KC ? r * (kMThreads / kMK) * (kMK + 4) : r * (kMThreads / kMT) * (kMT + 8)] = tf32r(x[r]);
    }
}
template <bool KC>
__device__ __forceinline__ float mma_at(const float* S, int row, int kk) {
    return S[KC ? row * (kMK + 4) + kk : kk * (kMT + 8) + row];
}
// four 8 x 4 (32-bit) matrices of a [row][k] tile: lane L addresses row base_row(L) of matrix L / 8
__device__ __forceinline__ void ldsm_x4(uint32_t (&r)[4], const float* p) {
    const uint32_t a = (uint32_t)__cvta_generic_to_shared(p);
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(a));
}

// 16-byte cp.async of a vector-mode tile straight into its shared layout (zero-filled
// outside [rows) x [K2)); the MMA then reads fp32 bits as TF32 (truncation)
template <int MODE>
__device__ __forceinline__ void mma_issue_async(float* S, const float* P, int64_t s_row, int64_t s_k, int r0,
                                                int rows, int k0, int K2, int tid) {
    if (MODE < 2) {   // scalar modes: 4-byte cp.async per element, same element map as mma_load
#pragma unroll
        for (int r = 0; r < kMT * kMK / kMThreads; ++r) {
            const int row = MODE == 1 ? tid / kMK + (kMThreads / kMK) * r : tid % kMT;
            const int kk = MODE == 1 ? tid % kMK : tid / kMT + (kMThreads / kMT) * r;
            const bool ok = r0 + row < rows && k0 + kk < K2;
            const float* src = P + (int64_t)(r0 + row) * s_row + (int64_t)(k0 + kk) * s_k;
            float* dst = MODE == 1 ? S + row * (kMK + 4) + kk : S + kk * (kMT + 8) + row;
            asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(
                             (uint32_t)__cvta_generic_to_shared(dst)),
                         "l"(ok ? src : P), "r"(ok ? 4 : 0)
                         : "memory");
        }
        return;
    }
#pragma unroll
    for (int r = 0; r < kMT * kMK / kMThreads / 4; ++r) {
        int row, kk;
        const float* src;
        float* dst;
        if (MODE == 3) {
            row = tid / 8 + 16 * r;
            kk = 4 * (tid % 8);
            src = P + (int64_t)(r0 + row) * s_row + k0 + kk;
            dst = S + row * (kMK + 4) + kk;
        } else {
            row = 4 * (tid % 16);
            kk = tid / 16 + 8 * r;
            src = P + (r0 + row) + (int64_t)(k0 + kk) * s_k;
            dst = S + kk * (kMT + 8) + row;
        }
        const bool ok = r0 + row < rows && k0 + kk < K2;
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)),
                     "l"(ok ? src : P), "r"(ok ? 16 : 0)
                     : "memory");
    }
}
#ifndef MBX_BWD_ASYNC_ALL
#define MBX_BWD_ASYNC_ALL 1   // 0: registers-staged steps unless both operands are 16-byte aligned
#endif
#ifndef MBX_BWD_MINB
#define MBX_BWD_MINB 6
#endif
#ifndef MBX_BWD_STAGES
#define MBX_BWD_STAGES 2
#endif
constexpr int kMStages = MBX_BWD_STAGES;
constexpr int kMTile = kMT * (kMK + 4);   // floats per operand tile, both layouts (64 x 36 = 32 x 72)
__host__ __device__ constexpr size_t mma_smem_bytes(bool async) {
    return (async ? kMStages : 1) * 2 * kMTile * sizeof(float);
}

template <int AM, int BM>
__global__ void __launch_bounds__(kMThreads, MBX_BWD_MINB) gemm_batched_tf32(Gemm G) {
    constexpr bool AK = AM & 1, BK = BM & 1;
    // both operands 16-byte aligned: a kMStages-deep cp.async ring, else registers-staged steps
    constexpr bool ASYNC = MBX_BWD_ASYNC_ALL ? true : (AM >= 2 && BM >= 2);
    extern __shared__ __align__(16) float mma_smem[];
    const int tiles_n = (G.N + kMT - 1) / kMT;
    int64_t bx = blockIdx.x;
    const int tn = (int)(bx % tiles_n);
    bx /= tiles_n;
    int bi[4];
    bi[3] = (int)(bx % G.nb[3]); bx /= G.nb[3];
    bi[2] = (int)(bx % G.nb[2]); bx /= G.nb[2];
    bi[1] = (int)(bx % G.nb[1]); bx /= G.nb[1];
    bi[0] = (int)bx;
    const int m0 = blockIdx.y * kMT, n0 = tn * kMT;
    const float* A = G.A.p;
    const float* B = G.B.p;
    float* C = const_cast<float*>(G.C.p);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        A += bi[i] * G.A.b[i];
        B += bi[i] * G.B.b[i];
        C += bi[i] * G.C.b[i];
    }
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int g = lane >> 2, t = lane & 3;
    const int wm = (warp & 1) * 32, wn = (warp >> 1) * 32;
    float acc[2][4][4] = {};
    float ra[ASYNC ? 1 : kMT * kMK / kMThreads], rb[ASYNC ? 1 : kMT * kMK / kMThreads];
    const int ksteps = (G.K2 + kMK - 1) / kMK, total = G.K1 * ksteps;
    auto issue = [&](int step) {   // ASYNC: step -> ring slot step % kMStages
        const int k1 = step / ksteps, k0 = (step - k1 * ksteps) * kMK;
        float* sa = mma_smem + (step % kMStages) * 2 * kMTile;
        if constexpr (ASYNC) {
            mma_issue_async<AM>(sa, A + (int64_t)k1 * G.A.s1, G.A.s0, G.A.s2, m0, G.M, k0, G.K2, tid);
            mma_issue_async<BM>(sa + kMTile, B + (int64_t)k1 * G.B.s1, G.B.s0, G.B.s2, n0, G.N, k0, G.K2, tid);
        }
    };
    if constexpr (ASYNC) {
#pragma unroll
        for (int p = 0; p < kMStages - 1; ++p) {
            if (p < total) issue(p);
            asm volatile("cp.async.commit_group;" ::: "memory");
        }
    } else {
        mma_load<AM>(ra, A, G.A.s0, G.A.s2, m0, G.M, 0, G.K2, tid);
        mma_load<BM>(rb, B, G.B.s0, G.B.s2, n0, G.N, 0, G.K2, tid);
    }
    for (int s = 0; s < total; ++s) {
        const float* As = mma_smem + (ASYNC ? (s % kMStages) * 2 * kMTile : 0);
        const float* Bs = As + kMTile;
        if constexpr (ASYNC) {
            asm volatile("cp.async.wait_group %0;" ::"n"(kMStages - 2) : "memory");
            __syncthreads();   // step s landed for every thread; slot (s - 1) % kMStages is free
            if (s + kMStages - 1 < total) issue(s + kMStages - 1);
            asm volatile("cp.async.commit_group;" ::: "memory");
        } else {
            mma_store<AM>(mma_smem, ra, tid);
            mma_store<BM>(mma_smem + kMTile, rb, tid);
            __syncthreads();
            if (s + 1 < total) {   // next step's loads in flight while this one computes
                const int k1 = (s + 1) / ksteps, k0 = ((s + 1) - k1 * ksteps) * kMK;
                mma_load<AM>(ra, A + (int64_t)k1 * G.A.s1, G.A.s0, G.A.s2, m0, G.M, k0, G.K2, tid);
                mma_load<BM>(rb, B + (int64_t)k1 * G.B.s1, G.B.s0, G.B.s2, n0, G.N, k0, G.K2, tid);
            }
        }
#pragma unroll
        for (int kb = 0; kb < kMK; kb += 8) {
            uint32_t af[2][4], bf[4][2];
#pragma unroll
            for (int i = 0; i < 2; ++i) {
                const int m = wm + 16 * i + g;
                if (AK) {   // matrices (rows 0-7 | 8-15) x (k 0-3 | 4-7) -> a0..a3
                    const int q = lane >> 3;
                    ldsm_x4(af[i], As + (wm + 16 * i + (lane & 7) + 8 * (q & 1)) * (kMK + 4) + kb + 4 * (q >> 1));
                } else {
                    af[i][0] = __float_as_uint(mma_at<AK>(As, m, kb + t));
                    af[i][1] = __float_as_uint(mma_at<AK>(As, m + 8, kb + t));
                    af[i][2] = __float_as_uint(mma_at<AK>(As, m, kb + t + 4));
                    af[i][3] = __float_as_uint(mma_at<AK>(As, m + 8, kb + t + 4));
                }
            }
            if (BK) {   // matrices (n block j | j + 1) x (k 0-3 | 4-7) -> b0, b1 of j, j + 1
#pragma unroll
                for (int j = 0; j < 4; j += 2) {
                    const int q = lane >> 3;
                    uint32_t r[4];
                    ldsm_x4(r, Bs + (wn + 8 * (j + (q >> 1)) + (lane & 7)) * (kMK + 4) + kb + 4 * (q & 1));
                    bf[j][0] = r[0];
                    bf[j][1] = r[1];
                    bf[j + 1][0] = r[2];
                    bf[j + 1][1] = r[3];
                }
            } else {
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const int n = wn + 8 * j + g;
                    bf[j][0] = __float_as_uint(mma_at<BK>(Bs, n, kb + t));
                    bf[j][1] = __float_as_uint(mma_at<BK>(Bs, n, kb + t + 4));
                }
            }
#pragma unroll
            for (int i = 0; i < 2; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    asm volatile(
                        "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
                        "{%8,%9}, {%0,%1,%2,%3};"
                        : "+f"(acc[i][j][0]), "+f"(acc[i][j][1]), "+f"(acc[i][j][2]), "+f"(acc[i][j][3])
                        : "r"(af[i][0]), "r"(af[i][1]), "r"(af[i][2]), "r"(af[i][3]), "r"(bf[j][0]),
                          "r"(bf[j][1]));
        }
        if constexpr (!ASYNC) __syncthreads();
    }
    // accumulate: every previous C value is loaded before the first store (a read-modify-write
    // per element would serialise 32 round trips, the stores possibly aliasing later loads)
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int j = 0; j < 4; ++j)
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const int m = m0 + wm + 16 * i + g + 8 * h, n = n0 + wn + 8 * j + 2 * t + e;
                    float& a = acc[i][j][2 * h + e];
                    a *= G.alpha;
                    if (G.acc && m < G.M && n < G.N) a += __ldg(C + (int64_t)m * G.C.s0 + (int64_t)n * G.C.s1);
                }
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int m = m0 + wm + 16 * i + g + 8 * h;
            if (m >= G.M) continue;
#pragma unroll
            for (int j = 0; j < 4; ++j)
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const int n = n0 + wn + 8 * j + 2 * t + e;
                    if (n < G.N) C[(int64_t)m * G.C.s0 + (int64_t)n * G.C.s1] = acc[i][j][2 * h + e];
                }
        }
}

// launch of the TF32 kernel: the reduction folded to one k stride when (k1, k2) allow it
bool gemm_mma(Gemm G, cudaStream_t st) {
    auto fold = [&](const Operand& o) { return G.K1 == 1 || o.s1 == (int64_t)G.K2 * o.s2; };
    if (G.K1 > 1 && G.K2 == 1) {   // k1 alone: it becomes the k2 index
        G.A.s2 = G.A.s1;
        G.B.s2 = G.B.s1;
        G.K2 = G.K1;
        G.K1 = 1;
    } else if (G.K1 > 1 && fold(G.A) && fold(G.B)) {
        G.K2 *= G.K1;
        G.K1 = 1;
    }
    const int64_t batches = (int64_t)G.nb[0] * G.nb[1] * G.nb[2] * G.nb[3];
    const int64_t gx = batches * ((G.N + kMT - 1) / kMT);
    if (gx > INT32_MAX) return false;
    dim3 grid((unsigned)gx, (unsigned)((G.M + kMT - 1) / kMT));
    // operand mode: bit 0 k-contiguous staging, bit 1 16-byte loads (every offset a multiple of 4)
    auto mode = [&](const Operand& o, int rows) {
        const bool kc = o.s2 == 1 || o.s0 != 1;
        bool vec = ((uintptr_t)o.p % 16) == 0 && (G.K1 == 1 || o.s1 % 4 == 0);
        for (int i = 0; i < 4; ++i) vec = vec && o.b[i] % 4 == 0;
        vec = vec && (kc ? o.s2 == 1 && o.s0 % 4 == 0 && G.K2 % 4 == 0 : o.s0 == 1 && o.s2 % 4 == 0 && rows % 4 == 0);
        return (kc ? 1 : 0) | (vec ? 2 : 0);
    };
    const int am = mode(G.A, G.M), bm = mode(G.B, G.N);
#define MBX_TF32_CASE(X, Y) \
    if (am == X && bm == Y) {                                                                          \
        constexpr size_t smem = mma_smem_bytes(MBX_BWD_ASYNC_ALL ? true : (X >= 2 && Y >= 2));                                      \
        if (smem > 48 * 1024 &&                                                                        \
            cudaFuncSetAttribute(gemm_batched_tf32<X, Y>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                                 (int)smem) != cudaSuccess)                                            \
            return false;                                                                              \
        gemm_batched_tf32<X, Y><<<grid, kMThreads, smem, st>>>(G);                                     \
        return true;                                                                                   \
    }
    MBX_TF32_CASE(0, 0) MBX_TF32_CASE(0, 1) MBX_TF32_CASE(0, 2) MBX_TF32_CASE(0, 3)
    MBX_TF32_CASE(1, 0) MBX_TF32_CASE(1, 1) MBX_TF32_CASE(1, 2) MBX_TF32_CASE(1, 3)
    MBX_TF32_CASE(2, 0) MBX_TF32_CASE(2, 1) MBX_TF32_CASE(2, 2) MBX_TF32_CASE(2, 3)
    MBX_TF32_CASE(3, 0) MBX_TF32_CASE(3, 1) MBX_TF32_CASE(3, 2) MBX_TF32_CASE(3, 3)
#undef MBX_TF32_CASE
    return false;
}

// ---------------------------------------------------------------- row kernels
// dS = L (dL - D), D = sum_(c,k) L dL, in place over dL.  One warp per (bh a, j, l).
// L, dL: [bha][c][j][l][k]
__global__ void softmax_bwd_cols(const float* __restrict__ L, float* __restrict__ dL, int64_t rows, int gk, int s2,
                                 int s1) {
    const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (w >= rows) return;
    const int l = (int)(w % s1), j = (int)((w / s1) % s2);
    const int64_t bha = w / ((int64_t)s1 * s2);
    const int64_t cst = (int64_t)s2 * s1 * s1;
    const int64_t base = bha * gk * cst + ((int64_t)j * s1 + l) * s1;
    const int n = gk * s1;
    float D = 0.f;
    if (n <= 128) {   // the row in registers: one round of loads, no re-read
        float lv[4], dv[4];
        int64_t off[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int x = lane + 32 * u;
            off[u] = base + (int64_t)(x / s1) * cst + x % s1;
            lv[u] = x < n ? L[off[u]] : 0.f;
            dv[u] = x < n ? dL[off[u]] : 0.f;
            D += lv[u] * dv[u];
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) D += __shfl_xor_sync(0xffffffffu, D, o);
#pragma unroll
        for (int u = 0; u < 4; ++u)
            if (lane + 32 * u < n) dL[off[u]] = lv[u] * (dv[u] - D);
        return;
    }
    for (int x = lane; x < n; x += 32) {
        const int64_t o = base + (x / s1) * cst + x % s1;
        D += L[o] * dL[o];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) D += __shfl_xor_sync(0xffffffffu, D, o);
    for (int x = lane; x < n; x += 32) {
        const int64_t o = base + (x / s1) * cst + x % s1;
        dL[o] = L[o] * (dL[o] - D);
    }
}

// out[bha][c][k][j] = sign * sum_l X[bha][c][j][l][k]  (c_L / c_R reductions over the query rows)
__global__ void sum_over_l(const float* __restrict__ X, float* __restrict__ out, int64_t n, int s2, int s1,
                           float sign) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n) return;
    // k fastest across threads: each step over l reads consecutive k (coalesced)
    const int k = (int)(t % s1), j = (int)((t / s1) % s2);
    const int64_t bhac = t / ((int64_t)s2 * s1);
    const float* x = X + (bhac * s2 + j) * s1 * s1 + k;
    float s = 0.f;
    for (int l = 0; l < s1; ++l) s += x[(int64_t)l * s1];
    out[(bhac * s1 + k) * s2 + j] = sign * s;
}

// Row softmax backward of the row stage, in place over dR:
//   dz = R (dR - sum R dR) + dcL R (z - sum R z),  one warp per row (bh,a,c,k,j) of s2 entries.
__global__ void softmax_bwd_rows(const float* __restrict__ R, const float* __restrict__ z, float* __restrict__ dR,
                                 const float* __restrict__ dcl, int64_t rows, int s2) {
    const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (w >= rows) return;
    const float* r = R + w * s2;
    const float* zz = z + w * s2;
    float* d = dR + w * s2;
    const float c = dcl[w];
    float srd = 0.f, srz = 0.f;
    if (s2 <= 64) {   // the row in registers: one round of loads, no re-read
        float rv[2], dv[2], zv[2];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            const int i = lane + 32 * u;
            const bool in = i < s2;
            rv[u] = in ? r[i] : 0.f;
            dv[u] = in ? d[i] : 0.f;
            zv[u] = in ? zz[i] : 0.f;
            srd += rv[u] * dv[u];
            srz += rv[u] * zv[u];
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            srd += __shfl_xor_sync(0xffffffffu, srd, o);
            srz += __shfl_xor_sync(0xffffffffu, srz, o);
        }
#pragma unroll
        for (int u = 0; u < 2; ++u)
            if (lane + 32 * u < s2) d[lane + 32 * u] = rv[u] * (dv[u] - srd) + c * rv[u] * (zv[u] - srz);
        return;
    }
    for (int i = lane; i < s2; i += 32) {
        srd += r[i] * d[i];
        srz += r[i] * zz[i];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        srd += __shfl_xor_sync(0xffffffffu, srd, o);
        srz += __shfl_xor_sync(0xffffffffu, srz, o);
    }
    for (int i = lane; i < s2; i += 32) d[i] = r[i] * (d[i] - srd) + c * r[i] * (zz[i] - srz);
}

// A_t = alpha_R / max(c_R, eps) (rows of d features), in place.
__global__ void normalize_rows(float* __restrict__ a, const float* __restrict__ cr, int64_t n, int d, float eps) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n) return;
    a[t] /= fmaxf(cr[t / d], eps);
}

// dalpha_R = dA / m and dc_R = -(dA . A) / m (0 where c_R was clamped); in place over dA.
__global__ void normalize_bwd(float* __restrict__ dA, const float* __restrict__ A, const float* __restrict__ cr,
                              float* __restrict__ dcr, int64_t rows, int d, float eps) {
    const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (w >= rows) return;
    const float m = fmaxf(cr[w], eps);
    float s = 0.f;
    for (int e = lane; e < d; e += 32) {
        s += dA[w * d + e] * A[w * d + e];
        dA[w * d + e] /= m;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) dcr[w] = cr[w] > eps ? -s / m : 0.f;
}

// dL[bha][c][j][l][k] += dcr[bha][c][k][j]  (c_R = sum_l L)
__global__ void add_dcr(float* __restrict__ dL, const float* __restrict__ dcr, int64_t n, int s2, int s1) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n) return;
    const int k = (int)(t % s1), j = (int)((t / ((int64_t)s1 * s1)) % s2);
    const int64_t bhac = t / ((int64_t)s1 * s1 * s2);
    dL[t] += dcr[(bhac * s1 + k) * s2 + j];
}

// ---------------------------------------------------------------- gathers / scatters
__device__ __forceinline__ int64_t slot_row(const Geometry& g, const int32_t* order, int tile, int r, int j) {
    const int l1 = tile / g.c2, j1 = tile - (tile / g.c2) * g.c2;
    const int64_t p = ((int64_t)(l1 * g.s1 + r) * g.c2 + j1) * g.s2 + j;
    return order ? (int64_t)order[p] : p;
}

// token-order offset of slot row w (bh, tile, r, j) in a (B, H, N, width) tensor with strides st
__device__ __forceinline__ int64_t slot_offset(const Geometry& g, const int32_t* order, int tiles, uint32_t w,
                                               int64_t s0, int64_t s1, int64_t s2) {
    const int j = (int)(w % (uint32_t)g.s2); w /= (uint32_t)g.s2;
    const int r = (int)(w % (uint32_t)g.s1); w /= (uint32_t)g.s1;
    const int tile = (int)(w % (uint32_t)tiles);
    const int bh = (int)(w / (uint32_t)tiles);
    const int b = bh / g.heads, h = bh - (bh / g.heads) * g.heads;
    return b * s0 + h * s1 + slot_row(g, order, tile, r, j) * s2;
}

// dst[bh][tile][r][j][e] = scale * src[b, h, row(tile, r, j), e] (gather) and back (scatter):
// one warp per kRowsPerWarp slot rows, lanes over e.  With width 128 and 16-byte aligned rows
// all of a warp's rows are loaded before any is stored (4 x 16 B in flight per lane: with one
// row per warp the copy ran at ~2 TB/s, latency-bound); otherwise a scalar loop per row.
constexpr int kRowsPerWarp = 4;
template <typename T, bool GATHER>
__global__ void copy_tiles(const Geometry g, const void* __restrict__ src_, const int64_t* st, const int32_t* order,
                           int tiles, int width, float scale, void* __restrict__ dst_) {
    using S = typename std::conditional<GATHER, T, float>::type;   // source element
    using D = typename std::conditional<GATHER, float, T>::type;   // destination element
    const S* src = static_cast<const S*>(src_);
    D* dst = static_cast<D*>(dst_);
    const int64_t rows = (int64_t)g.bh * tiles * g.s1 * g.s2;
    const int lane = threadIdx.x & 31;
    const int64_t s0 = st[0], s1 = st[1], s2 = st[2];
    const bool vec = width == 128 && (s0 % 4) == 0 && (s1 % 4) == 0 && (s2 % 4) == 0 &&
                     ((uintptr_t)(GATHER ? (const void*)src : (const void*)dst) % (4 * sizeof(T))) == 0;
    for (int64_t w0 = (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5) * kRowsPerWarp; w0 < rows;
         w0 += (((int64_t)gridDim.x * blockDim.x) >> 5) * kRowsPerWarp) {
        int64_t tok[kRowsPerWarp];
#pragma unroll
        for (int u = 0; u < kRowsPerWarp; ++u)
            tok[u] = w0 + u < rows ? slot_offset(g, order, tiles, (uint32_t)(w0 + u), s0, s1, s2) : 0;
        if (vec) {
            float4 x[kRowsPerWarp];
#pragma unroll
            for (int u = 0; u < kRowsPerWarp; ++u)
                if (w0 + u < rows) x[u] = ld4(src + (GATHER ? tok[u] : (w0 + u) * width) + 4 * lane);
#pragma unroll
            for (int u = 0; u < kRowsPerWarp; ++u)
                if (w0 + u < rows)
                    store4(dst + (GATHER ? (w0 + u) * width : tok[u]) + 4 * lane,
                           make_float4(scale * x[u].x, scale * x[u].y, scale * x[u].z, scale * x[u].w));
        } else {
            for (int u = 0; u < kRowsPerWarp && w0 + u < rows; ++u) {
                const S* sp = src + (GATHER ? tok[u] : (w0 + u) * width);
                D* dp = dst + (GATHER ? (w0 + u) * width : tok[u]);
                for (int e = lane; e < width; e += 32) store(dp + e, scale * ld(sp + e));
            }
        }
    }
}

// ------------------------------------------------------------------ cuBLAS (bf16 I/O)
// For bf16 I/O (the 2e-2 tolerance) the contractions run as TF32 tensor-core batched
// GEMMs through cuBLAS (plain library GEMMs: per-batch pointers from a fill kernel, the
// two-level reduction index split into K1 accumulating calls when it is not contiguous).
// libcublas is opened at first use (dlopen of the soname PyTorch already loaded, else the
// CUDA toolkit's), so the forward library has no link-time dependency on it.  fp32 I/O
// (the 1e-4 parity mode) keeps the fp32 SIMT GEMM above.
typedef cublasStatus_t (*CreateFn)(cublasHandle_t*);
typedef cublasStatus_t (*SetStreamFn)(cublasHandle_t, cudaStream_t);
typedef cublasStatus_t (*GemmBatchedExFn)(cublasHandle_t, cublasOperation_t, cublasOperation_t, int, int, int,
                                          const void*, const void* const[], cudaDataType, int, const void* const[],
                                          cudaDataType, int, const void*, void* const[], cudaDataType, int, int,
                                          cublasComputeType_t, cublasGemmAlgo_t);
struct Cublas {
    CreateFn create = nullptr;
    SetStreamFn set_stream = nullptr;
    GemmBatchedExFn gemm = nullptr;
    bool ok = false;
};
const Cublas& cublas() {
    static Cublas c;
    static std::once_flag once;
    std::call_once(once, [] {
        const char* names[] = {"libcublas.so.12", "/usr/local/cuda/lib64/libcublas.so.12", "libcublas.so"};
        void* h = nullptr;
        for (const char* n : names)
            if ((h = dlopen(n, RTLD_NOW | RTLD_GLOBAL)) != nullptr) break;
        if (!h) return;
        c.create = reinterpret_cast<CreateFn>(dlsym(h, "cublasCreate_v2"));
        c.set_stream = reinterpret_cast<SetStreamFn>(dlsym(h, "cublasSetStream_v2"));
        c.gemm = reinterpret_cast<GemmBatchedExFn>(dlsym(h, "cublasGemmBatchedEx"));
        c.ok = c.create && c.set_stream && c.gemm;
    });
    return c;
}
// one handle per (thread, device): cuBLAS handles are not for concurrent use across threads
cublasHandle_t cublas_handle() {
    thread_local cublasHandle_t h[64] = {};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return nullptr;
    if (!h[dev] && cublas().ok && cublas().create(&h[dev]) != CUBLAS_STATUS_SUCCESS) h[dev] = nullptr;
    return h[dev];
}

// pointer arrays of one batched call: batch b = (b0, b1, b2, b3) row-major over nb
__global__ void fill_ptrs(Gemm G, int64_t a_off, int64_t b_off, const float** pa, const float** pb, float** pc,
                          int64_t n) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    int64_t x = i;
    int bi[4];
    bi[3] = (int)(x % G.nb[3]); x /= G.nb[3];
    bi[2] = (int)(x % G.nb[2]); x /= G.nb[2];
    bi[1] = (int)(x % G.nb[1]); x /= G.nb[1];
    bi[0] = (int)x;
    int64_t oa = a_off, ob = b_off, oc = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        oa += bi[k] * G.A.b[k];
        ob += bi[k] * G.B.b[k];
        oc += bi[k] * G.C.b[k];
    }
    pa[i] = G.A.p + oa;
    pb[i] = G.B.p + ob;
    pc[i] = const_cast<float*>(G.C.p) + oc;
}

// C (row-major M x N, ld C.s0) = alpha A B^T (+ C): cuBLAS column-major C^T = op(B) op(A^T)
bool gemm_tf32(const Gemm& G, void** ptrs, int64_t max_batches, cudaStream_t st) {
    const Cublas& cb = cublas();
    cublasHandle_t h = cublas_handle();
    if (!cb.ok || !h || G.C.s1 != 1) return false;
    const int64_t batches = (int64_t)G.nb[0] * G.nb[1] * G.nb[2] * G.nb[3];
    if (batches > max_batches || batches > INT32_MAX) return false;
    // K index: flattened when k1 and k2 form one stride (or one of them is trivial), else K1 calls
    auto kstride = [&](const Operand& o, int64_t& sk, bool& flat) {
        if (G.K1 == 1) { sk = o.s2; flat = true; }
        else if (G.K2 == 1) { sk = o.s1; flat = true; }
        else { sk = o.s2; flat = o.s1 == (int64_t)G.K2 * o.s2; }
    };
    int64_t ak, bk;
    bool af, bf;
    kstride(G.A, ak, af);
    kstride(G.B, bk, bf);
    const bool flat = af && bf;
    const int K = flat ? G.K1 * G.K2 : G.K2;
    const int calls = flat ? 1 : G.K1;
    cublasOperation_t ta, tb;
    int64_t lda, ldb;
    if (bk == 1) { ta = CUBLAS_OP_T; lda = G.B.s0; } else if (G.B.s0 == 1) { ta = CUBLAS_OP_N; lda = bk; } else return false;
    if (ak == 1) { tb = CUBLAS_OP_N; ldb = G.A.s0; } else if (G.A.s0 == 1) { tb = CUBLAS_OP_T; ldb = ak; } else return false;
    if (lda > INT32_MAX || ldb > INT32_MAX || G.C.s0 > INT32_MAX) return false;
    if (cb.set_stream(h, st) != CUBLAS_STATUS_SUCCESS) return false;
    const float** pa = (const float**)ptrs;
    const float** pb = pa + max_batches;
    float** pc = reinterpret_cast<float**>(ptrs + 2 * max_batches);
    for (int k1 = 0; k1 < calls; ++k1) {
        const int64_t a_off = flat ? 0 : (int64_t)k1 * G.A.s1, b_off = flat ? 0 : (int64_t)k1 * G.B.s1;
        fill_ptrs<<<(unsigned)((batches + 255) / 256), 256, 0, st>>>(G, a_off, b_off, pa, pb, pc, batches);
        const float alpha = G.alpha, beta = (G.acc || k1 > 0) ? 1.f : 0.f;
        if (cb.gemm(h, ta, tb, G.N, G.M, K, &alpha, (const void* const*)pb, CUDA_R_32F, (int)lda,
                    (const void* const*)pa, CUDA_R_32F, (int)ldb, &beta,
                    (void* const*)pc, CUDA_R_32F, (int)G.C.s0, (int)batches,
                    CUBLAS_COMPUTE_32F_FAST_TF32, CUBLAS_GEMM_DEFAULT) != CUBLAS_STATUS_SUCCESS)
            return false;
    }
    return true;
}

// ------------------------------------------------------------------ host
struct Buf {
    int64_t* strides;   // q, k, v, out element strides (read by the gather / scatter kernels)
    float *Qt, *Kt, *Vt, *dOt, *dQt, *dKt, *dVt;
    float *aL, *Y, *daL, *dY, *Ah, *dAh;
    float *cR, *dcL, *dcR;
    float *dL, *dLp, *z, *dR;
    void** ptrs;        // 3 x max_batches pointers (cuBLAS batched calls)
    int64_t max_batches;
};

size_t align_up(size_t x) { return (x + 255) & ~size_t(255); }

size_t layout(const Geometry& g, char* base, Buf* b) {
    const size_t bh = g.bh, gq = g.gq, gk = g.gk, s1 = g.s1, s2 = g.s2, d = g.d, dv = g.dv;
    const size_t tq = gq * s1 * s2, tk = gk * s1 * s2, pairs = gq * gk * s1 * s2;
    size_t off = 0;
    auto carve = [&](size_t floats) {
        float* p = base ? reinterpret_cast<float*>(base + off) : nullptr;
        off += align_up(floats * bh * sizeof(float));
        return p;
    };
    Buf x{};
    x.strides = base ? reinterpret_cast<int64_t*>(base) : nullptr;
    off += 256;
    x.Qt = carve(tq * d);
    x.Kt = carve(tk * d);
    x.Vt = carve(tk * dv);
    x.dOt = carve(tq * dv);
    x.dQt = carve(tq * d);
    x.dKt = carve(tk * d);
    x.dVt = carve(tk * dv);
    x.aL = carve(pairs * d);
    x.Y = carve(pairs * dv);
    x.daL = carve(pairs * d);
    x.dY = carve(pairs * dv);
    if (g.T > 1) {
        x.Ah = carve(pairs * d);
        x.dAh = carve(pairs * d);
        x.cR = carve(pairs);
        x.dcR = carve(pairs);
        x.dLp = carve(pairs * s1);
    }
    x.dcL = carve(pairs);
    x.dL = carve(pairs * s1);
    x.z = carve(pairs * s2);
    x.dR = carve(pairs * s2);
    // the largest batch count of any call is bh gq gk max(s1, s2)
    x.max_batches = (int64_t)bh * gq * gk * (s1 > s2 ? s1 : s2);
    x.ptrs = base ? reinterpret_cast<void**>(base + off) : nullptr;
    off += align_up((size_t)x.max_batches * 3 * sizeof(void*));
    if (b) *b = x;
    return off;
}

struct Ctx {
    const Geometry& g;
    cudaStream_t st;
    cudaError_t err = cudaSuccess;
    bool tf32 = false;          // bf16 I/O: TF32 tensor-core GEMMs through cuBLAS
    void** ptrs = nullptr;
    int64_t max_batches = 0;
};

Operand op(const float* p, int64_t s0, int64_t s1, int64_t s2, int64_t b0, int64_t b1, int64_t b2, int64_t b3) {
    Operand o;
    o.p = p;
    o.s0 = s0;
    o.s1 = s1;
    o.s2 = s2;
    o.b[0] = b0;
    o.b[1] = b1;
    o.b[2] = b2;
    o.b[3] = b3;
    return o;
}

void gemm(Ctx& c, const char* name, int M, int N, int K1, int K2, const int nb[4], Operand A, Operand B, Operand C,
          float alpha, int acc) {
    if (c.err != cudaSuccess) return;
    Gemm G;
    G.M = M; G.N = N; G.K1 = K1; G.K2 = K2;
    for (int i = 0; i < 4; ++i) G.nb[i] = nb[i];
    G.A = A; G.B = B; G.C = C;
    G.alpha = alpha;
    G.acc = acc;
    const int64_t batches = (int64_t)nb[0] * nb[1] * nb[2] * nb[3];
    ProfScope p(name, c.st);
    // bf16 I/O: the in-library TF32 kernel, except for the contractions where cuBLAS's
    // batched GEMM measured faster at C2 (scripts/bwd_profile.py, profiles/r2v_*): the two
    // with row-contiguous operands on both sides (the kernel's scalar fragment reads).
    // MBX_BWD_CUBLAS overrides the list ("all", "none", or comma-separated names; A/B only).
    static const char* cublas_names = [] {
        const char* e = getenv("MBX_BWD_CUBLAS");
        return e ? e : "bwd_dalpha_l,bwd_dy";
    }();
    if (c.tf32) {
        bool prefer_cublas = strcmp(cublas_names, "all") == 0;
        for (const char* p = cublas_names; !prefer_cublas && (p = strstr(p, name)) != nullptr; ++p)
            prefer_cublas = (p == cublas_names || p[-1] == ',') && (p[strlen(name)] == ',' || !p[strlen(name)]);
        if ((prefer_cublas && gemm_tf32(G, c.ptrs, c.max_batches, c.st)) || gemm_mma(G, c.st) ||
            gemm_tf32(G, c.ptrs, c.max_batches, c.st)) {
            c.err = cudaGetLastError();
            return;
        }
    }
    dim3 grid((unsigned)(batches * ((N + kTN - 1) / kTN)), (unsigned)((M + kTM - 1) / kTM));
    gemm_batched<<<grid, kGemmThreads, 0, c.st>>>(G);
    c.err = cudaGetLastError();
}

unsigned blocks_for(int64_t threads, int per_block = 256) { return (unsigned)((threads + per_block - 1) / per_block); }

template <typename T>
cudaError_t backward_t(const Geometry& g, const T* q, const T* k, const T* v, const T* dout, const float* lf,
                       const float* rf, T* dq_out, T* dk_out, T* dv_out, char* ws, cudaStream_t stream) {
    Buf b;
    layout(g, ws, &b);
    Ctx c{g, stream};
    c.tf32 = sizeof(T) == 2;
    c.ptrs = b.ptrs;
    c.max_batches = b.max_batches;
    const int64_t bh = g.bh, gq = g.gq, gk = g.gk, s1 = g.s1, s2 = g.s2, d = g.d, dv = g.dv;
    const int64_t bha = bh * gq;
    const int64_t tq = gq * s1 * s2, tk = gk * s1 * s2;
    const int64_t pairs = gq * gk * s1 * s2;            // per bh
    const int64_t rsz = pairs * s2, lsz = pairs * s1;   // R' / L' elements per bh
    // strides of the host q/k/v/out tensors, on the device (gather / scatter kernels read them there)
    int64_t* dstr = b.strides;
    {
        int64_t h[12];
        for (int i = 0; i < 3; ++i) {
            h[i] = g.qs[i];
            h[3 + i] = g.ks[i];
            h[6 + i] = g.vs[i];
            h[9 + i] = g.os[i];
        }
        cudaError_t e = cudaMemcpyAsync(dstr, h, sizeof(h), cudaMemcpyHostToDevice, stream);
        if (e != cudaSuccess) return e;
    }
    // gathers / scatters: one warp per slot row, all rows resident in one pass
    const int64_t slot_rows = bh * (gq > gk ? gq : gk) * s1 * s2;
    if (slot_rows >= (int64_t)UINT32_MAX) return cudaErrorInvalidValue;
    const unsigned gb = (unsigned)((slot_rows + 8 * kRowsPerWarp - 1) / (8 * kRowsPerWarp));
    { ProfScope ps_("bwd_gather", stream);
    copy_tiles<T, true><<<gb, 256, 0, stream>>>(g, q, dstr + 0, g.q_order, (int)gq, (int)d, g.scale, b.Qt); }
    { ProfScope ps_("bwd_gather", stream);
    copy_tiles<T, true><<<gb, 256, 0, stream>>>(g, k, dstr + 3, g.kv_order, (int)gk, (int)d, 1.f, b.Kt); }
    { ProfScope ps_("bwd_gather", stream);
    copy_tiles<T, true><<<gb, 256, 0, stream>>>(g, v, dstr + 6, g.kv_order, (int)gk, (int)dv, 1.f, b.Vt); }
    { ProfScope ps_("bwd_gather", stream);
    copy_tiles<T, true><<<gb, 256, 0, stream>>>(g, dout, dstr + 9, g.q_order, (int)gq, (int)dv, 1.f, b.dOt); }
    cudaMemsetAsync(b.dQt, 0, sizeof(float) * bh * tq * d, stream);
    cudaMemsetAsync(b.dKt, 0, sizeof(float) * bh * tk * d, stream);
    cudaMemsetAsync(b.dVt, 0, sizeof(float) * bh * tk * dv, stream);
    if ((c.err = cudaGetLastError()) != cudaSuccess) return c.err;
    // strides reused below (elements)
    const int64_t qt_a = s1 * s2 * d, kt_c = s1 * s2 * d, vt_c = s1 * s2 * dv, do_a = s1 * s2 * dv;
    const int64_t pd_a = gk * s1 * s2 * d, pd_c = s1 * s2 * d, pd_k = s2 * d;            // [a][c][k][j][d]
    const int64_t pv_a = gk * s1 * s2 * dv, pv_c = s1 * s2 * dv, pv_k = s2 * dv;
    const int64_t r_a = gk * s1 * s2 * s2, r_c = s1 * s2 * s2, r_k = s2 * s2;            // [a][c][k][j][i]
    const int64_t l_a = gk * s2 * s1 * s1, l_c = s2 * s1 * s1, l_j = s1 * s1;            // [a][c][j][l][k]
    const int64_t p_a = gk * s1 * s2, p_c = s1 * s2, p_k = s2;                            // [a][c][k][j]
    const int nb_ack[4] = {(int)bh, (int)gq, (int)gk, (int)s1};
    const int nb_acj[4] = {(int)bh, (int)gq, (int)gk, (int)s2};
    const int nb_aj[4] = {(int)bh, (int)gq, 1, (int)s2};
    const int nb_ak[4] = {(int)bh, (int)gq, 1, (int)s1};
    const int nb_ck[4] = {(int)bh, 1, (int)gk, (int)s1};

    for (int t = g.T - 1; t >= 0; --t) {
        const float* R = rf + (size_t)t * bh * rsz;
        const float* L = lf + (size_t)t * bh * lsz;
        const bool last = t == g.T - 1;
        // A_t rows: Q (t = 0) or alpha_R / max(c_R, eps) from L_{t-1} (recomputed)
        const float* At;
        Operand At_rows;   // as [bh][a][c][k][j][e]
        if (t == 0) {
            At = b.Qt;
            At_rows = op(b.Qt, d, 0, 1, gq * qt_a, qt_a, 0, s2 * d);
        } else {
            const float* Lp = lf + (size_t)(t - 1) * bh * lsz;
            // alpha_R[a][c][k][j][:] = sum_l L_{t-1}[a][c][j][l][k] Q[a][l][j][:]   (M = k, N = e, K = l)
            gemm(c, "bwd_alpha_r", (int)s1, (int)d, 1, (int)s1, nb_acj,
                 op(Lp, 1, 0, s1, gq * l_a, l_a, l_c, l_j), op(b.Qt, 1, 0, s2 * d, gq * qt_a, qt_a, 0, d),
                 op(b.Ah, pd_k, 1, 0, gq * pd_a, pd_a, pd_c, d), 1.f, 0);
            { ProfScope ps_("bwd_sum_l", stream);
            sum_over_l<<<blocks_for(bh * pairs), 256, 0, stream>>>(Lp, b.cR, bh * pairs, (int)s2, (int)s1, 1.f); }
            normalize_rows<<<blocks_for(bh * pairs * d), 256, 0, stream>>>(b.Ah, b.cR, bh * pairs * d, (int)d,
                                                                          g.eps_div);
            At = b.Ah;
            At_rows = op(b.Ah, d, 0, 1, gq * pd_a, pd_a, pd_c, pd_k);
        }
        // forward recompute: aL = R K (and Y = R V on the last refinement)   (M = j, N = e, K = i)
        gemm(c, "bwd_alpha_l", (int)s2, (int)d, 1, (int)s2, nb_ack, op(R, s2, 0, 1, gq * r_a, r_a, r_c, r_k),
             op(b.Kt, 1, 0, d, gk * kt_c, 0, kt_c, s2 * d), op(b.aL, d, 1, 0, gq * pd_a, pd_a, pd_c, pd_k), 1.f, 0);
        if (last) {
            gemm(c, "bwd_y", (int)s2, (int)dv, 1, (int)s2, nb_ack, op(R, s2, 0, 1, gq * r_a, r_a, r_c, r_k),
                 op(b.Vt, 1, 0, dv, gk * vt_c, 0, vt_c, s2 * dv), op(b.Y, dv, 1, 0, gq * pv_a, pv_a, pv_c, pv_k), 1.f,
                 0);
            // dL[a][c][j][l][k] = dO[a][l][j][:] . Y[a][c][k][j][:]   (M = l, N = k, K = e)
            gemm(c, "bwd_dl", (int)s1, (int)s1, 1, (int)dv, nb_acj, op(b.dOt, s2 * dv, 0, 1, gq * do_a, do_a, 0, dv),
                 op(b.Y, pv_k, 0, 1, gq * pv_a, pv_a, pv_c, dv), op(b.dL, s1, 1, 0, gq * l_a, l_a, l_c, l_j), 1.f, 0);
        }
        // dS = L (dL - sum L dL)
        { ProfScope ps_("bwd_softmax_cols", stream);
        softmax_bwd_cols<<<blocks_for(bha * s2 * s1 * 32), 256, 0, stream>>>(L, b.dL, bha * s2 * s1, (int)gk, (int)s2,
                                                                          (int)s1); }
        // dQ[a][l][j][:] += sum_(c,k) dS[a][c][j][l][k] aL[a][c][k][j][:]   (M = l, N = e, K = (c, k))
        gemm(c, "bwd_dq_col", (int)s1, (int)d, (int)gk, (int)s1, nb_aj, op(b.dL, s1, l_c, 1, gq * l_a, l_a, 0, l_j),
             op(b.aL, 1, pd_c, pd_k, gq * pd_a, pd_a, 0, d), op(b.dQt, s2 * d, 1, 0, gq * qt_a, qt_a, 0, d), 1.f, 1);
        // daL[a][c][k][j][:] = sum_l dS[a][c][j][l][k] Q[a][l][j][:]   (M = k, N = e, K = l)
        gemm(c, "bwd_dalpha_l", (int)s1, (int)d, 1, (int)s1, nb_acj, op(b.dL, 1, 0, s1, gq * l_a, l_a, l_c, l_j),
             op(b.Qt, 1, 0, s2 * d, gq * qt_a, qt_a, 0, d), op(b.daL, pd_k, 1, 0, gq * pd_a, pd_a, pd_c, d), 1.f, 0);
        // dc_L[a][c][k][j] = -sum_l dS
        { ProfScope ps_("bwd_sum_l", stream);
        sum_over_l<<<blocks_for(bh * pairs), 256, 0, stream>>>(b.dL, b.dcL, bh * pairs, (int)s2, (int)s1, -1.f); }
        if (last) {
            // dY[a][c][k][j][:] = sum_l L[a][c][j][l][k] dO[a][l][j][:]
            gemm(c, "bwd_dy", (int)s1, (int)dv, 1, (int)s1, nb_acj, op(L, 1, 0, s1, gq * l_a, l_a, l_c, l_j),
                 op(b.dOt, 1, 0, s2 * dv, gq * do_a, do_a, 0, dv), op(b.dY, pv_k, 1, 0, gq * pv_a, pv_a, pv_c, dv), 1.f,
                 0);
        }
        // z = A_t K^T  (M = j, N = i, K = e)
        gemm(c, "bwd_z", (int)s2, (int)s2, 1, (int)d, nb_ack, At_rows, op(b.Kt, d, 0, 1, gk * kt_c, 0, kt_c, s2 * d),
             op(b.z, s2, 1, 0, gq * r_a, r_a, r_c, r_k), 1.f, 0);
        // dR = dY V^T (last) + daL K^T
        if (last)
            gemm(c, "bwd_dr_v", (int)s2, (int)s2, 1, (int)dv, nb_ack, op(b.dY, dv, 0, 1, gq * pv_a, pv_a, pv_c, pv_k),
                 op(b.Vt, dv, 0, 1, gk * vt_c, 0, vt_c, s2 * dv), op(b.dR, s2, 1, 0, gq * r_a, r_a, r_c, r_k), 1.f, 0);
        gemm(c, "bwd_dr_k", (int)s2, (int)s2, 1, (int)d, nb_ack, op(b.daL, d, 0, 1, gq * pd_a, pd_a, pd_c, pd_k),
             op(b.Kt, d, 0, 1, gk * kt_c, 0, kt_c, s2 * d), op(b.dR, s2, 1, 0, gq * r_a, r_a, r_c, r_k), 1.f, last);
        // dz (in place over dR)
        { ProfScope ps_("bwd_softmax_rows", stream);
        softmax_bwd_rows<<<blocks_for(bh * pairs * 32), 256, 0, stream>>>(R, b.z, b.dR, b.dcL, bh * pairs, (int)s2); }
        // dK[c][k][i][:] += sum_(a,j) dz[a][c][k][j][i] A_t[a][c][k][j][:] + R daL   (M = i, N = e, K = (a, j))
        {
            Operand Ab = At_rows;   // as B[k1 = a][k2 = j][n = e]
            Operand B_at = op(At, 1, Ab.b[1], Ab.s0, Ab.b[0], 0, Ab.b[2], Ab.b[3]);
            gemm(c, "bwd_dk_z", (int)s2, (int)d, (int)gq, (int)s2, nb_ck, op(b.dR, 1, r_a, s2, gq * r_a, 0, r_c, r_k),
                 B_at, op(b.dKt, d, 1, 0, gk * kt_c, 0, kt_c, s2 * d), 1.f, 1);
        }
        gemm(c, "bwd_dk_r", (int)s2, (int)d, (int)gq, (int)s2, nb_ck, op(R, 1, r_a, s2, gq * r_a, 0, r_c, r_k),
             op(b.daL, 1, pd_a, d, gq * pd_a, 0, pd_c, pd_k), op(b.dKt, d, 1, 0, gk * kt_c, 0, kt_c, s2 * d), 1.f, 1);
        if (last)
            gemm(c, "bwd_dv", (int)s2, (int)dv, (int)gq, (int)s2, nb_ck, op(R, 1, r_a, s2, gq * r_a, 0, r_c, r_k),
                 op(b.dY, 1, pv_a, dv, gq * pv_a, 0, pv_c, pv_k), op(b.dVt, dv, 1, 0, gk * vt_c, 0, vt_c, s2 * dv), 1.f,
                 1);
        if (t == 0) {
            // dQ[a][k][j][:] += sum_(c,i) dz[a][c][k][j][i] K[c][k][i][:]   (M = j, N = e, K = (c, i))
            gemm(c, "bwd_dq_row", (int)s2, (int)d, (int)gk, (int)s2, nb_ak, op(b.dR, s2, r_c, 1, gq * r_a, r_a, 0, r_k),
                 op(b.Kt, 1, kt_c, d, gk * kt_c, 0, 0, s2 * d), op(b.dQt, d, 1, 0, gq * qt_a, qt_a, 0, s2 * d), 1.f,
                 1);
        } else {
            // dA_t = dz K  -> dalpha_R, dc_R -> dL_{t-1}, dQ
            gemm(c, "bwd_da", (int)s2, (int)d, 1, (int)s2, nb_ack, op(b.dR, s2, 0, 1, gq * r_a, r_a, r_c, r_k),
                 op(b.Kt, 1, 0, d, gk * kt_c, 0, kt_c, s2 * d), op(b.dAh, d, 1, 0, gq * pd_a, pd_a, pd_c, pd_k), 1.f, 0);
            normalize_bwd<<<blocks_for(bh * pairs * 32), 256, 0, stream>>>(b.dAh, b.Ah, b.cR, b.dcR, bh * pairs,
                                                                          (int)d, g.eps_div);
            const float* Lp = lf + (size_t)(t - 1) * bh * lsz;
            // dL_{t-1}[a][c][j][l][k] = Q[a][l][j][:] . dalpha_R[a][c][k][j][:] + dc_R   (M = l, N = k, K = e)
            gemm(c, "bwd_dl_prev", (int)s1, (int)s1, 1, (int)d, nb_acj, op(b.Qt, s2 * d, 0, 1, gq * qt_a, qt_a, 0, d),
                 op(b.dAh, pd_k, 0, 1, gq * pd_a, pd_a, pd_c, d), op(b.dLp, s1, 1, 0, gq * l_a, l_a, l_c, l_j), 1.f, 0);
            add_dcr<<<blocks_for(bh * lsz), 256, 0, stream>>>(b.dLp, b.dcR, bh * lsz, (int)s2, (int)s1);
            // dQ[a][l][j][:] += sum_(c,k) L_{t-1}[a][c][j][l][k] dalpha_R[a][c][k][j][:]
            gemm(c, "bwd_dq_alpha", (int)s1, (int)d, (int)gk, (int)s1, nb_aj, op(Lp, s1, l_c, 1, gq * l_a, l_a, 0, l_j),
                 op(b.dAh, 1, pd_c, pd_k, gq * pd_a, pd_a, 0, d), op(b.dQt, s2 * d, 1, 0, gq * qt_a, qt_a, 0, d), 1.f,
                 1);
            float* tmp = b.dL;   // dL_{t-1} becomes the next step's dL
            b.dL = b.dLp;
            b.dLp = tmp;
        }
        if (c.err != cudaSuccess) return c.err;
        if ((c.err = cudaGetLastError()) != cudaSuccess) return c.err;
    }
    // scatter back to token order: dq = scale * dQt (Q entered the solver as scale * q)
    { ProfScope ps_("bwd_scatter", stream);
    copy_tiles<T, false><<<gb, 256, 0, stream>>>(g, b.dQt, dstr + 0, g.q_order, (int)gq, (int)d, g.scale, dq_out); }
    { ProfScope ps_("bwd_scatter", stream);
    copy_tiles<T, false><<<gb, 256, 0, stream>>>(g, b.dKt, dstr + 3, g.kv_order, (int)gk, (int)d, 1.f, dk_out); }
    { ProfScope ps_("bwd_scatter", stream);
    copy_tiles<T, false><<<gb, 256, 0, stream>>>(g, b.dVt, dstr + 6, g.kv_order, (int)gk, (int)dv, 1.f, dv_out); }
    (void)nb_ak;
    return cudaGetLastError();
}

}  // namespace

size_t backward_workspace_bytes(const Geometry& g) { return layout(g, nullptr, nullptr); }

cudaError_t backward(const Geometry& g, int dtype, const void* q, const void* k, const void* v, const void* dout,
                     const float* l_factors, const float* r_factors, void* dq, void* dk, void* dv, void* ws,
                     cudaStream_t stream) {
    if (dtype == MBX_F32)
        return backward_t<float>(g, (const float*)q, (const float*)k, (const float*)v, (const float*)dout, l_factors,
                                 r_factors, (float*)dq, (float*)dk, (float*)dv, (char*)ws, stream);
    return backward_t<__nv_bfloat16>(g, (const __nv_bfloat16*)q, (const __nv_bfloat16*)k, (const __nv_bfloat16*)v,
                                     (const __nv_bfloat16*)dout, l_factors, r_factors, (__nv_bfloat16*)dq,
                                     (__nv_bfloat16*)dk, (__nv_bfloat16*)dv, (char*)ws, stream);
}

}  // namespace mbx
