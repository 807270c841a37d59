// tcgen05 / TMEM / TMA kernels of the tiled MonarchAttention forward (bf16,
// d = d_v = 128, T = 1, tile rows of <= 64 tokens, <= 4 query tiles).
//
// Two stages joined by a bf16 workspace W:
//
//   row stage  (tc_row_stage, persistent): one unit = key row (b,h,c,k).
//     TMA: K row, V row (64 x 128 boxes) and row k of every query tile.
//     MMA1  S[(a,j), i]   = Q_k . K_k^T             M=128 (2 query tiles), N=64, K=128
//     softmax_i in registers (one query row per thread), c_L = sum R z - lse
//     MMA2  [aL | Y]      = P . [K_k | V_k]          M=128, N=256 (K and V adjacent), K=64
//     epilogue: scale by 1/l, bf16, store W[b,h,a,j,(c,k),0:256], c_L -> Wc.
//     (solver.py:187-191, factors.py:123; tensorops.py:268-272)
//   column stage (tc_column_stage): one CTA per (b,h,a,j), keys (c,k) in
//     chunks of 128, transposed so keys fill the 128 TMEM lanes:
//     MMA3  S^T[key, l]   = aL . Q_col^T           M=128, N=32, K=128
//     joint softmax over keys (online across chunks) with bias -c_L
//     MMA4  O^T[v, l]    += Y^T . P^T               M=128, N=32, K=128
//     (solver.py:192-195, factors.py:124)
//
// The permutation of the plan is folded into addressing: tile rows are
// contiguous runs of s2 tokens for identity and neighborhood plans, so each
// row is one TMA box at the token coordinate row_base(tile, r).
#include "mbx_internal.h"
#include "mbx_sm100.cuh"

#include <cuda.h>
#include <math.h>
#include <string.h>

namespace mbx {
namespace {

using namespace sm100;

constexpr int kD = 128;          // head dim (q, k) and value dim
constexpr int kRowsPerTile = 64; // TMA box rows per tile row (s2 <= 64)
constexpr int kMaxGq = 4;        // query tiles handled per key row
constexpr int kThreads = 128;

// ---------------------------------------------------------------- row stage
struct RowSmem {
    // per stage: [K chunk0 | K chunk1 | V chunk0 | V chunk1] (8 KB each), then
    // Q: M-tile mt, d-chunk c at mt*32K + c*16K, query tile (a%2) at +8K.
    static constexpr int kKV = 32768;
    static constexpr int kQ = 65536;
    static constexpr int kStage = kKV + kQ;
    static constexpr int kP = 2 * kStage;            // P: 128 rows x 64 keys bf16 (16 KB)
    static constexpr int kBars = kP + 16384;         // full[2], mma
    static constexpr int kTmemSlot = kBars + 64;
    static constexpr int kTotal = kTmemSlot + 16;
};

__device__ __forceinline__ float fast_exp2(float x) { return exp2f(x); }

__global__ void __launch_bounds__(kThreads, 1)
tc_row_stage(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
             const __grid_constant__ CUtensorMap tm_v, Geometry g, __nv_bfloat16* __restrict__ W,
             float* __restrict__ Wc) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + RowSmem::kBars);
    uint64_t* mma_bar = full + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + RowSmem::kTmemSlot);
    const int tid = threadIdx.x, warp = tid >> 5;

    const int units = g.bh * g.gk * g.s1;
    const int n_mt = (g.gq + 1) / 2;
    const uint32_t stage_bytes = RowSmem::kKV + (uint32_t)g.gq * 16384u;

    if (tid == 0) {
        tma_prefetch(&tm_q);
        tma_prefetch(&tm_k);
        tma_prefetch(&tm_v);
        mbar_init(&full[0], 1);
        mbar_init(&full[1], 1);
        mbar_init(mma_bar, 1);
        fence_barrier_init();
    }
    if (warp == 0) tmem_alloc<512>(tmem_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const uint32_t tmem_S = tmem;        // 64 columns
    const uint32_t tmem_O = tmem + 64;   // 256 columns

    auto issue = [&](int u, int s) {
        const int kr = u % g.s1, c = (u / g.s1) % g.gk, bh = u / (g.s1 * g.gk);
        const int b = bh / g.heads, h = bh % g.heads;
        uint8_t* st = smem + s * RowSmem::kStage;
        mbar_expect_tx(&full[s], stage_bytes);
        const int kt = (int)row_base(g, false, c, kr);
        tma_load_4d(st + 0, &tm_k, &full[s], 0, kt, h, b);
        tma_load_4d(st + 8192, &tm_k, &full[s], 64, kt, h, b);
        tma_load_4d(st + 16384, &tm_v, &full[s], 0, kt, h, b);
        tma_load_4d(st + 24576, &tm_v, &full[s], 64, kt, h, b);
        for (int a = 0; a < g.gq; ++a) {
            const int qt = (int)row_base(g, true, a, kr);
            uint8_t* qd = st + RowSmem::kKV + (a >> 1) * 32768 + (a & 1) * 8192;
            tma_load_4d(qd, &tm_q, &full[s], 0, qt, h, b);
            tma_load_4d(qd + 16384, &tm_q, &full[s], 64, qt, h, b);
        }
    };

    int it = 0;
    if (tid == 0) {
        if ((int)blockIdx.x < units) issue(blockIdx.x, 0);
        if ((int)(blockIdx.x + gridDim.x) < units) issue(blockIdx.x + gridDim.x, 1);
    }
    uint32_t mma_phase = 0;
    const uint32_t idesc_s = idesc_bf16(128, 64, false, false);
    const uint32_t idesc_o = idesc_bf16(128, 256, false, true);
    const uint32_t lane_off = (uint32_t)(warp * 32) << 16;
    const float log2e = 1.4426950408889634f;
    uint8_t* Pbuf = smem + RowSmem::kP;
    const uint32_t p_row = smem_u32(Pbuf) + tid * 128;

    for (int u = blockIdx.x; u < units; u += gridDim.x, ++it) {
        const int s = it & 1;
        const uint32_t ph = (it >> 1) & 1;
        const int kr = u % g.s1, c = (u / g.s1) % g.gk, bh = u / (g.s1 * g.gk);
        uint8_t* st = smem + s * RowSmem::kStage;
        const uint32_t kv_base = smem_u32(st);
        mbar_wait(&full[s], ph);

        for (int mt = 0; mt < n_mt; ++mt) {
            const uint32_t q_base = kv_base + RowSmem::kKV + mt * 32768;
            // ---- MMA1: S = Q K^T ------------------------------------------------
            if (tid == 0) {
                tc_fence_after();
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) {
                    const uint32_t off = (kk >> 2) * 16384 + (kk & 3) * 32;
                    const uint64_t a = smem_desc(q_base + off, 16, 1024, 2);
                    const uint64_t bd = smem_desc(kv_base + (kk >> 2) * 8192 + (kk & 3) * 32, 16, 1024, 2);
                    mma_bf16(tmem_S, a, bd, idesc_s, kk > 0);
                }
                mma_commit(mma_bar);
            }
            mbar_wait(mma_bar, mma_phase);
            mma_phase ^= 1;
            tc_fence_after();

            // ---- softmax over the s2 keys of this row (one query row per thread) --
            const int a = mt * 2 + (tid >> 6), j = tid & 63;
            const bool row_ok = a < g.gq && j < g.s2;
            float z[64];
            tmem_ld32(tmem_S + lane_off, z);
            tmem_ld32(tmem_S + lane_off + 32, z + 32);
#pragma unroll
            for (int i = 0; i < 64; ++i) z[i] *= g.scale;   // logits of scale*Q (solver.py:104)
            float m = -INFINITY;
#pragma unroll
            for (int i = 0; i < 64; ++i)
                if (i < g.s2) m = fmaxf(m, z[i]);
            float l = 0.f, A = 0.f;
            uint32_t packed[32];
#pragma unroll
            for (int i = 0; i < 64; i += 2) {
                float p0 = (i < g.s2) ? fast_exp2((z[i] - m) * log2e) : 0.f;
                float p1 = (i + 1 < g.s2) ? fast_exp2((z[i + 1] - m) * log2e) : 0.f;
                l += p0 + p1;
                A += (i < g.s2 ? p0 * z[i] : 0.f) + (i + 1 < g.s2 ? p1 * z[i + 1] : 0.f);
                if (!row_ok) p0 = p1 = 0.f;
                packed[i >> 1] = pack_bf16(p0, p1);
            }
#pragma unroll
            for (int cc = 0; cc < 8; ++cc) {
                const uint32_t addr = p_row + ((cc ^ (tid & 7)) << 4);
                st_shared_v4(addr, packed[4 * cc], packed[4 * cc + 1], packed[4 * cc + 2], packed[4 * cc + 3]);
            }
            const float inv_l = 1.f / l;
            const float c_l = A * inv_l - (m + __logf(l));
            fence_proxy_async_smem();
            tc_fence_before();
            __syncthreads();

            // ---- MMA2: [aL | Y] = P [K | V] ----------------------------------------
            if (tid == 0) {
                tc_fence_after();
                const uint32_t p_base = smem_u32(Pbuf);
#pragma unroll
                for (int kk = 0; kk < 4; ++kk) {
                    const uint64_t ad = smem_desc(p_base + kk * 32, 16, 1024, 2);
                    const uint64_t bd = smem_desc(kv_base + kk * 2048, 8192, 1024, 2);
                    mma_bf16(tmem_O, ad, bd, idesc_o, kk > 0);
                }
                mma_commit(mma_bar);
            }
            mbar_wait(mma_bar, mma_phase);
            mma_phase ^= 1;
            tc_fence_after();

            // ---- epilogue: W[b,h,a,j,key,:] = bf16(acc / l) ------------------------
            const int key = c * g.s1 + kr;
            const int64_t wrow = ((((int64_t)bh * g.gq + (row_ok ? a : 0)) * g.s2 + (row_ok ? j : 0)) * g.nkeys) + key;
            uint4* dst = reinterpret_cast<uint4*>(W + wrow * 256);
#pragma unroll
            for (int q32 = 0; q32 < 8; ++q32) {
                float o[32];
                tmem_ld32(tmem_O + lane_off + q32 * 32, o);
                if (row_ok) {
#pragma unroll
                    for (int v4 = 0; v4 < 4; ++v4) {
                        uint4 pk;
                        pk.x = pack_bf16(o[8 * v4 + 0] * inv_l, o[8 * v4 + 1] * inv_l);
                        pk.y = pack_bf16(o[8 * v4 + 2] * inv_l, o[8 * v4 + 3] * inv_l);
                        pk.z = pack_bf16(o[8 * v4 + 4] * inv_l, o[8 * v4 + 5] * inv_l);
                        pk.w = pack_bf16(o[8 * v4 + 6] * inv_l, o[8 * v4 + 7] * inv_l);
                        dst[q32 * 4 + v4] = pk;
                    }
                }
            }
            if (row_ok) Wc[wrow] = c_l;
            tc_fence_before();
            __syncthreads();
        }
        // stage s fully consumed (last MMA completed): refill it
        if (tid == 0 && u + 2 * (int)gridDim.x < units) issue(u + 2 * gridDim.x, s);
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc<512>(tmem);
}

// ------------------------------------------------------------- column stage
struct ColSmem {
    static constexpr int kA = 0;          // aL chunk: 2 x [128 keys][64] (32 KB)
    static constexpr int kY = 32768;      // Y chunk:  2 x [128 keys][64] (32 KB)
    static constexpr int kQ = 65536;      // Q column: 2 x [32 l][64]     (8 KB)
    static constexpr int kP = 73728;      // P^T: [128 keys][32 l] bf16 SW64 (8 KB)
    static constexpr int kRed = 81920;    // [128][33] floats
    static constexpr int kStats = kRed + 128 * 33 * 4;   // m_run, s_run, scale, mnew (4 x 32)
    static constexpr int kBars = kStats + 4 * 32 * 4;
    static constexpr int kTmemSlot = kBars + 16;
    static constexpr int kTotal = kTmemSlot + 16;
};

__global__ void __launch_bounds__(kThreads)
tc_column_stage(const __grid_constant__ CUtensorMap tm_w, Geometry g, const __nv_bfloat16* __restrict__ q,
                const float* __restrict__ Wc, __nv_bfloat16* __restrict__ out) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    float* red = reinterpret_cast<float*>(smem + ColSmem::kRed);
    float* m_run = reinterpret_cast<float*>(smem + ColSmem::kStats);
    float* s_run = m_run + 32;
    float* scale_l = m_run + 64;
    float* m_new = m_run + 96;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + ColSmem::kBars);
    uint64_t* load_bar = bars;
    uint64_t* mma_bar = bars + 1;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + ColSmem::kTmemSlot);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

    const int j = blockIdx.x % g.s2;
    const int a = (blockIdx.x / g.s2) % g.gq;
    const int bh = blockIdx.x / (g.s2 * g.gq);
    const int b = bh / g.heads, h = bh % g.heads;

    if (tid == 0) {
        tma_prefetch(&tm_w);
        mbar_init(load_bar, 1);
        mbar_init(mma_bar, 1);
        fence_barrier_init();
    }
    if (warp == 0) tmem_alloc<64>(tmem_slot);
    if (tid < 32) {
        m_run[tid] = -INFINITY;
        s_run[tid] = 0.f;
    }
    // Q column (rows l < s1 of tile a at column j) into SW128 K-major [32][64] x 2
    {
        const __nv_bfloat16* qb = q + b * g.qs[0] + h * g.qs[1];
        const uint32_t qbase = smem_u32(smem + ColSmem::kQ);
        for (int idx = tid; idx < 32 * 16; idx += kThreads) {
            const int l = idx >> 4, cidx = idx & 15;
            uint4 v = make_uint4(0, 0, 0, 0);
            if (l < g.s1) {
                const int64_t tok = row_base(g, true, a, l) + j;
                v = *reinterpret_cast<const uint4*>(qb + tok * g.qs[2] + cidx * 8);
            }
            const int dch = cidx >> 3, cc = cidx & 7;
            st_shared_v4(qbase + dch * 4096 + l * 128 + ((cc ^ (l & 7)) << 4), v.x, v.y, v.z, v.w);
        }
    }
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const uint32_t tmem_S = tmem, tmem_O = tmem + 32;
    const uint32_t lane_off = (uint32_t)(warp * 32) << 16;
    const uint32_t idesc_s = idesc_bf16(128, 32, false, false);
    const uint32_t idesc_o = idesc_bf16(128, 32, true, true);
    const float log2e = 1.4426950408889634f;

    const int64_t col = ((int64_t)bh * g.gq + a) * g.s2 + j;
    const int64_t row0 = col * g.nkeys;
    const int nchunks = (g.nkeys + 127) / 128;
    uint32_t load_phase = 0, mma_phase = 0;
    const uint32_t sA = smem_u32(smem + ColSmem::kA), sY = smem_u32(smem + ColSmem::kY);
    const uint32_t sQ = smem_u32(smem + ColSmem::kQ), sP = smem_u32(smem + ColSmem::kP);

    for (int ch = 0; ch < nchunks; ++ch) {
        if (tid == 0) {
            mbar_expect_tx(load_bar, 65536);
            const int r = (int)(row0 + ch * 128);
            tma_load_2d(smem + ColSmem::kA, &tm_w, load_bar, 0, r);
            tma_load_2d(smem + ColSmem::kA + 16384, &tm_w, load_bar, 64, r);
            tma_load_2d(smem + ColSmem::kY, &tm_w, load_bar, 128, r);
            tma_load_2d(smem + ColSmem::kY + 16384, &tm_w, load_bar, 192, r);
        }
        const int key = ch * 128 + tid;
        const bool kv = key < g.nkeys;
        const float cl = kv ? Wc[row0 + key] : 0.f;
        mbar_wait(load_bar, load_phase);
        load_phase ^= 1;
        if (tid == 0) {
            tc_fence_after();
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) {
                const uint64_t ad = smem_desc(sA + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024, 2);
                const uint64_t bd = smem_desc(sQ + (kk >> 2) * 4096 + (kk & 3) * 32, 16, 1024, 2);
                mma_bf16(tmem_S, ad, bd, idesc_s, kk > 0);
            }
            mma_commit(mma_bar);
        }
        mbar_wait(mma_bar, mma_phase);
        mma_phase ^= 1;
        tc_fence_after();

        float sv[32];
        tmem_ld32(tmem_S + lane_off, sv);
#pragma unroll
        for (int l = 0; l < 32; ++l) sv[l] = (kv && l < g.s1) ? sv[l] * g.scale - cl : -INFINITY;
        // column max over the 128 keys
#pragma unroll
        for (int l = 0; l < 32; ++l) red[tid * 33 + l] = sv[l];
        __syncthreads();
        {
            float pm = -INFINITY;
            for (int r = 0; r < 32; ++r) pm = fmaxf(pm, red[(warp * 32 + r) * 33 + lane]);
            __syncthreads();
            red[warp * 33 + lane] = pm;
        }
        __syncthreads();
        if (tid < 32) {
            float cm = fmaxf(fmaxf(red[tid], red[33 + tid]), fmaxf(red[66 + tid], red[99 + tid]));
            const float mo = m_run[tid];
            const float mn = fmaxf(mo, cm);
            m_new[tid] = mn;
            scale_l[tid] = (mo == -INFINITY) ? 0.f : fast_exp2((mo - mn) * log2e);
            m_run[tid] = mn;
        }
        __syncthreads();
        float pv[32];
#pragma unroll
        for (int l = 0; l < 32; ++l) {
            const float mn = m_new[l];
            pv[l] = (sv[l] == -INFINITY || mn == -INFINITY) ? 0.f : fast_exp2((sv[l] - mn) * log2e);
        }
        // P^T row (key = tid): 32 bf16 = 64 B, SW64 swizzle: chunk c -> c ^ ((row >> 1) & 3)
#pragma unroll
        for (int c4 = 0; c4 < 4; ++c4) {
            const uint32_t addr = sP + tid * 64 + ((c4 ^ ((tid >> 1) & 3)) << 4);
            st_shared_v4(addr, pack_bf16(pv[8 * c4], pv[8 * c4 + 1]), pack_bf16(pv[8 * c4 + 2], pv[8 * c4 + 3]),
                         pack_bf16(pv[8 * c4 + 4], pv[8 * c4 + 5]), pack_bf16(pv[8 * c4 + 6], pv[8 * c4 + 7]));
        }
        // column sums
#pragma unroll
        for (int l = 0; l < 32; ++l) red[tid * 33 + l] = pv[l];
        __syncthreads();
        {
            float ps = 0.f;
            for (int r = 0; r < 32; ++r) ps += red[(warp * 32 + r) * 33 + lane];
            __syncthreads();
            red[warp * 33 + lane] = ps;
        }
        __syncthreads();
        if (tid < 32) s_run[tid] = s_run[tid] * scale_l[tid] + (red[tid] + red[33 + tid] + red[66 + tid] + red[99 + tid]);
        // rescale the running O^T (thread = value dim v, columns = l)
        if (ch > 0) {
            float o[32];
            tmem_ld32(tmem_O + lane_off, o);
#pragma unroll
            for (int l = 0; l < 32; ++l) o[l] *= scale_l[l];
            tmem_st32(tmem_O + lane_off, o);
        }
        fence_proxy_async_smem();
        tc_fence_before();
        __syncthreads();
        if (tid == 0) {
            tc_fence_after();
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) {
                const uint64_t ad = smem_desc(sY + kk * 2048, 16384, 1024, 2);
                const uint64_t bd = smem_desc(sP + kk * 1024, 4096, 512, 4);
                mma_bf16(tmem_O, ad, bd, idesc_o, ch > 0 || kk > 0);
            }
            mma_commit(mma_bar);
        }
        mbar_wait(mma_bar, mma_phase);
        mma_phase ^= 1;
        tc_fence_after();
    }
    // O[l, v] = O^T[v, l] / s_l
    float o[32];
    tmem_ld32(tmem_O + lane_off, o);
    __nv_bfloat16* ob = out + b * g.os[0] + h * g.os[1];
    for (int l = 0; l < g.s1 && l < 32; ++l) {
        const int64_t tok = row_base(g, true, a, l) + j;
        ob[tok * g.os[2] + tid] = __float2bfloat16_rn(o[l] / s_run[l]);
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc<64>(tmem);
}

// ------------------------------------------------------------------- host
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
    static EncodeTiledFn fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiledFn>(p);
    }
    return fn;
}

// 4D map over a (B, H, N, 128) bf16 tensor with arbitrary element strides; box (64, 64, 1, 1), SW128.
bool make_qkv_map(CUtensorMap* m, const void* base, int B, int H, int N, const int64_t* st) {
    EncodeTiledFn enc = encode_fn();
    if (!enc) return false;
    cuuint64_t dims[4] = {(cuuint64_t)kD, (cuuint64_t)N, (cuuint64_t)H, (cuuint64_t)B};
    cuuint64_t strides[3] = {(cuuint64_t)st[2] * 2, (cuuint64_t)st[1] * 2, (cuuint64_t)st[0] * 2};
    cuuint32_t box[4] = {64, (cuuint32_t)kRowsPerTile, 1, 1};
    cuuint32_t es[4] = {1, 1, 1, 1};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(base), dims, strides, box, es,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

bool make_w_map(CUtensorMap* m, const void* base, int64_t rows) {
    EncodeTiledFn enc = encode_fn();
    if (!enc) return false;
    cuuint64_t dims[2] = {256, (cuuint64_t)rows};
    cuuint64_t strides[1] = {512};
    cuuint32_t box[2] = {64, 128};
    cuuint32_t es[2] = {1, 1};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, es,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

int num_sms() {
    static int n = 0;
    if (!n) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        if (n <= 0) n = 148;
    }
    return n;
}

bool strides_ok(const int64_t* s) {
    return (s[0] * 2) % 16 == 0 && (s[1] * 2) % 16 == 0 && (s[2] * 2) % 16 == 0;
}

}  // namespace

bool tc_supported(const Geometry& g, int dtype, int flags) {
    if (flags & MBX_FLAG_FORCE_GENERIC) return false;
    if (dtype != MBX_BF16 || g.d != kD || g.dv != kD || g.T != 1) return false;
    if (g.s2 > kRowsPerTile || g.gq > kMaxGq || g.s1 > 32) return false;
    if (g.nf == 0 && (g.q_order || g.kv_order)) return false;   // no closed form for the rows
    if (!strides_ok(g.qs) || !strides_ok(g.ks) || !strides_ok(g.vs) || !strides_ok(g.os)) return false;
    const int64_t nq = (int64_t)g.c1q * g.s1 * g.c2 * g.s2, nk = (int64_t)g.c1k * g.s1 * g.c2 * g.s2;
    if (nq < kRowsPerTile || nk < kRowsPerTile) return false;
    if ((int64_t)g.bh * g.gq * g.s2 * g.nkeys >= ((int64_t)1 << 31)) return false;
    return encode_fn() != nullptr;
}

size_t tc_workspace_bytes(const Geometry& g) {
    const size_t rows = (size_t)g.bh * g.gq * g.s2 * g.nkeys;
    return align256(rows * 512) + align256(rows * 4);
}

cudaError_t tc_forward(const Geometry& g, const void* q, const void* k, const void* v, void* out,
                       void* workspace, cudaStream_t stream) {
    const int B = g.bh / g.heads;
    const int nq = g.c1q * g.s1 * g.c2 * g.s2, nk = g.c1k * g.s1 * g.c2 * g.s2;
    if (((uintptr_t)q | (uintptr_t)k | (uintptr_t)v | (uintptr_t)out | (uintptr_t)workspace) & 15)
        return cudaErrorInvalidValue;
    CUtensorMap tq, tk, tv, tw;
    if (!make_qkv_map(&tq, q, B, g.heads, nq, g.qs) || !make_qkv_map(&tk, k, B, g.heads, nk, g.ks) ||
        !make_qkv_map(&tv, v, B, g.heads, nk, g.vs))
        return cudaErrorInvalidValue;
    const int64_t rows = (int64_t)g.bh * g.gq * g.s2 * g.nkeys;
    __nv_bfloat16* W = reinterpret_cast<__nv_bfloat16*>(workspace);
    float* Wc = reinterpret_cast<float*>(reinterpret_cast<char*>(workspace) + align256(rows * 512));
    if (!make_w_map(&tw, W, rows)) return cudaErrorInvalidValue;

    cudaError_t e;
    const int smem_row = RowSmem::kTotal + 1024;
    const int smem_col = ColSmem::kTotal + 1024;
    if ((e = cudaFuncSetAttribute(tc_row_stage, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_row)) != cudaSuccess)
        return e;
    if ((e = cudaFuncSetAttribute(tc_column_stage, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_col)) !=
        cudaSuccess)
        return e;
    const int units = g.bh * g.gk * g.s1;
    const int grid_row = units < num_sms() ? units : num_sms();
    {
        ProfScope p("tc_row_stage", stream);
        tc_row_stage<<<grid_row, kThreads, smem_row, stream>>>(tq, tk, tv, g, W, Wc);
    }
    {
        ProfScope p("tc_column_stage", stream);
        tc_column_stage<<<g.bh * g.gq * g.s2, kThreads, smem_col, stream>>>(
            tw, g, reinterpret_cast<const __nv_bfloat16*>(q), Wc, reinterpret_cast<__nv_bfloat16*>(out));
    }
    return cudaGetLastError();
}

}  // namespace mbx
