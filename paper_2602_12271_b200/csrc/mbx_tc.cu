// tcgen05 / TMEM / TMA kernels of the tiled MonarchAttention forward (bf16,
// d = d_v = 128, T = 1, tile rows of <= 64 tokens, <= 32 rows per tile,
// <= 4 query tiles).  Two warp-specialized persistent kernels joined by a
// bf16 workspace W:
//
//   row stage (tc_row_stage): item = (b, h, in-tile row k); the Q rows k of all
//     query tiles stay in smem while the K/V rows k of every key tile c stream
//     through a 2-stage TMA ring.  Per (c, M-tile):
//       MMA1  S[(a,j), i] = Q_k . K_ck^T        128 x 64 x 128      -> TMEM buf b
//       softmax_i (warps 2-5, one query row per thread), c_L = sum R z - lse
//       MMA2  [aL | Y]    = P . [K_ck | V_ck]   128 x 256 x 64      -> TMEM buf b
//       epilogue (warps 6-9): * 1/l, bf16, W[b,h,a,j,(c,k),0:256], c_L -> Wc
//     (solver.py:187-191, factors.py:123; tensorops.py:268-272)
//   column stage (tc_column_stage): item = column (b, h, a, j), keys (c,k) in
//     chunks of 128 on the TMEM lanes (transposed):
//       MMA3  S^T[key, l] = aL . Q_col^T        128 x 32 x 128
//       joint softmax over keys (warps 2-5), online across chunks, bias -c_L
//       MMA4  O^T[v, l]  += Y^T . P^T            128 x 32 x 128
//     (solver.py:192-195, factors.py:124)
//
// Warp roles: 0 = TMA producer, 1 = MMA issuer (one elected lane),
// 2-5 = softmax, 6-9 = epilogue (row stage only).  Every hand-off is an
// mbarrier; TMEM accumulators are double-buffered so MMA1(t+1) overlaps the
// softmax / epilogue of t.  The plan's permutation is folded into TMA
// coordinates: each tile row is one box at token row_base(tile, r).
#include "mbx_internal.h"
#include "mbx_sm100.cuh"

#include <cuda.h>
#include <math.h>
#include <string.h>

namespace mbx {
namespace {

using namespace sm100;

constexpr int kD = 128;           // head dim (q, k) and value dim
constexpr int kMaxS2 = 64;        // tile-row tokens (MMA1 N, MMA2 K)
constexpr int kMaxS1 = 32;        // tile rows (column-stage N)
constexpr int kMaxGq = 4;         // query tiles per key row (2 M tiles)
constexpr float kLog2e = 1.4426950408889634f;

__device__ __forceinline__ uint32_t ring_parity(uint32_t n, uint32_t size) { return (n / size) & 1u; }

// c_L rows are padded to 32 floats so each column's row is a 16-byte aligned TMA box.
__host__ __device__ __forceinline__ int ckey_stride(const Geometry& g) { return (g.nkeys + 31) & ~31; }

// =============================================================== row stage
constexpr int kRowThreads = 320;   // 10 warps
struct RowSmem {
    static constexpr int kQ = 0;                      // Q[2]: 2 M tiles x 2 d-chunks x [128][64]  (64 KB each)
    static constexpr int kQBytes = 65536;
    static constexpr int kKV = 2 * kQBytes;           // KV[2]: [K c0 | K c1 | V c0 | V c1] 8 KB each (32 KB)
    static constexpr int kKVBytes = 32768;
    static constexpr int kP = kKV + 2 * kKVBytes;     // P: [128][64] bf16 (16 KB)
    static constexpr int kStats = kP + 16384;         // stats[2][128] float2 (inv_l, c_L)
    static constexpr int kBars = kStats + 2 * 128 * 8;
    static constexpr int kNumBars = 16;
    static constexpr int kTmemSlot = kBars + kNumBars * 8;
    static constexpr int kTotal = kTmemSlot + 16;
};

struct RowTask {            // decoded task t of this CTA
    int item, c, mt;
    bool first_of_item, last_of_item, first_of_c, last_of_c;
};

__device__ __forceinline__ RowTask row_task(int t, int n_mt, int gk, int first_item, int item_stride) {
    RowTask r;
    const int per_item = n_mt * gk;
    const int li = t / per_item, rem = t - li * per_item;
    r.item = first_item + li * item_stride;
    r.c = rem / n_mt;
    r.mt = rem - r.c * n_mt;
    r.first_of_item = rem == 0;
    r.last_of_item = rem == per_item - 1;
    r.first_of_c = r.mt == 0;
    r.last_of_c = r.mt == n_mt - 1;
    return r;
}

__global__ void __launch_bounds__(kRowThreads, 1)
tc_row_stage(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
             const __grid_constant__ CUtensorMap tm_v, Geometry g, __nv_bfloat16* __restrict__ W,
             float* __restrict__ Wc) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + RowSmem::kBars);
    uint64_t* q_full = bars + 0;    // [2]
    uint64_t* q_empty = bars + 2;   // [2]
    uint64_t* kv_full = bars + 4;   // [2]
    uint64_t* kv_empty = bars + 6;  // [2]
    uint64_t* s_full = bars + 8;    // [2]
    uint64_t* o_full = bars + 10;   // [2]
    uint64_t* t_empty = bars + 12;  // [2]
    uint64_t* p_full = bars + 14;   // [1]
    uint64_t* p_empty = bars + 15;  // [1]
    float2* stats = reinterpret_cast<float2*>(smem + RowSmem::kStats);
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + RowSmem::kTmemSlot);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

    const int items = g.bh * g.s1;
    const int first_item = blockIdx.x, item_stride = gridDim.x;
    const int my_items = first_item < items ? (items - first_item + item_stride - 1) / item_stride : 0;
    const int n_mt = (g.gq + 1) >> 1;
    const int my_tasks = my_items * g.gk * n_mt;
    const uint32_t box_bytes = (uint32_t)g.s2 * 128u;

    if (tid == 0) {
        tma_prefetch(&tm_q);
        tma_prefetch(&tm_k);
        tma_prefetch(&tm_v);
        for (int i = 0; i < 2; ++i) {
            mbar_init(&q_full[i], 1);
            mbar_init(&q_empty[i], 1);
            mbar_init(&kv_full[i], 1);
            mbar_init(&kv_empty[i], 1);
            mbar_init(&s_full[i], 1);
            mbar_init(&o_full[i], 1);
            mbar_init(&t_empty[i], 128);
        }
        mbar_init(p_full, 128);
        mbar_init(p_empty, 1);
        fence_barrier_init();
    }
    // rows s2..63 of every K/V/Q box slot (and unused query-tile slots) are never
    // written by TMA (box = s2 rows): zero them once so MMA padding reads zeros.
    for (int i = tid; i < (2 * RowSmem::kQBytes + 2 * RowSmem::kKVBytes) / 16; i += kRowThreads)
        reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
    if (warp == 0) tmem_alloc<512>(tmem_slot);
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        // ------------------------------------------------------ TMA producer
        if (lane == 0) {
            uint32_t nq = 0, nkv = 0;
            for (int t = 0; t < my_tasks; ++t) {
                const RowTask tk = row_task(t, n_mt, g.gk, first_item, item_stride);
                const int kr = tk.item % g.s1, bh = tk.item / g.s1;
                const int b = bh / g.heads, h = bh % g.heads;
                if (tk.first_of_item) {
                    const int qs = nq & 1;
                    mbar_wait(&q_empty[qs], ring_parity(nq, 2) ^ 1);
                    mbar_expect_tx(&q_full[qs], 2u * box_bytes * (uint32_t)g.gq);
                    uint8_t* qb = smem + RowSmem::kQ + qs * RowSmem::kQBytes;
                    for (int a = 0; a < g.gq; ++a) {
                        const int tok = (int)row_base(g, true, a, kr);
                        uint8_t* dst = qb + (a >> 1) * 32768 + (a & 1) * 8192;
                        tma_load_4d(dst, &tm_q, &q_full[qs], 0, tok, h, b);
                        tma_load_4d(dst + 16384, &tm_q, &q_full[qs], 64, tok, h, b);
                    }
                    ++nq;
                }
                if (tk.first_of_c) {
                    const int ks = nkv & 1;
                    mbar_wait(&kv_empty[ks], ring_parity(nkv, 2) ^ 1);
                    mbar_expect_tx(&kv_full[ks], 4u * box_bytes);
                    uint8_t* kb = smem + RowSmem::kKV + ks * RowSmem::kKVBytes;
                    const int tok = (int)row_base(g, false, tk.c, kr);
                    tma_load_4d(kb, &tm_k, &kv_full[ks], 0, tok, h, b);
                    tma_load_4d(kb + 8192, &tm_k, &kv_full[ks], 64, tok, h, b);
                    tma_load_4d(kb + 16384, &tm_v, &kv_full[ks], 0, tok, h, b);
                    tma_load_4d(kb + 24576, &tm_v, &kv_full[ks], 64, tok, h, b);
                    ++nkv;
                }
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------------ MMA issuer
        if (lane == 0) {
            const uint32_t idesc_s = idesc_bf16(128, 64, false, false);
            const uint32_t idesc_o = idesc_bf16(128, 256, false, true);
            const uint32_t p_base = smem_u32(smem + RowSmem::kP);
            uint32_t nq = 0, nkv = 0;
            // MMA1 for task t (needs Q, K/V and a free TMEM buffer)
            auto issue_s = [&](int t, const RowTask& tk) {
                const int qs = (nq - 1) & 1, ks = (nkv - 1) & 1;
                const int bsel = t & 1;
                mbar_wait(&t_empty[bsel], ring_parity(t, 2) ^ 1);
                tc_fence_after();
                const uint32_t qbase = smem_u32(smem + RowSmem::kQ + qs * RowSmem::kQBytes) + tk.mt * 32768;
                const uint32_t kbase = smem_u32(smem + RowSmem::kKV + ks * RowSmem::kKVBytes);
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) {
                    const uint64_t ad = smem_desc(qbase + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024, 2);
                    const uint64_t bd = smem_desc(kbase + (kk >> 2) * 8192 + (kk & 3) * 32, 16, 1024, 2);
                    mma_bf16(tmem + bsel * 256, ad, bd, idesc_s, kk > 0);
                }
                mma_commit(&s_full[bsel]);
            };
            RowTask cur{};
            for (int t = 0; t < my_tasks; ++t) {
                cur = row_task(t, n_mt, g.gk, first_item, item_stride);
                if (t == 0) {
                    if (cur.first_of_item) { mbar_wait(&q_full[nq & 1], ring_parity(nq, 2)); ++nq; }
                    if (cur.first_of_c) { mbar_wait(&kv_full[nkv & 1], ring_parity(nkv, 2)); ++nkv; }
                    issue_s(t, cur);
                }
                // look ahead: MMA1(t+1) before MMA2(t) so it overlaps softmax(t)
                if (t + 1 < my_tasks) {
                    const RowTask nx = row_task(t + 1, n_mt, g.gk, first_item, item_stride);
                    if (nx.first_of_item) { mbar_wait(&q_full[nq & 1], ring_parity(nq, 2)); ++nq; }
                    if (nx.first_of_c) { mbar_wait(&kv_full[nkv & 1], ring_parity(nkv, 2)); ++nkv; }
                    issue_s(t + 1, nx);
                }
                // MMA2(t): [aL | Y] = P . [K | V]
                const int bsel = t & 1;
                mbar_wait(p_full, ring_parity(t, 1));
                tc_fence_after();
                // K/V stage of task t: stage of its c (tasks t+1 may have advanced nkv)
                const int adv = (t + 1 < my_tasks) &&
                                row_task(t + 1, n_mt, g.gk, first_item, item_stride).first_of_c;
                const int ks = (nkv - 1 - adv) & 1;
                const uint32_t kbase = smem_u32(smem + RowSmem::kKV + ks * RowSmem::kKVBytes);
#pragma unroll
                for (int kk = 0; kk < 4; ++kk) {
                    const uint64_t ad = smem_desc(p_base + kk * 32, 16, 1024, 2);
                    const uint64_t bd = smem_desc(kbase + kk * 2048, 8192, 1024, 2);
                    mma_bf16(tmem + bsel * 256, ad, bd, idesc_o, kk > 0);
                }
                mma_commit(&o_full[bsel]);
                mma_commit(p_empty);
                if (cur.last_of_c) mma_commit(&kv_empty[ks]);
                if (cur.last_of_item) {
                    const int advq = (t + 1 < my_tasks) &&
                                     row_task(t + 1, n_mt, g.gk, first_item, item_stride).first_of_item;
                    mma_commit(&q_empty[(nq - 1 - advq) & 1]);
                }
            }
        }
    } else if (warp < 6) {
        // ------------------------------------------------------ softmax (rows = TMEM lanes)
        const int quad = warp & 3;
        const int r = quad * 32 + lane;
        const uint32_t lane_off = (uint32_t)(quad * 32) << 16;
        const uint32_t p_row = smem_u32(smem + RowSmem::kP) + r * 128;
        const float sl2 = g.scale * kLog2e;
        for (int t = 0; t < my_tasks; ++t) {
            const RowTask tk = row_task(t, n_mt, g.gk, first_item, item_stride);
            const int bsel = t & 1;
            const int a = tk.mt * 2 + (r >> 6), j = r & 63;
            const bool row_ok = a < g.gq && j < g.s2;
            mbar_wait(&s_full[bsel], ring_parity(t, 2));
            tc_fence_after();
            float z[64];
            tmem_ld32(tmem + bsel * 256 + lane_off, z);
            tmem_ld32(tmem + bsel * 256 + lane_off + 32, z + 32);
            float m = -INFINITY;
#pragma unroll
            for (int i = 0; i < 64; ++i)
                if (i < g.s2) m = fmaxf(m, z[i]);
            const float mb = m * sl2;
            float l = 0.f, A = 0.f;
            uint32_t packed[32];
#pragma unroll
            for (int i = 0; i < 64; i += 2) {
                float p0 = (i < g.s2) ? exp2f(fmaf(z[i], sl2, -mb)) : 0.f;
                float p1 = (i + 1 < g.s2) ? exp2f(fmaf(z[i + 1], sl2, -mb)) : 0.f;
                l += p0 + p1;
                A = fmaf(p0, (i < g.s2 ? z[i] : 0.f), A);
                A = fmaf(p1, (i + 1 < g.s2 ? z[i + 1] : 0.f), A);
                if (!row_ok) p0 = p1 = 0.f;
                packed[i >> 1] = pack_bf16(p0, p1);
            }
            const float inv_l = 1.f / l;
            // c_L = sum R z - lse with z = scale * S
            const float c_l = g.scale * (A * inv_l - m) - __logf(l);
            stats[bsel * 128 + r] = make_float2(inv_l, c_l);
            tc_fence_before();
            mbar_wait(p_empty, ring_parity(t, 1) ^ 1);
#pragma unroll
            for (int cc = 0; cc < 8; ++cc)
                st_shared_v4(p_row + ((cc ^ (r & 7)) << 4), packed[4 * cc], packed[4 * cc + 1],
                             packed[4 * cc + 2], packed[4 * cc + 3]);
            fence_proxy_async_smem();
            mbar_arrive(p_full);
        }
    } else {
        // ------------------------------------------------------ epilogue
        const int quad = warp & 3;
        const int r = quad * 32 + lane;
        const uint32_t lane_off = (uint32_t)(quad * 32) << 16;
        for (int t = 0; t < my_tasks; ++t) {
            const RowTask tk = row_task(t, n_mt, g.gk, first_item, item_stride);
            const int bsel = t & 1;
            const int a = tk.mt * 2 + (r >> 6), j = r & 63;
            const bool row_ok = a < g.gq && j < g.s2;
            const int kr = tk.item % g.s1, bh = tk.item / g.s1;
            mbar_wait(&o_full[bsel], ring_parity(t, 2));
            tc_fence_after();
            const float2 st = stats[bsel * 128 + r];
            const int64_t wrow = (((int64_t)bh * g.gq + (row_ok ? a : 0)) * g.s2 + (row_ok ? j : 0)) * g.nkeys +
                                 tk.c * g.s1 + kr;
            uint4* dst = reinterpret_cast<uint4*>(W + wrow * 256);
#pragma unroll
            for (int q32 = 0; q32 < 8; ++q32) {
                float o[32];
                tmem_ld32(tmem + bsel * 256 + lane_off + q32 * 32, o);
                if (row_ok) {
#pragma unroll
                    for (int v4 = 0; v4 < 4; ++v4) {
                        uint4 pk;
                        pk.x = pack_bf16(o[8 * v4 + 0] * st.x, o[8 * v4 + 1] * st.x);
                        pk.y = pack_bf16(o[8 * v4 + 2] * st.x, o[8 * v4 + 3] * st.x);
                        pk.z = pack_bf16(o[8 * v4 + 4] * st.x, o[8 * v4 + 5] * st.x);
                        pk.w = pack_bf16(o[8 * v4 + 6] * st.x, o[8 * v4 + 7] * st.x);
                        dst[q32 * 4 + v4] = pk;
                    }
                }
            }
            if (row_ok)
                Wc[(((int64_t)bh * g.gq + a) * g.s2 + j) * ckey_stride(g) + tk.c * g.s1 + kr] = st.y;
            tc_fence_before();
            mbar_arrive(&t_empty[bsel]);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc<512>(tmem);
}

// ============================================================ column stage
constexpr int kColThreads = 192;   // 6 warps
struct ColSmem {
    static constexpr int kW = 0;                       // W[2]: aL (2 x [128][64]) | Y (2 x [128][64]) = 64 KB
    static constexpr int kWBytes = 65536;
    static constexpr int kC = 2 * kWBytes;             // c_L[2][128] floats
    static constexpr int kQ = kC + 2 * 512;            // Qcol[2]: 2 x [32][64] (8 KB each)
    static constexpr int kQBytes = 8192;
    static constexpr int kP = kQ + 2 * kQBytes;        // P^T: [128][32] bf16 SW64 (8 KB)
    static constexpr int kRed = kP + 8192;             // [4 warps][32] partials
    static constexpr int kBars = kRed + 4 * 32 * 4;
    static constexpr int kNumBars = 16;
    static constexpr int kTmemSlot = kBars + kNumBars * 8;
    static constexpr int kTotal = kTmemSlot + 16;
};

// Reduce v[0..31] (one value per column l) over the 32 lanes of the warp;
// afterwards lane i holds the reduction of column i in v[0].
template <bool kMax>
__device__ __forceinline__ float warp_transpose_reduce(float (&v)[32], int lane) {
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
        const bool upper = (lane & o) != 0;
#pragma unroll
        for (int i = 0; i < o; ++i) {
            const float send = upper ? v[i] : v[i + o];
            const float keep = upper ? v[i + o] : v[i];
            const float recv = __shfl_xor_sync(0xffffffffu, send, o);
            v[i] = kMax ? fmaxf(keep, recv) : keep + recv;
        }
    }
    return v[0];
}

__global__ void __launch_bounds__(kColThreads, 1)
tc_column_stage(const __grid_constant__ CUtensorMap tm_w, const __grid_constant__ CUtensorMap tm_c,
                const __grid_constant__ CUtensorMap tm_qc, Geometry g, __nv_bfloat16* __restrict__ out) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + ColSmem::kBars);
    uint64_t* w_full = bars + 0;    // [2]
    uint64_t* w_empty = bars + 2;   // [2]
    uint64_t* q_full = bars + 4;    // [2]
    uint64_t* q_empty = bars + 6;   // [2]
    uint64_t* s_full = bars + 8;    // [1]
    uint64_t* p_full = bars + 9;    // [1]  softmax wrote P^T (and rescaled O)
    uint64_t* mma4_done = bars + 10;// [1]  MMA4 finished (O^T readable, P^T free)
    float* red = reinterpret_cast<float*>(smem + ColSmem::kRed);
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + ColSmem::kTmemSlot);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

    const int ncols = g.bh * g.gq * g.s2;
    const int nch = (g.nkeys + 127) / 128;
    const int first = blockIdx.x, stride = gridDim.x;
    const int my_cols = first < ncols ? (ncols - first + stride - 1) / stride : 0;
    const int my_tasks = my_cols * nch;

    if (tid == 0) {
        tma_prefetch(&tm_w);
        tma_prefetch(&tm_c);
        tma_prefetch(&tm_qc);
        for (int i = 0; i < 2; ++i) {
            mbar_init(&w_full[i], 1);
            mbar_init(&w_empty[i], 1);
            mbar_init(&q_full[i], 1);
            mbar_init(&q_empty[i], 1);
        }
        mbar_init(s_full, 1);
        mbar_init(p_full, 128);
        mbar_init(mma4_done, 1);
        fence_barrier_init();
    }
    if (warp == 0) tmem_alloc<64>(tmem_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const uint32_t tmem_S = tmem, tmem_O = tmem + 32;

    if (warp == 0) {
        // ------------------------------------------------------ TMA producer
        if (lane == 0) {
            for (int t = 0; t < my_tasks; ++t) {
                const int ci = t / nch, ch = t - ci * nch;
                const int col = first + ci * stride;
                if (ch == 0) {
                    const int qs = ci & 1;
                    mbar_wait(&q_empty[qs], ring_parity(ci, 2) ^ 1);
                    mbar_expect_tx(&q_full[qs], 2u * 32u * 128u);
                    const int j = col % g.s2, a = (col / g.s2) % g.gq, bh = col / (g.s2 * g.gq);
                    const int b = bh / g.heads, h = bh % g.heads;
                    // rows l of tile a at column j: token row_base(a, 0) + j + l * W (contiguous rows)
                    const int64_t tok0 = row_base(g, true, a, 0) + j;
                    const int wcol = (int)(tok0 % g.W), wrow = (int)(tok0 / g.W);
                    uint8_t* dst = smem + ColSmem::kQ + qs * ColSmem::kQBytes;
                    tma_load_4d(dst, &tm_qc, &q_full[qs], 0, wcol, wrow, bh);
                    tma_load_4d(dst + 4096, &tm_qc, &q_full[qs], 64, wcol, wrow, bh);
                    (void)b;
                    (void)h;
                }
                const int ws = t & 1;
                mbar_wait(&w_empty[ws], ring_parity(t, 2) ^ 1);
                mbar_expect_tx(&w_full[ws], 65536u + 512u);
                uint8_t* dst = smem + ColSmem::kW + ws * ColSmem::kWBytes;
                const int k0 = ch * 128;
                tma_load_3d(dst, &tm_w, &w_full[ws], 0, k0, col);
                tma_load_3d(dst + 16384, &tm_w, &w_full[ws], 64, k0, col);
                tma_load_3d(dst + 32768, &tm_w, &w_full[ws], 128, k0, col);
                tma_load_3d(dst + 49152, &tm_w, &w_full[ws], 192, k0, col);
                tma_load_2d(smem + ColSmem::kC + ws * 512, &tm_c, &w_full[ws], k0, col);
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------------ MMA issuer
        if (lane == 0) {
            const uint32_t idesc_s = idesc_bf16(128, 32, false, false);
            const uint32_t idesc_o = idesc_bf16(128, 32, true, true);
            const uint32_t sP = smem_u32(smem + ColSmem::kP);
            for (int t = 0; t < my_tasks; ++t) {
                const int ci = t / nch, ch = t - ci * nch;
                const int ws = t & 1, qs = ci & 1;
                const uint32_t sA = smem_u32(smem + ColSmem::kW + ws * ColSmem::kWBytes);
                const uint32_t sQ = smem_u32(smem + ColSmem::kQ + qs * ColSmem::kQBytes);
                if (ch == 0) mbar_wait(&q_full[qs], ring_parity(ci, 2));
                mbar_wait(&w_full[ws], ring_parity(t, 2));
                // S^T buffer is free once softmax(t-1) arrived on p_full (it read S first)
                if (t > 0) mbar_wait(p_full, ring_parity(t - 1, 1));
                tc_fence_after();
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) {
                    const uint64_t ad = smem_desc(sA + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024, 2);
                    const uint64_t bd = smem_desc(sQ + (kk >> 2) * 4096 + (kk & 3) * 32, 16, 1024, 2);
                    mma_bf16(tmem_S, ad, bd, idesc_s, kk > 0);
                }
                mma_commit(s_full);
                if (ch == nch - 1) mma_commit(&q_empty[qs]);
                // MMA4 once softmax(t) wrote P^T and rescaled O^T
                mbar_wait(p_full, ring_parity(t, 1));
                tc_fence_after();
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) {
                    const uint64_t ad = smem_desc(sA + 32768 + kk * 2048, 16384, 1024, 2);
                    const uint64_t bd = smem_desc(sP + kk * 1024, 4096, 512, 4);
                    mma_bf16(tmem_O, ad, bd, idesc_o, ch > 0 || kk > 0);
                }
                mma_commit(&w_empty[ws]);
                mma_commit(mma4_done);
            }
        }
    } else {
        // ------------------------------------------------------ softmax + output (keys / values on lanes)
        const int quad = warp & 3;
        const int r = quad * 32 + lane;                       // key within chunk / value dim
        const uint32_t lane_off = (uint32_t)(quad * 32) << 16;
        const uint32_t sP = smem_u32(smem + ColSmem::kP);
        const float sl2 = g.scale * kLog2e;
        float m_run[32], s_run[32];
        for (int t = 0; t < my_tasks; ++t) {
            const int ci = t / nch, ch = t - ci * nch;
            const int col = first + ci * stride;
            const int ws = t & 1;
            if (ch == 0) {
#pragma unroll
                for (int l = 0; l < 32; ++l) { m_run[l] = -INFINITY; s_run[l] = 0.f; }
            }
            const bool kv = ch * 128 + r < g.nkeys;
            mbar_wait(s_full, ring_parity(t, 1));
            tc_fence_after();
            float sv[32];
            tmem_ld32(tmem_S + lane_off, sv);
            const float cl2 = (kv ? reinterpret_cast<const float*>(smem + ColSmem::kC + ws * 512)[r] : 0.f) * kLog2e;
            // x = log2e * (scale * S - c_L), invalid keys / rows -> -inf
#pragma unroll
            for (int l = 0; l < 32; ++l) sv[l] = (kv && l < g.s1) ? fmaf(sv[l], sl2, -cl2) : -INFINITY;
            float tmp[32];
#pragma unroll
            for (int l = 0; l < 32; ++l) tmp[l] = sv[l];
            const float wmax = warp_transpose_reduce<true>(tmp, lane);   // lane l: max of column l in warp
            red[quad * 32 + lane] = wmax;
            named_sync(1, 128);
            const float cmax = fmaxf(fmaxf(red[lane], red[32 + lane]), fmaxf(red[64 + lane], red[96 + lane]));
            named_sync(1, 128);
            float scale_l[32], mnew[32];
#pragma unroll
            for (int l = 0; l < 32; ++l) {
                mnew[l] = fmaxf(m_run[l], __shfl_sync(0xffffffffu, cmax, l));
                scale_l[l] = (m_run[l] == -INFINITY) ? 0.f : exp2f(m_run[l] - mnew[l]);
                m_run[l] = mnew[l];
            }
            float pv[32];
#pragma unroll
            for (int l = 0; l < 32; ++l) pv[l] = (sv[l] == -INFINITY) ? 0.f : exp2f(sv[l] - mnew[l]);
#pragma unroll
            for (int l = 0; l < 32; ++l) tmp[l] = pv[l];
            const float wsum = warp_transpose_reduce<false>(tmp, lane);
            red[quad * 32 + lane] = wsum;
            named_sync(1, 128);
            const float csum = red[lane] + red[32 + lane] + red[64 + lane] + red[96 + lane];
#pragma unroll
            for (int l = 0; l < 32; ++l) s_run[l] = s_run[l] * scale_l[l] + __shfl_sync(0xffffffffu, csum, l);
            // P^T (and the O^T rescale) may only be written once MMA4(t-1) is done
            if (t > 0) mbar_wait(mma4_done, ring_parity(t - 1, 1));
            tc_fence_after();
            if (ch > 0) {
                float o[32];
                tmem_ld32(tmem_O + lane_off, o);
#pragma unroll
                for (int l = 0; l < 32; ++l) o[l] *= scale_l[l];
                tmem_st32(tmem_O + lane_off, o);
            } else if (t > 0) {
                // previous column finished: its O^T was consumed below before this point
            }
#pragma unroll
            for (int c4 = 0; c4 < 4; ++c4)
                st_shared_v4(sP + r * 64 + ((c4 ^ ((r >> 1) & 3)) << 4),
                             pack_bf16(pv[8 * c4], pv[8 * c4 + 1]), pack_bf16(pv[8 * c4 + 2], pv[8 * c4 + 3]),
                             pack_bf16(pv[8 * c4 + 4], pv[8 * c4 + 5]), pack_bf16(pv[8 * c4 + 6], pv[8 * c4 + 7]));
            fence_proxy_async_smem();
            tc_fence_before();
            named_sync(1, 128);   // everyone done with red[] / S^T before the next chunk
            mbar_arrive(p_full);
            if (ch == nch - 1) {
                // O[l, v] = O^T[v, l] / s_l  (thread r = value dim v)
                mbar_wait(mma4_done, ring_parity(t, 1));
                tc_fence_after();
                float o[32];
                tmem_ld32(tmem_O + lane_off, o);
                const int j = col % g.s2, a = (col / g.s2) % g.gq, bh = col / (g.s2 * g.gq);
                const int b = bh / g.heads, h = bh % g.heads;
                __nv_bfloat16* ob = out + b * g.os[0] + h * g.os[1];
#pragma unroll
                for (int l = 0; l < kMaxS1; ++l) {
                    if (l < g.s1) {
                        const int64_t tok = row_base(g, true, a, l) + j;
                        ob[tok * g.os[2] + r] = __float2bfloat16_rn(o[l] / s_run[l]);
                    }
                }
                tc_fence_before();
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc<64>(tmem);
}

// ===================================================================== host
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

bool encode(CUtensorMap* m, CUtensorMapDataType dt, int rank, const void* base, const cuuint64_t* dims,
            const cuuint64_t* strides, const cuuint32_t* box, CUtensorMapSwizzle sw) {
    EncodeTiledFn enc = encode_fn();
    if (!enc) return false;
    cuuint32_t es[5] = {1, 1, 1, 1, 1};
    return enc(m, dt, rank, const_cast<void*>(base), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// (B, H, N, 128) bf16 with element strides st[b,h,token]; box (64 features, rows tokens).
bool make_rows_map(CUtensorMap* m, const void* base, int B, int H, int N, const int64_t* st, int rows) {
    cuuint64_t dims[4] = {(cuuint64_t)kD, (cuuint64_t)N, (cuuint64_t)H, (cuuint64_t)B};
    cuuint64_t strides[3] = {(cuuint64_t)st[2] * 2, (cuuint64_t)st[1] * 2, (cuuint64_t)st[0] * 2};
    cuuint32_t box[4] = {64, (cuuint32_t)rows, 1, 1};
    return encode(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, base, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B);
}

// Query columns: q viewed as (d, w-column, grid row of W tokens, b*H+h); box (64, 1, 32, 1).
bool make_qcol_map(CUtensorMap* m, const void* base, const Geometry& g, int nq) {
    cuuint64_t dims[4] = {(cuuint64_t)kD, (cuuint64_t)g.W, (cuuint64_t)(nq / g.W), (cuuint64_t)g.bh};
    cuuint64_t strides[3] = {(cuuint64_t)g.qs[2] * 2, (cuuint64_t)g.qs[2] * 2 * g.W, (cuuint64_t)g.qs[1] * 2};
    cuuint32_t box[4] = {64, 1, (cuuint32_t)kMaxS1, 1};
    return encode(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, base, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B);
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

// Geometry with identity plans expressed as a (1, s1, s2)-neighborhood grid so the
// column-stage map can address tile columns uniformly.
bool column_grid(const Geometry& g, int* F, int* H, int* W) {
    if (g.nf > 0) {
        // rows of a tile are contiguous W-token grid rows iff nf == 1 or nh == H
        if (!(g.nf == 1 || g.nh == g.H)) return false;
        *F = g.F; *H = g.H; *W = g.W;
        return true;
    }
    if (g.c2 != 1) return false;          // identity with c2 > 1: rows interleave tile columns
    *F = g.c1k; *H = g.s1; *W = g.s2;
    return true;
}

}  // namespace

bool tc_supported(const Geometry& g, int dtype, int flags) {
    if (flags & MBX_FLAG_FORCE_GENERIC) return false;
    if (dtype != MBX_BF16 || g.d != kD || g.dv != kD || g.T != 1) return false;
    if (g.s2 > kMaxS2 || g.s1 > kMaxS1 || g.gq > kMaxGq) return false;
    if (g.nf == 0 && (g.q_order || g.kv_order)) return false;   // rows need a closed form
    int F, H, W;
    if (!column_grid(g, &F, &H, &W)) return false;
    if (!strides_ok(g.qs) || !strides_ok(g.ks) || !strides_ok(g.vs) || !strides_ok(g.os)) return false;
    if (g.bh > 1 && g.qs[0] != (int64_t)g.heads * g.qs[1]) return false;   // qcol map folds (b, h)
    if ((int64_t)g.bh * g.gq * g.s2 * g.nkeys >= ((int64_t)1 << 31)) return false;
    return encode_fn() != nullptr;
}

size_t tc_workspace_bytes(const Geometry& g) {
    const size_t rows = (size_t)g.bh * g.gq * g.s2 * g.nkeys;
    return align256(rows * 512) + align256((size_t)g.bh * g.gq * g.s2 * ckey_stride(g) * 4);
}

cudaError_t tc_forward(const Geometry& g0, const void* q, const void* k, const void* v, void* out,
                       void* workspace, cudaStream_t stream) {
    Geometry g = g0;
    int F, H, W;
    if (!column_grid(g, &F, &H, &W)) return cudaErrorInvalidValue;
    if (g.nf == 0) {   // express the identity plan as a (1, s1, s2) neighborhood grid
        g.F = F; g.H = H; g.W = W;
        g.nf = 1; g.nh = g.s1; g.nw = g.s2;
    }
    const int B = g.bh / g.heads;
    const int nq = g.c1q * g.s1 * g.c2 * g.s2, nk = g.c1k * g.s1 * g.c2 * g.s2;
    if (((uintptr_t)q | (uintptr_t)k | (uintptr_t)v | (uintptr_t)out | (uintptr_t)workspace) & 15)
        return cudaErrorInvalidValue;
    CUtensorMap tq, tk, tv, tqc, tw, tc;
    if (!make_rows_map(&tq, q, B, g.heads, nq, g.qs, g.s2) || !make_rows_map(&tk, k, B, g.heads, nk, g.ks, g.s2) ||
        !make_rows_map(&tv, v, B, g.heads, nk, g.vs, g.s2) || !make_qcol_map(&tqc, q, g, nq))
        return cudaErrorInvalidValue;
    const int64_t ncols = (int64_t)g.bh * g.gq * g.s2;
    const int64_t rows = ncols * g.nkeys;
    __nv_bfloat16* Wp = reinterpret_cast<__nv_bfloat16*>(workspace);
    float* Wc = reinterpret_cast<float*>(reinterpret_cast<char*>(workspace) + align256(rows * 512));
    {
        cuuint64_t dims[3] = {256, (cuuint64_t)g.nkeys, (cuuint64_t)ncols};
        cuuint64_t strides[2] = {512, (cuuint64_t)g.nkeys * 512};
        cuuint32_t box[3] = {64, 128, 1};
        if (!encode(&tw, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, Wp, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B))
            return cudaErrorInvalidValue;
        cuuint64_t cdims[2] = {(cuuint64_t)ckey_stride(g), (cuuint64_t)ncols};
        cuuint64_t cstrides[1] = {(cuuint64_t)ckey_stride(g) * 4};
        cuuint32_t cbox[2] = {128, 1};
        if (!encode(&tc, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, Wc, cdims, cstrides, cbox, CU_TENSOR_MAP_SWIZZLE_NONE))
            return cudaErrorInvalidValue;
    }

    cudaError_t e;
    const int smem_row = RowSmem::kTotal + 1024;
    const int smem_col = ColSmem::kTotal + 1024;
    if ((e = cudaFuncSetAttribute(tc_row_stage, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_row)) != cudaSuccess)
        return e;
    if ((e = cudaFuncSetAttribute(tc_column_stage, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_col)) !=
        cudaSuccess)
        return e;
    const int items = g.bh * g.s1;
    const int grid_row = items < num_sms() ? items : num_sms();
    {
        ProfScope p("tc_row_stage", stream);
        tc_row_stage<<<grid_row, kRowThreads, smem_row, stream>>>(tq, tk, tv, g, Wp, Wc);
    }
    const int grid_col = ncols < num_sms() ? (int)ncols : num_sms();
    {
        ProfScope p("tc_column_stage", stream);
        tc_column_stage<<<grid_col, kColThreads, smem_col, stream>>>(tw, tc, tqc, g,
                                                                      reinterpret_cast<__nv_bfloat16*>(out));
    }
    return cudaGetLastError();
}

}  // namespace mbx
