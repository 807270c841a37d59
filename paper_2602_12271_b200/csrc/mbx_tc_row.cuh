// Row stage (included by mbx_tc.cu).
//
// Item = (b, h, in-tile row k, M-tile mt): the Q rows k of query tiles
// 2mt, 2mt+1 (one 128-row M tile) stay in smem while the K/V rows k of every
// key tile c stream through a 2-stage TMA ring.  Per task (key tile c):
//   MMA1  S[(a,j), i] = Q_k . K_ck^T        128 x 64 x 128      -> TMEM buffer t%2
//   softmax_i (warps 2-5, one query row per thread), c_L = sum R z - lse,
//   R = p / l written as bf16 P (double-buffered)
//   MMA2  [aL | Y]    = P . [K_ck | V_ck]   128 x 256 x 64      -> same TMEM buffer
//   epilogue (warps 6-9): TMEM -> bf16 -> per-warp smem staging -> TMA store into the
//   blocked workspace W[col][part][key][64] (part 0,1 = aL halves, 2,3 = Y halves),
//   so the column stage reads contiguous 12 KB boxes.
// (solver.py:187-191 R update and c_L; factors.py:123 Y = R V; tensorops.py:268-272)
constexpr int kRowThreads = 320;   // 10 warps
struct RowSmem {
    // Q[2] (32 KB each): d-chunk c at c*16K, query tile 2mt+la at rows la*64.. (+la*8K)
    static constexpr int kQ = 0;
    static constexpr int kQBytes = 32768;
    static constexpr int kKV = 2 * kQBytes;           // KV[2]: [K c0 | K c1 | V c0 | V c1] 8 KB each (32 KB)
    static constexpr int kKVBytes = 32768;
    static constexpr int kP = kKV + 2 * kKVBytes;     // P[2]: [128][64] bf16 (16 KB each)
    static constexpr int kStage = kP + 2 * 16384;     // epilogue staging [4 warps][2] x [32][64] bf16 (4 KB each)
    static constexpr int kStats = kStage + 2 * 16384; // c_L[2][128] floats
    static constexpr int kBars = kStats + 2 * 128 * 4;
    static constexpr int kNumBars = 18;
    static constexpr int kTmemSlot = kBars + kNumBars * 8;
    static constexpr int kTotal = kTmemSlot + 16;
};

struct RowTask {            // decoded task t of this CTA: item (b,h,k,mt), key tile c
    int bh, kr, mt, c;
    bool first_of_item, last_of_item;
};

__device__ __forceinline__ RowTask row_task(const Geometry& g, int t, int n_mt, int first_item, int item_stride) {
    RowTask r;
    const int li = t / g.gk;
    r.c = t - li * g.gk;
    const int item = first_item + li * item_stride;   // item = (bh * s1 + k) * n_mt + mt
    r.mt = item % n_mt;
    r.kr = (item / n_mt) % g.s1;
    r.bh = item / (n_mt * g.s1);
    r.first_of_item = r.c == 0;
    r.last_of_item = r.c == g.gk - 1;
    return r;
}

__device__ __forceinline__ void tma_store_4d(const CUtensorMap* map, const void* src, int c0, int c1, int c2, int c3) {
    asm volatile("cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%2, %3, %4, %5}], [%1];" ::"l"(
                     reinterpret_cast<uint64_t>(map)),
                 "r"(smem_u32(src)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait() { asm volatile("cp.async.bulk.wait_group %0;" ::"n"(N) : "memory"); }

__global__ void __launch_bounds__(kRowThreads, 1)
tc_row_stage(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
             const __grid_constant__ CUtensorMap tm_v, const __grid_constant__ CUtensorMap tm_wst,
             const __grid_constant__ CUtensorMap tm_wst_b, Geometry g, float* __restrict__ Wc) {
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
    uint64_t* p_full = bars + 14;   // [2]
    uint64_t* p_empty = bars + 16;  // [2]
    float* stats = reinterpret_cast<float*>(smem + RowSmem::kStats);
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + RowSmem::kTmemSlot);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

    const int n_mt = (g.gq + 1) >> 1;
    const int items = g.bh * g.s1 * n_mt;
    const int first_item = blockIdx.x, item_stride = gridDim.x;
    const int my_items = first_item < items ? (items - first_item + item_stride - 1) / item_stride : 0;
    const int my_tasks = my_items * g.gk;
    const uint32_t box_bytes = (uint32_t)g.s2 * 128u;

    if (tid == 0) {
        tma_prefetch(&tm_q);
        tma_prefetch(&tm_k);
        tma_prefetch(&tm_v);
        tma_prefetch(&tm_wst);
        tma_prefetch(&tm_wst_b);
        for (int i = 0; i < 2; ++i) {
            mbar_init(&q_full[i], 1);
            mbar_init(&q_empty[i], 1);
            mbar_init(&kv_full[i], 1);
            mbar_init(&kv_empty[i], 1);
            mbar_init(&s_full[i], 1);
            mbar_init(&o_full[i], 1);
            mbar_init(&t_empty[i], 128);
            mbar_init(&p_full[i], 128);
            mbar_init(&p_empty[i], 1);
        }
        fence_barrier_init();
    }
    // Rows s2..63 of every box slot (and the second query-tile slot of an odd last
    // M tile) are never written by TMA: zero them once so MMA padding reads zeros.
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
            int ti = 0;
            for (int t = 0; t < my_tasks; ++t) {
                const RowTask tk = row_task(g, t, n_mt, first_item, item_stride);
                const int b = tk.bh / g.heads, h = tk.bh % g.heads;
                if (tk.first_of_item) {
                    const int li = t / g.gk, qs = li & 1;
                    mbar_wait(&q_empty[qs], ring_parity(li, 2) ^ 1);
                    TR(0, ti, 1);
                    const int nqa = min(2, g.gq - 2 * tk.mt);
                    mbar_expect_tx(&q_full[qs], 2u * box_bytes * (uint32_t)nqa);
                    uint8_t* qb = smem + RowSmem::kQ + qs * RowSmem::kQBytes;
                    for (int la = 0; la < nqa; ++la) {
                        const int tok = (int)row_base(g, true, 2 * tk.mt + la, tk.kr);
                        tma_load_4d(qb + la * 8192, &tm_q, &q_full[qs], 0, tok, h, b);
                        tma_load_4d(qb + 16384 + la * 8192, &tm_q, &q_full[qs], 64, tok, h, b);
                    }
                }
                const int ks = t & 1;
                mbar_wait(&kv_empty[ks], ring_parity(t, 2) ^ 1);
                TR(0, ti, 2);
                mbar_expect_tx(&kv_full[ks], 4u * box_bytes);
                uint8_t* kb = smem + RowSmem::kKV + ks * RowSmem::kKVBytes;
                const int tok = (int)row_base(g, false, tk.c, tk.kr);
                tma_load_4d(kb, &tm_k, &kv_full[ks], 0, tok, h, b);
                tma_load_4d(kb + 8192, &tm_k, &kv_full[ks], 64, tok, h, b);
                tma_load_4d(kb + 16384, &tm_v, &kv_full[ks], 0, tok, h, b);
                tma_load_4d(kb + 24576, &tm_v, &kv_full[ks], 64, tok, h, b);
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------------ MMA issuer
        if (lane == 0) {
            const uint32_t idesc_s = idesc_bf16(128, 64, false, false);
            const uint32_t idesc_o = idesc_bf16(128, 256, false, true);
            int ti = 0;
            auto issue_s = [&](int t) {   // MMA1(t): TMEM buffer t%2 must be free
                const RowTask tk = row_task(g, t, n_mt, first_item, item_stride);
                const int li = t / g.gk;
                if (tk.first_of_item) mbar_wait(&q_full[li & 1], ring_parity(li, 2));
                mbar_wait(&kv_full[t & 1], ring_parity(t, 2));
                TR(1, ti, 11);
                tc_fence_after();
                const uint32_t qbase = smem_u32(smem + RowSmem::kQ + (li & 1) * RowSmem::kQBytes);
                const uint32_t kbase = smem_u32(smem + RowSmem::kKV + (t & 1) * RowSmem::kKVBytes);
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) {
                    const uint64_t ad = smem_desc(qbase + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024, 2);
                    const uint64_t bd = smem_desc(kbase + (kk >> 2) * 8192 + (kk & 3) * 32, 16, 1024, 2);
                    mma_bf16(tmem + (t & 1) * 256, ad, bd, idesc_s, kk > 0);
                }
                mma_commit(&s_full[t & 1]);
            };
            if (my_tasks > 0) issue_s(0);
            for (int t = 0; t < my_tasks; ++t) {
                const RowTask cur = row_task(g, t, n_mt, first_item, item_stride);
                // MMA1(t+1) waits for the epilogue of t-1 to free TMEM buffer (t+1)%2, MMA2(t)
                // for softmax(t): issue whichever is ready first so neither chain stalls the other.
                bool s_done = t + 1 >= my_tasks, o_done = false;
                while (!o_done) {
                    if (!s_done && mbar_test(&t_empty[(t + 1) & 1], ring_parity(t + 1, 2) ^ 1)) {
                        issue_s(t + 1);
                        s_done = true;
                    }
                    if (mbar_test(&p_full[t & 1], ring_parity(t, 2))) {
                        TR(1, ti, 12);
                        tc_fence_after();
                        const uint32_t pbase = smem_u32(smem + RowSmem::kP + (t & 1) * 16384);
                        const uint32_t kbase = smem_u32(smem + RowSmem::kKV + (t & 1) * RowSmem::kKVBytes);
#pragma unroll
                        for (int kk = 0; kk < 4; ++kk) {
                            const uint64_t ad = smem_desc(pbase + kk * 32, 16, 1024, 2);
                            const uint64_t bd = smem_desc(kbase + kk * 2048, 8192, 1024, 2);
                            mma_bf16(tmem + (t & 1) * 256, ad, bd, idesc_o, kk > 0);
                        }
                        mma_commit(&o_full[t & 1]);
                        mma_commit(&p_empty[t & 1]);
                        mma_commit(&kv_empty[t & 1]);
                        if (cur.last_of_item) mma_commit(&q_empty[(t / g.gk) & 1]);
                        o_done = true;
                    }
                }
                if (!s_done) {
                    mbar_wait(&t_empty[(t + 1) & 1], ring_parity(t + 1, 2) ^ 1);
                    issue_s(t + 1);
                }
            }
        }
    } else if (warp < 6) {
        // ------------------------------------------------------ softmax (rows = TMEM lanes)
        const int quad = warp & 3;
        const int r = quad * 32 + lane;
        const uint32_t lane_off = (uint32_t)(quad * 32) << 16;
        const float sl2 = g.scale * kLog2e;
        int ti = 0;
        for (int t = 0; t < my_tasks; ++t) {
            const RowTask tk = row_task(g, t, n_mt, first_item, item_stride);
            const int bsel = t & 1;
            const int a = tk.mt * 2 + (r >> 6), j = r & 63;
            const bool row_ok = a < g.gq && j < g.s2;
            mbar_wait(&s_full[bsel], ring_parity(t, 2));
            if (lane == 0) TR(warp, ti, 21);
            tc_fence_after();
            float z[64];
            tmem_ld32(tmem + bsel * 256 + lane_off, z);
            tmem_ld32(tmem + bsel * 256 + lane_off + 32, z + 32);
            // padded keys -> -1e30 (finite: exp2 -> 0 and 0 * z stays 0)
            if (g.s2 < 64) {
#pragma unroll
                for (int i = 0; i < 64; ++i) z[i] = i < g.s2 ? z[i] : -1e30f;
            }
            float mq[4] = {-1e30f, -1e30f, -1e30f, -1e30f};
#pragma unroll
            for (int i = 0; i < 64; ++i) mq[i & 3] = fmaxf(mq[i & 3], z[i]);
            const float m = fmaxf(fmaxf(mq[0], mq[1]), fmaxf(mq[2], mq[3]));
            const float mb = m * sl2;
            float lq[4] = {0.f, 0.f, 0.f, 0.f}, aq[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
            for (int i = 0; i < 64; i += 2) {
                const float p0 = ex2(fmaf(z[i], sl2, -mb)), p1 = ex2(fmaf(z[i + 1], sl2, -mb));
                lq[(i >> 1) & 3] += p0 + p1;
                aq[(i >> 1) & 3] = fmaf(p1, z[i + 1], fmaf(p0, z[i], aq[(i >> 1) & 3]));
                z[i] = p0;
                z[i + 1] = p1;
            }
            const float l = (lq[0] + lq[1]) + (lq[2] + lq[3]);
            const float A = (aq[0] + aq[1]) + (aq[2] + aq[3]);
            const float inv_l = 1.f / l;
            // c_L = sum R z - lse with z = scale * S
            stats[bsel * 128 + r] = g.scale * (A * inv_l - m) - __logf(l);
            // R = p / l goes into P (bf16, <= 1), so MMA2 yields normalised aL and Y
            const float pscale = row_ok ? inv_l : 0.f;
            uint32_t packed[32];
#pragma unroll
            for (int i = 0; i < 64; i += 2) packed[i >> 1] = pack_bf16(z[i] * pscale, z[i + 1] * pscale);
            tc_fence_before();
            mbar_wait(&p_empty[bsel], ring_parity(t, 2) ^ 1);   // MMA2(t-2) done with P[bsel]
            const uint32_t p_row = smem_u32(smem + RowSmem::kP + bsel * 16384) + r * 128;
#pragma unroll
            for (int cc = 0; cc < 8; ++cc)
                st_shared_v4(p_row + ((cc ^ (r & 7)) << 4), packed[4 * cc], packed[4 * cc + 1],
                             packed[4 * cc + 2], packed[4 * cc + 3]);
            fence_proxy_async_smem();
            mbar_arrive(&p_full[bsel]);
            if (lane == 0) TR(warp, ti, 22);
        }
    } else {
        // ------------------------------------------------------ epilogue: TMEM -> smem -> TMA store
        const int quad = warp & 3;
        const int r = quad * 32 + lane;
        const uint32_t lane_off = (uint32_t)(quad * 32) << 16;
        int nstore = 0;   // staging buffer uses of this warp
        int ti = 0;
        for (int t = 0; t < my_tasks; ++t) {
            const RowTask tk = row_task(g, t, n_mt, first_item, item_stride);
            const int bsel = t & 1;
            const int a = tk.mt * 2 + (r >> 6), j = r & 63;
            const bool row_ok = a < g.gq && j < g.s2;
            const int key = tk.c * g.s1 + tk.kr;
            mbar_wait(&o_full[bsel], ring_parity(t, 2));
            if (lane == 0 && warp < 8) TR(warp, ti, 31);
            tc_fence_after();
            const float c_l = stats[bsel * 128 + r];
            // per-warp staging (32 rows x 64 features) and per-warp TMA store: no cross-warp sync
            const int half = quad & 1;
            const int nrows = min(32, g.s2 - half * 32);
            const bool store_ok = a < g.gq && nrows > 0;
            const int col0 = (tk.bh * g.gq + (a < g.gq ? a : 0)) * g.s2 + half * 32;
            for (int part = 0; part < 4; ++part) {
                float o[64];
                tmem_ld32(tmem + bsel * 256 + lane_off + part * 64, o);
                tmem_ld32(tmem + bsel * 256 + lane_off + part * 64 + 32, o + 32);
                if (part == 3) {   // TMEM buffer fully read: MMA1(t+2) may reuse it
                    tc_fence_before();
                    mbar_arrive(&t_empty[bsel]);
                }
                // a warp whose rows are all padding (a >= G_q) writes nothing: touching the
                // staging buffer would race with this warp's in-flight TMA store from it
                if (!store_ok) continue;
                const int sb = nstore++ & 1;
                uint8_t* stg = smem + RowSmem::kStage + quad * 8192 + sb * 4096;
                if (lane == 0) bulk_wait_read<1>();   // previous store from this buffer has read it
                __syncwarp();
                const uint32_t srow = smem_u32(stg) + lane * 128;
#pragma unroll
                for (int cc = 0; cc < 8; ++cc)
                    st_shared_v4(srow + ((cc ^ (lane & 7)) << 4),
                                 pack_bf16(o[8 * cc], o[8 * cc + 1]), pack_bf16(o[8 * cc + 2], o[8 * cc + 3]),
                                 pack_bf16(o[8 * cc + 4], o[8 * cc + 5]), pack_bf16(o[8 * cc + 6], o[8 * cc + 7]));
                fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0) {
                    tma_store_4d(half ? &tm_wst_b : &tm_wst, stg, 0, key, part, col0);
                    bulk_commit();
                }
            }
            if (row_ok) Wc[(((int64_t)tk.bh * g.gq + a) * g.s2 + j) * ckey_stride(g) + key] = c_l;
            if (lane == 0 && warp < 8) TR(warp, ti, 32);
        }
        if (lane == 0) bulk_wait<0>();
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc<512>(tmem);
}
