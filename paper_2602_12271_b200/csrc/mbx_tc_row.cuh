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

