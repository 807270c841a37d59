// Row stage for long tile rows, s2 > 64 (included by mbx_tc.cu): the paper's 720p
// blockings (w = 80), the aligned (f, hw) configuration (s2 = h w = 1560 at N = 32760)
// and raw (b1, b2) blockings with wide b2.  One tile row is then a FlashAttention-sized
// problem, so the row softmax runs online over 128-key chunks (solver.py:187-191,
// factors.py:123):
//
//   task = (b h, query tile a, row k, M tile of 128 query columns j, key tile c)
//   for each 128-key chunk of K/V row (c, k):
//     MMA1  S = A . K_ch^T             M=128 (j), N=128 (i), K=128     A = Q (or hat_alpha_R) rows
//     softmax warps 2-5 (thread = row j): running max (lazy: rescale O only when the max grows
//       by > 8 in log2 units), running sum l and sum p z; P (bf16) back over S
//     MMA2  O_aL += P . K_ch,  O_Y += P . V_ch     M=128, N=128, K=128 keys, A = P in TMEM
//   epilogue warps 6-9: aL = O_aL / l, Y = O_Y / l (bf16, coalesced rows of W through a
//   per-warp transpose buffer), c_L = scale (sum p z / l - m) - ln l.
//
// TMEM: S/P [0,128) [128,256); O_aL [256,384); O_Y [384,512).  smem: A slots 2 x 32 KB,
// K/V ring 2 x 64 KB (K and V chunks, 2 d-halves of [128 keys][128 B] each), epilogue
// transpose buffers 4 x 4 KB, per-task row statistics.
constexpr int kFThreads = 320;   // producer, MMA, 4 softmax, 4 epilogue warps
constexpr int kFKC = 128;        // keys per chunk / query rows per M tile
struct RowFSmem {
    static constexpr int kA = 0;                 // [2] x [2 d-halves][128 rows][128 B]
    static constexpr int kASlot = 32768;
    static constexpr int kKV = 2 * kASlot;       // [2] x [K d0 | K d1 | V d0 | V d1], 16 KB each
    static constexpr int kKVStage = 65536;
    static constexpr int kStage = kKV + 2 * kKVStage;   // [4 warps] x [32 rows][128 B]
    static constexpr int kStat = kStage + 4 * 4096;     // [2 tasks][3][128] floats: m, l, sum p z
    static constexpr int kBars = kStat + 2 * 3 * 128 * 4;
    static constexpr int kNumBars = 21;
    static constexpr int kTmemSlot = kBars + kNumBars * 8;
    static constexpr int kTotal = kTmemSlot + 16;
};
static_assert(RowFSmem::kTotal + 1024 <= 232448, "flash row stage exceeds 227 KB of shared memory");
constexpr uint32_t kFS = 0, kFOA = 256, kFOY = 384;

// Task walker: (bh, a, k, mt, c) with c fastest; a contiguous range per CTA.
struct FlashCursor {
    int t, t1, bh, a, k, mt, c;
    int nmt;
    bool valid;
    __device__ __forceinline__ void init(const Geometry& g, int cta, int ctas) {
        nmt = (g.s2 + kFKC - 1) / kFKC;
        const long long tasks = (long long)g.bh * g.gq * g.s1 * nmt * g.gk;
        t = (int)(tasks * cta / ctas);
        t1 = (int)(tasks * (cta + 1) / ctas);
        int x = t;
        c = x % g.gk; x /= g.gk;
        mt = x % nmt; x /= nmt;
        k = x % g.s1; x /= g.s1;
        a = x % g.gq;
        bh = x / g.gq;
        valid = t < t1;
    }
    __device__ __forceinline__ void advance(const Geometry& g) {
        ++t;
        valid = t < t1;
        if (++c == g.gk) {
            c = 0;
            if (++mt == nmt) {
                mt = 0;
                if (++k == g.s1) {
                    k = 0;
                    if (++a == g.gq) {
                        a = 0;
                        ++bh;
                    }
                }
            }
        }
    }
    __device__ __forceinline__ bool first_of_item(int t0) const { return c == 0 || t == t0; }
    __device__ __forceinline__ bool last_of_item(const Geometry& g) const { return c == g.gk - 1 || t == t1 - 1; }
};

__global__ void __launch_bounds__(kFThreads, 1)
tc_row_flash(const __grid_constant__ TcParams P, Geometry g, int amode_i, int want_y_i) {
    const bool amode = amode_i != 0, want_y = want_y_i != 0;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + RowFSmem::kBars);
    uint64_t* a_full = bars;          // [2]
    uint64_t* a_empty = bars + 2;     // [2]
    uint64_t* kv_full = bars + 4;     // [2]
    uint64_t* kv_empty = bars + 6;    // [2]
    uint64_t* s_full = bars + 8;      // [2]  MMA1 wrote S
    uint64_t* p_full = bars + 10;     // [2]  softmax wrote P (128 arrivals)
    uint64_t* sp_empty = bars + 12;   // [2]  MMA2 read P: S/P buffer reusable
    uint64_t* o_step = bars + 14;     // every MMA2 completed (rescale waits)
    uint64_t* o_full = bars + 15;     // last chunk's MMA2 of a task completed
    uint64_t* o_empty = bars + 16;    // epilogue read O (128 arrivals)
    uint64_t* st_full = bars + 17;    // [2] row statistics of a task written (128)
    uint64_t* st_empty = bars + 19;   // [2] and read (128)
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + RowFSmem::kTmemSlot);
    float* stats = reinterpret_cast<float*>(smem + RowFSmem::kStat);   // [2][3][128]
    const int tid = threadIdx.x, lane = tid & 31;
    const int warp = __shfl_sync(0xffffffffu, tid >> 5, 0);
    const int nck = (g.s2 + kFKC - 1) / kFKC;
    const int ckey = ckey_stride(g);

    if (tid == 0) {
        tma_prefetch(&P.tq128);
        tma_prefetch(&P.tk128);
        tma_prefetch(&P.tv128);
        if (amode) tma_prefetch(&P.tar_ld128);
        for (int i = 0; i < 2; ++i) {
            mbar_init(&a_full[i], 1);
            mbar_init(&a_empty[i], 1);
            mbar_init(&kv_full[i], 1);
            mbar_init(&kv_empty[i], 1);
            mbar_init(&s_full[i], 1);
            mbar_init(&p_full[i], 128);
            mbar_init(&sp_empty[i], 1);
            mbar_init(&st_full[i], 128);
            mbar_init(&st_empty[i], 128);
        }
        mbar_init(o_step, 1);
        mbar_init(o_full, 1);
        mbar_init(o_empty, 128);
        fence_barrier_init();
    }
    if (warp == 0) tmem_alloc<512>(tmem_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    pdl_wait();
    pdl_trigger();

    FlashCursor cur;
    cur.init(g, blockIdx.x, gridDim.x);
    const int t0 = cur.t;

    if (warp == 0) {
        // ------------------------------------------------ TMA producer
        const bool leader = elect_one();
        int an = 0, n = 0;   // A slot uses, global chunk index
        for (FlashCursor pc = cur; pc.valid; pc.advance(g)) {
            const int b = pc.bh / g.heads, h = pc.bh % g.heads;
            const int j0 = pc.mt * kFKC;
            if (amode || pc.first_of_item(t0)) {
                const int sl = an & 1;
                mbar_wait(&a_empty[sl], ((an >> 1) & 1) ^ 1);
                if (leader) {
                    mbar_expect_tx(&a_full[sl], 32768u);
                    uint8_t* ab = smem + RowFSmem::kA + sl * RowFSmem::kASlot;
                    if (amode) {
                        const int key = pc.c * g.s1 + pc.k, ag = pc.bh * g.gq + pc.a;
                        tma_load_4d(ab, &P.tar_ld128, &a_full[sl], 0, j0, key, ag);
                        tma_load_4d(ab + 16384, &P.tar_ld128, &a_full[sl], 64, j0, key, ag);
                    } else {
                        const int tok = (int)row_base(g, true, pc.a, pc.k) + j0;
                        tma_load_4d(ab, &P.tq128, &a_full[sl], 0, tok, h, b);
                        tma_load_4d(ab + 16384, &P.tq128, &a_full[sl], 64, tok, h, b);
                    }
                }
                __syncwarp();
                ++an;
            }
            const int tokk = (int)row_base(g, false, pc.c, pc.k);
            for (int ch = 0; ch < nck; ++ch, ++n) {
                const int st = n & 1;
                mbar_wait(&kv_empty[st], ((n >> 1) & 1) ^ 1);
                if (leader) {
                    mbar_expect_tx(&kv_full[st], want_y ? 65536u : 32768u);   // V only for Y
                    uint8_t* kb = smem + RowFSmem::kKV + st * RowFSmem::kKVStage;
                    const int tok = tokk + ch * kFKC;
                    tma_load_4d(kb, &P.tk128, &kv_full[st], 0, tok, h, b);
                    tma_load_4d(kb + 16384, &P.tk128, &kv_full[st], 64, tok, h, b);
                    if (want_y) {
                        tma_load_4d(kb + 32768, &P.tv128, &kv_full[st], 0, tok, h, b);
                        tma_load_4d(kb + 49152, &P.tv128, &kv_full[st], 64, tok, h, b);
                    }
                }
                __syncwarp();
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------ MMA issuer (whole warp, uniform state)
        const bool leader = elect_one();
        const uint32_t id1 = idesc_bf16(128, 128, false, false);
        const uint32_t id2 = idesc_bf16(128, 128, false, true);
        constexpr uint32_t kHi = (1024u >> 4) | (1u << 14) | (2u << 29);
        auto desc = [](uint32_t lo) { return ((uint64_t)kHi << 32) | lo; };
        const uint32_t a_lo = ((smem_u32(smem + RowFSmem::kA) & 0x3FFFF) >> 4) | (1u << 16);
        const uint32_t kv_lo = (smem_u32(smem + RowFSmem::kKV) & 0x3FFFF) >> 4;
        // MMA1 cursor (task cs, chunk c1n) and MMA2 cursor (task co, chunk c2n); global chunk indices
        FlashCursor cs = cur, co = cur;
        int ch1 = 0, ch2 = 0, n1 = 0, n2 = 0, an = 0, to = 0;
        while (cs.valid || co.valid) {
            // MMA2(n2): P written; the task's first chunk also needs O drained by the epilogue
            if (co.valid && n2 < n1 && mbar_test_uniform(&p_full[n2 & 1], (n2 >> 1) & 1) &&
                (ch2 > 0 || mbar_test_uniform(o_empty, (to & 1) ^ 1))) {
                tc_fence_after();
                if (leader) {
                    const int st = n2 & 1;
                    const uint32_t pa = tmem + kFS + st * 128;
                    const uint32_t b_lo = kv_lo + (uint32_t)((st * RowFSmem::kKVStage) >> 4) + ((16384u >> 4) << 16);
                    for (int s = 0; s < (want_y ? 2 : 1); ++s) {
#pragma unroll
                        for (int kk = 0; kk < 8; ++kk)
                            mma_bf16_ts(tmem + (s ? kFOY : kFOA), pa + kk * 8,
                                        desc(b_lo + ((s * 32768 + kk * 2048) >> 4)), id2, ch2 > 0 || kk > 0);
                    }
                    mma_commit(&kv_empty[st]);
                    mma_commit(&sp_empty[st]);
                    mma_commit(o_step);
                    if (ch2 == nck - 1) mma_commit(o_full);
                }
                __syncwarp();
                ++n2;
                if (++ch2 == nck) {
                    ch2 = 0;
                    ++to;
                    co.advance(g);
                }
            }
            // MMA1(n1): A and K/V landed, S/P buffer released by MMA2(n1 - 2)
            if (cs.valid && n1 < n2 + 2) {
                const int sl = an & 1;
                const bool ready = mbar_test_uniform(&a_full[sl], (an >> 1) & 1) &&
                                   mbar_test_uniform(&kv_full[n1 & 1], (n1 >> 1) & 1) &&
                                   (n1 < 2 || mbar_test_uniform(&sp_empty[n1 & 1], ((n1 >> 1) - 1) & 1));
                if (ready) {
                    tc_fence_after();
                    const bool last_use = ch1 == nck - 1 && (amode || cs.last_of_item(g));
                    if (leader) {
                        const int st = n1 & 1;
                        const uint32_t aa = a_lo + (uint32_t)sl * (RowFSmem::kASlot >> 4);
                        const uint32_t b_lo = kv_lo + (uint32_t)((st * RowFSmem::kKVStage) >> 4) + (1u << 16);
#pragma unroll
                        for (int kk = 0; kk < 8; ++kk)
                            mma_bf16(tmem + kFS + st * 128, desc(aa + (((kk >> 2) * 16384 + (kk & 3) * 32) >> 4)),
                                     desc(b_lo + (((kk >> 2) * 16384 + (kk & 3) * 32) >> 4)), id1, kk > 0);
                        mma_commit(&s_full[st]);
                        if (last_use) mma_commit(&a_empty[sl]);
                    }
                    __syncwarp();
                    ++n1;
                    if (++ch1 == nck) {
                        ch1 = 0;
                        if (amode || cs.last_of_item(g)) ++an;
                        cs.advance(g);
                    }
                }
            }
        }
    } else if (warp < 6) {
        // ------------------------------------------------ online softmax: thread = row j of the M tile
        const int quad = warp & 3;
        const int r = quad * 32 + lane;
        const uint32_t lane_off = (uint32_t)(quad * 32) << 16;
        const float sl2 = g.scale * kLog2e;
        const float thr = 8.f / sl2;   // lazy rescale threshold (raw logit units)
        int n = 0, task = 0;
        for (FlashCursor sc = cur; sc.valid; sc.advance(g), ++task) {
            float m = -1e30f, l = 0.f, A = 0.f;
            for (int ch = 0; ch < nck; ++ch, ++n) {
                const int st = n & 1;
                const uint32_t sbuf = tmem + kFS + st * 128 + lane_off;
                mbar_wait(&s_full[st], (n >> 1) & 1);
                tc_fence_after();
                const int kvalid = min(kFKC, g.s2 - ch * kFKC);
                float mx = -1e30f;
                float z[128];
                {   // the four 32-column loads in flight before one wait
                    uint32_t* zr = reinterpret_cast<uint32_t*>(z);
#pragma unroll
                    for (int q4 = 0; q4 < 4; ++q4) tmem_ld32_nw(sbuf + q4 * 32, zr + q4 * 32);
                    tmem_wait_ld();
                }
                if (kvalid < kFKC) {
#pragma unroll
                    for (int i = 0; i < kFKC; ++i) z[i] = i < kvalid ? z[i] : -1e30f;
                }
#pragma unroll
                for (int i = 0; i < kFKC; ++i) mx = fmaxf(mx, z[i]);
                float fac = 1.f;
                int need = 0;
                if (ch == 0) {
                    m = mx;
                } else if (mx > m + thr) {
                    fac = ex2((m - mx) * sl2);
                    m = mx;
                    need = 1;
                }
                l *= fac;
                A *= fac;
                if (__any_sync(0xffffffffu, need)) {
                    // rescale this warp's rows of O_aL / O_Y once MMA2(n - 1) has accumulated into them
                    mbar_wait(o_step, (n - 1) & 1);
                    tc_fence_after();
#pragma unroll 1
                    for (int part = 0; part < (want_y ? 8 : 4); ++part) {
                        float o[32];
                        const uint32_t oa = tmem + kFOA + part * 32 + lane_off;
                        tmem_ld32(oa, o);
#pragma unroll
                        for (int i = 0; i < 32; ++i) o[i] *= fac;
                        tmem_st32(oa, o);
                    }
                }
                const float mb = m * sl2;
                float lq[4] = {0.f, 0.f, 0.f, 0.f}, aq[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
                for (int hf = 0; hf < 2; ++hf) {   // 64 keys -> 32 packed columns at a time
                    uint32_t packed[32];
#pragma unroll
                    for (int i = 0; i < 64; i += 2) {
                        const int kk = hf * 64 + i;
                        const float p0 = ex2(fmaf(z[kk], sl2, -mb)), p1 = ex2(fmaf(z[kk + 1], sl2, -mb));
                        lq[(i >> 1) & 3] += p0 + p1;
                        aq[(i >> 1) & 3] = fmaf(p1, z[kk + 1], fmaf(p0, z[kk], aq[(i >> 1) & 3]));
                        packed[i >> 1] = pack_bf16(p0, p1);
                    }
                    tmem_st32(sbuf + hf * 32, reinterpret_cast<const float*>(packed));
                }
                l += (lq[0] + lq[1]) + (lq[2] + lq[3]);
                A += (aq[0] + aq[1]) + (aq[2] + aq[3]);
                tc_fence_before();
                mbar_arrive(&p_full[st]);
            }
            // per-row statistics of the task for the epilogue
            const int ss = task & 1;
            mbar_wait(&st_empty[ss], ((task >> 1) & 1) ^ 1);
            stats[(ss * 3 + 0) * 128 + r] = m;
            stats[(ss * 3 + 1) * 128 + r] = l;
            stats[(ss * 3 + 2) * 128 + r] = A;
            mbar_arrive(&st_full[ss]);
        }
    } else {
        // ------------------------------------------------ epilogue: thread = row j
        const int quad = warp & 3;
        const int r = quad * 32 + lane;
        const uint32_t lane_off = (uint32_t)(quad * 32) << 16;
        const uint64_t w_policy = (P.l2hint & 1) ? l2_evict_last() : l2_evict_normal();
        __nv_bfloat16* W = const_cast<__nv_bfloat16*>(P.w);
        const uint32_t stg = smem_u32(smem + RowFSmem::kStage + quad * 4096);
        const int64_t rstride = (int64_t)4 * g.nkeys * 64;   // bf16 elements between rows j, j + 1
        int task = 0;
        for (FlashCursor ec = cur; ec.valid; ec.advance(g), ++task) {
            const int ss = task & 1;
            mbar_wait(o_full, task & 1);
            mbar_wait(&st_full[ss], (task >> 1) & 1);
            tc_fence_after();
            const float m = stats[(ss * 3 + 0) * 128 + r], l = stats[(ss * 3 + 1) * 128 + r],
                        A = stats[(ss * 3 + 2) * 128 + r];
            mbar_arrive(&st_empty[ss]);
            const float inv_l = 1.f / l;
            const int j0 = ec.mt * kFKC;
            const int j = j0 + r;
            const int key = ec.c * g.s1 + ec.k;
            const int64_t col0 = (int64_t)(ec.bh * g.gq + ec.a) * g.s2 + j0 + quad * 32;   // this warp's first row
            const int nrows = min(32, g.s2 - (j0 + quad * 32));
            const int nparts = want_y ? 4 : 2;
#pragma unroll 1
            for (int part = 0; part < nparts; ++part) {
                float o[64];
                const uint32_t ob = tmem + (part < 2 ? kFOA : kFOY) + (part & 1) * 64 + lane_off;
                tmem_ld32(ob, o);
                tmem_ld32(ob + 32, o + 32);
                if (part == nparts - 1) {
                    tc_fence_before();
                    mbar_arrive(o_empty);   // O fully read: the next task's MMA2 may overwrite it
                }
                if (nrows <= 0 || (P.dbg & 1)) continue;
                // transpose through the warp's buffer: lane writes its row, then 4 rows per instruction
                const uint32_t srow = stg + lane * 128;
#pragma unroll
                for (int cc = 0; cc < 8; ++cc)
                    st_shared_v4(srow + ((cc ^ (lane & 7)) << 4), pack_bf16(o[8 * cc] * inv_l, o[8 * cc + 1] * inv_l),
                                 pack_bf16(o[8 * cc + 2] * inv_l, o[8 * cc + 3] * inv_l),
                                 pack_bf16(o[8 * cc + 4] * inv_l, o[8 * cc + 5] * inv_l),
                                 pack_bf16(o[8 * cc + 6] * inv_l, o[8 * cc + 7] * inv_l));
                __syncwarp();
                __nv_bfloat16* base = W + ((col0 * 4 + part) * g.nkeys + key) * 64;
                const int chn = lane & 7;
#pragma unroll
                for (int it = 0; it < 8; ++it) {
                    const int rr = it * 4 + (lane >> 3);
                    if (rr < nrows) {
                        const uint4 v4 = ld_shared_v4u(stg + rr * 128 + ((chn ^ (rr & 7)) << 4));
                        st_global_v4_hint(base + rr * rstride + chn * 8, v4.x, v4.y, v4.z, v4.w, w_policy);
                    }
                }
                __syncwarp();
            }
            if (j < g.s2) {   // c_L = sum R z - lse with z = scale * S (solver.py:191)
                const int64_t col = (int64_t)(ec.bh * g.gq + ec.a) * g.s2 + j;
                P.wc[col * ckey + key] = g.scale * (A * inv_l - m) - __logf(l);
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc<512>(tmem);
}
