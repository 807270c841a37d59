// Row stage, half-packed variant (included by mbx_tc.cu).  A 128-lane M tile of the
// classic row stage holds whole query tiles (s2 <= 64 rows each), so a plan with one
// (or an odd number of) query tiles leaves up to 60% of every softmax / epilogue pass
// idle.  Here a task is two independent M=64 "halves", each one (query tile qt, in-tile
// row k) combination of the same (b,h) and key tile c, with its own K/V row (c,k): the
// two MMAs' accumulators interleave in TMEM (M=64 row r -> lane 32 (r / 16) + r % 16,
// the second MMA at lane offset 16), so every 128-lane pass carries 2 s2 useful rows.
// Halves enumerate idx = k * G_q + qt; task pair p holds idx 2p, 2p+1, and halves with the
// same k share one K/V ring stage.  Per task:
//   MMA1  S_h = A_h . K_{c,k_h}^T     2 x (64 x 64 x 128)  A = Q (or hat_alpha_R) rows from smem
//   softmax over i: two warpgroups (warps 2-5 even tasks, 6-9 odd tasks) so one group's
//   TMEM load / store latency hides behind the other's arithmetic; c_L to the
//   workspace, P (bf16) back over S
//   MMA2  [aL | Y]_h = P_h . [K | V]_{c,k_h}   2 x 2 x (64 x 128 x 64), A = P in TMEM
//   epilogue: warps 10-13 (aL) / 14-17 (Y), per warp two 16-row TMA stores (one per half)
// (solver.py:187-191 R update and c_L; factors.py:123 Y = R V)
constexpr int kPKV = 5;   // K/V ring stages (one key row each), at most
#ifndef MBX_PAIR_SOFT_WG
#define MBX_PAIR_SOFT_WG 1
#endif
constexpr int kPairSoftWG = MBX_PAIR_SOFT_WG;        // softmax warpgroups (tasks alternate between them)
constexpr int kPSB = kPairSoftWG == 1 ? 3 : 4;       // S/P buffers: MMA1 runs up to kPSB tasks ahead of MMA2
constexpr int kPairEpi = 2 + 4 * kPairSoftWG;        // first epilogue warp
constexpr int kPairThreads = 32 * (kPairEpi + 8);
struct RowPSmem {
    static constexpr int kA = 0;                         // A slots [2] x [2 d-chunks][2 halves][64 rows][128 B]
    static constexpr int kASlot = 32768;
    static constexpr int kKV = 2 * kASlot;               // K/V rows [4] x [K c0 | K c1 | V c0 | V c1]
    // K/V ring: nkv stages of 4 chunks [K d0-63 | K d64-127 | V d0-63 | V d64-127], each
    // chunk ceil(s2 / 8) x 8 rows of 128 B (7 KB at s2 = 52: five stages; 8 KB: four),
    // then 1 KB of zeros that the last chunk's MMA reads of rows >= s2 may touch
    static constexpr int kKVRegion = 5 * 4 * 7168 + 1024;
    static constexpr int kStage = kKV + kKVRegion;       // per epilogue warp: [16 rows][128 B] transpose buffer
    static constexpr int kBars = kStage + 8 * 2048;
    static constexpr int kNumBars = 4 + 2 * kPKV + 2 * kPSB + 4;
    static constexpr int kTmemSlot = kBars + kNumBars * 8;
    static constexpr int kTotal = kTmemSlot + 16;
};
static_assert(RowPSmem::kTotal + 1024 <= 232448, "paired row stage exceeds 227 KB of shared memory");
// TMEM: S/P buffers [0,64) .. [192,256); O_aL [256,384); O_Y [384,512)
constexpr uint32_t kPS = 0, kPOA = 64 * kPSB, kPOY = kPOA + 128;

// Task walker: tasks (bh, p, c) in order, a contiguous range per CTA; item = (bh, p).
// Half h of pair p is idx = 2p + h = k * G_q + qt (valid while idx < G_q * s1).
struct PairCursor {
    int t, t1, bh, kp, c, n_kp, gk, gq, nidx;
    int k0, q0, k1, q1;       // (row, query tile) of the two halves
    int kvi, kst, kph;        // K/V ring position of this task's first row
    int nkv;                  // K/V ring stages
    bool valid;
    __device__ __forceinline__ void halves() {
        k0 = (2 * kp) / gq;
        q0 = 2 * kp - k0 * gq;
        q1 = q0 + 1;
        k1 = k0;
        if (q1 == gq) {
            q1 = 0;
            ++k1;
        }
    }
    __device__ __forceinline__ void init(const Geometry& g, int cta, int ctas, int stages) {
        nkv = stages;
        gq = g.gq;
        nidx = g.gq * g.s1;
        n_kp = (nidx + 1) / 2;
        gk = g.gk;
        const long long tasks = (long long)g.bh * n_kp * g.gk;
        t = (int)(tasks * cta / ctas);
        t1 = (int)(tasks * (cta + 1) / ctas);
        c = t % gk;
        kp = (t / gk) % n_kp;
        bh = t / (gk * n_kp);
        halves();
        kvi = kst = kph = 0;
        valid = t < t1;
    }
    __device__ __forceinline__ int nh() const { return 2 * kp + 1 < nidx ? 2 : 1; }   // valid halves
    __device__ __forceinline__ int nrows() const { return nh() == 2 && k1 != k0 ? 2 : 1; }   // distinct K/V rows
    __device__ __forceinline__ int kr(int hh) const { return hh ? k1 : k0; }
    __device__ __forceinline__ int qt(int hh) const { return hh ? q1 : q0; }
    __device__ __forceinline__ bool first_of_item(int t0) const { return c == 0 || t == t0; }
    __device__ __forceinline__ bool last_of_item() const { return c == gk - 1 || t == t1 - 1; }
    __device__ __forceinline__ void advance() {
        for (int h = nrows(); h > 0; --h) {
            ++kvi;
            if (++kst == nkv) {
                kst = 0;
                kph ^= 1;
            }
        }
        ++t;
        valid = t < t1;
        if (++c == gk) {
            c = 0;
            if (++kp == n_kp) {
                kp = 0;
                ++bh;
            }
            halves();
        }
    }
};

__global__ void __launch_bounds__(kPairThreads, 1)
tc_row_pair(const __grid_constant__ TcParams P, Geometry g, int amode_i, int want_y_i) {
    const bool amode = amode_i != 0, want_y = want_y_i != 0;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + RowPSmem::kBars);
    uint64_t* a_full = bars;                       // [2] A slot landed (Q per item, hat_alpha_R per task)
    uint64_t* a_empty = bars + 2;                  // [2] MMA1s done with it
    uint64_t* kv_full = bars + 4;                  // [nkv]
    uint64_t* kv_empty = kv_full + kPKV;           // [nkv]
    uint64_t* s_full = kv_empty + kPKV;            // [kPSB]
    uint64_t* p_full = s_full + kPSB;              // [kPSB]
    uint64_t* o_full = p_full + kPSB;              // [2]
    uint64_t* o_empty = o_full + 2;                // [2]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + RowPSmem::kTmemSlot);
    const int tid = threadIdx.x, lane = tid & 31;
    const int warp = __shfl_sync(0xffffffffu, tid >> 5, 0);
    const uint32_t box_bytes = (uint32_t)g.s2 * 128u;
    const int cpitch = ((g.s2 + 7) / 8) * 1024;              // K/V chunk pitch (rows rounded to 8)
    const int nkv = cpitch <= 7168 ? 5 : 4;                  // stages that fit the ring region
    const int kvbytes = 4 * cpitch;
    const int ckey = ckey_stride(g);
    SPAN_AT(0, 0);

    if (tid == 0) {
        tma_prefetch(&P.tq);
        tma_prefetch(&P.tk);
        tma_prefetch(&P.tv);
        for (int i = 0; i < 2; ++i) {
            mbar_init(&a_full[i], 1);
            mbar_init(&a_empty[i], 1);
            mbar_init(&o_full[i], 1);
            mbar_init(&o_empty[i], 128);
        }
        for (int i = 0; i < kPSB; ++i) {
            mbar_init(&s_full[i], 1);
            mbar_init(&p_full[i], 128);
        }
        for (int i = 0; i < nkv; ++i) {
            mbar_init(&kv_full[i], 1);
            mbar_init(&kv_empty[i], 1);
        }
        fence_barrier_init();
    }
    // K/V rows s2..63 and A rows s2..63 are never written by TMA: MMA2 multiplies K/V
    // padding by P = 0 (must be finite); A padding only feeds rows that are never stored.
    for (int i = tid; i < RowPSmem::kKVRegion / 16; i += blockDim.x)
        reinterpret_cast<uint4*>(smem + RowPSmem::kKV)[i] = make_uint4(0, 0, 0, 0);
    if (warp == 0) tmem_alloc<512>(tmem_slot);
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    pdl_wait();      // predecessor kernels complete and visible
    pdl_trigger();   // only then may dependents start (they read q before their own wait)

    PairCursor cur;
    cur.init(g, blockIdx.x, gridDim.x, nkv);
    const int t0 = cur.t;
    int ti = 0;   // trace event index (MBX_TRACE builds)

    if (warp == 0) {
        // ------------------------------------------------ TMA producer (whole warp, elected lane issues)
        const bool leader = elect_one();
        // A slot of (item or task) n: the halves' Q rows (per item) or hat_alpha_R rows (per task)
        int an = 0;
        auto load_a = [&](const PairCursor& pc) {
            const int sl = an & 1;
            mbar_wait(&a_empty[sl], ((an >> 1) & 1) ^ 1);
            const int b = pc.bh / g.heads, h = pc.bh % g.heads, nh = pc.nh();
            if (leader) {
                mbar_expect_tx(&a_full[sl], 2u * box_bytes * (uint32_t)nh);
                uint8_t* ab = smem + RowPSmem::kA + sl * RowPSmem::kASlot;
                for (int hh = 0; hh < nh; ++hh) {
                    const int kr = pc.kr(hh), qt = pc.qt(hh);
                    if (amode) {
                        const int key = pc.c * g.s1 + kr, ag = pc.bh * g.gq + qt;
                        tma_load_4d(ab + hh * 8192, &P.tar_ld, &a_full[sl], 0, 0, key, ag);
                        tma_load_4d(ab + 16384 + hh * 8192, &P.tar_ld, &a_full[sl], 64, 0, key, ag);
                    } else {
                        const int tok = (int)row_base(g, true, qt, kr);
                        tma_load_4d(ab + hh * 8192, &P.tq, &a_full[sl], 0, tok, h, b);
                        tma_load_4d(ab + 16384 + hh * 8192, &P.tq, &a_full[sl], 64, tok, h, b);
                    }
                }
            }
            __syncwarp();
            ++an;
        };
        PairCursor pc = cur;
        while (pc.valid) {
            const int b = pc.bh / g.heads, h = pc.bh % g.heads;
            int kvi = pc.kvi, kst = pc.kst, kph = pc.kph;
            for (int r = 0; r < pc.nrows(); ++r) {
                mbar_wait(&kv_empty[kst], kph ^ 1);
                // dbg 8 (timing only): every K/V load reads the same (L2-resident) row
                const int tok = (P.dbg & 8) ? 0 : (int)row_base(g, false, pc.c, pc.kr(r));
                if (leader) {
                    mbar_expect_tx(&kv_full[kst], (want_y ? 4u : 2u) * box_bytes);   // V only for Y
                    uint8_t* kb = smem + RowPSmem::kKV + kst * kvbytes;
                    tma_load_4d(kb, &P.tk, &kv_full[kst], 0, tok, h, b);
                    tma_load_4d(kb + cpitch, &P.tk, &kv_full[kst], 64, tok, h, b);
                    if (want_y) {
                        tma_load_4d(kb + 2 * cpitch, &P.tv, &kv_full[kst], 0, tok, h, b);
                        tma_load_4d(kb + 3 * cpitch, &P.tv, &kv_full[kst], 64, tok, h, b);
                    }
                }
                if (leader) TR(0, ti, 2);
                __syncwarp();
                ++kvi;
                if (++kst == nkv) {
                    kst = 0;
                    kph ^= 1;
                }
            }
            // the task's K/V rows go out before its A rows: an A issue can block ~1 us (C2 -1 %)
            if (amode || pc.first_of_item(t0)) {
                load_a(pc);
                if (leader) TR(0, ti, 1);
            }
            pc.advance();
        }
    } else if (warp == 1) {
        // ------------------------------------------------ MMA issuer (whole warp, uniform descriptors)
        const bool leader = elect_one();
        const uint32_t id1 = idesc_bf16(64, 64, false, false);
        const uint32_t id2 = idesc_bf16(64, 128, false, true);
        const uint32_t id1w = idesc_bf16(128, 64, false, false);    // shared-row tasks: one M=128 MMA
        const uint32_t id2w = idesc_bf16(128, 128, false, true);
        constexpr uint32_t kHi = (1024u >> 4) | (1u << 14) | (2u << 29);
        auto desc = [](uint32_t lo) { return ((uint64_t)kHi << 32) | lo; };
        const uint32_t a_lo = ((smem_u32(smem + RowPSmem::kA) & 0x3FFFF) >> 4) | (1u << 16);
        const uint32_t kv_lo = (smem_u32(smem + RowPSmem::kKV) & 0x3FFFF) >> 4;
        PairCursor cs = cur, co = cur;
        int ts = 0, to = 0, an_s = 0;   // an_s: A slot uses consumed by MMA1
        int sb_s = 0, sph_s = 0, sb_o = 0, sph_o = 0;   // S/P buffer + phase of task ts / to
        while (cs.valid || co.valid) {
            // MMA2(to): softmax done with S/P buffer to%2, O buffers drained by task to-1
            if (co.valid && to < ts && mbar_test_uniform(&p_full[sb_o], sph_o) &&
                mbar_test_uniform(&o_empty[0], (to & 1) ^ 1) &&
                (!want_y || mbar_test_uniform(&o_empty[1], (to & 1) ^ 1))) {
                if (leader) TR(1, ti, 13);
                tc_fence_after();
                if (leader) {
                    const int two = co.nrows() == 2;
                    const bool wide = co.nh() == 2 && !two;   // both halves on one K/V row: M=128
                    const int nm = wide ? 1 : co.nh();
                    const uint32_t id = wide ? id2w : id2;
                    for (int hh = 0; hh < nm; ++hh) {
                        int kst = co.kst + (hh & two);
                        if (kst >= nkv) kst -= nkv;
                        const uint32_t lane_h = (uint32_t)(hh * 16) << 16;
                        // MN-major B: the two 64-wide d chunks of K (or V) are LBO = cpitch apart
                        const uint32_t b_lo = kv_lo + (uint32_t)((kst * kvbytes) >> 4) + ((uint32_t)(cpitch >> 4) << 16);
                        const uint32_t pa = tmem + kPS + sb_o * 64 + lane_h;
                        for (int s = 0; s < (want_y ? 2 : 1); ++s) {
#pragma unroll
                            for (int kk = 0; kk < 4; ++kk)
                                mma_bf16_ts(tmem + (s ? kPOY : kPOA) + lane_h, pa + kk * 8,
                                            desc(b_lo + ((s * 2 * cpitch + kk * 2048) >> 4)), id, kk > 0);
                        }
                        if (hh == nm - 1 || two) mma_commit(&kv_empty[kst]);
                    }
                    mma_commit(&o_full[0]);
                    if (want_y) mma_commit(&o_full[1]);
                    TR(1, ti, 12);
                }
                __syncwarp();
                co.advance();
                ++to;
                if (++sb_o == kPSB) {
                    sb_o = 0;
                    sph_o ^= 1;
                }
            }
            // MMA1(ts): S/P buffer ts%2 released by MMA2(ts-2), A slot and K/V rows landed
            if (cs.valid && ts < to + kPSB) {
                const int sl = an_s & 1;
                bool ready = mbar_test_uniform(&a_full[sl], (an_s >> 1) & 1);
                int kst = cs.kst, kph = cs.kph;
                for (int r = 0; r < cs.nrows() && ready; ++r) {
                    ready = mbar_test_uniform(&kv_full[kst], kph);
                    if (++kst == nkv) {
                        kst = 0;
                        kph ^= 1;
                    }
                }
                if (ready) {
                    if (leader) TR(1, ti, 10);
                    tc_fence_after();
                    const bool last_use = amode || cs.last_of_item();
                    if (leader) {
                        const int two = cs.nrows() == 2;
                        const bool wide = cs.nh() == 2 && !two;   // rows of both halves stacked: M=128
                        const int nm = wide ? 1 : cs.nh();
                        const uint32_t id = wide ? id1w : id1;
                        for (int hh = 0; hh < nm; ++hh) {
                            int ks = cs.kst + (hh & two);
                            if (ks >= nkv) ks -= nkv;
                            const uint32_t aa = a_lo + (uint32_t)sl * (RowPSmem::kASlot >> 4) + ((hh * 8192) >> 4);
                            const uint32_t b_lo = kv_lo + (uint32_t)((ks * kvbytes) >> 4) + (1u << 16);
                            const uint32_t d = tmem + kPS + sb_s * 64 + ((uint32_t)(hh * 16) << 16);
#pragma unroll
                            for (int kk = 0; kk < 8; ++kk)
                                mma_bf16(d, desc(aa + (((kk >> 2) * 16384 + (kk & 3) * 32) >> 4)),
                                         desc(b_lo + (((kk >> 2) * cpitch + (kk & 3) * 32) >> 4)), id, kk > 0);
                        }
                        mma_commit(&s_full[sb_s]);
                        if (last_use) mma_commit(&a_empty[sl]);
                        TR(1, ti, 11);
                    }
                    __syncwarp();
                    if (last_use) ++an_s;
                    cs.advance();
                    ++ts;
                    if (++sb_s == kPSB) {
                        sb_s = 0;
                        sph_s ^= 1;
                    }
                }
            }
        }
    } else if (warp < kPairEpi) {
        // ------------------------------------------------ softmax: lane = (half h, row j); tasks alternate
        const int wg = (warp - 2) >> 2;       // between the warpgroups: t % kPairSoftWG == wg
        const int quad = warp & 3;
        const uint32_t lane_off = (uint32_t)(quad * 32) << 16;
        const float sl2 = g.scale * kLog2e;
        int bsel = 0, bph = 0;   // S/P buffer + phase of task t
        for (int t = 0; cur.valid; ++t, cur.advance()) {
            if (t % kPairSoftWG == wg) {
                const uint32_t sbuf = tmem + kPS + bsel * 64 + lane_off;
                // M=64 pair: lane = (half lane/16, row 16 quad + lane%16); shared-row M=128: (quad/2, 32 (quad%2) + lane)
                const bool wide = cur.nh() == 2 && cur.nrows() == 1;
                const int hh = wide ? quad >> 1 : lane >> 4;
                const int j = wide ? 32 * (quad & 1) + lane : quad * 16 + (lane & 15);
                const int kr = cur.kr(hh), qt = cur.qt(hh);
                const bool row_ok = j < g.s2 && hh < cur.nh();
                mbar_wait(&s_full[bsel], bph);
                if (lane == 0) TR(warp, ti, 21);
                tc_fence_after();
                float z[64];
                {
                    uint32_t zr[64];
                    tmem_ld32_nw(sbuf, zr);
                    tmem_ld32_nw(sbuf + 32, zr + 32);
                    tmem_wait_ld();
#pragma unroll
                    for (int i = 0; i < 64; ++i) z[i] = __uint_as_float(zr[i]);
                }
#pragma unroll
                for (int blk = 0; blk < 4; ++blk) {   // only the 16-column blocks that reach past s2
                    if (16 * blk + 16 > g.s2) {
#pragma unroll
                        for (int i = 16 * blk; i < 16 * blk + 16; ++i) z[i] = i < g.s2 ? z[i] : -1e30f;
                    }
                }
                float mq[8];
#pragma unroll
                for (int e = 0; e < 8; ++e) mq[e] = fmaxf(z[e], z[e + 8]);
#pragma unroll
                for (int i = 16; i < 64; i += 8)
#pragma unroll
                    for (int e = 0; e < 8; ++e) mq[e] = fmaxf(mq[e], z[i + e]);
                const float m = fmaxf(fmaxf(fmaxf(mq[0], mq[1]), fmaxf(mq[2], mq[3])),
                                      fmaxf(fmaxf(mq[4], mq[5]), fmaxf(mq[6], mq[7])));
                const float mb = m * sl2;
                // p overwrites z once its z term is in the partial sums (register pressure: 18 warps)
                float lq[8], aq[8];
#pragma unroll
                for (int e = 0; e < 8; ++e) {
                    lq[e] = 0.f;
                    aq[e] = 0.f;
                }
#pragma unroll
                for (int i = 0; i < 64; i += 8)
#pragma unroll
                    for (int e = 0; e < 8; ++e) {
                        const float pe = ex2(fmaf(z[i + e], sl2, -mb));
                        lq[e] += pe;
                        aq[e] = fmaf(pe, z[i + e], aq[e]);
                        z[i + e] = pe;
                    }
                const float l = ((lq[0] + lq[1]) + (lq[2] + lq[3])) + ((lq[4] + lq[5]) + (lq[6] + lq[7]));
                const float A = ((aq[0] + aq[1]) + (aq[2] + aq[3])) + ((aq[4] + aq[5]) + (aq[6] + aq[7]));
                const float inv_l = 1.f / l;
                const float pscale = row_ok ? inv_l : 0.f;
                uint32_t packed[32];
#pragma unroll
                for (int i = 0; i < 64; i += 2) packed[i >> 1] = pack_bf16(z[i] * pscale, z[i + 1] * pscale);
                tmem_st32(sbuf, reinterpret_cast<const float*>(packed));
                tc_fence_before();
                mbar_arrive(&p_full[bsel]);
                if (lane == 0) TR(warp, ti, 22);
                if (P.rfac && row_ok)   // R' row (final, or this refinement's slice) [bh][a][c][k][j][:] (factors.py:57-79)
                    store_r_row(P.rfac + ((((int64_t)(cur.bh * g.gq + qt) * g.gk + cur.c) * g.s1 + kr) * g.s2 + j) * g.s2,
                                z, inv_l, g.s2);
                if (row_ok) {   // c_L = sum R z - lse with z = scale * S (solver.py:191)
                    const int col = (cur.bh * g.gq + qt) * g.s2 + j;
                    P.wc[(int64_t)col * ckey + cur.c * g.s1 + kr] = g.scale * (A * inv_l - m) - __logf(l);
                }
            }
            if (++bsel == kPSB) {
                bsel = 0;
                bph ^= 1;
            }
        }
    } else {
        // ------------------------------------------------ epilogue: 4 warps O_aL, 4 warps O_Y
        // Each lane owns one row (TMEM lane) and writes its 128 contiguous bytes per part straight
        // from registers (st.global.v4 with the L2 evict_last policy): no staging round trips.
        const int set = warp >= kPairEpi + 4 ? 1 : 0;
        if (set == 1 && !want_y) cur.valid = false;
        // the column stage reads W right after this launch: keep it in L2 ahead of q / k / v
        const uint64_t w_policy = (P.l2hint & 1) ? l2_evict_last() : l2_evict_normal();
        const int quad = warp & 3;
        const uint32_t lane_off = (uint32_t)(quad * 32) << 16;
        const uint32_t obuf = tmem + (set ? kPOY : kPOA) + lane_off;
        __nv_bfloat16* W = const_cast<__nv_bfloat16*>(P.w);
        for (int t = 0; cur.valid; ++t, cur.advance()) {
            const bool wide = cur.nh() == 2 && cur.nrows() == 1;
            mbar_wait(&o_full[set], t & 1);
            if (lane == 0) TR(warp, ti, 31);
            tc_fence_after();
            uint32_t pk[2][32];
            if (P.dbg & 2) {   // timing experiment: O released undrained (wrong results)
#pragma unroll
                for (int i = 0; i < 32; ++i) pk[0][i] = pk[1][i] = 0u;
            } else {
                uint32_t o[2][32];
                tmem_ld32_nw(obuf, o[0]);
                tmem_ld32_nw(obuf + 32, o[1]);
                tmem_wait_ld();
#pragma unroll
                for (int q2 = 0; q2 < 2; ++q2)
#pragma unroll
                    for (int i = 0; i < 16; ++i)
                        pk[0][q2 * 16 + i] = pack_bf16(__uint_as_float(o[q2][2 * i]), __uint_as_float(o[q2][2 * i + 1]));
                tmem_ld32_nw(obuf + 64, o[0]);
                tmem_ld32_nw(obuf + 96, o[1]);
                tmem_wait_ld();
#pragma unroll
                for (int q2 = 0; q2 < 2; ++q2)
#pragma unroll
                    for (int i = 0; i < 16; ++i)
                        pk[1][q2 * 16 + i] = pack_bf16(__uint_as_float(o[q2][2 * i]), __uint_as_float(o[q2][2 * i + 1]));
            }
            tc_fence_before();
            mbar_arrive(&o_empty[set]);
            if (lane == 0) TR(warp, ti, 32);
            if (!(P.dbg & 1)) {   // dbg 1: timing experiment without the workspace stores
                // 16 rows at a time through the warp's 2 KB buffer: each lane writes its row (swizzled
                // 16-byte chunks), then every instruction stores 4 whole 128-byte rows (coalesced
                // st.global.v4, L2 evict_last) -- no bulk-copy round trips between the groups.
                const uint32_t stg = smem_u32(smem + RowPSmem::kStage + (warp - kPairEpi) * 2048);
                const int nh = cur.nh();
                const int64_t rstride = (int64_t)4 * g.nkeys * 64;   // bf16 elements between rows j, j + 1
#pragma unroll
                for (int sub = 0; sub < 2; ++sub) {
                    const int hs = wide ? quad >> 1 : sub;
                    const int j0 = wide ? 32 * (quad & 1) + 16 * sub : quad * 16;
                    const int nrows = hs < nh ? min(16, g.s2 - j0) : 0;
                    if (nrows <= 0) continue;
                    const int64_t col0 = (int64_t)(cur.bh * g.gq + cur.qt(hs)) * g.s2 + j0;
                    const int key = cur.c * g.s1 + cur.kr(hs);
#pragma unroll
                    for (int part = 0; part < 2; ++part) {
                        if ((lane >> 4) == sub) {
                            const uint32_t srow = stg + (lane & 15) * 128;
#pragma unroll
                            for (int cc = 0; cc < 8; ++cc)
                                st_shared_v4(srow + ((cc ^ (lane & 7)) << 4), pk[part][4 * cc], pk[part][4 * cc + 1],
                                             pk[part][4 * cc + 2], pk[part][4 * cc + 3]);
                        }
                        __syncwarp();
                        __nv_bfloat16* base = W + ((col0 * 4 + 2 * set + part) * g.nkeys + key) * 64;
                        const int ch = lane & 7;
#pragma unroll
                        for (int it = 0; it < 4; ++it) {
                            const int r = it * 4 + (lane >> 3);
                            if (r < nrows) {
                                const uint4 v4 = ld_shared_v4u(stg + r * 128 + ((ch ^ (r & 7)) << 4));
                                st_global_v4_hint(base + r * rstride + ch * 8, v4.x, v4.y, v4.z, v4.w, w_policy);
                            }
                        }
                        __syncwarp();
                    }
                }
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc<512>(tmem);
    SPAN_AT(0, 1);
}
