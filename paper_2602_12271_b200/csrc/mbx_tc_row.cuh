// Row stage (included by mbx_tc.cu).
//
// Item = (b, h, in-tile row k, query group qg): the Q rows k of up to three query
// tiles 3qg.. are copied (tcgen05.cp) from a smem staging tile into TMEM, where
// they are the A operand of every MMA1 of the item; the K/V rows k of the item's
// key tiles c stream through a 3-stage TMA ring and each serves the item's one or
// two M tiles (tiles 3qg,3qg+1 | 3qg+2).  Per task (key tile c, M tile mt):
//   MMA1  S[(a,j), i] = Q_k . K_ck^T        128 x 64 x 128  (A: TMEM, B: smem) -> S/P buffer t%2
//   softmax_i (warps 2-5, one query row per thread), c_L = sum R z - lse straight to the
//   workspace, R = p / l written back over S as packed bf16 P (tcgen05.st)
//   MMA2a aL = P . K_ck                     128 x 128 x 64  (A = P in TMEM)  -> O_aL
//   MMA2b Y  = P . V_ck                     128 x 128 x 64                   -> O_Y
//   epilogue: warps 6-9 drain O_aL, warps 10-13 drain O_Y: TMEM -> bf16 -> per-warp
//   SW128 staging -> TMA store into the blocked workspace W[col][part][key][64]
//   (part 0,1 = aL halves, 2,3 = Y halves).
// The MMA warp issues MMA1 and MMA2 in readiness order from two independent
// cursors, so the tensor pipe never idles behind one stage's wait.
// (solver.py:187-191 R update and c_L; factors.py:123 Y = R V; tensorops.py:268-272)
constexpr int kRowThreads = 448;   // 14 warps
constexpr int kQG = 3;             // query tiles per item
constexpr int kKVStages = 3;
struct RowSmem {
    // Q staging (48 KB): [d-chunk 2][query tile 3][64 rows][128 B], SW128 (tcgen05.cp source)
    static constexpr int kQ = 0;
    static constexpr int kQChunk = kQG * 8192;
    static constexpr int kQBytes = 2 * kQChunk;
    // refinements t >= 1: A ring of two [2 d-chunks][128 rows][128 B] tiles (hat_alpha_R rows) in the same region
    static constexpr int kASlot = 32768;
    static constexpr int kQRegion = 2 * kASlot;
    static constexpr int kKV = kQRegion;              // KV[3]: [K c0 | K c1 | V c0 | V c1] 8 KB each
    static constexpr int kKVBytes = 32768;
    static constexpr int kStage = kKV + kKVStages * kKVBytes;   // staging [8 warps][2] x [32][64] bf16
    static constexpr int kBars = kStage + 16 * 4096;
    static constexpr int kNumBars = 6 + 2 * kKVStages + 2 + 2 + 4 + 4;
    static constexpr int kTmemSlot = kBars + kNumBars * 8;
    static constexpr int kTotal = kTmemSlot + 16;
};
static_assert(RowSmem::kTotal + 1024 <= 232448, "row stage exceeds 227 KB of shared memory");

// TMEM columns: Q M tiles [0,64) [64,128); S/P buffers [128,192) [192,256); O_aL [256,384); O_Y [384,512).
constexpr uint32_t kRowQ = 0, kRowS = 128, kRowO = 256;

// Walks the (item, key tile c, M tile mt) task sequence of one CTA: a contiguous
// range [L0, L1) of key rows, items ordered (b*h, query group qg, row k), equal
// key-row counts per CTA, the item's Q reloaded only at item boundaries.
struct RowCursor {
    int li, c, mt, kvi, n_mt, nt, bh, kr, qg, cc, c0, c1, unit, my_items, first, stride, n_qg, n_cc, cpi;
    int L0, L1;   // range schedule (stride == 0)
    int kst, kph; // K/V ring stage (kvi % kKVStages) and its phase parity, kept incrementally
    bool valid;
    __device__ __forceinline__ void load(const Geometry& g) {
        valid = li < my_items;
        if (!valid) return;
        const int item = stride ? first + li * stride : L0 / cpi + li;
        kr = item % g.s1;
        unit = item / g.s1;
        cc = unit % n_cc;
        qg = (unit / n_cc) % n_qg;
        bh = unit / (n_cc * n_qg);
        nt = min(kQG, g.gq - kQG * qg);
        n_mt = (nt + 1) >> 1;
        c0 = cc * cpi;
        c1 = min(g.gk, c0 + cpi);
        if (!stride) {
            if (li == 0) c0 = L0 % cpi;
            if (li == my_items - 1) c1 = (L1 - 1) % cpi + 1;
        }
        c = c0;
    }
    // Range schedule: CTA `cta` of `ctas` takes an equal share of all key rows.
    __device__ __forceinline__ void init_range(const Geometry& g, int cta, int ctas) {
        stride = 0;
        first = 0;
        n_qg = row_groups(g);
        cpi = g.gk;
        n_cc = 1;
        const long long rows = (long long)g.bh * n_qg * g.s1 * g.gk;
        L0 = (int)(rows * cta / ctas);
        L1 = (int)(rows * (cta + 1) / ctas);
        my_items = L1 > L0 ? (L1 - 1) / cpi - L0 / cpi + 1 : 0;
        li = mt = kvi = kst = kph = 0;
        load(g);
    }
    __device__ __forceinline__ bool last_mt() const { return mt == n_mt - 1; }
    __device__ __forceinline__ bool last_of_item() const { return last_mt() && c == c1 - 1; }
    __device__ __forceinline__ void advance(const Geometry& g) {
        if (++mt < n_mt) return;
        mt = 0;
        ++kvi;
        if (++kst == kKVStages) {
            kst = 0;
            kph ^= 1;
        }
        if (++c < c1) return;
        ++li;
        if (stride) {
            load(g);
            return;
        }
        // range schedule: items are consecutive, so decode incrementally (no divisions on
        // the issue path): item = ((bh * n_qg + qg) * n_cc + cc) * s1 + kr with n_cc = 1
        valid = li < my_items;
        if (!valid) return;
        if (++kr == g.s1) {
            kr = 0;
            ++unit;
            if (++qg == n_qg) {
                qg = 0;
                ++bh;
            }
            nt = min(kQG, g.gq - kQG * qg);
            n_mt = (nt + 1) >> 1;
        }
        c0 = 0;
        c1 = li == my_items - 1 ? (L1 - 1) % cpi + 1 : g.gk;
        c = 0;
    }
};

__device__ __forceinline__ void tma_store_4d(const CUtensorMap* map, const void* src, int c0, int c1, int c2, int c3) {
    asm volatile("cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%2, %3, %4, %5}], [%1];" ::"l"(
                     reinterpret_cast<uint64_t>(map)),
                 "r"(smem_u32(src)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
                 : "memory");
}
__device__ __forceinline__ void tma_store_4d_hint(const CUtensorMap* map, const void* src, int c0, int c1, int c2,
                                                  int c3, uint64_t policy) {
    asm volatile(
        "cp.async.bulk.tensor.4d.global.shared::cta.bulk_group.L2::cache_hint [%0, {%2, %3, %4, %5}], [%1], %6;" ::"l"(
            reinterpret_cast<uint64_t>(map)),
        "r"(smem_u32(src)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "l"(policy)
        : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait() { asm volatile("cp.async.bulk.wait_group %0;" ::"n"(N) : "memory"); }

// D[tmem] (+)= A[tmem] * B[smem]; issued by ONE thread.
__device__ __forceinline__ void mma_bf16_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                            bool accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
        "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"((uint32_t)accumulate));
}

__device__ __forceinline__ void tmem_cp_128x256b(uint32_t taddr, uint64_t sdesc) {
    asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;" ::"r"(taddr), "l"(sdesc));
}

// Row-stage role of CTA `first` among `stride` row CTAs (contiguous key-row ranges).
// amode: MMA1's A rows come from hat_alpha_R of the previous refinement (per task,
// smem) instead of Q (per item, TMEM); want_y: compute Y = R V (last refinement only).
__device__ __forceinline__ void row_role(uint8_t* smem, const TcParams& P, const Geometry& g, int first, int stride,
                                         bool amode = false, bool want_y = true) {
    const CUtensorMap& tm_q = P.tq;
    const CUtensorMap& tm_k = P.tk;
    const CUtensorMap& tm_v = P.tv;
    const CUtensorMap& tm_wst = P.tws;
    const CUtensorMap& tm_wst_b = P.tws_b;
    float* __restrict__ Wc = P.wc;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + RowSmem::kBars);
    uint64_t* q_full = bars + 0;                  // [3] Q staging slot landed
    uint64_t* q_empty = bars + 3;                 // [3] Q staging slot copied into TMEM
    uint64_t* kv_full = bars + 6;                 // [3]
    uint64_t* kv_empty = kv_full + kKVStages;     // [3]
    uint64_t* s_full = kv_empty + kKVStages;      // [2]
    uint64_t* p_full = s_full + 2;                // [2]
    uint64_t* o_full = p_full + 2;                // [2] O_aL / O_Y written
    uint64_t* o_empty = o_full + 2;               // [2] O_aL / O_Y drained
    uint64_t* a_full = o_empty + 2;               // [2] amode: A tile of task landed
    uint64_t* a_empty = a_full + 2;               // [2] amode: MMA1 done with it
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + RowSmem::kTmemSlot);
    const int tid = threadIdx.x, lane = tid & 31;
    const int warp = __shfl_sync(0xffffffffu, tid >> 5, 0);   // provably warp-uniform

    const uint32_t box_bytes = (uint32_t)g.s2 * 128u;
    const int ckey = ckey_stride(g);
    // Q staging: slots of [2 d-chunks][nt_max tiles][64 rows][128 B]; with one query tile per
    // item (the (3h,w) / untiled plans) three slots let Q loads run two items ahead
    const int nt_max = g.gq < kQG ? g.gq : kQG;
    const int qchunk = nt_max * 8192;
    const int nqs = kQG / nt_max;

    if (tid == 0) {
        tma_prefetch(&tm_q);
        tma_prefetch(&tm_k);
        tma_prefetch(&tm_v);
        tma_prefetch(&tm_wst);
        tma_prefetch(&tm_wst_b);
        for (int i = 0; i < 3; ++i) {
            mbar_init(&q_full[i], 1);
            mbar_init(&q_empty[i], 1);
        }
        for (int i = 0; i < kKVStages; ++i) {
            mbar_init(&kv_full[i], 1);
            mbar_init(&kv_empty[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&s_full[i], 1);
            mbar_init(&p_full[i], 128);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&o_full[i], 1);
            mbar_init(&o_empty[i], 128);
            mbar_init(&a_full[i], 1);
            mbar_init(&a_empty[i], 1);
        }
        fence_barrier_init();
    }
    // Rows s2..63 of the K/V slots are never written by TMA; MMA2 multiplies them by
    // P = 0, so they must be finite: zero them once.
    for (int i = tid; i < kKVStages * RowSmem::kKVBytes / 16; i += kRowThreads)
        reinterpret_cast<uint4*>(smem + RowSmem::kKV)[i] = make_uint4(0, 0, 0, 0);
    if (warp == 0) tmem_alloc<512>(tmem_slot);
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    pdl_wait();      // predecessor kernels (previous stage) complete and visible
    pdl_trigger();   // only then may dependents start (they read q before their own wait)

#define WAITX(bar, par) do { if (P.dbg & 64) mbar_spin(bar, par); else if (P.dbg & 128) mbar_wait_nohint(bar, par); else mbar_wait(bar, par); } while (0)
    RowCursor cur;
    cur.init_range(g, first, stride);

    if (warp == 0) {
        // ------------------------------------------------------ TMA producer
        // whole warp on warp-uniform state (TMA coordinates in uniform registers), the
        // elected lane issues
        {
            const bool leader = elect_one();
            int ti = 0, kvi = 0;
            // Q rows of item li into the staging tile (free once the previous item's Q was copied)
            auto load_q = [&](int li) {
                RowCursor qc = cur;
                qc.li = li;
                qc.load(g);
                const int b = qc.bh / g.heads, h = qc.bh % g.heads;
                const int sl = li % nqs;
                WAITX(&q_empty[sl], ((li / nqs) & 1) ^ 1);
                if (leader) {
                    TR(0, ti, 1);
                    mbar_expect_tx(&q_full[sl], 2u * box_bytes * (uint32_t)qc.nt);
                    uint8_t* qb = smem + RowSmem::kQ + sl * 2 * qchunk;
                    for (int la = 0; la < qc.nt; ++la) {
                        const int tok = (int)row_base(g, true, kQG * qc.qg + la, qc.kr);
                        tma_load_4d(qb + la * 8192, &tm_q, &q_full[sl], 0, tok, h, b);
                        tma_load_4d(qb + qchunk + la * 8192, &tm_q, &q_full[sl], 64, tok, h, b);
                    }
                }
                __syncwarp();
            };
            int ta = 0;   // amode: tasks whose A tile was issued
            // amode: A tile of task (key tile c, M tile mt) = hat_alpha_R rows j of tiles 2mt, 2mt+1
            auto load_a = [&](int c, int mt) {
                const int sl = ta & 1;
                WAITX(&a_empty[sl], ((ta >> 1) & 1) ^ 1);
                const int nla = min(2, cur.nt - 2 * mt);
                if (leader) {
                    mbar_expect_tx(&a_full[sl], 2u * box_bytes * (uint32_t)nla);
                    uint8_t* ab = smem + RowSmem::kQ + sl * RowSmem::kASlot;
                    const int key = c * g.s1 + cur.kr;
                    for (int la = 0; la < nla; ++la) {
                        const int ag = cur.bh * g.gq + kQG * cur.qg + 2 * mt + la;
                        tma_load_4d(ab + la * 8192, &P.tar_ld, &a_full[sl], 0, 0, key, ag);
                        tma_load_4d(ab + 16384 + la * 8192, &P.tar_ld, &a_full[sl], 64, 0, key, ag);
                    }
                }
                __syncwarp();
                ++ta;
            };
            // Q loads are issued whenever a staging slot is free, interleaved with the K/V
            // waits (never blocking a K/V load behind a Q slot)
            int q_next = amode ? cur.my_items : 0;
            auto try_q = [&]() {
                while (q_next < cur.my_items &&
                       mbar_test_uniform(&q_empty[q_next % nqs], (((q_next / nqs) & 1) ^ 1))) load_q(q_next++);
            };
            try_q();
            for (int li = 0; li < cur.my_items; ++li) {
                cur.li = li;
                cur.load(g);
                const int b = cur.bh / g.heads, h = cur.bh % g.heads;
                for (int c = cur.c0; c < cur.c1; ++c, ++kvi) {
                    const int ks = kvi % kKVStages;
                    const uint32_t kpar = ring_parity(kvi, kKVStages) ^ 1;
                    while (!mbar_test_uniform(&kv_empty[ks], kpar)) try_q();
                    const int tok = (int)row_base(g, false, c, cur.kr);
                    if (leader) {
                        TR(0, ti, 2);
                        mbar_expect_tx(&kv_full[ks], (want_y ? 4u : 2u) * box_bytes);   // V only for Y
                        uint8_t* kb = smem + RowSmem::kKV + ks * RowSmem::kKVBytes;
                        tma_load_4d(kb, &tm_k, &kv_full[ks], 0, tok, h, b);
                        tma_load_4d(kb + 8192, &tm_k, &kv_full[ks], 64, tok, h, b);
                        if (want_y) {
                            tma_load_4d(kb + 16384, &tm_v, &kv_full[ks], 0, tok, h, b);
                            tma_load_4d(kb + 24576, &tm_v, &kv_full[ks], 64, tok, h, b);
                        }
                    }
                    __syncwarp();
                    if (amode)
                        for (int mt = 0; mt < cur.n_mt; ++mt) load_a(c, mt);
                    try_q();
                }
            }
            while (q_next < cur.my_items) load_q(q_next++);   // (blocking) remaining Q rows
        }
    } else if (warp == 1) {
        // ------------------------------------------------------ MMA issuer (readiness order)
        // The whole warp runs the loop on warp-uniform state (so descriptors live in uniform
        // registers) and one elected lane issues the tcgen05 ops; descriptors are precomputed
        // (only the 14-bit start-address field moves) and ring positions kept incrementally.
        {
            const bool leader = elect_one();
            const uint32_t idesc_s = idesc_bf16(128, 64, false, false);
            const uint32_t idesc_o = idesc_bf16(128, 128, false, true);
            constexpr uint32_t kHi = (1024u >> 4) | (1u << 14) | (2u << 29);   // SBO 1024, v1, SW128
            const uint32_t kv_lo = (smem_u32(smem + RowSmem::kKV) & 0x3FFFF) >> 4;
            const uint32_t q_lo = ((smem_u32(smem + RowSmem::kQ) & 0x3FFFF) >> 4) | (1u << 16);
            auto desc = [](uint32_t lo) { return ((uint64_t)kHi << 32) | lo; };
            int ti = 0;
            RowCursor cs = cur, co = cur;   // next MMA1 task ts, next MMA2 task to
            int ts = 0, to = 0, q_item = -1;
            bool s_kv_ok = false;           // K/V of cs's key row known to have landed
            while (cs.valid || co.valid) {
                bool did = false;
                // MMA2(to): softmax done with S/P buffer to%2, both O buffers drained by task to-1
                if (co.valid && to < ts && ((P.dbg & 32) || (mbar_test_uniform(&p_full[to & 1], (to >> 1) & 1) &&
                    mbar_test_uniform(&o_empty[0], (to & 1) ^ 1) && (!want_y || mbar_test_uniform(&o_empty[1], (to & 1) ^ 1))))) {
                    if (leader) TR(1, ti, 12);
                    tc_fence_after();
                    // B = [K | V] row, MN-major SW128 (LBO 8192 between 64-feature atoms)
                    const uint32_t b_lo = kv_lo + (uint32_t)co.kst * (RowSmem::kKVBytes >> 4) + (8192u >> 4 << 16);
                    const uint32_t pa = tmem + kRowS + (to & 1) * 64;
                    if (leader) {
#pragma unroll
                        for (int s = 0; s < 2; ++s) {   // s = 0: aL = P K, s = 1: Y = P V
                            if (s == 1 && !want_y) break;
#pragma unroll
                            for (int kk = 0; kk < 4; ++kk)
                                mma_bf16_ts(tmem + kRowO + s * 128, pa + kk * 8,
                                            desc(b_lo + ((s * 16384 + kk * 2048) >> 4)), idesc_o, kk > 0);
                            mma_commit(&o_full[s]);
                        }
                        if (co.last_mt()) mma_commit(&kv_empty[co.kst]);
                    }
                    __syncwarp();
                    co.advance(g);
                    ++to;
                    did = true;
                }
                // MMA1(ts): S/P buffer ts%2 released by MMA2(ts-2), Q of its item in TMEM, K/V landed
                if (cs.valid && ts < to + 2) {
                    bool ready = true;
                    if (amode) {
                        ready = mbar_test_uniform(&a_full[ts & 1], (ts >> 1) & 1);
                    } else if (cs.li != q_item) {
                        // first task of a new item: all MMA1 of the previous item are issued,
                        // so (tensor-pipe order) the copy cannot overtake their reads of Q
                        const int qsl = cs.li % nqs;
                        if (mbar_test_uniform(&q_full[qsl], (cs.li / nqs) & 1)) {
                            tc_fence_after();
                            if (leader) {
                                for (int mt = 0; mt < cs.n_mt; ++mt)
#pragma unroll
                                    for (int kk = 0; kk < 8; ++kk)
                                        tmem_cp_128x256b(tmem + kRowQ + mt * 64 + kk * 8,
                                                         desc(q_lo + ((qsl * 2 * qchunk + (kk >> 2) * qchunk +
                                                                       mt * 16384 + (kk & 3) * 32) >> 4)));
                                mma_commit(&q_empty[qsl]);
                            }
                            __syncwarp();
                            q_item = cs.li;
                        } else {
                            ready = false;
                        }
                    }
                    if (ready && cs.mt == 0 && !s_kv_ok) {
                        s_kv_ok = mbar_test_uniform(&kv_full[cs.kst], cs.kph);
                        ready = s_kv_ok;
                    }
                    if (ready) {
                        if (leader) TR(1, ti, 11);
                        tc_fence_after();
                        // B = K row, K-major SW128 (LBO 16)
                        const uint32_t b_lo = kv_lo + (uint32_t)cs.kst * (RowSmem::kKVBytes >> 4) + (1u << 16);
                        const uint32_t a_t = tmem + kRowQ + cs.mt * 64;
                        const uint32_t d_t = tmem + kRowS + (ts & 1) * 64;
                        if (leader) {
                            if (amode) {   // A = hat_alpha_R rows of this task, K-major SW128 in smem
                                const uint32_t a_lo = q_lo + (uint32_t)(ts & 1) * (RowSmem::kASlot >> 4);
#pragma unroll
                                for (int kk = 0; kk < 8; ++kk)
                                    mma_bf16(d_t, desc(a_lo + (((kk >> 2) * 16384 + (kk & 3) * 32) >> 4)),
                                             desc(b_lo + (((kk >> 2) * 8192 + (kk & 3) * 32) >> 4)), idesc_s, kk > 0);
                                mma_commit(&a_empty[ts & 1]);
                            } else {
#pragma unroll
                                for (int kk = 0; kk < 8; ++kk)
                                    mma_bf16_ts(d_t, a_t + kk * 8,
                                                desc(b_lo + (((kk >> 2) * 8192 + (kk & 3) * 32) >> 4)), idesc_s,
                                                kk > 0);
                            }
                            mma_commit(&s_full[ts & 1]);
                        }
                        __syncwarp();
                        if (cs.last_mt()) s_kv_ok = false;
                        cs.advance(g);
                        ++ts;
                        did = true;
                    }
                }
                if (!did) __nanosleep(20);
            }
        }
    } else if (warp < 6) {
        // ------------------------------------------------------ softmax (rows = TMEM lanes)
        const int quad = warp & 3;
        const int r = quad * 32 + lane;
        const uint32_t lane_off = (uint32_t)(quad * 32) << 16;
        const float sl2 = g.scale * kLog2e;
        int ti = 0;
        for (int t = 0; cur.valid; ++t, cur.advance(g)) {
            const int bsel = t & 1;
            const uint32_t sbuf = tmem + kRowS + bsel * 64 + lane_off;
            const int al = cur.mt * 2 + (r >> 6), j = r & 63;
            const bool row_ok = al < cur.nt && j < g.s2;
            WAITX(&s_full[bsel], ring_parity(t, 2));
            if (lane == 0) TR(warp, ti, 21);
            tc_fence_after();
            if (P.dbg & 4) {   // timing experiment: no softmax arithmetic
                float zz[32];
                for (int i = 0; i < 32; ++i) zz[i] = 0.f;
                tmem_st32(sbuf, zz);
                tc_fence_before();
                mbar_arrive(&p_full[bsel]);
                continue;
            }
            float z[64];
            {
                uint32_t zr[64];
                tmem_ld32_nw(sbuf, zr);
                tmem_ld32_nw(sbuf + 32, zr + 32);
                tmem_wait_ld();
#pragma unroll
                for (int i = 0; i < 64; ++i) z[i] = __uint_as_float(zr[i]);
            }
            // padded keys -> -1e30 (finite: exp2 -> 0 and 0 * z stays 0)
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
            // p = 2^(z sl2 - m sl2); l = sum p; A = sum p z -- eight independent partial sums
            float p[64];
#pragma unroll
            for (int i = 0; i < 64; ++i) p[i] = ex2(fmaf(z[i], sl2, -mb));
            float lq[8], aq[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) {
                lq[e] = p[e] + p[e + 8];
                aq[e] = fmaf(p[e + 8], z[e + 8], p[e] * z[e]);
            }
#pragma unroll
            for (int i = 16; i < 64; i += 8)
#pragma unroll
                for (int e = 0; e < 8; ++e) {
                    lq[e] += p[i + e];
                    aq[e] = fmaf(p[i + e], z[i + e], aq[e]);
                }
            const float l = ((lq[0] + lq[1]) + (lq[2] + lq[3])) + ((lq[4] + lq[5]) + (lq[6] + lq[7]));
            const float A = ((aq[0] + aq[1]) + (aq[2] + aq[3])) + ((aq[4] + aq[5]) + (aq[6] + aq[7]));
            const float inv_l = 1.f / l;
            // R = p / l (bf16, <= 1) over S's first 32 columns: MMA2 reads it as its A operand
            const float pscale = row_ok ? inv_l : 0.f;
            uint32_t packed[32];
#pragma unroll
            for (int i = 0; i < 64; i += 2) packed[i >> 1] = pack_bf16(p[i] * pscale, p[i + 1] * pscale);
            tmem_st32(sbuf, reinterpret_cast<const float*>(packed));
            tc_fence_before();
            mbar_arrive(&p_full[bsel]);
            if (P.rfac && row_ok)   // R' row (final, or this refinement's slice) [bh][a][c][k][j][:] (factors.py:57-79)
                store_r_row(P.rfac + ((((int64_t)(cur.bh * g.gq + kQG * cur.qg + al) * g.gk + cur.c) * g.s1 + cur.kr) *
                                          g.s2 + j) * g.s2,
                            p, inv_l, g.s2);
            // c_L = sum R z - lse with z = scale * S (solver.py:191)
            if (row_ok) {
                const int col = (cur.bh * g.gq + kQG * cur.qg + al) * g.s2 + j;
                Wc[(int64_t)col * ckey + cur.c * g.s1 + cur.kr] = g.scale * (A * inv_l - m) - __logf(l);
            }
            if (lane == 0) TR(warp, ti, 22);
        }
    } else {
        // ------------------------------------------------------ epilogue: TMEM -> smem -> TMA store
        const int set = warp >= 10 ? 1 : 0;   // warps 6-9: O_aL, 10-13: O_Y
        // the column stage reads W right after this launch: keep it in L2 ahead of q / k / v
        const uint64_t w_policy = (P.l2hint & 1) ? l2_evict_last() : l2_evict_normal();
        if (set == 1 && !want_y) cur.valid = false;   // no Y this refinement
        const int quad = warp & 3;
        const uint32_t lane_off = (uint32_t)(quad * 32) << 16;
        const uint32_t obuf = tmem + kRowO + set * 128 + lane_off;
        const int half = quad & 1;
        const int nrows = min(32, g.s2 - half * 32);
        uint8_t* stg_base = smem + RowSmem::kStage + (warp - 6) * 8192;
        int nstore = 0;   // staging buffer uses (== bulk groups committed) of this warp
        int ti = 0;
        for (int t = 0; cur.valid; ++t, cur.advance(g)) {
            const int al = cur.mt * 2 + (quad >> 1);
            const bool store_ok = al < cur.nt && nrows > 0;
            const int key = cur.c * g.s1 + cur.kr;
            const int col0 = (cur.bh * g.gq + kQG * cur.qg + (al < cur.nt ? al : 0)) * g.s2 + half * 32;
            mbar_wait(&o_full[set], t & 1);
            if (lane == 0) TR(warp, ti, 31);
            tc_fence_after();
            if (P.dbg & 2) {   // timing experiment: no drain
                tc_fence_before();
                mbar_arrive(&o_empty[set]);
                continue;
            }
            // both 64-feature parts to registers as packed bf16, then release the buffer
            uint32_t pk[2][32];
#pragma unroll
            for (int q4 = 0; q4 < 4; ++q4) {
                uint32_t o[32];
                tmem_ld32_nw(obuf + q4 * 32, o);
                tmem_wait_ld();
#pragma unroll
                for (int i = 0; i < 16; ++i)
                    pk[q4 >> 1][(q4 & 1) * 16 + i] = pack_bf16(__uint_as_float(o[2 * i]), __uint_as_float(o[2 * i + 1]));
            }
            tc_fence_before();
            mbar_arrive(&o_empty[set]);
            // a warp whose rows are all padding writes nothing: touching the staging
            // buffer would race with this warp's in-flight TMA store from it
            if (store_ok && !(P.dbg & 1)) {
#pragma unroll
                for (int part = 0; part < 2; ++part) {
                    uint8_t* stg = stg_base + (nstore++ & 1) * 4096;
                    if (lane == 0) bulk_wait_read<1>();   // previous store from this buffer has read it
                    __syncwarp();
                    const uint32_t srow = smem_u32(stg) + lane * 128;
#pragma unroll
                    for (int cc = 0; cc < 8; ++cc)
                        st_shared_v4(srow + ((cc ^ (lane & 7)) << 4), pk[part][4 * cc], pk[part][4 * cc + 1],
                                     pk[part][4 * cc + 2], pk[part][4 * cc + 3]);
                    fence_proxy_async_smem();
                    __syncwarp();
                    if (lane == 0) {
                        tma_store_4d_hint(half ? &tm_wst_b : &tm_wst, stg, 0, key, 2 * set + part, col0, w_policy);
                        bulk_commit();
                    }
                }
            }
            if (lane == 0 && warp < 16) TR(warp, ti, 32);
        }
        if (lane == 0) bulk_wait<0>();
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc<512>(tmem);
}
