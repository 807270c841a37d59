// Column stage (included by mbx_tc.cu).
//
// Item = group of 4 consecutive query columns (b, h, a, j..j+3).  The Q
// columns are stacked on the four TMEM lane quadrants (rows 32i..32i+31 of
// the A operand), so after
//     MMA_S_i  S_i[(rows), key] = Qstack . aL_i^T      M=128, N=96 (one key chunk)
// warp i (lane quadrant i) owns exactly the 32 query rows l of column i and
// does an in-thread softmax over the keys (no cross-lane reductions); the other
// 96 rows of S_i are discarded.  The joint softmax over (c, k) is online across
// 96-key chunks with lazy rescaling (FA4 style: rescale only when the running
// max grows by > 8 in log2 units).  The value product runs transposed so all
// 128 lanes carry value dims:
//     MMA_O_i  O^T_i[v, l] += Y_i^T . P_i^T            M=128, N=32, K=96
// (solver.py:192-195 joint softmax with bias -c_L; factors.py:124 O = L Y).
constexpr int kColThreads = 192;   // 6 warps: producer, MMA, 4 x softmax/output
constexpr int kKC = 96;            // keys per chunk (S_i is 96 TMEM columns)
#ifndef MBX_COL_RING6
#define MBX_COL_RING6 1
#endif
// MBX_COL_RING6: six ring slots, paid for by one output staging buffer per warp (reused
// column by column) instead of four
template <int mode>
struct ColSmemT {
    static constexpr bool kSix = MBX_COL_RING6 && mode == 0;   // mode 2 needs the 4-column staging
    static constexpr int kRing = kSix ? 6 : 5;           // aL / Y chunk slots
    static constexpr int kQ = 0;                          // Qstack: 2 d-chunks x [128][64] (32 KB)
    static constexpr int kSlot = 2 * kKC * 128;           // [96 keys][128 feat] as 2 x [96][64] (24 KB)
    static constexpr int kRingOff = 32768;
    static constexpr int kP = kRingOff + kRing * kSlot;   // P_i: 2 x [32 l][64 keys] (8 KB each)
    static constexpr int kC = kP + 4 * 8192;              // c_L chunks: [4 columns][2 buffers] x 96 floats (512 B pitch)
    static constexpr int kOut = kC + 8 * 512;             // output staging [4 warps][4 columns] x [32 rows][64 B]
    static constexpr int kStat = kOut + (kSix ? 4 : 16) * 2048;   // row sums [4][32], rescale [4][32], flags [4], rb[32]
    static constexpr int kBars = kStat + 4 * 32 * 4 * 2 + 4 * 4 + 32 * 8;
    static constexpr int kNumBars = 2 * kRing + 2 + 4 * 4 + 1 + 16;
    static constexpr int kTmemSlot = kBars + kNumBars * 8;
    static constexpr int kTotal = kTmemSlot + 16;
};
using ColSmem = ColSmemT<1>;

// Column-stage role of CTA `first` among `stride` column CTAs.
// mode 0: O = L Y (last refinement); mode 1 (T >= 2, earlier refinements): only the
// per-row softmax statistics (running max, sum) of L, for the alpha_R stage.
// mode 2 (T >= 2, earlier refinements, all keys of a column in one 96-key chunk): the
// alpha_R hand-off fused in (solver.py:185-186 of the next refinement): the softmax is
// exact in one pass, so P_i = L (normalised, bf16) goes to shared memory and
//     MMA_A_i  alpha_R_i[key, v] = P_i^T . Q_col_i      M=128 keys, N=128, K=32 rows l
// runs into TMEM (D_i at columns 128 i, over the consumed S regions); c_R = sum_l L is a
// warp transpose-reduce of the fp32 L row; the epilogue writes hat_alpha_R = alpha_R /
// max(c_R, eps) (bf16) for the next row stage -- no statistics pass, no alpha_R stage.
template <int mode>   // compile-time: each mode gets its own register allocation
__device__ __forceinline__ void col_role(uint8_t* smem, const TcParams& P, const Geometry& g, int first, int stride) {
    using ColSmem = ColSmemT<mode>;
    constexpr int kRing = ColSmem::kRing;
    constexpr bool kSix = ColSmem::kSix;
    constexpr bool outm = mode == 0;
    constexpr bool hand = mode == 2;
    const CUtensorMap& tm_w = P.tw;
    const CUtensorMap& tm_c = P.tc;
    const CUtensorMap& tm_qc = P.tqc;
    const CUtensorMap& tm_out = P.tout;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + ColSmem::kBars);
    uint64_t* ring_full = bars;                   // [6]
    uint64_t* ring_empty = bars + kRing;          // [6]
    uint64_t* q_full = bars + 2 * kRing;          // [1]
    uint64_t* q_empty = q_full + 1;               // [1]
    uint64_t* s_full = q_full + 2;                // [4]
    uint64_t* s_free = s_full + 4;                // [4]  softmax i read S_i and c_L_i
    uint64_t* p_full = s_free + 4;                // [4]
    uint64_t* o_done = p_full + 4;                // [4]  MMA_O_i of the chunk completed
    uint64_t* o_free = o_done + 4;                // [1]  all four O^T regions read out
    uint64_t* c_full = o_free + 1;                // [4][2]  c_L chunk of column i landed
    uint64_t* c_empty = c_full + 8;               // [4][2]  softmax i read it
    float* stat_sum = reinterpret_cast<float*>(smem + ColSmem::kStat);   // [4][32]
    float* stat_fac = stat_sum + 128;                                    // [4][32]
    int* flags = reinterpret_cast<int*>(stat_fac + 128);                 // [4]
    int64_t* rb = reinterpret_cast<int64_t*>(flags + 4);                 // [32] row_base(a, l)
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + ColSmem::kTmemSlot);
    const int tid = threadIdx.x, lane = tid & 31;
    const int warp = __shfl_sync(0xffffffffu, tid >> 5, 0);   // provably warp-uniform

    const int gpt = (g.s2 + 3) >> 2;                       // column groups per query tile
    const int groups = g.bh * g.gq * gpt;
    const int nch = (g.nkeys + kKC - 1) / kKC;
    const int my_groups = first < groups ? (groups - first + stride - 1) / stride : 0;

    if (tid == 0) {
        tma_prefetch(&tm_w);
        tma_prefetch(&tm_c);
        tma_prefetch(&tm_qc);
        tma_prefetch(&tm_out);
        for (int i = 0; i < kRing; ++i) {
            mbar_init(&ring_full[i], 1);
            mbar_init(&ring_empty[i], 1);
        }
        mbar_init(q_full, 1);
        mbar_init(q_empty, 1);
        for (int i = 0; i < 4; ++i) {
            mbar_init(&s_full[i], 1);
            mbar_init(&s_free[i], 32);
            mbar_init(&p_full[i], 32);
            mbar_init(&o_done[i], 1);
        }
        for (int i = 0; i < 8; ++i) {
            mbar_init(&c_full[i], 1);
            mbar_init(&c_empty[i], 32);
        }
        mbar_init(o_free, 128);
        fence_barrier_init();
    }
    if (warp == 0) tmem_alloc<512>(tmem_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    // Dependents may start their prologue once every CTA got here.  The predecessor (the
    // row stage) is waited for by the producer alone, right before its first workspace
    // read: q columns are inputs the row stage does not write, and the row stage only
    // triggers after its own wait, so they are already final.
    pdl_trigger();

    auto decode = [&](int grp, int& bh, int& a, int& j0) {
        const int jg = grp % gpt;
        a = (grp / gpt) % g.gq;
        bh = grp / (gpt * g.gq);
        j0 = jg * 4;
    };

    if (warp == 0) {
        // ------------------------------------------------------ TMA producer
        // whole warp on warp-uniform state (TMA coordinates in uniform registers), one elected lane issues
        const bool leader = elect_one();
        int slot = 0, sph = 0;   // ring position of use n: n % kRing and (n / kRing) & 1
        // the final pass is W's last reader: stream it through L2 without displacing the rest
        const uint64_t w_policy = (P.l2hint & 2) && mode == 0 ? l2_evict_first() : l2_evict_normal();
        int ti = 0;
        auto next_slot = [&]() {
            if (++slot == kRing) {
                slot = 0;
                sph ^= 1;
            }
        };
        // Ring order = MMA order: aL(u) [+ Q at a group start], then Y(u-1) -- the aL of the next
        // chunk is in flight while the current chunk's softmax runs (u = global chunk index)
        const int U = my_groups * nch;
        // one-chunk lookahead only pays with several chunks per group (MBX_DBG 2048 / 4096 force off / on)
        const bool look = (nch > 1 || (P.dbg & 4096)) && !(P.dbg & 2048);
        int bh = 0, a = 0, j0 = 0, col0 = 0;
        auto load_y = [&](int up) {   // Y_i of chunk up (its group's columns col0p .. +3)
            int bhp, ap, j0p;
            decode(first + (up / nch) * stride, bhp, ap, j0p);
            const int col0p = (bhp * g.gq + ap) * g.s2 + j0p, k0 = (up % nch) * kKC;
            for (int i = 0; i < 4; ++i) {
                mbar_wait(&ring_empty[slot], sph ^ 1);
                if (leader) {
                    TRC(0, ti, 2);
                    mbar_expect_tx(&ring_full[slot], 2u * kKC * 128u);
                    uint8_t* dst = smem + ColSmem::kRingOff + slot * ColSmem::kSlot;
                    tma_load_4d_hint(dst, &tm_w, &ring_full[slot], 0, k0, 2, col0p + i, w_policy);
                    tma_load_4d_hint(dst + kKC * 128, &tm_w, &ring_full[slot], 0, k0, 3, col0p + i, w_policy);
                }
                __syncwarp();
                next_slot();
            }
        };
        for (int u = 0; u < U; ++u) {
            const int gi = u / nch, ch = u - gi * nch;
            if (ch == 0) {
                decode(first + gi * stride, bh, a, j0);
                col0 = (bh * g.gq + a) * g.s2 + j0;
                mbar_wait(q_empty, (gi & 1) ^ 1);
                if (leader) TRC(0, ti, 5);
                const int64_t tq0 = row_base(g, true, a, 0) + j0;
                if (leader) {
                    mbar_expect_tx(q_full, 4u * 2u * 32u * 128u);
                    for (int i = 0; i < 4; ++i) {
                        const int64_t tok0 = tq0 + i;
                        const int wcol = (int)(tok0 % g.W), wrow = (int)(tok0 / g.W);
                        uint8_t* dst = smem + ColSmem::kQ + i * 4096;
                        tma_load_4d(dst, &tm_qc, q_full, 0, wcol, wrow, bh);
                        tma_load_4d(dst + 16384, &tm_qc, q_full, 64, wcol, wrow, bh);
                    }
                }
                __syncwarp();
            }
            const int k0 = ch * kKC;
            if (u == 0) pdl_wait();   // W and c_L of the row stage complete and visible
            for (int i = 0; i < 4; ++i) {   // aL_i + c_L_i
                mbar_wait(&ring_empty[slot], sph ^ 1);
                const int cb = i * 2 + (u & 1);
                mbar_wait(&c_empty[cb], ((u >> 1) & 1) ^ 1);
                if (leader) {
                    TRC(0, ti, 1);
                    mbar_expect_tx(&ring_full[slot], 2u * kKC * 128u);
                    uint8_t* dst = smem + ColSmem::kRingOff + slot * ColSmem::kSlot;
                    tma_load_4d_hint(dst, &tm_w, &ring_full[slot], 0, k0, 0, col0 + i, w_policy);
                    tma_load_4d_hint(dst + kKC * 128, &tm_w, &ring_full[slot], 0, k0, 1, col0 + i, w_policy);
                    mbar_expect_tx(&c_full[cb], kKC * 4u);
                    tma_load_2d(smem + ColSmem::kC + cb * 512, &tm_c, &c_full[cb], k0, col0 + i);
                }
                __syncwarp();
                next_slot();
            }
            if (outm && look && u > 0) load_y(u - 1);
            if (outm && !look) load_y(u);
        }
        if (outm && look && U > 0) load_y(U - 1);
    } else if (warp == 1) {
        // ------------------------------------------------------ MMA issuer
        // whole warp on warp-uniform state (descriptors in uniform registers), one elected lane issues
        const bool leader = elect_one();
        const uint32_t idesc_s = idesc_bf16(128, kKC, false, false);
        const uint32_t idesc_o = idesc_bf16(128, 32, true, false);
        constexpr uint32_t kHi = (1024u >> 4) | (1u << 14) | (2u << 29);   // SBO 1024, v1, SW128
        auto desc = [](uint32_t lo) { return ((uint64_t)kHi << 32) | lo; };
        const uint32_t q_lo = ((smem_u32(smem + ColSmem::kQ) & 0x3FFFF) >> 4) | (1u << 16);
        const uint32_t ring_lo = (smem_u32(smem + ColSmem::kRingOff) & 0x3FFFF) >> 4;
        const uint32_t p_lo = ((smem_u32(smem + ColSmem::kP) & 0x3FFFF) >> 4) | (1u << 16);
        int ti = 0;
        int slot = 0, sph = 0;   // ring position of use n: n % kRing and (n / kRing) & 1
        auto next_slot = [&]() {
            if (++slot == kRing) {
                slot = 0;
                sph ^= 1;
            }
        };
        // order: S(0), then S(u), O(u-1) for u = 1 .. U-1, then O(U-1) -- the next chunk's
        // S MMAs are queued before this chunk's O MMAs, matching the producer's ring order
        const int U = my_groups * nch;
        const bool look = (nch > 1 || (P.dbg & 4096)) && !(P.dbg & 2048);
        auto issue_o = [&](int up) {
            const int gp = up / nch, cp = up - gp * nch;
            for (int i = 0; i < 4; ++i) {
                mbar_wait(&ring_full[slot], sph);
                mbar_wait(&p_full[i], up & 1);
                if (cp == 0 && gp > 0 && i == 0) mbar_wait(o_free, (gp - 1) & 1);
                tc_fence_after();
                if (leader) {
                    TRC(1, ti, 13);
                    // A = Y^T (MN-major, LBO kKC*128 between the two 64-value halves), B = P_i (K-major)
                    const uint32_t y_lo = ring_lo + (uint32_t)slot * (ColSmem::kSlot >> 4) + ((kKC * 128) >> 4 << 16);
                    const uint32_t pb = p_lo + (uint32_t)i * (8192 >> 4);
#pragma unroll
                    for (int kk = 0; kk < kKC / 16; ++kk)
                        mma_bf16(tmem + 4 * kKC + i * 32, desc(y_lo + ((kk * 2048) >> 4)),
                                 desc(pb + (((kk >> 2) * 4096 + (kk & 3) * 32) >> 4)), idesc_o, cp > 0 || kk > 0);
                    mma_commit(&ring_empty[slot]);
                    mma_commit(&o_done[i]);
                }
                __syncwarp();
                next_slot();
            }
        };
        const uint32_t idesc_a = idesc_bf16(128, 128, true, true);   // A = P^T (MN-major), B = Q_col (MN-major)
        for (int u = 0; u < U; ++u) {
            const int gi = u / nch, ch = u - gi * nch;
            if (ch == 0) mbar_wait(q_full, gi & 1);
            if (hand && gi > 0) mbar_wait(o_free, (gi - 1) & 1);   // D_i (over the S regions) drained
            for (int i = 0; i < 4; ++i) {
                mbar_wait(&ring_full[slot], sph);
                if (u > 0) mbar_wait(&s_free[i], (u - 1) & 1);
                tc_fence_after();
                if (leader) {
                    TRC(1, ti, 11);
                    const uint32_t a_lo = ring_lo + (uint32_t)slot * (ColSmem::kSlot >> 4) + (1u << 16);
#pragma unroll
                    for (int kk = 0; kk < 8; ++kk)
                        mma_bf16(tmem + i * kKC, desc(q_lo + (((kk >> 2) * 16384 + (kk & 3) * 32) >> 4)),
                                 desc(a_lo + (((kk >> 2) * (kKC * 128) + (kk & 3) * 32) >> 4)), idesc_s, kk > 0);
                    mma_commit(&s_full[i]);
                    mma_commit(&ring_empty[slot]);
                }
                __syncwarp();
                next_slot();
            }
            if (hand) {   // nch == 1: alpha_R_i = P_i^T Q_col_i once every softmax wrote its P_i
                // (D_i spans S regions of other columns: all four must have been read first)
                for (int i = 0; i < 4; ++i) mbar_wait(&p_full[i], u & 1);
                tc_fence_after();
                for (int i = 0; i < 4; ++i) {
                    if (leader) {
                        const uint32_t pa = p_lo + (uint32_t)i * (8192 >> 4);   // [32 l][64 keys] x 2 key chunks
#pragma unroll
                        for (int kk = 0; kk < 2; ++kk)   // K = 32 rows l: two k-steps of 16 rows (2 KB)
                            mma_bf16(tmem + i * 128,
                                     desc((pa & ~(0x3FFFu << 16)) + ((kk * 2048) >> 4) + ((4096u >> 4) << 16)),
                                     desc((q_lo & ~(0x3FFFu << 16)) + ((i * 4096 + kk * 2048) >> 4) + ((16384u >> 4) << 16)),
                                     idesc_a, kk > 0);
                        mma_commit(&o_done[i]);
                    }
                    __syncwarp();
                }
            }
            if (ch == nch - 1) {
                if (leader) mma_commit(q_empty);
                __syncwarp();
            }
            if (outm && look && u > 0) issue_o(u - 1);
            if (outm && !look) issue_o(u);
        }
        if (outm && look && U > 0) issue_o(U - 1);
    } else if (warp < 6) {
        // ------------------------------------------------------ softmax (warp i = column i) + output
        const int quad = warp & 3;                       // column i within the group == lane quadrant
        const uint32_t lane_off = (uint32_t)(quad * 32) << 16;
        const int l = lane;                              // query row of column i
        const uint32_t sP = smem_u32(smem + ColSmem::kP + quad * 8192);
        const float sl2 = g.scale * kLog2e;

        int ti = 0;
        for (int gi = 0; gi < my_groups; ++gi) {
            int bh, a, j0;
            decode(first + gi * stride, bh, a, j0);
            float m_run = -INFINITY, s_run = 0.f;
            for (int ch = 0; ch < nch; ++ch) {
                const int u = gi * nch + ch;
                const int kvalid = min(kKC, g.nkeys - ch * kKC);
                const int cb = quad * 2 + (u & 1);
                const uint32_t cbuf = smem_u32(smem + ColSmem::kC + cb * 512);
                mbar_wait(&c_full[cb], (u >> 1) & 1);
                if (lane == 0) TRC(warp + 8, ti, 21);
                mbar_wait(&s_full[quad], u & 1);
                if (lane == 0) TRC(warp + 8, ti, 22);
                tc_fence_after();
                float x[kKC];
                tmem_ld32(tmem + quad * kKC + lane_off, x);
                tmem_ld32(tmem + quad * kKC + 32 + lane_off, x + 32);
                tmem_ld32(tmem + quad * kKC + 64 + lane_off, x + 64);
                float mq[4] = {-1e30f, -1e30f, -1e30f, -1e30f};
#pragma unroll
                for (int k4 = 0; k4 < kKC; k4 += 4) {
                    const float4 c4 = ld_shared_v4f(cbuf + k4 * 4);
                    x[k4] = fmaf(x[k4], sl2, -c4.x * kLog2e);
                    x[k4 + 1] = fmaf(x[k4 + 1], sl2, -c4.y * kLog2e);
                    x[k4 + 2] = fmaf(x[k4 + 2], sl2, -c4.z * kLog2e);
                    x[k4 + 3] = fmaf(x[k4 + 3], sl2, -c4.w * kLog2e);
                }
                if (kvalid < kKC) {   // padded keys -> -1e30 (exp2 -> 0)
#pragma unroll
                    for (int k = 0; k < kKC; ++k) x[k] = k < kvalid ? x[k] : -1e30f;
                }
#pragma unroll
                for (int k = 0; k < kKC; ++k) mq[k & 3] = fmaxf(mq[k & 3], x[k]);
                const float mx = fmaxf(fmaxf(mq[0], mq[1]), fmaxf(mq[2], mq[3]));
                tc_fence_before();
                mbar_arrive(&s_free[quad]);
                mbar_arrive(&c_empty[cb]);
                // lazy online max: keep m_run unless the chunk max exceeds it by > 8 (x 256)
                float fac = 1.f;
                int need = 0;
                if (ch == 0) {
                    m_run = mx;
                } else if (mx > m_run + 8.f) {
                    fac = ex2(m_run - mx);
                    m_run = mx;
                    need = 1;
                }
                s_run *= fac;
                if (hand) {   // one chunk: exact softmax, normalised P_i, c_R, optional L' export
                    float sq[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
                    for (int k = 0; k < kKC; ++k) {
                        x[k] = ex2(x[k] - m_run);
                        sq[k & 3] += x[k];
                    }
                    const float inv = 1.f / ((sq[0] + sq[1]) + (sq[2] + sq[3]));
                    const bool lrow = l < g.s1 && j0 + quad < g.s2;
#pragma unroll
                    for (int k = 0; k < kKC; ++k) x[k] = lrow ? x[k] * inv : 0.f;
                    if (u > 0) mbar_wait(&o_done[quad], (u - 1) & 1);   // MMA_A_i(u-1) done with P_i
#pragma unroll
                    for (int cc = 0; cc < kKC / 8; ++cc) {
                        const uint32_t dst = sP + (cc >> 3) * 4096 + l * 128 + (((cc & 7) ^ (l & 7)) << 4);
                        st_shared_v4(dst, pack_bf16(x[cc * 8], x[cc * 8 + 1]), pack_bf16(x[cc * 8 + 2], x[cc * 8 + 3]),
                                     pack_bf16(x[cc * 8 + 4], x[cc * 8 + 5]), pack_bf16(x[cc * 8 + 6], x[cc * 8 + 7]));
                    }
                    fence_proxy_async_smem();
                    mbar_arrive(&p_full[quad]);
                    if (P.lfac && lrow) {   // L'[bh][a][c][j][l][k], key = c s1 + k
                        const int j = j0 + quad;
                        float* lrow0 = P.lfac + ((((int64_t)(bh * g.gq + a) * g.gk) * g.s2 + j) * g.s1 + l) * g.s1;
                        const int64_t cstride = (int64_t)g.s2 * g.s1 * g.s1;
                        int c = 0, kk = 0;
#pragma unroll
                        for (int key = 0; key < kKC; ++key) {   // constant indices keep x in registers
                            if (key < kvalid) lrow0[c * cstride + kk] = x[key];
                            if (++kk == g.s1) {
                                kk = 0;
                                ++c;
                            }
                        }
                    }
                    // c_R[key] = sum_l L[l, key]: transpose-reduce over the warp, 32 keys per pass
                    float* crs = reinterpret_cast<float*>(smem + ColSmem::kOut + 16384) + quad * 128;
#pragma unroll
                    for (int pass = 0; pass < kKC / 32; ++pass) {
                        float v[32];
#pragma unroll
                        for (int e = 0; e < 32; ++e) v[e] = x[pass * 32 + e];
#pragma unroll
                        for (int sh = 16; sh >= 1; sh >>= 1) {
#pragma unroll
                            for (int e = 0; e < sh; ++e) {
                                const bool up = (lane & sh) != 0;
                                const float send = up ? v[e] : v[e + sh];
                                const float keep = up ? v[e + sh] : v[e];
                                v[e] = keep + __shfl_xor_sync(0xffffffffu, send, sh);
                            }
                        }
                        crs[pass * 32 + lane] = v[0];
                    }
                    continue;
                }
                if (!outm) {   // statistics only: running sum of this chunk, no P, no O
                    float sq[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
                    for (int k = 0; k < kKC; k += 4) {
                        sq[0] += ex2(x[k] - m_run);
                        sq[1] += ex2(x[k + 1] - m_run);
                        sq[2] += ex2(x[k + 2] - m_run);
                        sq[3] += ex2(x[k + 3] - m_run);
                    }
                    s_run += (sq[0] + sq[1]) + (sq[2] + sq[3]);
                    continue;
                }
                if (ch > 0) {
                    const int any = __any_sync(0xffffffffu, need);
                    stat_fac[quad * 32 + l] = fac;
                    if (lane == 0) flags[quad] = any;
                    named_sync(1, 128);
                    const int f = flags[0] | flags[1] | flags[2] | flags[3];
                    if (f) {   // rescale O^T of every flagged column: thread = value lane
                        for (int i = 0; i < 4; ++i) {
                            if (!flags[i]) continue;
                            mbar_wait(&o_done[i], (u - 1) & 1);
                            tc_fence_after();
                            float o[32];
                            tmem_ld32(tmem + 4 * kKC + i * 32 + lane_off, o);
#pragma unroll
                            for (int q = 0; q < 32; ++q) o[q] *= stat_fac[i * 32 + q];
                            tmem_st32(tmem + 4 * kKC + i * 32 + lane_off, o);
                        }
                        tc_fence_before();
                    }
                    named_sync(1, 128);
                }
                // P_i row l (bf16, K-major SW128: keys 0-63 chunk 0, keys 64-95 chunk 1), written
                // 8 keys at a time so only one 16-byte group of packed values is live
                if (u > 0) mbar_wait(&o_done[quad], (u - 1) & 1);   // MMA_O_i(u-1) done with P_i
                float sq[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
                for (int cc = 0; cc < kKC / 8; ++cc) {
                    uint32_t pk[4];
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const int k = cc * 8 + 2 * e;
                        const float p0 = ex2(x[k] - m_run), p1 = ex2(x[k + 1] - m_run);
                        sq[e] += p0 + p1;
                        pk[e] = pack_bf16(p0, p1);
                    }
                    const uint32_t dst = sP + (cc >> 3) * 4096 + l * 128 + (((cc & 7) ^ (l & 7)) << 4);
                    st_shared_v4(dst, pk[0], pk[1], pk[2], pk[3]);
                }
                const float sum = (sq[0] + sq[1]) + (sq[2] + sq[3]);
                s_run += sum;
                fence_proxy_async_smem();
                mbar_arrive(&p_full[quad]);
                if (lane == 0) TRC(warp + 8, ti, 23);
            }
            if (hand) {
                // ---- hat_alpha_R of the 4 columns: thread = key (its TMEM lane), D_i row / c_R ----
                named_sync(1, 128);   // every column's c_R in shared memory
                const int key = quad * 32 + lane;
                const int u = gi;     // nch == 1
                if (lane == 0) bulk_wait_read<0>();
                __syncwarp();
                for (int i = 0; i < 4; ++i) {
                    mbar_wait(&o_done[i], u & 1);
                    tc_fence_after();
                    const float cr = reinterpret_cast<const float*>(smem + ColSmem::kOut + 16384)[i * 128 + key];
                    const float inv = 1.f / fmaxf(cr, g.eps_div);
                    const bool store = j0 + i < g.s2 && quad * 32 < g.nkeys;
#pragma unroll 1
                    for (int part = 0; part < 2; ++part) {
                        float o[64];
                        tmem_ld32(tmem + i * 128 + part * 64 + lane_off, o);
                        tmem_ld32(tmem + i * 128 + part * 64 + 32 + lane_off, o + 32);
                        if (!store) continue;
                        uint8_t* stg = smem + ColSmem::kOut + quad * 4096;   // [32 keys][64 values], SW128
                        if (lane == 0) bulk_wait_read<0>();
                        __syncwarp();
                        const uint32_t srow = smem_u32(stg) + lane * 128;
#pragma unroll
                        for (int cc = 0; cc < 8; ++cc)
                            st_shared_v4(srow + ((cc ^ (lane & 7)) << 4), pack_bf16(o[8 * cc] * inv, o[8 * cc + 1] * inv),
                                         pack_bf16(o[8 * cc + 2] * inv, o[8 * cc + 3] * inv),
                                         pack_bf16(o[8 * cc + 4] * inv, o[8 * cc + 5] * inv),
                                         pack_bf16(o[8 * cc + 6] * inv, o[8 * cc + 7] * inv));
                        fence_proxy_async_smem();
                        __syncwarp();
                        if (lane == 0) {   // box rows past nkeys are clipped
                            tma_store_4d(&P.tar_st, stg, part * 64, j0 + i, quad * 32, bh * g.gq + a);
                            bulk_commit();
                        }
                    }
                }
                tc_fence_before();
                mbar_arrive(o_free);
                named_sync(1, 128);   // c_R smem reused by the next group
                continue;
            }
            if (!outm) {   // L statistics of row l of column j0 + quad (log2 units, x = S sl2 - c_L log2e)
                if (j0 + quad < g.s2) {
                    const int col = (bh * g.gq + a) * g.s2 + j0 + quad;
                    P.stats[(int64_t)col * P.stats_pitch + l] = m_run;
                    P.stats[(int64_t)col * P.stats_pitch + P.stats_pitch / 2 + l] = 1.f / s_run;
                }
                continue;
            }
            // ---- output of the 4 columns: O[l, v] = O^T_i[v, l] / s_l ----
            // tile rows are contiguous W-token grid rows: token(l, j) = row_base(a,0) + j + l*W
            const uint32_t sinv = smem_u32(stat_sum);
            st_shared_f32(sinv + (quad * 32 + l) * 4, 1.f / s_run);
            named_sync(1, 128);
            const int v = quad * 32 + lane;              // this thread's TMEM lane = value dim
            const int b = bh / g.heads, h = bh % g.heads;
            (void)b;
            (void)h;
            (void)v;
            const int64_t tok0 = row_base(g, true, a, 0) + j0;
            // this warp's output staging (its 32 value dims of each row l) must have been read
            // by the previous group's TMA stores before it is rewritten
            if (lane == 0) bulk_wait_read<0>();
            __syncwarp();
            const int ulast = gi * nch + nch - 1;
            if (lane == 0) TRC(warp + 8, ti, 25);
            for (int i = 0; i < 4; ++i) {
                mbar_wait(&o_done[i], ulast & 1);
                if (lane == 0) TRC(warp + 8, ti, 26);
                tc_fence_after();
                float o[32];
                tmem_ld32(tmem + 4 * kKC + i * 32 + lane_off, o);
                if (lane == 0) TRC(warp + 8, ti, 28);
                float inv[32];
#pragma unroll
                for (int q4 = 0; q4 < 32; q4 += 4) {
                    const float4 t4 = ld_shared_v4f(sinv + (i * 32 + q4) * 4);
                    inv[q4] = t4.x; inv[q4 + 1] = t4.y; inv[q4 + 2] = t4.z; inv[q4 + 3] = t4.w;
                }
                if (j0 + i < g.s2) {
                    // rows l of column j: smem [l][64 B] (this warp's value dims), one TMA store
                    const int ob = kSix ? quad : quad * 4 + i;
                    if (kSix && i > 0) {   // one buffer per warp: the previous column's store read it
                        if (lane == 0) bulk_wait_read<0>();
                        __syncwarp();
                    }
                    const uint32_t stg = smem_u32(smem + ColSmem::kOut + ob * 2048) + lane * 2;
#pragma unroll
                    for (int q = 0; q < 32; ++q) {
                        const __nv_bfloat16 hv = __float2bfloat16_rn(o[q] * inv[q]);
                        asm volatile("st.shared.b16 [%0], %1;" ::"r"(stg + q * 64),
                                     "h"(*reinterpret_cast<const unsigned short*>(&hv))
                                     : "memory");
                    }
                    fence_proxy_async_smem();
                    __syncwarp();
                    if (lane == 0) {
                        const int64_t tok = tok0 + i;
                        tma_store_4d(&tm_out, smem + ColSmem::kOut + ob * 2048, quad * 32,
                                     (int)(tok % g.W), (int)(tok / g.W), bh);
                        bulk_commit();
                    }
                }
                if (lane == 0) TRC(warp + 8, ti, 29);
            }
            tc_fence_before();
            if (lane == 0) TRC(warp + 8, ti, 27);
            mbar_arrive(o_free);
            named_sync(1, 128);   // stat_sum / rb reused by the next group
        }
    }
    if (warp >= 2 && lane == 0) bulk_wait<0>();
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc<512>(tmem);
}
