// Wide column stage (included by mbx_tc.cu): tile plans with s1 > 32 rows per
// tile -- e.g. the (3h, w) plan of the paper's s = 0.97 configuration (s1 = 90)
// and untiled (fh, w) configs -- where stacking four 32-row columns on the TMEM
// lane quadrants (mbx_tc_col.cuh) no longer fits.  Item = (column (b,h,a,j),
// M tile of up to 128 query rows l); per 128-key chunk:
//   MMA_S  S[l, key] = Q_col[l,:] . aL[key,:]            128 x 128 x 128  -> S buffer ch%2
//   softmax (warps 2-5, thread = query row l): bias -c_L, online max with lazy
//   rescaling of its own O row in TMEM, P = 2^(x - m) as bf16 into TMEM
//   MMA_O  O[l, v] += P[l, keys] . Y[keys, v]            128 x 128 x 128  (A = P in TMEM)
// i.e. FlashAttention over the keys (c, k) of one column with the c_L bias.  The softmax
// reads a thread's 128 scores in one TMEM round trip (four loads, one wait) and keeps them
// in registers for the max and the exponentials (two passes over TMEM cost 3-7 % at N=32k)
// (solver.py:192-195 joint softmax; factors.py:124 O = L Y).  mode 1 writes the
// row statistics (max, 1/sum) instead of O (refinements t < T-1).
constexpr int kWideThreads = 192;
constexpr int kWKC = 128;   // keys per chunk
struct WideSmem {
    static constexpr int kQ = 0;                          // Q tile [2][2 d-chunks][128 rows][128 B] (64 KB)
    static constexpr int kRing = 65536;                   // 4 slots x 32 KB: aL / Y chunks [2 d-chunks][128 keys][128 B]
    static constexpr int kC = kRing + 4 * 32768;          // c_L chunks [2][128] f32
    static constexpr int kStage = kC + 1024;              // output staging [4 warps][2] x [32 rows][128 B]
    static constexpr int kBars = kStage + 8 * 4096;
    static constexpr int kNumBars = 24;
    static constexpr int kTmemSlot = kBars + kNumBars * 8;
    static constexpr int kTotal = kTmemSlot + 16;
};
static_assert(WideSmem::kTotal + 1024 <= 232448, "wide column stage exceeds 227 KB of shared memory");
// TMEM: S buffers [0,128) [128,256); P buffers (bf16 pairs) [256,320) [320,384); O [384,512)
constexpr uint32_t kWS = 0, kWP = 256, kWO = 384;

__global__ void __launch_bounds__(kWideThreads, 1)
tc_column_wide(const __grid_constant__ TcParams P, Geometry g, int mode) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + WideSmem::kBars);
    uint64_t* q_full = bars;          // [2]
    uint64_t* q_empty = bars + 2;     // [2]
    uint64_t* r_full = bars + 4;      // [4] ring slots
    uint64_t* r_empty = bars + 8;     // [4]
    uint64_t* c_full = bars + 12;     // [2]
    uint64_t* c_empty = bars + 14;    // [2]  (128 softmax threads)
    uint64_t* s_full = bars + 16;     // [2]
    uint64_t* p_full = bars + 18;     // [2]  (128)
    uint64_t* o_done = bars + 20;     // [2] MMA_O of chunk u completed (barrier u & 1: one phase per
                                      //     two chunks, so a wait can never be two phases behind)
    uint64_t* o_free = bars + 22;     // (128) O rows read out after an item
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + WideSmem::kTmemSlot);
    const int tid = threadIdx.x, lane = tid & 31;
    const int warp = __shfl_sync(0xffffffffu, tid >> 5, 0);   // provably warp-uniform
    const bool outm = mode == 0;
    const int n_mt = (g.s1 + 127) / 128;
    const int nch = (g.nkeys + kWKC - 1) / kWKC;
    const int items = g.bh * g.gq * g.s2 * n_mt;
    const int first = blockIdx.x, stride = gridDim.x;
    const int my_items = first < items ? (items - first + stride - 1) / stride : 0;

    if (tid == 0) {
        tma_prefetch(&P.tw128);
        tma_prefetch(&P.tc128);
        tma_prefetch(&P.tqcw);
        tma_prefetch(&P.toutw);
        for (int i = 0; i < 2; ++i) {
            mbar_init(&q_full[i], 1);
            mbar_init(&q_empty[i], 1);
            mbar_init(&c_full[i], 1);
            mbar_init(&c_empty[i], 128);
            mbar_init(&s_full[i], 1);
            mbar_init(&p_full[i], 128);
        }
        for (int i = 0; i < 4; ++i) {
            mbar_init(&r_full[i], 1);
            mbar_init(&r_empty[i], 1);
        }
        mbar_init(&o_done[0], 1);
        mbar_init(&o_done[1], 1);
        mbar_init(o_free, 128);
        fence_barrier_init();
    }
    if (warp == 0) tmem_alloc<512>(tmem_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    // dependents may start their prologue once every CTA got here; the producer alone waits
    // for the row stage, after its first q-column load (q is final: see mbx_tc_col.cuh)
    pdl_trigger();

    // item -> (column col, M tile mt); column -> (bh, a, j)
    auto decode = [&](int it, int& col, int& mt) {
        const int item = first + it * stride;
        mt = item % n_mt;
        col = item / n_mt;
    };

    // Ring order = MMA order with a one-chunk lookahead when a column has several key chunks:
    // aL(0), then aL(u), Y(u-1) for u >= 1, then Y(U-1) (u = global chunk index over the CTA's
    // items) -- MMA_S of chunk u+1 is issued before MMA_O of chunk u, so the next scores are
    // ready when the softmax finishes a chunk (N=32k raw (1260,26) 0.671 -> 0.566 ms, (3h,w)
    // 0.822 -> 0.759 ms, KV21 (3h,w) 156 -> 146 us; one-chunk columns, e.g. the C2 (3h,w)
    // plan, keep aL(u), Y(u): 46.6 -> 48.2 us with the lookahead).
    const int U = my_items * nch;
    const bool look = nch > 1;
    if (warp == 0) {
        // ------------------------------------------ TMA producer (whole warp, elected lane issues)
        const bool leader = elect_one();
        // the final pass is W's last reader: stream it through L2 without displacing the rest
        const uint64_t w_policy = (P.l2hint & 2) && mode == 0 ? l2_evict_first() : l2_evict_normal();
        uint32_t n = 0;   // ring uses
        auto load_part = [&](int uu, int part) {
            int col, mt;
            decode(uu / nch, col, mt);
            const int k0 = (uu % nch) * kWKC;
            const int sl = n & 3;
            mbar_wait(&r_empty[sl], ((n >> 2) & 1) ^ 1);
            if (leader) {
                mbar_expect_tx(&r_full[sl], 2u * kWKC * 128u);
                uint8_t* dst = smem + WideSmem::kRing + sl * 32768;
                tma_load_4d_hint(dst, &P.tw128, &r_full[sl], 0, k0, 2 * part, col, w_policy);
                tma_load_4d_hint(dst + 16384, &P.tw128, &r_full[sl], 0, k0, 2 * part + 1, col, w_policy);
            }
            __syncwarp();
            ++n;
        };
        for (int u = 0; u < U; ++u) {
            const int it = u / nch, ch = u - it * nch;
            if (ch == 0) {   // the item's Q tile (double-buffered)
                int col, mt;
                decode(it, col, mt);
                const int bh = col / (g.gq * g.s2), a = (col / g.s2) % g.gq, j = col % g.s2;
                const int64_t tok = row_base(g, true, a, 0) + j + (int64_t)mt * 128 * g.W;
                const int wcol = (int)(tok % g.W), wrow = (int)(tok / g.W);
                const int qb = it & 1;
                mbar_wait(&q_empty[qb], ((it >> 1) & 1) ^ 1);
                if (leader) {
                    mbar_expect_tx(&q_full[qb], 2u * 128u * 128u);
                    uint8_t* qd = smem + WideSmem::kQ + qb * 32768;
                    tma_load_4d(qd, &P.tqcw, &q_full[qb], 0, wcol, wrow, bh);
                    tma_load_4d(qd + 16384, &P.tqcw, &q_full[qb], 64, wcol, wrow, bh);
                }
                __syncwarp();
                if (it == 0) pdl_wait();   // W and c_L of the row stage complete and visible
            }
            load_part(u, 0);                                   // aL(u)
            if (outm && look && u > 0) load_part(u - 1, 1);   // Y(u-1)
            if (outm && !look) load_part(u, 1);                // Y(u)
            {   // c_L(u) last: its buffer waits for the softmax of chunk u-2, the W loads must not
                int col, mt;
                decode(it, col, mt);
                const int cb = u & 1;
                mbar_wait(&c_empty[cb], ((u >> 1) & 1) ^ 1);
                if (leader) {
                    mbar_expect_tx(&c_full[cb], kWKC * 4u);
                    tma_load_2d(smem + WideSmem::kC + cb * 512, &P.tc128, &c_full[cb], ch * kWKC, col);
                }
                __syncwarp();
            }
        }
        if (outm && look && U > 0) load_part(U - 1, 1);
    } else if (warp == 1) {
        // ------------------------------------------ MMA issuer: whole warp on warp-uniform
        // state (descriptors in uniform registers), one elected lane issues
        const bool leader = elect_one();
        const uint32_t id_s = idesc_bf16(128, kWKC, false, false);
        const uint32_t id_o = idesc_bf16(128, 128, false, true);
        constexpr uint32_t kHi = (1024u >> 4) | (1u << 14) | (2u << 29);   // SBO 1024, v1, SW128
        auto desc = [](uint32_t lo) { return ((uint64_t)kHi << 32) | lo; };
        const uint32_t q_lo = ((smem_u32(smem + WideSmem::kQ) & 0x3FFFF) >> 4) | (1u << 16);
        const uint32_t ring_lo = (smem_u32(smem + WideSmem::kRing) & 0x3FFFF) >> 4;
        uint32_t n = 0;
        auto issue_s = [&](int u) {
            const int it = u / nch, ch = u - it * nch;
            const int qb = it & 1, sb = u & 1;
            if (ch == 0) mbar_wait(&q_full[qb], (it >> 1) & 1);
            // S buffer sb free: the softmax read S(u-2) before arriving p_full(u-2)
            if (u >= 2) mbar_wait(&p_full[sb], ((u >> 1) - 1) & 1);
            const int sl = n & 3;
            mbar_wait(&r_full[sl], (n >> 2) & 1);
            tc_fence_after();
            if (leader) {
                const uint32_t sq = q_lo + (uint32_t)qb * (32768 >> 4);
                const uint32_t sa = ring_lo + (uint32_t)sl * (32768 >> 4) + (1u << 16);
#pragma unroll
                for (int kk = 0; kk < 8; ++kk)
                    mma_bf16(tmem + kWS + sb * 128, desc(sq + (((kk >> 2) * 16384 + (kk & 3) * 32) >> 4)),
                             desc(sa + (((kk >> 2) * 16384 + (kk & 3) * 32) >> 4)), id_s, kk > 0);
                mma_commit(&s_full[sb]);
                mma_commit(&r_empty[sl]);
                if (ch == nch - 1) mma_commit(&q_empty[qb]);
            }
            __syncwarp();
            ++n;
        };
        auto issue_o = [&](int u) {
            // MMA_O(u): P(u) in TMEM, Y chunk landed; the first chunk of an item
            // overwrites O, which the previous item's epilogue must have read
            const int it = u / nch, ch = u - it * nch;
            const int sb = u & 1;
            mbar_wait(&p_full[sb], (u >> 1) & 1);
            if (ch == 0 && it > 0) mbar_wait(o_free, (it - 1) & 1);
            const int yl = n & 3;
            mbar_wait(&r_full[yl], (n >> 2) & 1);
            tc_fence_after();
            if (leader) {
                const uint32_t sy = ring_lo + (uint32_t)yl * (32768 >> 4) + (16384u >> 4 << 16);
#pragma unroll
                for (int kk = 0; kk < 8; ++kk)   // K = keys 16 kk .. 16 kk + 15; B = Y MN-major (v atoms 16 KB apart)
                    mma_bf16_ts(tmem + kWO, tmem + kWP + sb * 64 + kk * 8, desc(sy + ((kk * 2048) >> 4)), id_o,
                                ch > 0 || kk > 0);
                mma_commit(&r_empty[yl]);
                mma_commit(&o_done[sb]);
            }
            __syncwarp();
            ++n;
        };
        for (int u = 0; u < U; ++u) {
            issue_s(u);
            if (outm && look && u > 0) issue_o(u - 1);
            if (outm && !look) issue_o(u);
        }
        if (outm && look && U > 0) issue_o(U - 1);
    } else if (warp < 6) {
        // ------------------------------------------ softmax (thread = query row l) + output
        const int quad = warp & 3;
        const uint32_t lane_off = (uint32_t)(quad * 32) << 16;
        const float sl2 = g.scale * kLog2e;
        uint8_t* stg_base = smem + WideSmem::kStage + quad * 8192;
        int nstore = 0;
        int u = 0;
        for (int it = 0; it < my_items; ++it) {
            int col, mt;
            decode(it, col, mt);
            const int l = mt * 128 + quad * 32 + lane;   // query row within the tile
            float m_run = -INFINITY, s_run = 0.f;
            for (int ch = 0; ch < nch; ++ch, ++u) {
                const int sb = u & 1, cb = u & 1;
                const int kvalid = min(kWKC, g.nkeys - ch * kWKC);
                const uint32_t cbuf = smem_u32(smem + WideSmem::kC + cb * 512);
                mbar_wait(&c_full[cb], (u >> 1) & 1);
                mbar_wait(&s_full[sb], (u >> 1) & 1);
                tc_fence_after();
                const uint32_t srow = tmem + kWS + sb * 128 + lane_off;
                // one TMEM round trip for the whole 128-key row: x = S sl2 - c_L log2e in registers
                float x[kWKC];
                {
                    uint32_t* xr = reinterpret_cast<uint32_t*>(x);
#pragma unroll
                    for (int q4 = 0; q4 < 4; ++q4) tmem_ld32_nw(srow + q4 * 32, xr + q4 * 32);
                    tmem_wait_ld();
                }
                float mq[4] = {-1e30f, -1e30f, -1e30f, -1e30f};
#pragma unroll
                for (int k4 = 0; k4 < kWKC; k4 += 4) {
                    const float4 c4 = ld_shared_v4f(cbuf + k4 * 4);
                    const float cv[4] = {c4.x, c4.y, c4.z, c4.w};
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        x[k4 + e] = (k4 + e < kvalid) ? fmaf(x[k4 + e], sl2, -cv[e] * kLog2e) : -1e30f;
                        mq[e] = fmaxf(mq[e], x[k4 + e]);
                    }
                }
                const float mx = fmaxf(fmaxf(mq[0], mq[1]), fmaxf(mq[2], mq[3]));
                // lazy online max: keep m_run unless the chunk max exceeds it by > 8 (x 256)
                if (ch == 0) {
                    m_run = mx;
                } else if (mx > m_run + 8.f) {
                    const float fac = ex2(m_run - mx);
                    m_run = mx;
                    s_run *= fac;
                    if (outm) {   // rescale this thread's O row once MMA_O(u-1) finished
                        mbar_wait(&o_done[(u - 1) & 1], ((u - 1) >> 1) & 1);
                        tc_fence_after();
#pragma unroll 1
                        for (int q4 = 0; q4 < 4; ++q4) {
                            float o[32];
                            tmem_ld32(tmem + kWO + lane_off + q4 * 32, o);
#pragma unroll
                            for (int i = 0; i < 32; ++i) o[i] *= fac;
                            tmem_st32(tmem + kWO + lane_off + q4 * 32, o);
                        }
                    }
                }
                // P = 2^(x - m) (0 for padded keys) as bf16 pairs into TMEM
                if (outm && u >= 2) mbar_wait(&o_done[sb], ((u - 2) >> 1) & 1);   // MMA_O(u-2) done with P buffer sb
                float ssum = 0.f;
                {
                    float sq[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
                    for (int q4 = 0; q4 < 4; ++q4) {
                        uint32_t pk[16];
#pragma unroll
                        for (int k2 = 0; k2 < 32; k2 += 2) {
                            const float p0 = ex2(x[q4 * 32 + k2] - m_run), p1 = ex2(x[q4 * 32 + k2 + 1] - m_run);
                            sq[(k2 >> 1) & 3] += p0 + p1;
                            pk[k2 >> 1] = pack_bf16(p0, p1);
                        }
                        if (outm) tmem_st16(tmem + kWP + sb * 64 + lane_off + q4 * 16, pk);
                    }
                    ssum = (sq[0] + sq[1]) + (sq[2] + sq[3]);
                }
                s_run += ssum;
                tc_fence_before();
                mbar_arrive(&c_empty[cb]);
                mbar_arrive(&p_full[sb]);
            }
            const int col_j = col;
            if (!outm) {   // L statistics of row l (log2 units)
                if (l < g.s1) {
                    P.stats[(int64_t)col_j * P.stats_pitch + l] = m_run;
                    P.stats[(int64_t)col_j * P.stats_pitch + P.stats_pitch / 2 + l] = 1.f / s_run;
                }
                continue;
            }
            // output row l: O[l, :] / s_run -> bf16 -> staging -> TMA store (rows at stride W tokens)
            mbar_wait(&o_done[(u - 1) & 1], ((u - 1) >> 1) & 1);
            tc_fence_after();
            const float inv = 1.f / s_run;
            const int bh = col / (g.gq * g.s2), a = (col / g.s2) % g.gq, j = col % g.s2;
            const int l0 = mt * 128 + quad * 32;                 // first row of this warp
            const int nrows = min(32, g.s1 - l0);
            const int64_t tok0 = row_base(g, true, a, 0) + j + (int64_t)l0 * g.W;
#pragma unroll 1
            for (int part = 0; part < 2; ++part) {
                float o[64];
                tmem_ld32(tmem + kWO + lane_off + part * 64, o);
                tmem_ld32(tmem + kWO + lane_off + part * 64 + 32, o + 32);
                if (part == 1) {
                    tc_fence_before();
                    mbar_arrive(o_free);
                }
                if (nrows <= 0) continue;
                if (nrows < 32) {   // partial last warp: direct stores of the valid rows
                    if (lane < nrows) {
                        __nv_bfloat16* dst = reinterpret_cast<__nv_bfloat16*>(P.out) +
                                             (int64_t)bh * P.out_bh_stride + (tok0 + (int64_t)lane * g.W) * P.out_tok_stride +
                                             part * 64;
#pragma unroll
                        for (int cc = 0; cc < 8; ++cc)
                            *reinterpret_cast<uint4*>(dst + cc * 8) =
                                make_uint4(pack_bf16(o[8 * cc] * inv, o[8 * cc + 1] * inv),
                                           pack_bf16(o[8 * cc + 2] * inv, o[8 * cc + 3] * inv),
                                           pack_bf16(o[8 * cc + 4] * inv, o[8 * cc + 5] * inv),
                                           pack_bf16(o[8 * cc + 6] * inv, o[8 * cc + 7] * inv));
                    }
                    continue;
                }
                uint8_t* stg = stg_base + (nstore++ & 1) * 4096;
                if (lane == 0) bulk_wait_read<1>();
                __syncwarp();
                const uint32_t srw = smem_u32(stg) + lane * 128;
#pragma unroll
                for (int cc = 0; cc < 8; ++cc)
                    st_shared_v4(srw + ((cc ^ (lane & 7)) << 4), pack_bf16(o[8 * cc] * inv, o[8 * cc + 1] * inv),
                                 pack_bf16(o[8 * cc + 2] * inv, o[8 * cc + 3] * inv),
                                 pack_bf16(o[8 * cc + 4] * inv, o[8 * cc + 5] * inv),
                                 pack_bf16(o[8 * cc + 6] * inv, o[8 * cc + 7] * inv));
                fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0) {
                    tma_store_4d(&P.toutw, stg, part * 64, (int)(tok0 % g.W), (int)(tok0 / g.W), bh);
                    bulk_commit();
                }
            }
        }
        if (lane == 0) bulk_wait<0>();
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc<512>(tmem);
}
