// Wide column stage, ping-pong variant (included by mbx_tc.cu).  mode 0: O = L Y;
// mode 1 (refinements t < T-1): the row statistics (max, 1/sum) of L only, no Y, no O.
// Same FlashAttention over the keys (c, k) of one column as tc_column_wide
// (mbx_tc_colw.cuh, solver.py:192-195 joint softmax with bias -c_L, factors.py:124
// O = L Y), with two item streams per CTA so one softmax warpgroup's exponentials
// overlap the other's score MMA: the CTA's items alternate between streams s = 0, 1;
// stream s owns TMEM columns [256 s, 256 s + 256) -- S (fp32, 128 columns) with P
// written over it in place as packed bf16, then O (128 columns) -- and softmax warps
// 4 + 4 s .. 7 + 4 s.
//
// One global step list interleaves the streams' chunks, (s0,c0) (s1,c0) (s0,c1) ...;
// the MMA warp issues MMA_S of step k before MMA_O of step k-1 unless both belong to
// the same stream (then O first: S overwrites that stream's P).  A commit after MMA_S
// of a stream's chunk c therefore also covers its MMA_O of chunk c-1, so the softmax
// may rescale O and overwrite P as soon as it sees the new scores.  The producer
// loads in exactly the MMA order (aL for S, Y for O) through one 3-slot ring.
// Warpgroups: [producer, MMA, 2 idle] at 48 registers, then one softmax / output
// warpgroup per stream at 224 (setmaxnreg), so the 128-score rows stay in registers.
constexpr int kW2Threads = 384;
struct Wide2Smem {
    static constexpr int kQ = 0;                    // Q tiles [2 streams][2 d-chunks][128 rows][128 B] (64 KB)
    static constexpr int kNRing = 3;
    static constexpr int kRing = 65536;             // aL / Y chunks [slot][2 d-chunks][128 keys][128 B] (32 KB)
    static constexpr int kC = kRing + kNRing * 32768;   // c_L [2 streams][2 buffers][128] f32
    static constexpr int kStage = kC + 4 * 512;     // output staging [8 warps][32 rows][128 B]
    static constexpr int kBars = kStage + 8 * 4096;
    static constexpr int kNumBars = 2 * kNRing + 2 * 10;
    static constexpr int kTmemSlot = kBars + kNumBars * 8;
    static constexpr int kTotal = kTmemSlot + 16;
};
static_assert(Wide2Smem::kTotal + 1024 <= 232448, "ping-pong wide column stage exceeds 227 KB of shared memory");

// Step k of the interleaved list -> (stream, chunk index within the stream).
struct W2Steps {
    int u0, u1, m;   // chunks of each stream, min of both
    __device__ __forceinline__ void at(int k, int& s, int& c) const {
        if (k < 2 * m) {
            s = k & 1;
            c = k >> 1;
        } else {
            s = u0 > u1 ? 0 : 1;
            c = m + (k - 2 * m);
        }
    }
    __device__ __forceinline__ int total() const { return u0 + u1; }
};

template <int mode>
__global__ void __launch_bounds__(kW2Threads, 1)
tc_column_wide2(const __grid_constant__ TcParams P, Geometry g) {
    constexpr bool outm = mode == 0;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + Wide2Smem::kBars);
    uint64_t* r_full = bars;                         // [3] ring slots
    uint64_t* r_empty = bars + Wide2Smem::kNRing;    // [3]
    uint64_t* sb = bars + 2 * Wide2Smem::kNRing;     // per stream s: 10 barriers at sb + 10 s
    auto q_full = [&](int s) { return sb + 10 * s + 0; };
    auto q_empty = [&](int s) { return sb + 10 * s + 1; };
    auto s_full = [&](int s) { return sb + 10 * s + 2; };
    auto p_full = [&](int s) { return sb + 10 * s + 3; };    // 128 softmax threads
    auto o_full = [&](int s) { return sb + 10 * s + 4; };    // last MMA_O of an item done
    auto o_free = [&](int s) { return sb + 10 * s + 5; };    // 128: O read out after an item
    auto c_full = [&](int s, int b) { return sb + 10 * s + 6 + b; };
    auto c_empty = [&](int s, int b) { return sb + 10 * s + 8 + b; };   // 128
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + Wide2Smem::kTmemSlot);
    const int tid = threadIdx.x, lane = tid & 31;
    const int warp = __shfl_sync(0xffffffffu, tid >> 5, 0);   // provably warp-uniform
    const int n_mt = (g.s1 + 127) / 128;
    const int nch = (g.nkeys + kWKC - 1) / kWKC;
    const int items = g.bh * g.gq * g.s2 * n_mt;
    const int first = blockIdx.x, stride = gridDim.x;
    const int my_items = first < items ? (items - first + stride - 1) / stride : 0;
    W2Steps steps;
    steps.u0 = ((my_items + 1) / 2) * nch;   // stream 0: items 0, 2, 4, ...
    steps.u1 = (my_items / 2) * nch;         // stream 1: items 1, 3, 5, ...
    steps.m = steps.u0 < steps.u1 ? steps.u0 : steps.u1;
    const int K = steps.total();

    if (tid == 0) {
        tma_prefetch(&P.tw128);
        tma_prefetch(&P.tc128);
        tma_prefetch(&P.tqcw);
        tma_prefetch(&P.toutw);
        for (int i = 0; i < Wide2Smem::kNRing; ++i) {
            mbar_init(&r_full[i], 1);
            mbar_init(&r_empty[i], 1);
        }
        for (int s = 0; s < 2; ++s) {
            mbar_init(q_full(s), 1);
            mbar_init(q_empty(s), 1);
            mbar_init(s_full(s), 1);
            mbar_init(p_full(s), 128);
            mbar_init(o_full(s), 1);
            mbar_init(o_free(s), 128);
            for (int b = 0; b < 2; ++b) {
                mbar_init(c_full(s, b), 1);
                mbar_init(c_empty(s, b), 128);
            }
        }
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

    // item of stream s, its i-th -> (column col, M tile mt)
    auto decode = [&](int s, int i, int& col, int& mt) {
        const int item = first + (s + 2 * i) * stride;
        mt = item % n_mt;
        col = item / n_mt;
    };
    // the op sequence shared by producer and MMA issuer: S(k) preceded by O(k-1) when both
    // are of one stream, followed by it otherwise; visit(is_o, step)
    auto schedule = [&](auto&& visit) {
        if (!outm) {   // statistics: score MMAs only
            for (int k = 0; k < K; ++k) visit(false, k);
            return;
        }
        int pending = -1, ps = -1;
        for (int k = 0; k < K; ++k) {
            int s, c;
            steps.at(k, s, c);
            if (pending >= 0 && ps == s) {
                visit(true, pending);
                pending = -1;
            }
            visit(false, k);
            if (pending >= 0) visit(true, pending);
            pending = k;
            ps = s;
        }
        if (pending >= 0) visit(true, pending);
    };

    if (warp < 4) {
      reg_dealloc<48>();
      if (warp == 0) {
        // ------------------------------------------ TMA producer (whole warp, elected lane issues)
        const bool leader = elect_one();
        const uint64_t w_policy = (P.l2hint & 2) && outm ? l2_evict_first() : l2_evict_normal();   // W's last reader
        uint32_t n = 0;   // ring uses
        bool waited = false;
        schedule([&](bool is_o, int k) {
            int s, c;
            steps.at(k, s, c);
            const int i = c / nch, ch = c - i * nch;
            int col, mt;
            decode(s, i, col, mt);
            if (!is_o && ch == 0) {   // the item's Q tile
                const int bh = col / (g.gq * g.s2), a = (col / g.s2) % g.gq, j = col % g.s2;
                const int64_t tok = row_base(g, true, a, 0) + j + (int64_t)mt * 128 * g.W;
                const int wcol = (int)(tok % g.W), wrow = (int)(tok / g.W);
                mbar_wait(q_empty(s), (i & 1) ^ 1);
                if (leader) {
                    mbar_expect_tx(q_full(s), 2u * 128u * 128u);
                    uint8_t* qd = smem + Wide2Smem::kQ + s * 32768;
                    tma_load_4d(qd, &P.tqcw, q_full(s), 0, wcol, wrow, bh);
                    tma_load_4d(qd + 16384, &P.tqcw, q_full(s), 64, wcol, wrow, bh);
                }
                __syncwarp();
                if (!waited) {
                    pdl_wait();   // W and c_L of the row stage complete and visible
                    waited = true;
                }
            }
            const int sl = n % Wide2Smem::kNRing;
            mbar_wait(&r_empty[sl], ((n / Wide2Smem::kNRing) & 1) ^ 1);
            if (leader) {
                const int part = is_o ? 1 : 0;   // aL for MMA_S, Y for MMA_O
                mbar_expect_tx(&r_full[sl], 2u * kWKC * 128u);
                uint8_t* dst = smem + Wide2Smem::kRing + sl * 32768;
                tma_load_4d_hint(dst, &P.tw128, &r_full[sl], 0, ch * kWKC, 2 * part, col, w_policy);
                tma_load_4d_hint(dst + 16384, &P.tw128, &r_full[sl], 0, ch * kWKC, 2 * part + 1, col, w_policy);
            }
            __syncwarp();
            ++n;
            if (!is_o) {   // c_L of the chunk, after its aL (its buffer waits for the softmax)
                const int cb = c & 1;
                mbar_wait(c_empty(s, cb), ((c >> 1) & 1) ^ 1);
                if (leader) {
                    mbar_expect_tx(c_full(s, cb), kWKC * 4u);
                    tma_load_2d(smem + Wide2Smem::kC + (s * 2 + cb) * 512, &P.tc128, c_full(s, cb), ch * kWKC, col);
                }
                __syncwarp();
            }
        });
    } else if (warp == 1) {
        // ------------------------------------------ MMA issuer (whole warp, uniform descriptors)
        const bool leader = elect_one();
        const uint32_t id_s = idesc_bf16(128, kWKC, false, false);
        const uint32_t id_o = idesc_bf16(128, 128, false, true);
        constexpr uint32_t kHi = (1024u >> 4) | (1u << 14) | (2u << 29);   // SBO 1024, v1, SW128
        auto desc = [](uint32_t lo) { return ((uint64_t)kHi << 32) | lo; };
        const uint32_t q_lo = ((smem_u32(smem + Wide2Smem::kQ) & 0x3FFFF) >> 4) | (1u << 16);
        const uint32_t ring_lo = (smem_u32(smem + Wide2Smem::kRing) & 0x3FFFF) >> 4;
        uint32_t n = 0;
        schedule([&](bool is_o, int k) {
            int s, c;
            steps.at(k, s, c);
            const int i = c / nch, ch = c - i * nch;
            const uint32_t sp = tmem + (uint32_t)s * 256;   // S / P of stream s; O at + 128
            const int sl = n % Wide2Smem::kNRing;
            if (!is_o) {
                if (ch == 0) mbar_wait(q_full(s), i & 1);
                // statistics mode has no MMA_O between a stream's score MMAs: S(c) may only
                // overwrite S(c-1) once the softmax read it
                if (!outm && c > 0) mbar_wait(p_full(s), (c - 1) & 1);
                mbar_wait(&r_full[sl], (n / Wide2Smem::kNRing) & 1);
                tc_fence_after();
                if (leader) {
                    const uint32_t sq = q_lo + (uint32_t)s * (32768 >> 4);
                    const uint32_t sa = ring_lo + (uint32_t)sl * (32768 >> 4) + (1u << 16);
#pragma unroll
                    for (int kk = 0; kk < 8; ++kk)
                        mma_bf16(sp, desc(sq + (((kk >> 2) * 16384 + (kk & 3) * 32) >> 4)),
                                 desc(sa + (((kk >> 2) * 16384 + (kk & 3) * 32) >> 4)), id_s, kk > 0);
                    mma_commit(s_full(s));
                    mma_commit(&r_empty[sl]);
                    if (ch == nch - 1) mma_commit(q_empty(s));
                }
            } else {
                // P(c) written; the first chunk of an item overwrites O, read out by then
                mbar_wait(p_full(s), c & 1);
                if (ch == 0 && i > 0) mbar_wait(o_free(s), (i - 1) & 1);
                mbar_wait(&r_full[sl], (n / Wide2Smem::kNRing) & 1);
                tc_fence_after();
                if (leader) {
                    const uint32_t sy = ring_lo + (uint32_t)sl * (32768 >> 4) + (16384u >> 4 << 16);
#pragma unroll
                    for (int kk = 0; kk < 8; ++kk)   // K = keys 16 kk .. 16 kk + 15; B = Y MN-major
                        mma_bf16_ts(sp + 128, sp + kk * 8, desc(sy + ((kk * 2048) >> 4)), id_o, ch > 0 || kk > 0);
                    mma_commit(&r_empty[sl]);
                    if (ch == nch - 1) mma_commit(o_full(s));
                }
            }
            __syncwarp();
            ++n;
        });
      }
    } else {
        reg_alloc<224>();
        // ------------------------------------------ softmax (thread = query row l) + output, stream s
        const int s = (warp - 4) >> 2;
        const int quad = warp & 3;
        const uint32_t lane_off = (uint32_t)(quad * 32) << 16;
        const uint32_t sp = tmem + (uint32_t)s * 256 + lane_off;
        const float sl2 = g.scale * kLog2e;
        uint8_t* stg = smem + Wide2Smem::kStage + (warp - 4) * 4096;
        const int n_items = s == 0 ? (my_items + 1) / 2 : my_items / 2;
        int c = 0;
        for (int i = 0; i < n_items; ++i) {
            int col, mt;
            decode(s, i, col, mt);
            const int l = mt * 128 + quad * 32 + lane;   // query row within the tile
            float m_run = -INFINITY, s_run = 0.f;
            for (int ch = 0; ch < nch; ++ch, ++c) {
                const int cb = c & 1;
                const int kvalid = min(kWKC, g.nkeys - ch * kWKC);
                const uint32_t cbuf = smem_u32(smem + Wide2Smem::kC + (s * 2 + cb) * 512);
                mbar_wait(c_full(s, cb), (c >> 1) & 1);
                mbar_wait(s_full(s), c & 1);   // also: MMA_O of chunk c-1 is done (commit order)
                tc_fence_after();
                float x[kWKC];
                {
                    uint32_t* xr = reinterpret_cast<uint32_t*>(x);
#pragma unroll
                    for (int q4 = 0; q4 < 4; ++q4) tmem_ld32_nw(sp + q4 * 32, xr + q4 * 32);
                    tmem_wait_ld();
                }
                if (!outm) {   // scores in registers: the next score MMA of this stream may start
                    tc_fence_before();
                    mbar_arrive(p_full(s));
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
#pragma unroll 1
                    for (int q4 = 0; q4 < (outm ? 4 : 0); ++q4) {   // this thread's O row
                        float o[32];
                        tmem_ld32(sp + 128 + q4 * 32, o);
#pragma unroll
                        for (int e = 0; e < 32; ++e) o[e] *= fac;
                        tmem_st32(sp + 128 + q4 * 32, o);
                    }
                }
                // P = 2^(x - m) (0 for padded keys) as bf16 pairs over the first 64 S columns
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
                    if (outm) tmem_st16(sp + q4 * 16, pk);
                }
                s_run += (sq[0] + sq[1]) + (sq[2] + sq[3]);
                tc_fence_before();
                mbar_arrive(c_empty(s, cb));
                if (outm) mbar_arrive(p_full(s));
            }
            if (!outm) {   // L statistics of row l (log2 units)
                if (l < g.s1) {
                    P.stats[(int64_t)col * P.stats_pitch + l] = m_run;
                    P.stats[(int64_t)col * P.stats_pitch + P.stats_pitch / 2 + l] = 1.f / s_run;
                }
                continue;
            }
            // output row l: O[l, :] / s_run -> bf16 -> staging -> TMA store (rows at stride W tokens)
            mbar_wait(o_full(s), i & 1);
            tc_fence_after();
            const float inv = 1.f / s_run;
            const int bh = col / (g.gq * g.s2), a = (col / g.s2) % g.gq, j = col % g.s2;
            const int l0 = mt * 128 + quad * 32;                 // first row of this warp
            const int nrows = min(32, g.s1 - l0);
            const int64_t tok0 = row_base(g, true, a, 0) + j + (int64_t)l0 * g.W;
            float o[2][64];
#pragma unroll
            for (int part = 0; part < 2; ++part) {
                uint32_t* orr = reinterpret_cast<uint32_t*>(o[part]);
                tmem_ld32_nw(sp + 128 + part * 64, orr);
                tmem_ld32_nw(sp + 128 + part * 64 + 32, orr + 32);
            }
            tmem_wait_ld();
            tc_fence_before();
            mbar_arrive(o_free(s));
            if (nrows <= 0) continue;
#pragma unroll
            for (int part = 0; part < 2; ++part) {
                if (nrows < 32) {   // partial last warp: direct stores of the valid rows
                    if (lane < nrows) {
                        __nv_bfloat16* dst = reinterpret_cast<__nv_bfloat16*>(P.out) + (int64_t)bh * P.out_bh_stride +
                                             (tok0 + (int64_t)lane * g.W) * P.out_tok_stride + part * 64;
#pragma unroll
                        for (int cc = 0; cc < 8; ++cc)
                            *reinterpret_cast<uint4*>(dst + cc * 8) =
                                make_uint4(pack_bf16(o[part][8 * cc] * inv, o[part][8 * cc + 1] * inv),
                                           pack_bf16(o[part][8 * cc + 2] * inv, o[part][8 * cc + 3] * inv),
                                           pack_bf16(o[part][8 * cc + 4] * inv, o[part][8 * cc + 5] * inv),
                                           pack_bf16(o[part][8 * cc + 6] * inv, o[part][8 * cc + 7] * inv));
                    }
                    continue;
                }
                if (lane == 0) bulk_wait_read<0>();   // the previous store from the buffer has read it
                __syncwarp();
                const uint32_t srw = smem_u32(stg) + lane * 128;
#pragma unroll
                for (int cc = 0; cc < 8; ++cc)
                    st_shared_v4(srw + ((cc ^ (lane & 7)) << 4), pack_bf16(o[part][8 * cc] * inv, o[part][8 * cc + 1] * inv),
                                 pack_bf16(o[part][8 * cc + 2] * inv, o[part][8 * cc + 3] * inv),
                                 pack_bf16(o[part][8 * cc + 4] * inv, o[part][8 * cc + 5] * inv),
                                 pack_bf16(o[part][8 * cc + 6] * inv, o[part][8 * cc + 7] * inv));
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
