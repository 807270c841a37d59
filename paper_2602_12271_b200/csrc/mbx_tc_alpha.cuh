// alpha_R stage (included by mbx_tc.cu): the hand-off from refinement t to
// t + 1 when T >= 2 (solver.py:185-186 at the next iteration):
//     alpha_R[c,k,j,:] = sum_l L[l,(c,k)] Q[a,l,j,:],   c_R[c,k,j] = sum_l L[l,(c,k)]
// written normalised, hat_alpha_R = alpha_R / max(c_R, eps_div) (bf16), so the next
// row stage computes z = scale * hat_alpha_R . K exactly like the first one with Q.
//
// Item = (column (b,h,a,j), chunk of 128 keys).  Keys sit on the TMEM lanes:
//   MMA1  S^T[key, l] = aL[key,:] . Q_col[l,:]          128 x s1p x 128   (s1p = s1 rounded to 32, <= 128)
//   P^T[key, l] = 2^(S^T sl2 - c_L log2e - m_l) / sum_l  (row statistics from the column
//   stage's statistics pass), c_R = sum_l P^T -- both thread-local (one key per thread)
//   MMA2  alpha_R[key, :] = P^T . Q_col                  128 x 128 x s1p
//   epilogue: / max(c_R, eps) -> bf16 -> staging -> TMA store into
//   hat_alpha_R[bh][a][key][j][128] (the next row stage's A rows).
// mode 1 (factor export after the last refinement's statistics pass): only the
// normalised P^T = L is needed; each thread writes its key's L[l] for every query
// row l straight into L' (c1_q, c2, c1_kv, c2, s2, s1, s1) (factors.py:57-79) and
// MMA2 / the alpha_R epilogue are skipped.
#ifndef MBX_ALPHA_PP
#define MBX_ALPHA_PP 1
#endif
// MBX_ALPHA_PP: two softmax / epilogue warpgroups, items alternating (warpgroup b owns the
// S^T / D2 / P^T buffers of parity b), so one item's epilogue overlaps the next's softmax;
// the epilogue stages its stores in the item's own P^T buffer, which MMA2 has finished with
#ifndef MBX_ALPHA_IL
#define MBX_ALPHA_IL 1   // interleave the steps of item pairs (build option, for A/B)
#endif
constexpr int kAlphaThreads = MBX_ALPHA_PP ? 320 : 192;   // producer, MMA, (1 or 2) x 4 softmax / epilogue
constexpr int kAKC = 128;            // keys per item
struct AlphaSmem {
    // per buffer b (2): aL [2 d-chunks][128 keys][128 B] (32 KB), Q_col [2 d-chunks][128 l][128 B]
    // (32 KB), P^T [2 l-chunks][128 keys][128 B] (32 KB), c_L [128] f32 (1 KB slot)
    static constexpr int kA = 0, kQc = 32768, kP = 65536, kC = 98304;
    static constexpr int kBuf = kC + 1024;               // keeps buffer 1 on a 1024 B (SW128) boundary
    static constexpr int kStage = 2 * kBuf;              // [4 warps] x [32 keys][64] bf16 (one slot each)
    static constexpr int kBars = kStage + 4 * 4096;
    static constexpr int kNumBars = 12;
    static constexpr int kTmemSlot = kBars + kNumBars * 8;
    static constexpr int kTotal = kTmemSlot + 16;
};
static_assert(AlphaSmem::kTotal + 1024 <= 232448, "alpha_R stage exceeds 227 KB of shared memory");

__global__ void __launch_bounds__(kAlphaThreads, 1)
tc_alpha_r_stage(const __grid_constant__ TcParams P, Geometry g, int mode) {
    const bool lexp = mode == 1;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + AlphaSmem::kBars);
    uint64_t* ld_full = bars;        // [2]
    uint64_t* ld_empty = bars + 2;   // [2]  MMA2 done with the buffer
    uint64_t* s_full = bars + 4;     // [2]
    uint64_t* p_full = bars + 6;     // [2]  128 softmax threads wrote P^T, read S^T
    uint64_t* o_full = bars + 8;     // [2]  (D2 buffer b; drained before the next s_full of b)
    uint64_t* p_empty = bars + 10;   // [2]  MMA2 of a step done reading P^T (rows l beyond 128: next step)
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + AlphaSmem::kTmemSlot);
    const int tid = threadIdx.x, lane = tid & 31;
    const int warp = __shfl_sync(0xffffffffu, tid >> 5, 0);   // provably warp-uniform
    const int nch = (g.nkeys + kAKC - 1) / kAKC;
    const int items = g.bh * g.gq * g.s2 * nch;
    const int first = blockIdx.x, stride = gridDim.x;
    const int my_items = first < items ? (items - first + stride - 1) / stride : 0;

    if (tid == 0) {
        tma_prefetch(&P.tw128);
        tma_prefetch(&P.tc128);
        tma_prefetch(&P.tqa);
        tma_prefetch(&P.tar_st);
        for (int i = 0; i < 2; ++i) {
            mbar_init(&ld_full[i], 1);
            mbar_init(&ld_empty[i], 1);
            mbar_init(&s_full[i], 1);
            mbar_init(&p_full[i], 128);
            mbar_init(&o_full[i], 1);
            mbar_init(&p_empty[i], 1);
        }
        fence_barrier_init();
    }
    // l padded to s1p (multiple of 32): Q_col rows >= s1 (TMA loads s1p rows: finite data or OOB
    // zeros) meet P^T columns that are written as zeros below, so nothing needs pre-zeroing.
    // Rows l beyond 128 (untiled / misaligned plans) run in steps of 128 l per item: S^T, P^T and
    // Q_col per step, alpha_R accumulated in D2 across the steps, c_R in registers.
    const int s1p = ((g.s1 + 31) / 32) * 32;
    const int nlc = (s1p + 127) / 128;                  // l steps per item
    auto step_l = [&](int lc) { return min(128, s1p - lc * 128); };   // rows l of step lc
    if (warp == 0) tmem_alloc<512>(tmem_slot);
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;   // S^T buffers at 128 b, D2 buffers at 256 + 128 b
    pdl_trigger();   // dependents may start their prologue once every CTA got here
    pdl_wait();      // predecessor kernels (previous stage) complete and visible

    auto decode = [&](int it, int& col, int& ch) {
        const int item = first + it * stride;
        ch = item % nch;
        col = item / nch;
    };
    // Step order of the producer and the MMA warp: with two softmax warpgroups the steps of
    // items 2g and 2g+1 interleave ((2g,0), (2g+1,0), (2g,1), ...), so one item's softmax,
    // Q load and MMA2 overlap the other's; a trailing odd item runs alone.
    const int nsteps = my_items * nlc;
    auto seq = [&](int q, int& it, int& lc) {
        const int paired = MBX_ALPHA_PP && MBX_ALPHA_IL ? (my_items & ~1) * nlc : 0;
        if (q < paired) {
            const int r = q % (2 * nlc);
            it = 2 * (q / (2 * nlc)) + (r & 1);
            lc = r >> 1;
        } else {
            const int q2 = q - paired;
            it = (paired / nlc) + q2 / nlc;
            lc = q2 % nlc;
        }
    };

    if (warp == 0) {
        // ------------------------------------------ TMA producer (whole warp, elected lane issues)
        const bool leader = elect_one();
        for (int q = 0; q < nsteps; ++q) {
            int it, lc, col, ch;
            seq(q, it, lc);
            decode(it, col, ch);
            const int b = it & 1;
            const int bh = col / (g.gq * g.s2), a = (col / g.s2) % g.gq, j = col % g.s2;
            const int64_t tok = row_base(g, true, a, 0) + j;
            const int wcol = (int)(tok % g.W), wrow = (int)(tok / g.W);
            {
                const int sidx = (it >> 1) * nlc + lc;   // step of buffer b
                mbar_wait(&ld_empty[b], (sidx & 1) ^ 1);
                if (leader) {
                    uint8_t* base = smem + b * AlphaSmem::kBuf;
                    // q columns: one box of min(s1p, 128) rows (tensor map P.tqa) per step -- a
                    // full box even on the last step (rows past the column are zero-filled, and
                    // MMA1's N / MMA2's K stop at the step's rows)
                    const uint32_t qbytes = 2u * (uint32_t)(s1p < 128 ? s1p : 128) * 128u;
                    mbar_expect_tx(&ld_full[b], qbytes + (lc == 0 ? 2u * kAKC * 128u + kAKC * 4u : 0u));
                    if (lc == 0) {
                        tma_load_4d(base + AlphaSmem::kA, &P.tw128, &ld_full[b], 0, ch * kAKC, 0, col);
                        tma_load_4d(base + AlphaSmem::kA + 16384, &P.tw128, &ld_full[b], 0, ch * kAKC, 1, col);
                        tma_load_2d(base + AlphaSmem::kC, &P.tc128, &ld_full[b], ch * kAKC, col);
                    }
                    tma_load_4d(base + AlphaSmem::kQc, &P.tqa, &ld_full[b], 0, wcol, wrow + lc * 128, bh);
                    tma_load_4d(base + AlphaSmem::kQc + 16384, &P.tqa, &ld_full[b], 64, wcol, wrow + lc * 128, bh);
                }
                __syncwarp();
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------ MMA issuer (whole warp, uniform descriptors)
        const bool leader = elect_one();
        const uint32_t id2 = idesc_bf16(128, 128, false, true);
        constexpr uint32_t kHi = (1024u >> 4) | (1u << 14) | (2u << 29);   // SBO 1024, v1, SW128
        auto desc = [](uint32_t lo) { return ((uint64_t)kHi << 32) | lo; };
        const uint32_t base_lo = (smem_u32(smem) & 0x3FFFF) >> 4;
        // MMA2 of step (it, lc), once the softmax wrote its P^T (and D2 buffer b was drained by
        // item it-2's epilogue, which the softmax threads finish before arriving on p_full)
        auto mma2 = [&](int it, int lc) {
            const int b = it & 1;
            const uint32_t lo = base_lo + (uint32_t)b * (AlphaSmem::kBuf >> 4);
            const int sidx = (it >> 1) * nlc + lc;
            const int nl = step_l(lc);
            mbar_wait(&p_full[b], sidx & 1);
            tc_fence_after();
            if (leader && lexp) {   // L export: no alpha_R product (and no o_full: nobody drains D2)
                mma_commit(&ld_empty[b]);
                if (lc < nlc - 1) mma_commit(&p_empty[b]);   // waited by the item's next step only
            } else if (leader) {
                for (int kk = 0; kk < nl / 16; ++kk)   // K = l: A = P^T (K-major, 64-l chunks 16 KB apart)
                    mma_bf16(tmem + 256 + b * 128,
                             desc(lo + ((AlphaSmem::kP + (kk >> 2) * 16384 + (kk & 3) * 32) >> 4) + (1u << 16)),
                             desc(lo + ((AlphaSmem::kQc + kk * 2048) >> 4) + (16384u >> 4 << 16)), id2,
                             lc > 0 || kk > 0);
                if (lc == nlc - 1) mma_commit(&o_full[b]);
                mma_commit(&ld_empty[b]);
                if (lc < nlc - 1) mma_commit(&p_empty[b]);
            }
            __syncwarp();
        };
        // MMA1 of step q is issued before MMA2 of step q-1 (software pipeline over the step
        // order), unless both use the same buffer: its next Q load waits for that MMA2
        int pit = -1, plc = 0;
        for (int q = 0; q < nsteps; ++q) {
            int it, lc;
            seq(q, it, lc);
            const int b = it & 1;
            if (pit >= 0 && (!MBX_ALPHA_IL || (pit & 1) == b)) {
                mma2(pit, plc);
                pit = -1;
            }
            const uint32_t lo = base_lo + (uint32_t)b * (AlphaSmem::kBuf >> 4);
            const int sidx = (it >> 1) * nlc + lc;
            const int nl = step_l(lc);
            // wait for this step's loads and a free S^T buffer b (the softmax read the previous
            // step's S^T: p_full precedes it); the pending MMA2 goes first if its P^T is ready
            // meanwhile, so the next load into its buffer never waits behind this step's loads
            for (;;) {
                if (pit >= 0 && mbar_test_uniform(&p_full[pit & 1], ((((pit >> 1) * nlc) + plc) & 1))) {
                    mma2(pit, plc);
                    pit = -1;
                }
                if (mbar_test_uniform(&ld_full[b], sidx & 1) &&
                    (sidx < 1 || mbar_test_uniform(&p_full[b], (sidx - 1) & 1)))
                    break;
            }
            tc_fence_after();
            if (leader) {
                const uint32_t id1 = idesc_bf16(128, nl, false, false);
#pragma unroll
                for (int kk = 0; kk < 8; ++kk)
                    mma_bf16(tmem + b * 128, desc(lo + ((AlphaSmem::kA + (kk >> 2) * 16384 + (kk & 3) * 32) >> 4) + (1u << 16)),
                             desc(lo + ((AlphaSmem::kQc + (kk >> 2) * 16384 + (kk & 3) * 32) >> 4) + (1u << 16)), id1,
                             kk > 0);
                mma_commit(&s_full[b]);
            }
            __syncwarp();
            if (pit >= 0) mma2(pit, plc);
            pit = it;
            plc = lc;
        }
        if (pit >= 0) mma2(pit, plc);
    } else if (warp < kAlphaThreads / 32) {
        // ------------------------------------------ softmax (thread = key) + epilogue
        const int quad = warp & 3;
        const int r = quad * 32 + lane;   // key within the chunk
        const uint32_t lane_off = (uint32_t)(quad * 32) << 16;
        const float sl2 = g.scale * kLog2e;
        const int wgi = MBX_ALPHA_PP ? (warp - 2) >> 2 : 0;
        for (int it = wgi; it < my_items; it += (MBX_ALPHA_PP ? 2 : 1)) {
            int col, ch;
            decode(it, col, ch);
            const int b = it & 1;
            uint8_t* base = smem + b * AlphaSmem::kBuf;
            // epilogue staging: in the two-warpgroup layout the warp's own P^T rows of the item's
            // buffer (4 KB in each 64-l chunk: only this warp writes them), else a 4 KB slot per warp
            uint8_t* stg_base = MBX_ALPHA_PP ? base + AlphaSmem::kP + quad * 4096 : smem + AlphaSmem::kStage + quad * 4096;
            if (MBX_ALPHA_PP) {   // this warp's stores from the buffer (item it-2) have read it
                if (lane == 0) bulk_wait_read<0>();
                __syncwarp();
            }
            const int key = ch * kAKC + r;
            const bool key_ok = key < g.nkeys;
            // row statistics of this column (written by the statistics pass)
            const float* st = P.stats + (int64_t)col * P.stats_pitch;
            float cr = 0.f;
            float cl = 0.f;
            const uint32_t prow = smem_u32(base + AlphaSmem::kP) + r * 128;
            // L' row of this key: [bh][a][c][j][l][k] with key = c s1 + k
            float* lrow = nullptr;
            if (P.lfac && key_ok) {
                const int bh = col / (g.gq * g.s2), a = (col / g.s2) % g.gq, j = col % g.s2;
                const int c = key / g.s1, kk = key - c * g.s1;
                lrow = P.lfac + ((((int64_t)(bh * g.gq + a) * g.gk + c) * g.s2 + j) * g.s1) * g.s1 + kk;
            }
            for (int lc = 0; lc < nlc; ++lc) {
                const int sidx = (it >> 1) * nlc + lc;
                const int nl = step_l(lc);
                mbar_wait(&s_full[b], sidx & 1);
                tc_fence_after();
                if (lc == 0) cl = reinterpret_cast<const float*>(base + AlphaSmem::kC)[r] * kLog2e;
                // P^T of the previous step read by its MMA2 (the first step's region was last
                // read by item it-2's MMA2, complete before that item's epilogue)
                if (lc > 0) mbar_wait(&p_empty[b], ((it >> 1) * (nlc - 1) + lc - 1) & 1);
                for (int l0 = 0; l0 < nl; l0 += 32) {   // 32 query rows l per pass
                    float x[32];
                    tmem_ld32(tmem + b * 128 + lane_off + l0, x);
                    float p[32];
#pragma unroll
                    for (int i = 0; i < 32; ++i) {
                        const int l = lc * 128 + l0 + i;
                        const float e = ex2(fmaf(x[i], sl2, -cl) - __ldg(st + l)) * __ldg(st + P.stats_pitch / 2 + l);
                        p[i] = (l < g.s1 && key_ok) ? e : 0.f;
                        cr += p[i];
                    }
                    if (lrow) {
#pragma unroll
                        for (int i = 0; i < 32; ++i)
                            if (lc * 128 + l0 + i < g.s1) lrow[(int64_t)(lc * 128 + l0 + i) * g.s1] = p[i];
                    }
                    if (lexp) continue;
                    // P^T row (keys on rows, l along K): 64-l chunk l0 / 64, logical 16 B chunks (l0 % 64) / 8 ..
                    const uint32_t pr = prow + (l0 >> 6) * 16384;
#pragma unroll
                    for (int cc = 0; cc < 4; ++cc) {
                        const int lq = ((l0 & 63) >> 3) + cc;
                        st_shared_v4(pr + ((lq ^ (r & 7)) << 4), pack_bf16(p[8 * cc], p[8 * cc + 1]),
                                     pack_bf16(p[8 * cc + 2], p[8 * cc + 3]), pack_bf16(p[8 * cc + 4], p[8 * cc + 5]),
                                     pack_bf16(p[8 * cc + 6], p[8 * cc + 7]));
                    }
                }
                fence_proxy_async_smem();
                tc_fence_before();
                mbar_arrive(&p_full[b]);
            }
            if (lexp) continue;
            // epilogue of this item: hat_alpha_R[key, :] = D2[key, :] / max(c_R, eps)
            mbar_wait(&o_full[b], (it >> 1) & 1);   // one o_full per item
            tc_fence_after();
            const float inv = 1.f / fmaxf(cr, g.eps_div);
            const int bh = col / (g.gq * g.s2), a = (col / g.s2) % g.gq, j = col % g.s2;
#pragma unroll 1
            for (int part = 0; part < 2; ++part) {
                float o[64];
                tmem_ld32(tmem + 256 + b * 128 + lane_off + part * 64, o);
                tmem_ld32(tmem + 256 + b * 128 + lane_off + part * 64 + 32, o + 32);
                uint8_t* stg = stg_base + (MBX_ALPHA_PP ? part * 16384 : 0);
                if (!MBX_ALPHA_PP) {
                    if (lane == 0) bulk_wait_read<0>();
                    __syncwarp();
                }
                const uint32_t srow = smem_u32(stg) + lane * 128;
#pragma unroll
                for (int cc = 0; cc < 8; ++cc)
                    st_shared_v4(srow + ((cc ^ (lane & 7)) << 4), pack_bf16(o[8 * cc] * inv, o[8 * cc + 1] * inv),
                                 pack_bf16(o[8 * cc + 2] * inv, o[8 * cc + 3] * inv),
                                 pack_bf16(o[8 * cc + 4] * inv, o[8 * cc + 5] * inv),
                                 pack_bf16(o[8 * cc + 6] * inv, o[8 * cc + 7] * inv));
                fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0 && ch * kAKC + quad * 32 < g.nkeys) {   // box rows past nkeys are clipped
                    tma_store_4d(&P.tar_st, stg, part * 64, j, ch * kAKC + quad * 32, bh * g.gq + a);
                    bulk_commit();
                }
            }
            tc_fence_before();
        }
        if (lane == 0) bulk_wait<0>();
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc<512>(tmem);
}
