// tcgen05 / TMEM / TMA kernels of the tiled MonarchAttention forward (bf16,
// d = d_v = 128, tile rows of <= 64 tokens, any number of tiles, any T; T >= 2
// and factor export step over rows in chunks of 128).  Warp-specialized persistent kernels
// joined by a bf16 workspace W[b,h,a,j,(c,k),0:256] = [aL | Y] and c_L
// (SURVEY.md Appendix B):
//   row stage    (mbx_tc_row.cuh, mbx_tc_rowp.cuh)  solver.py:187-191, factors.py:123
//   column stage (mbx_tc_col.cuh, mbx_tc_colw.cuh)  solver.py:192-195, factors.py:124
//   alpha_R hand-off / L export (mbx_tc_alpha.cuh)  solver.py:185-186
// The plan's permutation is folded into TMA coordinates: each tile row is one
// box at token row_base(tile, r); each tile column is one strided box.
#include "mbx_internal.h"
#include "mbx_sm100.cuh"

#include <cuda.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <mutex>

namespace mbx {
namespace {

using namespace sm100;

constexpr int kD = 128;           // head dim (q, k) and value dim
constexpr int kMaxS2 = 64;        // tile-row tokens (MMA1 N, MMA2 K)
constexpr int kMaxS1 = 32;        // tile rows (column-stage N)
constexpr float kLog2e = 1.4426950408889634f;

__device__ __forceinline__ uint32_t ring_parity(uint32_t n, uint32_t size) { return (n / size) & 1u; }

// c_L rows are padded to 32 floats so each column's row is a 16-byte aligned TMA box.
__host__ __device__ __forceinline__ int ckey_stride(const Geometry& g) { return (g.nkeys + 31) & ~31; }

#ifdef MBX_TRACE
// Event timestamps of the first kTraceCtas CTAs: [cta][role][event] = (globaltimer << 8) | tag.
constexpr int kTraceCtas = 4, kTraceRoles = 16, kTraceEvents = 2048;
__device__ unsigned long long g_trace[kTraceCtas][kTraceRoles][kTraceEvents];
__device__ __forceinline__ void trace_ev(int role, int& idx, int tag) {
    if (blockIdx.x < kTraceCtas && idx < kTraceEvents) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        g_trace[blockIdx.x][role][idx++] = (t << 8) | (unsigned)tag;
    }
}
#define TR(role, idx, tag) trace_ev(role, idx, tag)
// column-stage events (separate buffer: the row stage owns g_trace)
__device__ unsigned long long g_trace_col[kTraceCtas][kTraceRoles][kTraceEvents];
__device__ __forceinline__ void trace_col(int role, int& idx, int tag) {
    if (blockIdx.x < kTraceCtas && idx < kTraceEvents) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        g_trace_col[blockIdx.x][role][idx++] = (t << 8) | (unsigned)tag;
    }
}
#define TRC(role, idx, tag) trace_col(role, idx, tag)
// Start / end timestamps of every CTA of the last launch of each kernel: [kernel][cta][2].
constexpr int kSpanCtas = 256;
__device__ unsigned long long g_span[2][kSpanCtas][2];
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#define SPAN_AT(kern, which) \
    do { if (threadIdx.x == 0 && blockIdx.x < kSpanCtas) g_span[kern][blockIdx.x][which] = gtimer(); } while (0)
#else
#define TR(role, idx, tag) ((void)0)
#define TRC(role, idx, tag) ((void)0)
#define SPAN_AT(kern, which) ((void)0)
#endif
#define SPAN_BEGIN() SPAN_AT(0, 0)
#define SPAN_END() SPAN_AT(0, 1)

// Every tensor map and pointer of one forward (kernel parameter, 64-byte aligned maps).
struct TcParams {
    CUtensorMap tq, tk, tv, tws, tws_b;   // row stage: q/k/v rows, workspace store boxes
    CUtensorMap tw, tc, tqc, tout;        // column stage: workspace, c_L, q columns, output columns
    CUtensorMap tw128, tc128;             // alpha_R stage: 128-key workspace / c_L boxes
    CUtensorMap tar_st, tar_ld;           // hat_alpha_R [bh*gq][key][j][128]: store (32 keys), load (s2 rows)
    float* wc;                            // c_L [col][ckey_stride]
    const __nv_bfloat16* w;               // workspace W[col][part][key][64]
    float* stats;                         // T >= 2: per (col, l) running max and 1/sum of L
    int stats_pitch;                      // floats per column: [max x s1p | 1/sum x s1p]
    CUtensorMap tqcw, toutw;              // wide column stage: q columns (128 rows), output rows (32 x 64)
    CUtensorMap tqa;                      // alpha_R stage: q columns, s1 rounded up to 32 rows
    __nv_bfloat16* out;                   // output base (wide stage's partial-warp stores)
    int64_t out_bh_stride, out_tok_stride;
    int dbg;                              // MBX_DBG bit mask: timing experiments only (wrong results)
    int l2hint;                           // bit 0: W stores evict_last, bit 1: W last reads evict_first; -1 auto
    CUtensorMap tq128, tk128, tv128;      // flash row stage (s2 > 64): 128-row boxes of q / k / v
    CUtensorMap tar_ld128;                // flash row stage, T >= 2: 128 hat_alpha_R rows of one key
    float* rfac;                          // optional R' export (fp32, factors.py:57-79 layout), last row stage
    float* lfac;                          // optional L' export, written by the alpha kernel in mode 1
};

// Row-stage query groups (<= 3 query tiles each) of the classic row stage.
__host__ __device__ __forceinline__ int row_groups(const Geometry& g) { return (g.gq + 2) / 3; }

// One softmax row of the final R' (fp32, before the bf16 rounding the MMA operand gets).
__device__ __forceinline__ void store_r_row(float* dst, const float* p, float inv_l, int s2) {
#pragma unroll
    for (int i = 0; i < 64; ++i)
        if (i < s2) dst[i] = p[i] * inv_l;
}

#include "mbx_tc_row.cuh"
#include "mbx_tc_col.cuh"
#include "mbx_tc_alpha.cuh"
#include "mbx_tc_colw.cuh"
#include "mbx_tc_colw2.cuh"
#include "mbx_tc_rowp.cuh"
#include "mbx_tc_rowf.cuh"

__device__ __forceinline__ uint8_t* aligned_smem() {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    return reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
}

__global__ void __launch_bounds__(kRowThreads, 1)
tc_row_stage(const __grid_constant__ TcParams P, Geometry g, int amode, int want_y) {
    SPAN_AT(0, 0);
    row_role(aligned_smem(), P, g, blockIdx.x, gridDim.x, amode != 0, want_y != 0);
    SPAN_AT(0, 1);
}

template <int mode>
__global__ void __launch_bounds__(kColThreads, 1)
tc_column_stage(const __grid_constant__ TcParams P, Geometry g) {
    SPAN_AT(1, 0);
    col_role<mode>(aligned_smem(), P, g, blockIdx.x, gridDim.x);
    SPAN_AT(1, 1);
}
template __global__ void tc_column_stage<0>(const __grid_constant__ TcParams, Geometry);
template __global__ void tc_column_stage<1>(const __grid_constant__ TcParams, Geometry);
template __global__ void tc_column_stage<2>(const __grid_constant__ TcParams, Geometry);

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
    const CUresult r = enc(m, dt, rank, const_cast<void*>(base), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS && getenv("MBX_VERBOSE")) {
        fprintf(stderr, "mbx: cuTensorMapEncodeTiled failed (%d): base %p rank %d dims", (int)r, base, rank);
        for (int i = 0; i < rank; ++i) fprintf(stderr, " %llu", (unsigned long long)dims[i]);
        fprintf(stderr, " strides");
        for (int i = 0; i + 1 < rank; ++i) fprintf(stderr, " %llu", (unsigned long long)strides[i]);
        fprintf(stderr, " box");
        for (int i = 0; i < rank; ++i) fprintf(stderr, " %u", box[i]);
        fprintf(stderr, "\n");
    }
    return r == CUDA_SUCCESS;
}

// (B, H, N, 128) bf16 with element strides st[b,h,token]; box (64 features, rows tokens).
bool make_rows_map(CUtensorMap* m, const void* base, int B, int H, int N, const int64_t* st, int rows) {
    cuuint64_t dims[4] = {(cuuint64_t)kD, (cuuint64_t)N, (cuuint64_t)H, (cuuint64_t)B};
    cuuint64_t strides[3] = {(cuuint64_t)st[2] * 2, (cuuint64_t)st[1] * 2, (cuuint64_t)st[0] * 2};
    cuuint32_t box[4] = {64, (cuuint32_t)rows, 1, 1};
    return encode(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, base, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B);
}

// Query columns: q viewed as (d, w-column, grid row of W tokens, b*H+h); box (64, 1, 32, 1).
// Output columns: out viewed like q; box (32 value dims, 1, s1 rows, 1), no swizzle.
bool make_outcol_map(CUtensorMap* m, const void* base, const Geometry& g, int nq) {
    cuuint64_t dims[4] = {(cuuint64_t)kD, (cuuint64_t)g.W, (cuuint64_t)(nq / g.W), (cuuint64_t)g.bh};
    cuuint64_t strides[3] = {(cuuint64_t)g.os[2] * 2, (cuuint64_t)g.os[2] * 2 * g.W, (cuuint64_t)g.os[1] * 2};
    cuuint32_t box[4] = {32, 1, (cuuint32_t)(g.s1 < kMaxS1 ? g.s1 : kMaxS1), 1};   // stacked stage only (s1 <= 32)
    return encode(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, base, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_NONE);
}

bool make_qcol_map(CUtensorMap* m, const void* base, const Geometry& g, int nq) {
    cuuint64_t dims[4] = {(cuuint64_t)kD, (cuuint64_t)g.W, (cuuint64_t)(nq / g.W), (cuuint64_t)g.bh};
    cuuint64_t strides[3] = {(cuuint64_t)g.qs[2] * 2, (cuuint64_t)g.qs[2] * 2 * g.W, (cuuint64_t)g.qs[1] * 2};
    cuuint32_t box[4] = {64, 1, (cuuint32_t)kMaxS1, 1};
    return encode(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, base, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B);
}

constexpr size_t kPairKvBytes = (size_t)48 << 20;   // K + V of a launch the half-packed stage re-reads from L2
constexpr long long kWavePairTasks = 2000;           // per-head pair tasks that make L2-sized waves pay

size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

int num_sms(int dev) {   // per device (mixed-GPU hosts)
    static int n[64] = {};
    if (dev < 0 || dev >= 64) return 148;
    if (!n[dev]) {
        int v = 0;
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
        n[dev] = v > 0 ? v : 148;
    }
    return n[dev];
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

// The geometry of a permuted plan's gathered copy: q, k, v (and out) in slot order, one
// contiguous (b h) slab of rows of 128 features each, identity orders.
Geometry slot_geometry(const Geometry& g) {
    Geometry s = g;
    const int64_t nq = (int64_t)g.c1q * g.s1 * g.c2 * g.s2, nk = (int64_t)g.c1k * g.s1 * g.c2 * g.s2;
    s.q_order = s.kv_order = nullptr;
    s.qs[0] = (int64_t)g.heads * nq * kD; s.qs[1] = nq * kD; s.qs[2] = kD;
    s.os[0] = s.qs[0]; s.os[1] = s.qs[1]; s.os[2] = s.qs[2];
    s.ks[0] = (int64_t)g.heads * nk * kD; s.ks[1] = nk * kD; s.ks[2] = kD;
    s.vs[0] = s.ks[0]; s.vs[1] = s.ks[1]; s.vs[2] = s.ks[2];
    return s;
}
size_t gather_bytes(const Geometry& g) {
    const size_t nq = (size_t)g.c1q * g.s1 * g.c2 * g.s2, nk = (size_t)g.c1k * g.s1 * g.c2 * g.s2;
    return align256((size_t)g.bh * (2 * nq + 2 * nk) * kD * 2);
}

// dst[bh][p][:] = src[b, h, order[p], :] (or the reverse with scatter): 16 threads per 256-byte row
__global__ void gather_rows(const __nv_bfloat16* __restrict__ src, __nv_bfloat16* __restrict__ dst,
                            const int32_t* __restrict__ order, int64_t n, int bh, int heads, int64_t s0, int64_t s1,
                            int64_t s2, int scatter) {
    const int64_t total = (int64_t)bh * n * 16;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int c = (int)(i & 15);
        const int64_t row = i >> 4;
        const int64_t p = row % n;
        const int u = (int)(row / n);
        const int b = u / heads, h = u - (u / heads) * heads;
        const int64_t tok = order ? order[p] : p;
        const uint4* a = reinterpret_cast<const uint4*>(src + b * s0 + h * s1 + tok * s2) + c;
        uint4* slot = reinterpret_cast<uint4*>(dst + row * kD) + c;
        if (scatter)
            *const_cast<uint4*>(a) = *slot;
        else
            *slot = *a;
    }
}

}  // namespace

// ------------------------------------------------------------------ options
static Options g_opts;
static std::once_flag g_opts_once;
static std::mutex g_opts_mu;

static void init_options() {
    auto env = [](const char* n, int dflt) {
        const char* e = getenv(n);
        return e && e[0] ? atoi(e) : dflt;
    };
    g_opts.pdl = env("MBX_PDL", 1);
    g_opts.l2hint = env("MBX_L2HINT", -1);
    g_opts.dbg = env("MBX_DBG", 0);
    g_opts.pair = env("MBX_PAIR", -1);
    g_opts.wide = env("MBX_WIDE", 0);
    g_opts.split = env("MBX_SPLIT", -1);
    g_opts.verbose = env("MBX_VERBOSE", 0);
    g_opts.fusedhand = env("MBX_FUSEDHAND", 1);
    g_opts.wave = env("MBX_WAVE", -1);
    g_opts.ws_cap_mb = env("MBX_WS_CAP_MB", 2048);
    g_opts.wide2 = env("MBX_WIDE2", 1);
}

const Options& options() {
    std::call_once(g_opts_once, init_options);
    return g_opts;
}

int set_option(const char* name, int value) {
    std::call_once(g_opts_once, init_options);
    if (!name) return -1000;
    std::lock_guard<std::mutex> lock(g_opts_mu);
    struct { const char* n; int* p; } tab[] = {
        {"MBX_PDL", &g_opts.pdl}, {"MBX_L2HINT", &g_opts.l2hint}, {"MBX_DBG", &g_opts.dbg},
        {"MBX_PAIR", &g_opts.pair}, {"MBX_WIDE", &g_opts.wide}, {"MBX_SPLIT", &g_opts.split},
        {"MBX_VERBOSE", &g_opts.verbose}, {"MBX_FUSEDHAND", &g_opts.fusedhand},
        {"MBX_WAVE", &g_opts.wave}, {"MBX_WS_CAP_MB", &g_opts.ws_cap_mb}, {"MBX_WIDE2", &g_opts.wide2}};
    for (auto& t : tab)
        if (strcmp(t.n, name) == 0) {
            const int prev = *t.p;
            *t.p = value;
            ++g_opts.version;
            return prev;
        }
    return -1000;
}

// Why a problem is not on the tcgen05 path (nullptr: it is); MBX_VERBOSE=1 prints it.
static const char* tc_unsupported_reason(const Geometry& g, int dtype, int flags, bool factors) {
    if (flags & MBX_FLAG_FORCE_GENERIC) return "forced generic";
    if (flags & MBX_FLAG_NO_OUTPUT) return "factors without output";
    if (dtype != MBX_BF16 || g.d != kD || g.dv != kD || g.T < 1) return "needs bf16 with d = dv = 128";
    if (factors && g.s2 > kMaxS2) return "factor export with s2 > 64";   // online row softmax (flash row stage)
    // permuted plans without a closed form (the aligned (w, fh), (hw, f), (fw, h), (h, fw)
    // configurations, misaligned raw orders) run gathered into slot order (tc_forward), where
    // the identity plan's tile rows are contiguous -- possible when c2 == 1
    const bool gathered = g.nf == 0 && (g.q_order || g.kv_order);
    if (gathered && g.c2 != 1) return "permuted plan with c2 > 1 and no closed form";
    Geometry gs = g;
    if (gathered) gs = slot_geometry(g);
    int F, H, W;
    if (!column_grid(gs, &F, &H, &W)) return "tile rows are not contiguous grid rows";
    if (!strides_ok(g.qs) || !strides_ok(g.ks) || !strides_ok(g.vs) || !strides_ok(g.os))
        return "strides not 16-byte aligned";
    // the q-column / output maps fold (b, h) into one dim; a size-1 batch has no stride to fold
    // (PyTorch keeps the parent's batch stride on head slices of a B = 1 tensor)
    if (gs.bh > gs.heads && gs.qs[0] != (int64_t)gs.heads * gs.qs[1]) return "q batch stride != heads * head stride";
    if (gs.bh > gs.heads && gs.os[0] != (int64_t)gs.heads * gs.os[1]) return "out batch stride != heads * head stride";
    if ((int64_t)g.bh * g.gq * g.s2 * g.nkeys >= ((int64_t)1 << 31)) return "workspace rows exceed 2^31";
    if (encode_fn() == nullptr) return "cuTensorMapEncodeTiled unavailable";
    return nullptr;
}

bool tc_supported(const Geometry& g, int dtype, int flags, bool factors) {
    const char* why = tc_unsupported_reason(g, dtype, flags, factors);
    if (why && !(flags & MBX_FLAG_FORCE_GENERIC) && options().verbose)
        fprintf(stderr, "mbx: tcgen05 path not used: %s (bh=%d heads=%d qs=%lld,%lld,%lld os=%lld,%lld,%lld)\n", why,
                g.bh, g.heads, (long long)g.qs[0], (long long)g.qs[1], (long long)g.qs[2], (long long)g.os[0],
                (long long)g.os[1], (long long)g.os[2]);
    return why == nullptr;
}

// Workspace of one launch sequence: W [col][part][key][64] bf16, c_L [col][ckey] f32,
// L statistics [col][2 s1p] f32, and for T >= 2 hat_alpha_R [bh gq][key][j][128] bf16.
struct TcLayout {
    size_t w, wc, stats, ar, total;
};
static TcLayout tc_layout(const Geometry& g) {
    const size_t ncols = (size_t)g.bh * g.gq * g.s2;
    const size_t rows = ncols * g.nkeys;
    const size_t s1p = ((g.s1 + 31) / 32) * 32;
    TcLayout L;
    L.w = 0;
    L.wc = align256(rows * 512);
    L.stats = L.wc + align256(ncols * ckey_stride(g) * 4);
    L.ar = L.stats + align256(ncols * 2 * s1p * 4);
    L.total = L.ar + (g.T > 1 ? align256(rows * 256) : 0);
    return L;
}

// Failure of a host-side setup step: reported on stderr when MBX_VERBOSE is set.
static cudaError_t tc_fail(const char* what, int line) {
    if (options().verbose) fprintf(stderr, "mbx tc_forward: %s failed (mbx_tc.cu:%d)\n", what, line);
    return cudaErrorInvalidValue;
}
#define TC_FAIL(what) tc_fail(what, __LINE__)

// Everything one forward launch sequence needs, derived from the descriptor, the pointers
// and the options; cached so repeated calls skip the tensor-map encodes.
struct TcPlan {
    TcParams P;
    Geometry g;            // identity plans rewritten as a (1, s1, s2) neighborhood grid
    bool pair, wide;
    bool fused_hand;       // T >= 2 hand-off fused into the stacked column stage (mode 2)
    bool flash;            // s2 > 64: online-softmax row stage
    int grid_flash, smem_flash;
    int grid_pair, grid_row, grid_col, grid_wide, grid_alpha;
    int smem_row, smem_col, smem_pair, smem_wide, smem_alpha;
};

static cudaError_t build_plan(const Geometry& g0, const void* q, const void* k, const void* v, void* out,
                              float* l_factor, float* r_factor, void* workspace, int dev, TcPlan* T) {
    const Options& o = options();
    Geometry g = g0;
    int F, H, W;
    if (!column_grid(g, &F, &H, &W)) return TC_FAIL("tensor map / argument check");
    if (g.nf == 0) {   // express the identity plan as a (1, s1, s2) neighborhood grid
        g.F = F; g.H = H; g.W = W;
        g.nf = 1; g.nh = g.s1; g.nw = g.s2;
    }
    const bool factors = l_factor || r_factor;
    const int B = g.bh / g.heads;
    const int nq = g.c1q * g.s1 * g.c2 * g.s2, nk = g.c1k * g.s1 * g.c2 * g.s2;
    if (((uintptr_t)q | (uintptr_t)k | (uintptr_t)v | (uintptr_t)out | (uintptr_t)workspace) & 15)
        return TC_FAIL("tensor map / argument check");
    TcParams& P = T->P;
    memset(&P, 0, sizeof(P));
    P.dbg = o.dbg;
    // L2 policy of the W exchange: its last reads evict_first; its stores evict_last only when
    // the launch's W exceeds L2 (a W that fits stays resident anyway, and marking it evict_last
    // costs the row stage's K/V reuse: C2, 86 MB, 58.0 -> 56.5 us without it; KV21 halves,
    // 302 MB each, 280 -> 277 us with it; profiles/r2h_l2hint_ab.txt)
    const size_t w_bytes = (size_t)g.bh * g.gq * g.s1 * g.gk * g.s2 * 512;
    P.l2hint = o.l2hint >= 0 ? o.l2hint : 2 | (w_bytes > ((size_t)128 << 20) ? 1 : 0);
    P.rfac = r_factor;
    P.lfac = l_factor;
    const bool flash = g.s2 > kMaxS2;   // long tile rows: online-softmax row stage
    const int rbox = flash ? kMaxS2 : g.s2;
    if (!make_rows_map(&P.tq, q, B, g.heads, nq, g.qs, rbox) || !make_rows_map(&P.tk, k, B, g.heads, nk, g.ks, rbox) ||
        !make_rows_map(&P.tv, v, B, g.heads, nk, g.vs, rbox) || !make_qcol_map(&P.tqc, q, g, nq) ||
        !make_outcol_map(&P.tout, out, g, nq))
        return TC_FAIL("tensor map / argument check");
    if (flash && (!make_rows_map(&P.tq128, q, B, g.heads, nq, g.qs, kFKC) ||
                  !make_rows_map(&P.tk128, k, B, g.heads, nk, g.ks, kFKC) ||
                  !make_rows_map(&P.tv128, v, B, g.heads, nk, g.vs, kFKC)))
        return TC_FAIL("tensor map / argument check");
    const int64_t ncols = (int64_t)g.bh * g.gq * g.s2;
    const int64_t rows = ncols * g.nkeys;
    const TcLayout lay = tc_layout(g);
    char* wsb = reinterpret_cast<char*>(workspace);
    __nv_bfloat16* Wp = reinterpret_cast<__nv_bfloat16*>(wsb + lay.w);
    float* Wc = reinterpret_cast<float*>(wsb + lay.wc);
    P.wc = Wc;
    P.w = Wp;
    const int s1p = ((g.s1 + 31) / 32) * 32;
    P.stats = reinterpret_cast<float*>(wsb + lay.stats);
    P.stats_pitch = 2 * s1p;
    P.out = reinterpret_cast<__nv_bfloat16*>(out);
    P.out_bh_stride = g.os[1];
    P.out_tok_stride = g.os[2];
    const bool wide = g.s1 > kMaxS1 || (g.T == 1 && o.wide == 1);
    const bool stats = g.T > 1 || factors;   // statistics pass + alpha kernel (hand-off / L export)
    if (wide || stats) {   // q columns of up to 128 rows; output rows of one warp (32 rows x 64 values)
        cuuint64_t dims[4] = {(cuuint64_t)kD, (cuuint64_t)g.W, (cuuint64_t)(nq / g.W), (cuuint64_t)g.bh};
        cuuint64_t qstr[3] = {(cuuint64_t)g.qs[2] * 2, (cuuint64_t)g.qs[2] * 2 * g.W, (cuuint64_t)g.qs[1] * 2};
        cuuint32_t qbox[4] = {64, 1, 128, 1};
        cuuint64_t ostr[3] = {(cuuint64_t)g.os[2] * 2, (cuuint64_t)g.os[2] * 2 * g.W, (cuuint64_t)g.os[1] * 2};
        cuuint32_t obox[4] = {64, 1, 32, 1};
        cuuint32_t qabox[4] = {64, 1, (cuuint32_t)(s1p < 128 ? s1p : 128), 1};
        if (!encode(&P.tqcw, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, q, dims, qstr, qbox, CU_TENSOR_MAP_SWIZZLE_128B) ||
            !encode(&P.tqa, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, q, dims, qstr, qabox, CU_TENSOR_MAP_SWIZZLE_128B) ||
            !encode(&P.toutw, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, out, dims, ostr, obox, CU_TENSOR_MAP_SWIZZLE_128B))
            return TC_FAIL("tensor map / argument check");
    }
    {
        // blocked W[col][part][key][64]: part 0,1 = aL halves, 2,3 = Y halves
        cuuint64_t dims[4] = {64, (cuuint64_t)g.nkeys, 4, (cuuint64_t)ncols};
        cuuint64_t strides[3] = {128, (cuuint64_t)g.nkeys * 128, (cuuint64_t)g.nkeys * 512};
        cuuint32_t box[4] = {64, (cuuint32_t)kKC, 1, 1};          // column stage: contiguous 12 KB
        if (!encode(&P.tw, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, Wp, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B))
            return TC_FAIL("tensor map / argument check");
        if (!flash) {
            // classic row stage: one key, the columns j of one epilogue warp (rows 0..31 and 32..s2-1)
            cuuint32_t sbox[4] = {64, 1, 1, (cuuint32_t)(g.s2 < 32 ? g.s2 : 32)};
            if (!encode(&P.tws, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, Wp, dims, strides, sbox, CU_TENSOR_MAP_SWIZZLE_128B))
                return TC_FAIL("tensor map / argument check");
            cuuint32_t sbox_b[4] = {64, 1, 1, (cuuint32_t)(g.s2 > 32 ? g.s2 - 32 : 1)};
            if (!encode(&P.tws_b, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, Wp, dims, strides, sbox_b,
                        CU_TENSOR_MAP_SWIZZLE_128B))
                return TC_FAIL("tensor map / argument check");
        }
        cuuint64_t cdims[2] = {(cuuint64_t)ckey_stride(g), (cuuint64_t)ncols};
        cuuint64_t cstrides[1] = {(cuuint64_t)ckey_stride(g) * 4};
        cuuint32_t cbox[2] = {(cuuint32_t)kKC, 1};
        if (!encode(&P.tc, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, Wc, cdims, cstrides, cbox, CU_TENSOR_MAP_SWIZZLE_NONE))
            return TC_FAIL("tensor map / argument check");
        if (stats || wide) {
            cuuint32_t box128[4] = {64, (cuuint32_t)kAKC, 1, 1};
            if (!encode(&P.tw128, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, Wp, dims, strides, box128,
                        CU_TENSOR_MAP_SWIZZLE_128B))
                return TC_FAIL("tensor map / argument check");
            cuuint32_t cbox128[2] = {(cuuint32_t)kAKC, 1};
            if (!encode(&P.tc128, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, Wc, cdims, cstrides, cbox128,
                        CU_TENSOR_MAP_SWIZZLE_NONE))
                return TC_FAIL("tensor map / argument check");
        }
        if (g.T > 1) {
            // hat_alpha_R[bh*gq][key][j][128] bf16
            __nv_bfloat16* AR = reinterpret_cast<__nv_bfloat16*>(wsb + lay.ar);
            cuuint64_t adims[4] = {128, (cuuint64_t)g.s2, (cuuint64_t)g.nkeys, (cuuint64_t)g.bh * g.gq};
            cuuint64_t astr[3] = {256, (cuuint64_t)g.s2 * 256, (cuuint64_t)g.s2 * 256 * g.nkeys};
            cuuint32_t abox_st[4] = {64, 1, 32, 1};
            cuuint32_t abox_ld[4] = {64, (cuuint32_t)rbox, 1, 1};
            cuuint32_t abox_ld128[4] = {64, (cuuint32_t)kFKC, 1, 1};
            if (!encode(&P.tar_st, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, AR, adims, astr, abox_st,
                        CU_TENSOR_MAP_SWIZZLE_128B) ||
                !encode(&P.tar_ld, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, AR, adims, astr, abox_ld,
                        CU_TENSOR_MAP_SWIZZLE_128B) ||
                (flash && !encode(&P.tar_ld128, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, AR, adims, astr, abox_ld128,
                                  CU_TENSOR_MAP_SWIZZLE_128B)))
                return TC_FAIL("tensor map / argument check");
        }
    }
    (void)rows;
    const int sms = num_sms(dev);
    T->g = g;
    T->wide = wide;
    T->flash = flash;
    T->smem_flash = RowFSmem::kTotal + 1024;
    {
        const int64_t ftasks = (int64_t)g.bh * g.gq * g.s1 * ((g.s2 + kFKC - 1) / kFKC) * g.gk;
        T->grid_flash = ftasks < sms ? (int)ftasks : sms;
    }
    T->fused_hand = !wide && g.T > 1 && g.nkeys <= kKC && o.fusedhand != 0;
    T->smem_row = RowSmem::kTotal + 1024;
    T->smem_col = ColSmem::kTotal + 1024;
    T->smem_alpha = AlphaSmem::kTotal + 1024;
    T->smem_wide = WideSmem::kTotal + 1024;
    T->smem_pair = RowPSmem::kTotal + 1024;
    const int64_t witems = ncols * ((g.s1 + 127) / 128);
    T->grid_wide = witems < sms ? (int)witems : sms;
    const int64_t key_rows = (int64_t)g.bh * g.s1 * row_groups(g) * g.gk;   // row-stage key rows
    T->grid_row = key_rows < sms ? (int)key_rows : sms;
    // half-packed row stage (two M=64 (query tile, row) halves per 128-lane task).  MBX_PAIR=0
    // selects the classic stage (whole query tiles per M=128 task), MBX_PAIR=1 the packed one.  Packing pays when whole
    // query tiles leave M=128 lanes idle (odd G_q); for G_q > 1 a K/V row then serves halves
    // of two items, so it is re-read once more -- cheap only while K and V sit in L2.
    const size_t kv_bytes = (size_t)g.bh * g.gk * g.s1 * g.s2 * (size_t)(g.d + g.dv) * 2;
    T->pair = o.pair >= 0 ? o.pair == 1 : g.gq == 1 || (g.gq % 2 == 1 && kv_bytes <= kPairKvBytes);
    const int64_t pair_tasks = (int64_t)g.bh * ((g.gq * g.s1 + 1) / 2) * g.gk;
    T->grid_pair = pair_tasks < sms ? (int)pair_tasks : sms;
    const int64_t ngroups = (int64_t)g.bh * g.gq * ((g.s2 + 3) / 4);
    T->grid_col = ngroups < sms ? (int)ngroups : sms;
    const int64_t aitems = ncols * ((g.nkeys + kAKC - 1) / kAKC);
    T->grid_alpha = aitems < sms ? (int)aitems : sms;
    return cudaSuccess;
}

// Launch-parameter cache: keyed by the geometry, pointers, device and option version.
struct PlanKey {
    Geometry g;
    const void *q, *k, *v, *out, *ws;
    float *lf, *rf;
    int dev;
    unsigned opt_version;
};
static bool key_eq(const PlanKey& a, const PlanKey& b) { return memcmp(&a, &b, sizeof(PlanKey)) == 0; }

struct PlanCache {
    static constexpr int kSlots = 16;
    PlanKey key[kSlots];
    TcPlan plan[kSlots];
    unsigned long long used[kSlots] = {};
    unsigned long long tick = 0;
    int n = 0;
};
static PlanCache g_plans;
static std::mutex g_plans_mu;

static cudaError_t get_plan(const Geometry& g, const void* q, const void* k, const void* v, void* out,
                            float* lf, float* rf, void* ws, int dev, TcPlan* out_plan) {
    PlanKey key;
    memset(&key, 0, sizeof(key));   // padding bytes take part in the comparison
    key.g = g;
    key.q = q; key.k = k; key.v = v; key.out = out; key.ws = ws;
    key.lf = lf; key.rf = rf;
    key.dev = dev;
    key.opt_version = options().version;
    {
        std::lock_guard<std::mutex> lock(g_plans_mu);
        for (int i = 0; i < g_plans.n; ++i)
            if (key_eq(g_plans.key[i], key)) {
                g_plans.used[i] = ++g_plans.tick;
                *out_plan = g_plans.plan[i];
                return cudaSuccess;
            }
    }
    TcPlan p;
    cudaError_t e = build_plan(g, q, k, v, out, lf, rf, ws, dev, &p);
    if (e != cudaSuccess) return e;
    std::lock_guard<std::mutex> lock(g_plans_mu);
    int slot = g_plans.n < PlanCache::kSlots ? g_plans.n++ : 0;
    if (g_plans.n == PlanCache::kSlots)
        for (int i = 1; i < PlanCache::kSlots; ++i)
            if (g_plans.used[i] < g_plans.used[slot]) slot = i;
    g_plans.key[slot] = key;
    g_plans.plan[slot] = p;
    g_plans.used[slot] = ++g_plans.tick;
    *out_plan = p;
    return cudaSuccess;
}

// Dynamic shared-memory limits: set once per device (not per call).
static cudaError_t ensure_attributes(int dev) {
    static bool done[64] = {};
    static std::mutex mu;
    if (dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
    std::lock_guard<std::mutex> lock(mu);
    if (done[dev]) return cudaSuccess;
    cudaError_t e;
    const struct { const void* fn; int smem; } k[] = {
        {(const void*)tc_row_stage, RowSmem::kTotal + 1024},     {(const void*)tc_column_stage<0>, ColSmemT<0>::kTotal + 1024},
        {(const void*)tc_column_stage<1>, ColSmem::kTotal + 1024}, {(const void*)tc_column_stage<2>, ColSmem::kTotal + 1024},
        {(const void*)tc_column_wide, WideSmem::kTotal + 1024},  {(const void*)tc_alpha_r_stage, AlphaSmem::kTotal + 1024},
        {(const void*)tc_column_wide2<0>, Wide2Smem::kTotal + 1024},
        {(const void*)tc_column_wide2<1>, Wide2Smem::kTotal + 1024},
        {(const void*)tc_row_pair, RowPSmem::kTotal + 1024}, {(const void*)tc_row_flash, RowFSmem::kTotal + 1024}};
    for (auto& x : k)
        if ((e = cudaFuncSetAttribute(x.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, x.smem)) != cudaSuccess)
            return e;
    done[dev] = true;
    return cudaSuccess;
}

static cudaError_t tc_forward_one(const Geometry& g0, int flags, const void* q, const void* k, const void* v,
                                  void* out, float* l_factor, float* r_factor, void* workspace, int dev,
                                  cudaStream_t stream, bool pdl_first = false) {
    cudaError_t e = ensure_attributes(dev);
    if (e != cudaSuccess) return e;
    TcPlan T;
    if ((e = get_plan(g0, q, k, v, out, l_factor, r_factor, workspace, dev, &T)) != cudaSuccess) return e;
    const Geometry& g = T.g;
    TcParams& P = T.P;
    const bool pdl = options().pdl != 0;
    const bool verbose = options().verbose != 0;
    const bool factors = l_factor || r_factor;
    // Every launch after the first uses programmatic dependent launch: its CTAs set up
    // while the previous stage drains and wait (griddepcontrol.wait) before touching
    // the workspace.  The first launch is ordinary, so it never overlaps the previous
    // forward's readers of the workspace.
    int nlaunch = pdl_first ? 1 : 0;
    auto launch = [&](const void* fn, int grid, int threads, int smem, void** args) -> cudaError_t {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(grid);
        cfg.blockDim = dim3(threads);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = stream;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = attr;
        cfg.numAttrs = (nlaunch++ > 0 && pdl) ? 1 : 0;
        cudaError_t le = cudaLaunchKernelExC(&cfg, fn, args);
        if (le != cudaSuccess && verbose)
            fprintf(stderr, "mbx tc_forward: launch %d (grid %d, smem %d) failed: %s\n", nlaunch, grid, smem,
                    cudaGetErrorString(le));
        return le;
    };
    auto column = [&](int mode, TcParams& Pc) -> cudaError_t {
        if (T.wide && mode <= 1 && options().wide2 != 0) {   // two item streams per CTA (ping-pong)
            ProfScope p("tc_column_wide", stream);
            void* args[] = {(void*)&Pc, (void*)&g};
            const void* fn = mode == 0 ? (const void*)tc_column_wide2<0> : (const void*)tc_column_wide2<1>;
            return launch(fn, T.grid_wide, kW2Threads, Wide2Smem::kTotal + 1024, args);
        }
        if (T.wide) {
            ProfScope p("tc_column_wide", stream);
            void* args[] = {(void*)&Pc, (void*)&g, (void*)&mode};
            return launch((const void*)tc_column_wide, T.grid_wide, kWideThreads, T.smem_wide, args);
        }
        ProfScope p("tc_column_stage", stream);
        void* args[] = {(void*)&Pc, (void*)&g};
        const void* fn = mode == 0 ? (const void*)tc_column_stage<0>
                         : mode == 1 ? (const void*)tc_column_stage<1> : (const void*)tc_column_stage<2>;
        return launch(fn, T.grid_col, kColThreads, mode == 0 ? ColSmemT<0>::kTotal + 1024 : T.smem_col, args);
    };
    auto alpha = [&](int amode, TcParams& Pc) -> cudaError_t {
        ProfScope p(amode ? "tc_alpha_l_export" : "tc_alpha_r_stage", stream);
        void* args[] = {(void*)&Pc, (void*)&g, (void*)&amode};
        return launch((const void*)tc_alpha_r_stage, T.grid_alpha, kAlphaThreads, T.smem_alpha, args);
    };
    // refinements (solver.py:184-195): row stage (A = Q at t = 0, hat_alpha_R after), then either
    // the L statistics + alpha_R hand-off (t < T-1) or the output O = L Y (t = T-1).  With factor
    // export the last refinement also runs the statistics pass and writes L' from it
    // (factors.py:57-79 layout); R' comes from the last row stage's softmax.  With
    // MBX_FLAG_ALL_ITERS every refinement t writes slice t of both factors (the backward pass).
    const bool all_iters = (flags & MBX_FLAG_ALL_ITERS) != 0;
    const size_t rslice = (size_t)g0.bh * g.gq * g.gk * g.s1 * g.s2 * g.s2;
    const size_t lslice = (size_t)g0.bh * g.gq * g.gk * g.s2 * g.s1 * g.s1;
    TcParams Pt = P;   // per-refinement copy: factor slices
    for (int t = 0; t < g.T; ++t) {
        int last = t == g.T - 1, amode = t > 0;
        Pt.rfac = !r_factor ? nullptr : all_iters ? r_factor + t * rslice : last ? r_factor : nullptr;
        Pt.lfac = !l_factor ? nullptr : all_iters ? l_factor + t * lslice : last ? l_factor : nullptr;
        if (T.flash) {
            ProfScope p("tc_row_flash", stream);
            void* args[] = {(void*)&Pt, (void*)&g, (void*)&amode, (void*)&last};
            if ((e = launch((const void*)tc_row_flash, T.grid_flash, kFThreads, T.smem_flash, args)) != cudaSuccess)
                return e;
        } else if (T.pair) {
            ProfScope p("tc_row_pair", stream);
            void* args[] = {(void*)&Pt, (void*)&g, (void*)&amode, (void*)&last};
            if ((e = launch((const void*)tc_row_pair, T.grid_pair, kPairThreads, T.smem_pair, args)) != cudaSuccess)
                return e;
        } else {
            ProfScope p("tc_row_stage", stream);
            void* args[] = {(void*)&Pt, (void*)&g, (void*)&amode, (void*)&last};
            if ((e = launch((const void*)tc_row_stage, T.grid_row, kRowThreads, T.smem_row, args)) != cudaSuccess)
                return e;
        }
        if (!last) {
            if (T.fused_hand) {   // one key chunk per column: hand-off inside the column stage
                if ((e = column(2, Pt)) != cudaSuccess) return e;
            } else if ((e = column(1, Pt)) != cudaSuccess || (e = alpha(0, Pt)) != cudaSuccess) {
                return e;
            }
        } else {
            if (Pt.lfac && ((e = column(1, Pt)) != cudaSuccess || (e = alpha(1, Pt)) != cudaSuccess)) return e;
            if ((e = column(0, Pt)) != cudaSuccess) return e;
        }
    }
    return cudaGetLastError();
}

// Long problems run as two concurrent halves of the heads, one on the caller's stream and
// one on a side stream (fork / join through events, CUDA-graph capturable): the second
// half's launches fill the ramp-up and drain of the first's persistent grids (KV21: 303 ->
// 279 us with CUDA graphs, scripts/exp_streams.py), while short problems lose to the
// halved work per CTA (C2: 59 -> 68 us), hence the size threshold.  Halves are of the heads
// for one batch, of the batch otherwise (even counts only).  MBX_FLAG_SPLIT / NO_SPLIT (or
// the MBX_SPLIT option) override the threshold.
static bool tc_split(const Geometry& g, int flags) {
    const int B = g.bh / g.heads;
    if (B == 1 ? g.heads % 2 != 0 : B % 2 != 0) return false;   // halves of the heads (B = 1) or of the batch
    if (flags & MBX_FLAG_FACTORS) return false;
    if (flags & MBX_FLAG_NO_SPLIT) return false;
    if (flags & MBX_FLAG_SPLIT) return true;
    const int o = options().split;
    if (o >= 0) return o == 1;
    return (size_t)g.bh * g.gq * g.s2 * g.nkeys >= ((size_t)600 << 10);   // workspace rows
}
static Geometry half_heads(const Geometry& g) {   // B = 1: first half of the heads; else of the batch
    Geometry h = g;
    if (g.bh == g.heads) h.heads = g.heads / 2;
    h.bh = g.bh / 2;
    return h;
}

// Waves: the (b, h) slices of one launch sequence run as consecutive waves of nb batches x nh
// heads (nh < heads only with nb = 1) that reuse one workspace region, so the workspace is
// capped (the paper's mini-sequence chunking) and, for small waves, the W
// exchange of a wave can stay L2-resident between its row and column stages.  The wave
// size is MBX_WAVE (b, h) slices per wave when set, else the largest that keeps the
// workspace under MBX_WS_CAP_MB.  Factor export runs as one wave (factor slices are laid
// out for the whole problem).
struct WavePlan {
    int nb, nh;
};
static Geometry wave_geom(const Geometry& g, int nb, int nh) {
    Geometry w = g;
    w.heads = nh;
    w.bh = nb * nh;
    return w;
}
static WavePlan tc_wave_plan(const Geometry& g, int flags) {
    const int B = g.bh / g.heads, H = g.heads;
    WavePlan w{B, H};
    if (flags & MBX_FLAG_FACTORS) return w;
    const Options& o = options();
    long long per = o.wave;
    if (per == 0) return w;
    if (per < 0) {
        const size_t cap = (size_t)(o.ws_cap_mb > 0 ? o.ws_cap_mb : 1) << 20;
        const size_t one = tc_layout(wave_geom(g, 1, 1)).total;
        per = (long long)(cap / (one ? one : 1));
        // Long problems with an odd number of query tiles: one-head waves, whose K / V sit in
        // L2, run the half-packed row stage (a K/V row serves halves of two items from L2) --
        // N=32k (h,w) 2.03 -> 1.72 ms (waves of 3 / 2 heads: 1.96 / 1.85), (3h,w) 0.88 -> 0.85 ms;
        // only when one head still gives every SM dozens of row tasks (KV21 (h,w), 945 tasks
        // per head, loses: 0.276 -> 0.376 ms).
        const size_t kv_head = (size_t)g.gk * g.s1 * g.s2 * (size_t)(g.d + g.dv) * 2;
        const long long pair_tasks_head = (long long)((g.gq * g.s1 + 1) / 2) * g.gk;
        if (o.pair < 0 && g.gq > 1 && g.gq % 2 == 1 && g.s2 <= kMaxS2 && kv_head <= kPairKvBytes &&
            (size_t)g.bh * kv_head > kPairKvBytes && pair_tasks_head >= kWavePairTasks)
            per = 1;
        // Long tile rows (online-softmax row stage): one-head waves keep a head's K / V in L2
        // while its row tasks stream them -- Wan 720p layer (h,w) 8.67 -> 7.90 ms, (3h,w)
        // 3.74 -> 3.50 ms; KV21 720p (945 tasks per head) and (f,hw) N=32k (273) lose.
        const long long flash_tasks_head = (long long)g.gq * g.s1 * ((g.s2 + kFKC - 1) / kFKC) * g.gk;
        if (o.pair < 0 && g.s2 > kMaxS2 && g.bh > 1 && flash_tasks_head >= kWavePairTasks) per = 1;
        if (per < 1) per = 1;
    }
    if (per >= g.bh) return w;
    if (per >= H) {
        w.nb = (int)(per / H);
    } else {
        w.nb = 1;
        w.nh = (int)per;
    }
    return w;
}
static size_t tc_wave_bytes(const Geometry& g, int flags) {
    const WavePlan w = tc_wave_plan(g, flags);
    return tc_layout(wave_geom(g, w.nb, w.nh)).total;
}

static size_t tc_workspace_bytes_ordered(const Geometry& g, int flags) {
    if (tc_split(g, flags)) return 2 * align256(tc_wave_bytes(half_heads(g), flags));
    return tc_wave_bytes(g, flags);
}

size_t tc_workspace_bytes(const Geometry& g, int flags) {
    if (g.nf == 0 && (g.q_order || g.kv_order))   // gathered copies + the slot-order problem
        return gather_bytes(g) + tc_workspace_bytes_ordered(slot_geometry(g), flags);
    return tc_workspace_bytes_ordered(g, flags);
}

// One launch sequence per wave, in (batch, head) order on `stream`; later waves use PDL
// (every stage waits for its predecessor before it touches the shared workspace).
static cudaError_t tc_forward_waves(const Geometry& g, int flags, const void* q, const void* k, const void* v,
                                    void* out, float* l_factor, float* r_factor, void* workspace, int dev,
                                    cudaStream_t stream) {
    const WavePlan w = tc_wave_plan(g, flags);
    const int B = g.bh / g.heads, H = g.heads;
    if (w.nb == B && w.nh == H)
        return tc_forward_one(g, flags, q, k, v, out, l_factor, r_factor, workspace, dev, stream);
    auto at = [](const void* p, const int64_t* st, int b, int h) {
        return const_cast<char*>(reinterpret_cast<const char*>(p)) + ((size_t)b * st[0] + (size_t)h * st[1]) * 2;
    };
    bool first = true;
    for (int b0 = 0; b0 < B; b0 += w.nb) {
        const int nb = B - b0 < w.nb ? B - b0 : w.nb;
        for (int h0 = 0; h0 < H; h0 += w.nh) {
            const int nh = H - h0 < w.nh ? H - h0 : w.nh;
            const Geometry gw = wave_geom(g, nb, nh);
            cudaError_t e = tc_forward_one(gw, flags, at(q, g.qs, b0, h0), at(k, g.ks, b0, h0), at(v, g.vs, b0, h0),
                                           at(out, g.os, b0, h0), nullptr, nullptr, workspace, dev, stream, !first);
            if (e != cudaSuccess) return e;
            first = false;
        }
    }
    return cudaSuccess;
}

// Side stream + fork/join events of one (device, caller stream); created all-or-nothing.
struct SideStream {
    int dev;
    cudaStream_t caller;
    cudaStream_t side;
    cudaEvent_t fork, join;
};
static std::mutex g_side_mu;
static SideStream* g_sides = nullptr;
static int g_nsides = 0, g_cap_sides = 0;

static SideStream* side_for(int dev, cudaStream_t caller, bool may_create) {
    std::lock_guard<std::mutex> lock(g_side_mu);
    for (int i = 0; i < g_nsides; ++i)
        if (g_sides[i].dev == dev && g_sides[i].caller == caller) return &g_sides[i];
    if (!may_create) return nullptr;
    SideStream s{dev, caller, nullptr, nullptr, nullptr};
    int prio = 0;
    cudaStreamGetPriority(caller, &prio);   // the side stream inherits the caller's priority
    if (cudaStreamCreateWithPriority(&s.side, cudaStreamNonBlocking, prio) != cudaSuccess) return nullptr;
    if (cudaEventCreateWithFlags(&s.fork, cudaEventDisableTiming) != cudaSuccess) {
        cudaStreamDestroy(s.side);
        return nullptr;
    }
    if (cudaEventCreateWithFlags(&s.join, cudaEventDisableTiming) != cudaSuccess) {
        cudaEventDestroy(s.fork);
        cudaStreamDestroy(s.side);
        return nullptr;
    }
    if (g_nsides == g_cap_sides) {   // entries are never freed: pointers stay valid
        const int cap = g_cap_sides ? 2 * g_cap_sides : 8;
        SideStream* grown = new SideStream[cap];
        for (int i = 0; i < g_nsides; ++i) grown[i] = g_sides[i];
        // old array intentionally leaked: callers may hold pointers into it
        g_sides = grown;
        g_cap_sides = cap;
    }
    g_sides[g_nsides] = s;
    return &g_sides[g_nsides++];
}

static cudaError_t tc_forward_ordered(const Geometry& g, int flags, const void* q, const void* k, const void* v,
                                      void* out, float* l_factor, float* r_factor, void* workspace, cudaStream_t stream);

cudaError_t tc_forward(const Geometry& g, int flags, const void* q, const void* k, const void* v, void* out,
                       float* l_factor, float* r_factor, void* workspace, cudaStream_t stream) {
    if (!(g.nf == 0 && (g.q_order || g.kv_order)))
        return tc_forward_ordered(g, flags, q, k, v, out, l_factor, r_factor, workspace, stream);
    // permuted plan: gather q / k / v into slot order (the reference's q[order], solver.py:103-106),
    // run the identity-order problem, scatter the output back (attention_output, solver.py:216)
    const Geometry gs = slot_geometry(g);
    const int64_t nq = (int64_t)g.c1q * g.s1 * g.c2 * g.s2, nk = (int64_t)g.c1k * g.s1 * g.c2 * g.s2;
    __nv_bfloat16* qg = reinterpret_cast<__nv_bfloat16*>(workspace);
    __nv_bfloat16* og = qg + (size_t)g.bh * nq * kD;
    __nv_bfloat16* kg = og + (size_t)g.bh * nq * kD;
    __nv_bfloat16* vg = kg + (size_t)g.bh * nk * kD;
    char* rest = reinterpret_cast<char*>(workspace) + gather_bytes(g);
    int dev = 0;
    cudaError_t e0 = cudaGetDevice(&dev);
    if (e0 != cudaSuccess) return e0;
    if (((uintptr_t)q | (uintptr_t)k | (uintptr_t)v | (uintptr_t)out) & 15) return TC_FAIL("tensor map / argument check");
    // one 16-byte chunk per thread, no grid-stride loop: every load in flight at once
    auto grid_for = [&](int64_t rows) { return (unsigned)((rows * 16 + 255) / 256); };
    {
        ProfScope p("tc_gather", stream);
        gather_rows<<<grid_for(g.bh * nq), 256, 0, stream>>>(reinterpret_cast<const __nv_bfloat16*>(q), qg, g.q_order, nq, g.bh,
                                              g.heads, g.qs[0], g.qs[1], g.qs[2], 0);
        gather_rows<<<grid_for(g.bh * nk), 256, 0, stream>>>(reinterpret_cast<const __nv_bfloat16*>(k), kg, g.kv_order, nk, g.bh,
                                              g.heads, g.ks[0], g.ks[1], g.ks[2], 0);
        gather_rows<<<grid_for(g.bh * nk), 256, 0, stream>>>(reinterpret_cast<const __nv_bfloat16*>(v), vg, g.kv_order, nk, g.bh,
                                              g.heads, g.vs[0], g.vs[1], g.vs[2], 0);
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    e = tc_forward_ordered(gs, flags, qg, kg, vg, og, l_factor, r_factor, rest, stream);
    if (e != cudaSuccess) return e;
    {
        ProfScope p("tc_scatter", stream);
        gather_rows<<<grid_for(g.bh * nq), 256, 0, stream>>>(reinterpret_cast<const __nv_bfloat16*>(out), og, g.q_order, nq, g.bh,
                                              g.heads, g.os[0], g.os[1], g.os[2], 1);
    }
    return cudaGetLastError();
}

static cudaError_t tc_forward_ordered(const Geometry& g, int flags, const void* q, const void* k, const void* v,
                                      void* out, float* l_factor, float* r_factor, void* workspace, cudaStream_t stream) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    // The tensor-map encode is a driver call: it needs the device's primary context current on
    // this thread, which a thread that has only made runtime calls that do not touch the context
    // (e.g. PyTorch's autograd worker) may not have yet.  cudaSetDevice binds it (once per thread).
    thread_local int bound_dev = -1;
    if (bound_dev != dev) {
        if ((e = cudaSetDevice(dev)) != cudaSuccess) return e;
        bound_dev = dev;
    }
    const bool factors = l_factor || r_factor;
    SideStream* ss = nullptr;
    if (!factors && tc_split(g, flags)) {
        cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
        if ((e = cudaStreamIsCapturing(stream, &cs)) != cudaSuccess) return e;
        // never create streams/events inside a capture: split only if this caller's side exists
        ss = side_for(dev, stream, cs == cudaStreamCaptureStatusNone);
    }
    if (!ss) {
        return tc_forward_waves(g, flags, q, k, v, out, l_factor, r_factor, workspace, dev, stream);
    }
    const Geometry h = half_heads(g);
    const size_t wsh = align256(tc_wave_bytes(h, flags));
    auto at = [&](const void* p, const int64_t* st) {   // start of the second half (bf16 elements)
        const size_t off = g.bh == g.heads ? (size_t)h.heads * (size_t)st[1] : (size_t)(h.bh / h.heads) * (size_t)st[0];
        return reinterpret_cast<const char*>(p) + off * 2;
    };
    if ((e = cudaEventRecord(ss->fork, stream)) != cudaSuccess || (e = cudaStreamWaitEvent(ss->side, ss->fork, 0)) != cudaSuccess)
        return e;
    cudaError_t e1 = tc_forward_waves(h, flags, q, k, v, out, nullptr, nullptr, workspace, dev, stream);
    cudaError_t e2 = tc_forward_waves(h, flags, at(q, g.qs), at(k, g.ks), at(v, g.vs), const_cast<char*>(at(out, g.os)),
                                    nullptr, nullptr, reinterpret_cast<char*>(workspace) + wsh, dev, ss->side);
    // the join is recorded even if a half failed, so the side stream never dangles outside a capture
    if ((e = cudaEventRecord(ss->join, ss->side)) != cudaSuccess || (e = cudaStreamWaitEvent(stream, ss->join, 0)) != cudaSuccess)
        return e;
    return e1 != cudaSuccess ? e1 : e2;
}

}  // namespace mbx

#ifdef MBX_TRACE
extern "C" int mbx_trace_dump(void* host, size_t bytes) {
    if (bytes < sizeof(mbx::g_trace)) return -1;
    cudaDeviceSynchronize();
    cudaMemcpyFromSymbol(host, mbx::g_trace, sizeof(mbx::g_trace));
    cudaMemset(reinterpret_cast<void*>(0), 0, 0);
    static unsigned long long zeros[4 * 16 * 2048];
    cudaMemcpyToSymbol(mbx::g_trace, zeros, sizeof(zeros));
    return (int)sizeof(mbx::g_trace);
}
extern "C" int mbx_trace_col_dump(void* host, size_t bytes) {
    if (bytes < sizeof(mbx::g_trace_col)) return -1;
    cudaDeviceSynchronize();
    cudaMemcpyFromSymbol(host, mbx::g_trace_col, sizeof(mbx::g_trace_col));
    static unsigned long long zeros[4 * 16 * 2048];
    cudaMemcpyToSymbol(mbx::g_trace_col, zeros, sizeof(zeros));
    return (int)sizeof(mbx::g_trace_col);
}
extern "C" int mbx_span_dump(void* host, size_t bytes) {
    if (bytes < sizeof(mbx::g_span)) return -1;
    cudaDeviceSynchronize();
    cudaMemcpyFromSymbol(host, mbx::g_span, sizeof(mbx::g_span));
    return (int)sizeof(mbx::g_span);
}
#endif
