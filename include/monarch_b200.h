/*
 * monarch_b200.h — C ABI of the B200-native tiled MonarchAttention forward.
 *
 * This is the drop-in boundary for the reference's hot path
 * (/root/reference/pkg/src/monarchbench):
 *
 *   mbx_forward   replaces  solve_tiled(problem, plan, solver)  solver.py:161-204
 *                           + attention_output(factors, v)      solver.py:207-217
 *                           and, with c1 = c2 = 1, solve(...)   solver.py:114-158
 *                           (factors optional: L', R' in the TiledMonarchFactors
 *                           layout, factors.py:57-79)
 *   mbx_apply     replaces  apply_factors(factors, v)           factors.py:110-125
 *                           via attention_output                solver.py:207-217
 *
 * All pointers are DEVICE pointers owned by the caller (the library never
 * allocates or frees user memory).  Work is enqueued on `stream` (a
 * cudaStream_t passed as void*); no call synchronizes the device.  The
 * descriptor is read during the call and not retained.
 *
 * Library-owned resources (process lifetime, created on first use):
 *   - a cache of launch parameters (TMA tensor maps) keyed by the descriptor,
 *     the pointers and the device, so repeated calls skip the host-side encode;
 *   - for long tensor-core problems (see MBX_FLAG_SPLIT), one side stream and
 *     a fork/join event pair PER (device, caller stream): half of the heads run
 *     on the side stream, which first waits for an event recorded on `stream`
 *     and on completion is joined back into `stream` by a second event.  All
 *     work therefore stays ordered after everything previously enqueued on
 *     `stream`, and everything later enqueued on `stream` runs after it.  The
 *     fork/join is capturable: under stream capture the side stream joins the
 *     caller's capture (the split is skipped if the side stream for that caller
 *     stream does not exist yet, so no stream is created inside a capture).
 *
 * Errors: every entry point returns an mbx_status; a non-zero status leaves a
 * thread-local message readable with mbx_last_error().  The Python layer maps
 * MBX_ERR_BAD_SHAPE / BAD_PLAN / BAD_ITERS / BAD_EPS to the reference's
 * SolverError / LayoutError (ValueError subclasses, solver.py:25-26,
 * layout.py:21-22).
 */
#ifndef MONARCH_B200_H
#define MONARCH_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MBX_ABI_VERSION 1

typedef enum mbx_status {
    MBX_OK = 0,
    MBX_ERR_BAD_SHAPE = 1,   /* inconsistent sizes / strides (SolverError, ShapeError)   */
    MBX_ERR_BAD_PLAN = 2,    /* tiling does not divide the blocks (LayoutError)          */
    MBX_ERR_BAD_ITERS = 3,   /* iterations < 1 (SolverConfig, solver.py:73-74)           */
    MBX_ERR_BAD_EPS = 4,     /* eps outside (0, 1e-6] (solver.py:75-77)                  */
    MBX_ERR_BAD_DTYPE = 5,
    MBX_ERR_NULL = 6,        /* required pointer is NULL                                 */
    MBX_ERR_WORKSPACE = 7,   /* workspace smaller than mbx_workspace_bytes()             */
    MBX_ERR_UNSUPPORTED = 8, /* shape outside what the kernels implement (e.g. d > 256)  */
    MBX_ERR_CUDA = 9         /* a CUDA launch failed                                     */
} mbx_status;

typedef enum mbx_dtype {
    MBX_F32 = 0,   /* fp32 I/O, fp32 arithmetic (parity mode, 1e-4 rel-L2)   */
    MBX_BF16 = 1   /* bf16 I/O, fp32 accumulate / softmax (2e-2 rel-L2)       */
} mbx_dtype;

/* flags */
#define MBX_FLAG_FORCE_GENERIC 0x1  /* route to the SIMT kernels even if a tensor-core path applies */
#define MBX_FLAG_NO_OUTPUT 0x2      /* factors only (solve_tiled without attention_output)          */
#define MBX_FLAG_FACTORS 0x4        /* the forward will export L' and R': size the workspace and pick
                                       the path for it (mbx_workspace_bytes / mbx_selected_path)     */
#define MBX_FLAG_NO_SPLIT 0x8       /* never run the concurrent head/batch halves                   */
#define MBX_FLAG_SPLIT 0x10         /* always run the concurrent halves when the shape allows        */
#define MBX_FLAG_ALL_ITERS 0x20     /* export the factors of EVERY refinement: l_factor / r_factor hold
                                       T slices [T][B][H][...] (the backward pass needs them)        */

/*
 * One forward problem, batched over (batch, heads).  Tokens of a (b, h)
 * slice live at  base + b*stride[0] + h*stride[1] + row*stride[2] (+ feature,
 * contiguous).  Slot order: ordered index p of query tile-row l1, row l2,
 * tile-column j1, column j2 is p = ((l1*s1 + l2)*c2 + j1)*s2 + j2 (the
 * reshape of solver.py:178-179); q_order[p] / kv_order[p] give the token row
 * it reads (TokenOrdering.to_phi, layout.py:89-94); NULL = identity.
 *
 * Square problems have c1_q == c1_kv.  Chunked-KV (causal autoregressive
 * rollout) problems have c1_q < c1_kv: the queries are the last query-tile
 * rows of the key grid, every query tile attends to every key tile.
 */
typedef struct mbx_desc {
    int32_t abi_version;          /* must be MBX_ABI_VERSION */
    int32_t dtype;                /* mbx_dtype for q, k, v and out */
    int32_t batch, heads;
    int32_t head_dim;             /* d   (q, k) */
    int32_t v_dim;                /* d_v (v, out) */
    int32_t c1_q, c1_kv, c2;      /* tile grid */
    int32_t s1, s2;               /* tile shape (rows, columns) */
    int32_t iterations;           /* T >= 1 (SolverConfig.iterations) */
    int32_t flags;
    float scale;                  /* logit scale applied to q (solver.py:58-60, 104) */
    double eps_div;               /* SolverConfig.eps_div (solver.py:67, 188), in (0, 1e-6] */
    double eps_log;               /* SolverConfig.eps_log (solver.py:68, 191), in (0, 1e-6];
                                     c_L is evaluated as sum R z - lse, which equals
                                     sum R log max(R, eps_log) up to terms < eps_log*|log eps_log| */
    int64_t q_stride[3];          /* (batch, head, token) strides in elements */
    int64_t k_stride[3];
    int64_t v_stride[3];
    int64_t o_stride[3];
    const int32_t* q_order;       /* device, c1_q*s1*c2*s2 entries or NULL */
    const int32_t* kv_order;      /* device, c1_kv*s1*c2*s2 entries or NULL */
    /* Optional closed form of the orders for neighborhood tile plans
     * (make_tile_plan, layout.py:319-351): key grid (f_kv, h, w) and
     * neighborhood (n_f, n_h, n_w).  nbhd[0] == 0 means "orders only".  When
     * set, it must describe the same permutation as q_order / kv_order; the
     * tensor-core path addresses tile rows with it (permutation folded into
     * TMA coordinates, no gather). */
    int32_t grid[3];
    int32_t nbhd[3];
} mbx_desc;

/* Library / ABI version (== MBX_ABI_VERSION for a matching build). */
int mbx_version(void);

/* Thread-local message for the last non-OK status on this thread. */
const char* mbx_last_error(void);

/* Validate a descriptor without launching anything. */
int mbx_validate(const mbx_desc* desc);

/* Device workspace the forward needs (bytes, 256-byte aligned). */
size_t mbx_workspace_bytes(const mbx_desc* desc);

/* 0 = SIMT generic kernels, 1 = tcgen05 tensor-core kernels. */
int mbx_selected_path(const mbx_desc* desc);

/* Host-side: token row that slot `slot` of the query (is_query=1) or key grid
 * reads under the descriptor's closed-form addressing (identity when no
 * neighborhood is given).  -1 on invalid input.  Lets callers check the
 * closed form against their order arrays without a GPU. */
int64_t mbx_token_index(const mbx_desc* desc, int is_query, int64_t slot);

/*
 * Forward: T alternating R/L refinements followed by O = L (R V).
 * out (optional if MBX_FLAG_NO_OUTPUT) is written in token (phi) order.
 * l_factor / r_factor (optional, fp32, per (b,h) contiguous) receive the final
 * L' (c1_q,c2,c1_kv,c2,s2,s1,s1) and R' (c1_q,c2,c1_kv,c2,s1,s2,s2).
 */
int mbx_forward(const mbx_desc* desc, const void* q, const void* k, const void* v,
                void* out, float* l_factor, float* r_factor,
                void* workspace, size_t workspace_bytes, void* stream);

/*
 * Block-apply of given factors (apply_factors, factors.py:110-125):
 * out = L' (R' V) with V gathered through kv_order and out scattered through
 * q_order.  Only v_dim, dtype, grid/tile sizes, v/o strides and orders are read.
 */
int mbx_apply(const mbx_desc* desc, const float* l_factor, const float* r_factor,
              const void* v, void* out, void* workspace, size_t workspace_bytes,
              void* stream);

/* Workspace for mbx_apply (the Y = R V intermediate). */
size_t mbx_apply_workspace_bytes(const mbx_desc* desc);

/*
 * Backward pass (the paper's finetuning backward; not in the
 * reference package): gradients of sum(out * dout) with respect to q, k and v.
 * l_factors / r_factors are the factors of every refinement as written by
 * mbx_forward with MBX_FLAG_ALL_ITERS (T slices; for T = 1 the ordinary export).
 * dq / dk / dv use the q / k / v strides of the descriptor, dout uses o_stride.
 * fp32 arithmetic for both dtypes (bf16 tensors are read and written as bf16).
 */
int mbx_backward(const mbx_desc* desc, const void* q, const void* k, const void* v, const void* dout,
                 const float* l_factors, const float* r_factors, void* dq, void* dk, void* dv,
                 void* workspace, size_t workspace_bytes, void* stream);
size_t mbx_backward_workspace_bytes(const mbx_desc* desc);

/*
 * Per-kernel timing for benchmarks (thread-local).  While enabled, every
 * kernel the library launches is bracketed by CUDA events on its stream.
 * mbx_profile_collect synchronizes those events, writes up to `max_entries`
 * (name, milliseconds) pairs in launch order, clears the record and returns
 * the number of launches recorded.
 */
int mbx_profile_enable(int on);
int mbx_profile_collect(float* ms, const char** names, int max_entries);
/* Same, with each launch's start relative to the first recorded start (ms), so
 * launches that overlap on different streams can be merged into one span. */
int mbx_profile_collect_ex(float* start_ms, float* ms, const char** names, int max_entries);

/*
 * Process-wide diagnostic options (initialised from the environment variables
 * of the same name on first use): "MBX_PDL" (programmatic dependent launch,
 * default 1), "MBX_L2HINT" (L2 residency hints: bit 0 W stores evict_last, bit 1
 * the W exchange's last reads evict_first; default -1 = bit 1, plus bit 0 when a
 * launch's exchange exceeds 128 MiB), "MBX_PAIR" (row-stage
 * variant, -1 auto / 0 classic / 1 half-packed), "MBX_WIDE" (wide column stage
 * for s1 <= 32, 0), "MBX_SPLIT" (concurrent halves, -1 auto / 0 / 1),
 * "MBX_DBG" (timing bits, results wrong), "MBX_VERBOSE", "MBX_WAVE" ((b,h)
 * slices per wave of the tensor-core path, -1 automatic, 0 one wave) and
 * "MBX_WS_CAP_MB" (automatic waves keep the workspace under this many MiB,
 * default 2048; waves run in sequence on `stream` and reuse one workspace
 * region -- the mini-sequence chunking of the paper).  Options that change
 * the workspace size must not change between mbx_workspace_bytes and
 * mbx_forward.  Returns the previous
 * value, or -1000 for an unknown name.  Not for use while another thread is
 * enqueueing forwards.
 */
int mbx_set_option(const char* name, int value);

#ifdef __cplusplus
}
#endif

#endif /* MONARCH_B200_H */
