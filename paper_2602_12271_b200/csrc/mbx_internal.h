// Internal declarations shared by the C-ABI layer and the kernel files.
#pragma once

#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>
#include <stddef.h>

#include "../../include/monarch_b200.h"

namespace mbx {

// Derived geometry of one forward problem (all sizes per (b, h) slice).
struct Geometry {
    int bh, heads;              // batch*heads, heads
    int d, dv;
    int c1q, c1k, c2, s1, s2;
    int gq, gk;                 // query / key tiles
    int nkeys;                  // keys per column stage: gk * s1
    int T;
    float scale, eps_div, eps_log;
    int64_t qs[3], ks[3], vs[3], os[3];
    const int32_t* q_order;
    const int32_t* kv_order;
    int F, H, W;                // key grid (neighborhood plans)
    int nf, nh, nw;             // neighborhood; nf == 0 -> identity / orders only
};

// Token row of (tile, row r, column 0) under the closed-form addressing:
// identity slot order, or a neighborhood plan whose digits are
// (f/nf, h/nh, nf, nh, w/nw, nw) (layout.py:319-332).  Query tiles are the last
// c1q tile-rows of the key grid (chunked-KV), shifted to q's own frames.
__host__ __device__ inline int64_t row_base(const Geometry& g, bool is_q, int tile, int r) {
    const int l1 = tile / g.c2, j1 = tile - (tile / g.c2) * g.c2;
    if (g.nf == 0) return ((int64_t)(l1 * g.s1 + r) * g.c2 + j1) * g.s2;
    const int hcn = g.H / g.nh;
    const int L1 = is_q ? l1 + (g.c1k - g.c1q) : l1;
    const int fc = L1 / hcn, hc = L1 - (L1 / hcn) * hcn;
    const int ff = r / g.nh, hf = r - (r / g.nh) * g.nh;
    int64_t tok = ((int64_t)(fc * g.nf + ff) * g.H + hc * g.nh + hf) * g.W + j1 * g.nw;
    if (is_q) tok -= (int64_t)((g.c1k - g.c1q) / hcn) * g.nf * g.H * g.W;
    return tok;
}

// fp32 workspace carved out of the caller's buffer.
struct Workspace {
    float* alpha_l;   // [bh][gq][s2][nkeys][d]   alpha_L of the current iteration
    float* y;         // [bh][gq][s2][nkeys][dv]  Y = R V (last iteration only)
    float* c_l;       // [bh][gq][s2][nkeys]      entropy term c_L
    float* lse;       // [bh][gq][s2][s1]         log-normaliser of each L row
    float* alpha_r;   // [bh][gq][gk][s1][s2][d]  alpha_R for the next iteration
    float* c_r;       // [bh][gq][gk][s1][s2]     column mass c_R
};

size_t workspace_layout(const Geometry& g, char* base, Workspace* ws);

// Brackets one kernel launch with CUDA events when profiling is enabled
// (mbx_profile_enable); no-op otherwise.
struct ProfScope {
    ProfScope(const char* name, cudaStream_t s);
    ~ProfScope();
    int slot;
    cudaStream_t stream;
};

// SIMT kernels (mbx_generic.cu) -- any plan, fp32 or bf16 I/O.
cudaError_t generic_forward(const Geometry& g, int dtype, const void* q, const void* k,
                            const void* v, void* out, float* l_factor, float* r_factor,
                            const Workspace& ws, cudaStream_t stream, bool all_iters = false);
cudaError_t generic_apply(const Geometry& g, int dtype, const float* l_factor,
                          const float* r_factor, const void* v, void* out,
                          const Workspace& ws, cudaStream_t stream);

// Process-wide diagnostic options (mbx_set_option; initialised once from the
// MBX_* environment variables).  -1 = automatic choice.
struct Options {
    int pdl = 1;        // programmatic dependent launch between stages
    int l2hint = 1;     // W stores evict_last, last W reads evict_first
    int dbg = 0;        // MBX_DBG timing bits (wrong results by construction)
    int pair = -1;      // row stage: 0 classic, 1 half-packed
    int wide = 0;       // 1: FlashAttention-style column stage for s1 <= 32 too (T = 1)
    int split = -1;     // concurrent halves: 0 off, 1 on
    int verbose = 0;    // print why a problem leaves the tcgen05 path / setup failures
    int fusedhand = 1;  // T >= 2: alpha_R hand-off inside the column stage when a column is one key chunk
    int wave = -1;      // (b, h) slices per wave of the tensor-core path: -1 from the cap, 0 one wave
    int ws_cap_mb = 2048;   // automatic waves keep the tensor-core workspace under this many MiB
    int wide2 = 1;          // output pass of the wide column stage with two item streams per CTA (0: one)
    unsigned version = 0;   // bumped on every change (keys the launch-parameter cache)
};
const Options& options();
int set_option(const char* name, int value);

// tcgen05 tensor-core kernels (mbx_tc.cu) -- bf16, contiguous tile rows.
// `factors`: the call exports L' and R' (needs s1 <= 128 on this path).
bool tc_supported(const Geometry& g, int dtype, int flags, bool factors);
size_t tc_workspace_bytes(const Geometry& g, int flags);
cudaError_t tc_forward(const Geometry& g, int flags, const void* q, const void* k, const void* v,
                       void* out, float* l_factor, float* r_factor, void* workspace,
                       cudaStream_t stream);

// Backward pass (mbx_backward.cu): dq, dk, dv from dout and the factors of every refinement.
size_t backward_workspace_bytes(const Geometry& g);
cudaError_t backward(const Geometry& g, int dtype, const void* q, const void* k, const void* v, const void* dout,
                     const float* l_factors, const float* r_factors, void* dq, void* dk, void* dv, void* ws,
                     cudaStream_t stream);

}  // namespace mbx
