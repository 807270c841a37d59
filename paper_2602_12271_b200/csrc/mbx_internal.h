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
};

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
                            const Workspace& ws, cudaStream_t stream);
cudaError_t generic_apply(const Geometry& g, int dtype, const float* l_factor,
                          const float* r_factor, const void* v, void* out,
                          const Workspace& ws, cudaStream_t stream);

// tcgen05 tensor-core kernels (mbx_tc.cu) -- bf16, contiguous tile rows.
bool tc_supported(const Geometry& g, int dtype, int flags);
size_t tc_workspace_bytes(const Geometry& g);
cudaError_t tc_forward(const Geometry& g, const void* q, const void* k, const void* v,
                       void* out, void* workspace, cudaStream_t stream);

}  // namespace mbx
