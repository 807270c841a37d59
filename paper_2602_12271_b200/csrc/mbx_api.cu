// C-ABI entry points (include/monarch_b200.h): descriptor validation with the
// reference's error conditions, workspace carving, path selection.
#include "mbx_internal.h"

#include <stdarg.h>
#include <stdio.h>
#include <string>
#include <vector>

namespace {

thread_local std::string g_last_error;

int fail(int status, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_last_error = buf;
    return status;
}

size_t align_up(size_t x) { return (x + 255) & ~size_t(255); }

// Mirrors AttentionProblem / SolverConfig / TilePlan validation
// (solver.py:39-48, 72-77; layout.py:294-297).
int validate(const mbx_desc* d, mbx::Geometry* g) {
    if (!d) return fail(MBX_ERR_NULL, "descriptor is NULL");
    if (d->abi_version != MBX_ABI_VERSION)
        return fail(MBX_ERR_BAD_SHAPE, "abi_version %d != %d", d->abi_version, MBX_ABI_VERSION);
    if (d->dtype != MBX_F32 && d->dtype != MBX_BF16)
        return fail(MBX_ERR_BAD_DTYPE, "unknown dtype %d", d->dtype);
    if (d->iterations < 1) return fail(MBX_ERR_BAD_ITERS, "iterations must be >= 1");
    if (!(d->eps_div > 0.0 && d->eps_div <= 1e-6))
        return fail(MBX_ERR_BAD_EPS, "eps_div must lie in (0, 1e-6], got %g", d->eps_div);
    if (!(d->eps_log > 0.0 && d->eps_log <= 1e-6))
        return fail(MBX_ERR_BAD_EPS, "eps_log must lie in (0, 1e-6], got %g", d->eps_log);
    if (d->batch < 1 || d->heads < 1)
        return fail(MBX_ERR_BAD_SHAPE, "batch and heads must be >= 1");
    if (d->head_dim < 1 || d->v_dim < 1)
        return fail(MBX_ERR_BAD_SHAPE, "head_dim and v_dim must be >= 1");
    if (d->head_dim > 256 || d->v_dim > 256)
        return fail(MBX_ERR_UNSUPPORTED, "head_dim/v_dim > 256 not implemented");
    if (d->c1_q < 1 || d->c1_kv < 1 || d->c2 < 1 || d->s1 < 1 || d->s2 < 1)
        return fail(MBX_ERR_BAD_PLAN, "tile grid (%d,%d,%d) / tile (%d,%d) must be >= 1",
                    d->c1_q, d->c1_kv, d->c2, d->s1, d->s2);
    if (d->c1_q > d->c1_kv)
        return fail(MBX_ERR_BAD_PLAN, "more query tile-rows (%d) than key tile-rows (%d)",
                    d->c1_q, d->c1_kv);
    const int64_t nk = (int64_t)d->c1_kv * d->s1 * d->c2 * d->s2;
    if (nk > (int64_t)1 << 30) return fail(MBX_ERR_UNSUPPORTED, "too many tokens");
    if (!(d->scale == d->scale) || d->scale == 1.0f / 0.0f || d->scale == -1.0f / 0.0f)
        return fail(MBX_ERR_BAD_SHAPE, "non-finite logit scale");
    for (int i = 0; i < 3; ++i)
        if (d->q_stride[i] < 0 || d->k_stride[i] < 0 || d->v_stride[i] < 0 || d->o_stride[i] < 0)
            return fail(MBX_ERR_BAD_SHAPE, "negative stride");
    if (d->nbhd[0] > 0) {
        const int F = d->grid[0], H = d->grid[1], W = d->grid[2];
        const int nf = d->nbhd[0], nh = d->nbhd[1], nw = d->nbhd[2];
        if (F < 1 || H < 1 || W < 1 || nh < 1 || nw < 1 || F % nf || H % nh || W % nw)
            return fail(MBX_ERR_BAD_PLAN, "neighborhood (%d,%d,%d) must divide grid (%d,%d,%d)", nf, nh, nw,
                        F, H, W);
        if (d->s1 != nf * nh || d->s2 != nw || d->c2 != W / nw || d->c1_kv != (F / nf) * (H / nh) ||
            d->c1_q % (H / nh))
            return fail(MBX_ERR_BAD_PLAN, "neighborhood description inconsistent with the tile grid");
    }
    if (d->q_stride[2] < d->head_dim || d->k_stride[2] < d->head_dim || d->v_stride[2] < d->v_dim ||
        d->o_stride[2] < d->v_dim)
        return fail(MBX_ERR_BAD_SHAPE, "token stride smaller than the feature width");
    if (g) {
        g->bh = d->batch * d->heads;
        g->heads = d->heads;
        g->d = d->head_dim;
        g->dv = d->v_dim;
        g->c1q = d->c1_q;
        g->c1k = d->c1_kv;
        g->c2 = d->c2;
        g->s1 = d->s1;
        g->s2 = d->s2;
        g->gq = d->c1_q * d->c2;
        g->gk = d->c1_kv * d->c2;
        g->nkeys = g->gk * d->s1;
        g->T = d->iterations;
        g->scale = d->scale;
        g->eps_div = d->eps_div < 1e-37 ? 1e-37f : (float)d->eps_div;
        g->eps_log = (float)d->eps_log;
        for (int i = 0; i < 3; ++i) {
            g->qs[i] = d->q_stride[i];
            g->ks[i] = d->k_stride[i];
            g->vs[i] = d->v_stride[i];
            g->os[i] = d->o_stride[i];
        }
        g->q_order = d->q_order;
        g->kv_order = d->kv_order;
        g->F = d->grid[0];
        g->H = d->grid[1];
        g->W = d->grid[2];
        g->nf = d->nbhd[0] > 0 ? d->nbhd[0] : 0;
        g->nh = d->nbhd[1];
        g->nw = d->nbhd[2];
    }
    return MBX_OK;
}

struct ProfRecord {
    const char* name;
    cudaEvent_t start, stop;
};
thread_local bool g_prof_on = false;
thread_local std::vector<ProfRecord> g_prof;

}  // namespace

namespace mbx {

ProfScope::ProfScope(const char* name, cudaStream_t s) : slot(-1), stream(s) {
    if (!g_prof_on) return;
    ProfRecord r{name, nullptr, nullptr};
    cudaEventCreate(&r.start);
    cudaEventCreate(&r.stop);
    cudaEventRecord(r.start, s);
    slot = (int)g_prof.size();
    g_prof.push_back(r);
}

ProfScope::~ProfScope() {
    if (slot >= 0) cudaEventRecord(g_prof[slot].stop, stream);
}

size_t workspace_layout(const Geometry& g, char* base, Workspace* ws) {
    const size_t bh = g.bh;
    const size_t cols = bh * g.gq * g.s2;
    size_t off = 0;
    auto carve = [&](size_t floats) {
        float* p = base ? reinterpret_cast<float*>(base + off) : nullptr;
        off += align_up(floats * sizeof(float));
        return p;
    };
    Workspace w{};
    w.alpha_l = carve(cols * g.nkeys * g.d);
    w.y = carve(cols * g.nkeys * g.dv);
    w.c_l = carve(cols * g.nkeys);
    w.lse = carve(cols * g.s1);
    if (g.T > 1) {
        w.alpha_r = carve(bh * g.gq * g.gk * g.s1 * g.s2 * g.d);
        w.c_r = carve(bh * g.gq * g.gk * g.s1 * g.s2);
    }
    if (ws) *ws = w;
    return off;
}

}  // namespace mbx

extern "C" {

int mbx_version(void) { return MBX_ABI_VERSION; }

int mbx_profile_enable(int on) {
    const int prev = g_prof_on ? 1 : 0;
    g_prof_on = on != 0;
    return prev;
}

int mbx_profile_collect(float* ms, const char** names, int max_entries) {
    return mbx_profile_collect_ex(nullptr, ms, names, max_entries);
}

int mbx_profile_collect_ex(float* start_ms, float* ms, const char** names, int max_entries) {
    const int n = (int)g_prof.size();
    for (int i = 0; i < n; ++i) {
        ProfRecord& r = g_prof[i];
        if (i < max_entries) {
            float t = -1.f, t0 = 0.f;
            if (cudaEventSynchronize(r.stop) == cudaSuccess) cudaEventElapsedTime(&t, r.start, r.stop);
            if (start_ms && i > 0) cudaEventElapsedTime(&t0, g_prof[0].start, r.start);
            if (ms) ms[i] = t;
            if (start_ms) start_ms[i] = t0;
            if (names) names[i] = r.name;
        }
    }
    for (ProfRecord& r : g_prof) {
        cudaEventDestroy(r.start);
        cudaEventDestroy(r.stop);
    }
    g_prof.clear();
    return n;
}

const char* mbx_last_error(void) { return g_last_error.c_str(); }

int mbx_set_option(const char* name, int value) { return mbx::set_option(name, value); }

int mbx_validate(const mbx_desc* desc) { return validate(desc, nullptr); }

int64_t mbx_token_index(const mbx_desc* desc, int is_query, int64_t slot) {
    mbx::Geometry g;
    if (validate(desc, &g) != MBX_OK || slot < 0) return -1;
    const int64_t per_row = (int64_t)g.c2 * g.s2;
    const int64_t rows = (int64_t)(is_query ? g.c1q : g.c1k) * g.s1;
    if (slot >= rows * per_row) return -1;
    // slot = ((l1*s1 + r)*c2 + j1)*s2 + j
    const int64_t j = slot % g.s2, j1 = (slot / g.s2) % g.c2, lr = slot / per_row;
    const int l1 = (int)(lr / g.s1), r = (int)(lr % g.s1);
    return mbx::row_base(g, is_query != 0, l1 * g.c2 + (int)j1, r) + j;
}

int mbx_selected_path(const mbx_desc* desc) {
    mbx::Geometry g;
    if (validate(desc, &g) != MBX_OK) return -1;
    return mbx::tc_supported(g, desc->dtype, desc->flags, (desc->flags & MBX_FLAG_FACTORS) != 0) ? 1 : 0;
}

size_t mbx_workspace_bytes(const mbx_desc* desc) {
    mbx::Geometry g;
    if (validate(desc, &g) != MBX_OK) return 0;
    if (mbx::tc_supported(g, desc->dtype, desc->flags, (desc->flags & MBX_FLAG_FACTORS) != 0))
        return mbx::tc_workspace_bytes(g, desc->flags);
    return mbx::workspace_layout(g, nullptr, nullptr);
}

int mbx_forward(const mbx_desc* desc, const void* q, const void* k, const void* v, void* out,
                float* l_factor, float* r_factor, void* workspace, size_t workspace_bytes,
                void* stream) {
    mbx::Geometry g;
    int st = validate(desc, &g);
    if (st != MBX_OK) return st;
    const bool want_out = !(desc->flags & MBX_FLAG_NO_OUTPUT);
    if (!q || !k || (want_out && (!v || !out)))
        return fail(MBX_ERR_NULL, "q, k, v and out must be non-NULL");
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    const bool factors = l_factor || r_factor;
    const int flags = desc->flags | (factors ? MBX_FLAG_FACTORS : 0);
    const bool tc = want_out && mbx::tc_supported(g, desc->dtype, flags, factors);
    cudaError_t e;
    if (tc) {
        const size_t need = mbx::tc_workspace_bytes(g, flags);
        if (need && (!workspace || workspace_bytes < need))
            return fail(MBX_ERR_WORKSPACE, "workspace %zu < required %zu bytes", workspace_bytes, need);
        e = mbx::tc_forward(g, flags, q, k, v, out, l_factor, r_factor, workspace, s);
    } else {
        mbx::Workspace ws;
        const size_t need = mbx::workspace_layout(g, (char*)workspace, &ws);
        if (!workspace || workspace_bytes < need)
            return fail(MBX_ERR_WORKSPACE, "workspace %zu < required %zu bytes", workspace_bytes, need);
        if (!want_out) ws.y = nullptr;
        e = mbx::generic_forward(g, desc->dtype, q, k, v, want_out ? out : nullptr, l_factor,
                                 r_factor, ws, s, (desc->flags & MBX_FLAG_ALL_ITERS) != 0);
    }
    if (e != cudaSuccess) return fail(MBX_ERR_CUDA, "CUDA error: %s", cudaGetErrorString(e));
    return MBX_OK;
}

size_t mbx_backward_workspace_bytes(const mbx_desc* desc) {
    mbx::Geometry g;
    if (validate(desc, &g) != MBX_OK) return 0;
    return mbx::backward_workspace_bytes(g);
}

int mbx_backward(const mbx_desc* desc, const void* q, const void* k, const void* v, const void* dout,
                 const float* l_factors, const float* r_factors, void* dq, void* dk, void* dv,
                 void* workspace, size_t workspace_bytes, void* stream) {
    mbx::Geometry g;
    int st = validate(desc, &g);
    if (st != MBX_OK) return st;
    if (!q || !k || !v || !dout || !l_factors || !r_factors || !dq || !dk || !dv)
        return fail(MBX_ERR_NULL, "q, k, v, dout, factors, dq, dk and dv must be non-NULL");
    const size_t need = mbx::backward_workspace_bytes(g);
    if (!workspace || workspace_bytes < need)
        return fail(MBX_ERR_WORKSPACE, "workspace %zu < required %zu bytes", workspace_bytes, need);
    cudaError_t e = mbx::backward(g, desc->dtype, q, k, v, dout, l_factors, r_factors, dq, dk, dv, workspace,
                                  reinterpret_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return fail(MBX_ERR_CUDA, "CUDA error: %s", cudaGetErrorString(e));
    return MBX_OK;
}

size_t mbx_apply_workspace_bytes(const mbx_desc* desc) {
    mbx::Geometry g;
    if (validate(desc, &g) != MBX_OK) return 0;
    g.T = 1;
    return mbx::workspace_layout(g, nullptr, nullptr);
}

int mbx_apply(const mbx_desc* desc, const float* l_factor, const float* r_factor, const void* v,
              void* out, void* workspace, size_t workspace_bytes, void* stream) {
    mbx::Geometry g;
    int st = validate(desc, &g);
    if (st != MBX_OK) return st;
    if (!l_factor || !r_factor || !v || !out)
        return fail(MBX_ERR_NULL, "factors, v and out must be non-NULL");
    g.T = 1;
    mbx::Workspace ws;
    const size_t need = mbx::workspace_layout(g, (char*)workspace, &ws);
    if (!workspace || workspace_bytes < need)
        return fail(MBX_ERR_WORKSPACE, "workspace %zu < required %zu bytes", workspace_bytes, need);
    cudaError_t e = mbx::generic_apply(g, desc->dtype, l_factor, r_factor, v, out, ws,
                                       reinterpret_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return fail(MBX_ERR_CUDA, "CUDA error: %s", cudaGetErrorString(e));
    return MBX_OK;
}

}  // extern "C"
