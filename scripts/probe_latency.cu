// Probe: mbarrier hand-off latency between warps of one CTA (arrive -> waiter
// wakes), for try_wait with / without the suspend hint and test_wait spinning,
// and tcgen05.commit -> waiter latency after a small MMA.  Clock64 cycles.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_2602_12271_b200/csrc -o probe_latency probe_latency.cu -lcuda
#include <cstdio>
#include "mbx_sm100.cuh"

using namespace mbx::sm100;

template <int MODE>
__device__ __forceinline__ void wait_mode(uint64_t* bar, uint32_t par) {
    if (MODE == 0) mbar_wait(bar, par);
    if (MODE == 1) mbar_wait_nohint(bar, par);
    if (MODE == 2) mbar_spin(bar, par);
}

template <int MODE>
__global__ void probe(long long* out, int reps, int busy_warps) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t ping, pong, mbar;
    __shared__ uint32_t slot;
    __shared__ long long t_send[64], t_recv[64], m_send[64], m_recv[64];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == 0) tmem_alloc<512>(&slot);
    if (threadIdx.x == 0) {
        mbar_init(&ping, 1);
        mbar_init(&pong, 1);
        mbar_init(&mbar, 1);
        fence_barrier_init();
    }
    for (int i = threadIdx.x; i < 32768 / 16; i += blockDim.x) reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = slot;
    if (warp == 0 && lane == 0) {
        for (int r = 0; r < reps; ++r) {
            t_send[r] = clock64();
            mbar_arrive(&ping);
            wait_mode<MODE>(&pong, r & 1);
        }
        // MMA commit latency: one 128x64x16 MMA, commit, waiter in warp 1
        const uint32_t id = idesc_bf16(128, 64, false, false);
        for (int r = 0; r < reps; ++r) {
            m_send[r] = clock64();
            mma_bf16(tmem, smem_desc(smem_u32(smem), 16, 1024, 2), smem_desc(smem_u32(smem) + 16384, 16, 1024, 2), id,
                     false);
            mma_commit(&mbar);
            wait_mode<MODE>(&pong, (reps + r) & 1);
        }
    } else if (warp == 1) {
        for (int r = 0; r < reps; ++r) {
            wait_mode<MODE>(&ping, r & 1);
            if (lane == 0) t_recv[r] = clock64();
            __syncwarp();
            if (lane == 0) mbar_arrive(&pong);
        }
        for (int r = 0; r < reps; ++r) {
            wait_mode<MODE>(&mbar, r & 1);
            if (lane == 0) m_recv[r] = clock64();
            __syncwarp();
            if (lane == 0) mbar_arrive(&pong);
        }
    } else if (warp < 2 + busy_warps) {
        // background ALU load on the other sub-partitions
        float a = threadIdx.x;
        for (int i = 0; i < 200000; ++i) a = fmaf(a, 1.0000001f, 0.5f);
        if (a == 12345.f) out[100] = 1;
    }
    tc_fence_before();
    __syncthreads();
    if (threadIdx.x == 0) {
        long long s1 = 0, s2 = 0;
        for (int r = 1; r < reps; ++r) {
            s1 += t_recv[r] - t_send[r];
            s2 += m_recv[r] - m_send[r];
        }
        out[0] = s1 / (reps - 1);
        out[1] = s2 / (reps - 1);
    }
    if (warp == 0) tmem_dealloc<512>(tmem);
}

template <int MODE>
void run(const char* name, int busy) {
    long long* d;
    cudaMalloc(&d, 8 * 128);
    cudaFuncSetAttribute(probe<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 40000);
    probe<MODE><<<1, 32 * (2 + busy), 40000>>>(d, 32, busy);
    cudaError_t e = cudaDeviceSynchronize();
    long long h[2];
    cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    printf("{\"wait\": \"%s\", \"busy_warps\": %d, \"err\": \"%s\", \"arrive_to_wake_clk\": %lld, "
           "\"mma_issue_to_wake_clk\": %lld}\n",
           name, busy, cudaGetErrorString(e), h[0], h[1]);
    cudaFree(d);
}

int main() {
    for (int busy : {0, 8}) {
        run<0>("try_wait+hint", busy);
        run<1>("try_wait", busy);
        run<2>("test_wait spin", busy);
    }
    return 0;
}
