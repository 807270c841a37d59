// TMEM read / write throughput per SM: W warps (lane quadrant = warp % 4) loop
// tcgen05.ld.32x32b.x32 (+ wait) over 128 columns, or tcgen05.st; reports bytes per cycle.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_2602_12271_b200/csrc -o ubench_tmem ubench_tmem.cu
#include <cstdio>
#include "mbx_sm100.cuh"

using namespace mbx::sm100;

__global__ void probe(int iters, int mode, long long* cycles, float* sink) {
    __shared__ uint32_t slot;
    const int warp = threadIdx.x >> 5;
    if (warp == 0) tmem_alloc<512>(&slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = slot;
    const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
    const uint32_t base = tmem + lane_off + (uint32_t)((warp >> 2) * 128);
    float acc = 0.f;
    uint32_t v[32];
    for (int i = 0; i < 32; ++i) v[i] = __float_as_uint((float)i);
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        for (int c = 0; c < 128; c += 32) {
            if (mode == 0) {
                tmem_ld32_nw(base + c, v);
                tmem_wait_ld();
#pragma unroll
                for (int i = 0; i < 32; ++i) acc += __uint_as_float(v[i]);
            } else if (mode == 1) {   // two loads in flight per wait
                uint32_t w[32];
                tmem_ld32_nw(base + c, v);
                tmem_ld32_nw(base + ((c + 32) & 127), w);
                tmem_wait_ld();
#pragma unroll
                for (int i = 0; i < 32; ++i) acc += __uint_as_float(v[i]) + __uint_as_float(w[i]);
                c += 32;
            } else {
                tmem_st32(base + c, reinterpret_cast<const float*>(v));
            }
        }
    }
    long long t1 = clock64();
    __syncthreads();
    if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
    sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc<512>(tmem);
}

int main() {
    long long* cyc;
    float* sink;
    cudaMalloc(&cyc, 148 * 8);
    cudaMalloc(&sink, 148 * 512 * 4);
    const int iters = 2000;
    for (int mode = 0; mode < 3; ++mode) {
        for (int warps : {1, 4, 8, 16}) {
            probe<<<148, warps * 32>>>(iters, mode, cyc, sink);
            cudaError_t e = cudaDeviceSynchronize();
            long long h[148];
            cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
            long long mx = 0;
            for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
            const double bytes = (double)iters * 128 * 32 * 4 * warps;   // per SM
            printf("{\"mode\": \"%s\", \"warps\": %d, \"err\": \"%s\", \"bytes_per_cycle_per_sm\": %.1f}\n",
                   mode == 0 ? "ld x32 + wait" : mode == 1 ? "2 x ld x32 + wait" : "st x32 + wait", warps,
                   cudaGetErrorString(e), bytes / (double)mx);
        }
    }
    return 0;
}
