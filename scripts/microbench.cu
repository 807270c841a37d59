// Memory-system microbenchmarks that shape the kernel design:
//   l2_read   : read-only 128-bit loads over a working set of W MB, many passes
//   l2_write  : 128-bit stores over W MB
//   dsmem     : cluster CTAs write 64 KB blocks into a peer's shared memory
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o microbench scripts/microbench.cu
#include <cstdio>
#include <cstdlib>
#include <cooperative_groups.h>
#include <cuda_runtime.h>

namespace cg = cooperative_groups;

__global__ void l2_read(const int4* __restrict__ p, size_t n, int passes, int4* sink) {
    int4 acc = make_int4(0, 0, 0, 0);
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    for (int it = 0; it < passes; ++it) {
        for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += stride) {
            int4 v;
            asm volatile("ld.global.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
                         : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p + i));
            acc.x ^= v.x; acc.y ^= v.y; acc.z ^= v.z; acc.w ^= v.w;
        }
    }
    if (acc.x == 0x12345678) sink[0] = acc;
}

__global__ void l2_write(int4* __restrict__ p, size_t n, int passes) {
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    for (int it = 0; it < passes; ++it)
        for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += stride)
            p[i] = make_int4(it, (int)i, 0, 0);
}

template <int CL>
__global__ void __cluster_dims__(CL, 1, 1) dsmem_write(int reps, int* sink) {
    extern __shared__ int4 buf[];
    cg::cluster_group cluster = cg::this_cluster();
    const unsigned rank = cluster.block_rank();
    int4* peer = cluster.map_shared_rank(buf, (rank + 1) % CL);
    const int n = 64 * 1024 / 16;
    cluster.sync();
    for (int r = 0; r < reps; ++r)
        for (int i = threadIdx.x; i < n; i += blockDim.x) peer[i] = make_int4(r, i, 0, 0);
    cluster.sync();
    if (threadIdx.x == 0 && buf[5].x == 0x7fffffff) sink[0] = 1;
}

static float time_ms(cudaEvent_t a, cudaEvent_t b) {
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    return ms;
}

int main() {
    int dev = 0, sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    int4* buf;
    int4* sink;
    const size_t max_bytes = (size_t)1 << 30;
    cudaMalloc(&buf, max_bytes);
    cudaMalloc(&sink, 64);
    cudaMemset(buf, 1, max_bytes);
    printf("{\"sms\": %d, \"l2_read_GBps\": {", sms);
    const int mbs[] = {8, 16, 24, 32, 48, 64, 96, 1024};
    for (int t = 0; t < 8; ++t) {
        size_t bytes = (size_t)mbs[t] << 20;
        size_t n = bytes / 16;
        int passes = mbs[t] >= 1024 ? 3 : 40;
        l2_read<<<sms * 4, 512>>>(buf, n, 2, sink);
        cudaEventRecord(a);
        l2_read<<<sms * 4, 512>>>(buf, n, passes, sink);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        printf("%s\"%d\": %.0f", t ? ", " : "", mbs[t], bytes * (double)passes / (time_ms(a, b) * 1e-3) / 1e9);
    }
    printf("}, \"l2_write_GBps\": {");
    for (int t = 0; t < 8; ++t) {
        size_t bytes = (size_t)mbs[t] << 20;
        size_t n = bytes / 16;
        int passes = mbs[t] >= 1024 ? 3 : 40;
        l2_write<<<sms * 4, 512>>>(buf, n, 2);
        cudaEventRecord(a);
        l2_write<<<sms * 4, 512>>>(buf, n, passes);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        printf("%s\"%d\": %.0f", t ? ", " : "", mbs[t], bytes * (double)passes / (time_ms(a, b) * 1e-3) / 1e9);
    }
    printf("}, \"dsmem_write_GBps\": {");
    const int reps = 200;
    cudaFuncSetAttribute(dsmem_write<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
    cudaFuncSetAttribute(dsmem_write<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
    cudaFuncSetAttribute(dsmem_write<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
    int grid = (sms / 8) * 8;
    dsmem_write<2><<<grid, 512, 65536>>>(2, (int*)sink);
    cudaEventRecord(a);
    dsmem_write<2><<<grid, 512, 65536>>>(reps, (int*)sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    printf("\"cl2\": %.0f", grid * 65536.0 * reps / (time_ms(a, b) * 1e-3) / 1e9);
    cudaEventRecord(a);
    dsmem_write<4><<<grid, 512, 65536>>>(reps, (int*)sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    printf(", \"cl4\": %.0f", grid * 65536.0 * reps / (time_ms(a, b) * 1e-3) / 1e9);
    cudaEventRecord(a);
    dsmem_write<8><<<grid, 512, 65536>>>(reps, (int*)sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    printf(", \"cl8\": %.0f", grid * 65536.0 * reps / (time_ms(a, b) * 1e-3) / 1e9);
    cudaError_t e = cudaDeviceSynchronize();
    printf("}, \"err\": \"%s\"}\n", cudaGetErrorString(e));
    return 0;
}
