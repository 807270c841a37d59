// tcgen05.mma issue-rate probe on one SM: back-to-back MMAs of the row-stage
// shapes, one commit at the end, clock64 around.  Prints clocks per MMA and
// achieved MAC/clk.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../paper_2602_12271_b200/csrc -o ubench_mma ubench_mma.cu -lcuda
#include <cstdio>
#include "mbx_sm100.cuh"

using namespace mbx::sm100;

__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, bool acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
        "r"(a), "l"(b), "r"(idesc), "r"((uint32_t)acc));
}

template <int MODE>
__global__ void probe(long long* out, int iters) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t bar;
    __shared__ uint64_t bar2[4];
    __shared__ uint32_t slot;
    for (int i = threadIdx.x; i < 65536 / 16; i += blockDim.x) reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
    if (threadIdx.x < 32) tmem_alloc<512>(&slot);
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        for (int i = 0; i < 4; ++i) mbar_init(&bar2[i], 1);
        fence_barrier_init();
    }
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = slot;
    if (threadIdx.x == 0) {
        const uint32_t sa = smem_u32(smem), sb = smem_u32(smem + 32768);
        const uint32_t id1 = idesc_bf16(128, 64, false, false);
        const uint32_t id2 = idesc_bf16(128, 128, false, true);
        const uint32_t id3 = idesc_bf16(128, 256, false, false);
        long long t0 = clock64();
        for (int it = 0; it < iters; ++it) {
            if (MODE == 0) {   // MMA1: 128x64, K=128 as 8 x K16, A,B K-major SW128 smem
#pragma unroll
                for (int kk = 0; kk < 8; ++kk)
                    mma_bf16(tmem + (it & 1) * 64, smem_desc(sa + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024, 2),
                             smem_desc(sb + (kk >> 2) * 8192 + (kk & 3) * 32, 16, 1024, 2), id1, kk > 0);
            } else if (MODE == 1) {   // MMA2 half: 128x128, K=64, A in TMEM, B MN-major SW128
#pragma unroll
                for (int kk = 0; kk < 4; ++kk)
                    mma_ts(tmem + 128 + (it & 1) * 128, tmem + kk * 8, smem_desc(sb + kk * 2048, 8192, 1024, 2), id2,
                           kk > 0);
            } else if (MODE == 2) {   // MMA2 half with A from smem (K-major)
#pragma unroll
                for (int kk = 0; kk < 4; ++kk)
                    mma_bf16(tmem + 128 + (it & 1) * 128, smem_desc(sa + kk * 32, 16, 1024, 2),
                             smem_desc(sb + kk * 2048, 8192, 1024, 2), id2, kk > 0);
            } else if (MODE == 4 || MODE == 5) {   // row-stage task sequence, optionally committing each group
#pragma unroll
                for (int kk = 0; kk < 8; ++kk)
                    mma_bf16(tmem + (it & 1) * 64, smem_desc(sa + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024, 2),
                             smem_desc(sb + (kk >> 2) * 8192 + (kk & 3) * 32, 16, 1024, 2), id1, kk > 0);
                if (MODE == 5) mma_commit(&bar2[0]);
#pragma unroll
                for (int h = 0; h < 2; ++h) {
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk)
                        mma_ts(tmem + 128 + ((2 * it + h) % 3) * 128, tmem + (it & 1) * 64 + kk * 8,
                               smem_desc(sb + h * 16384 + kk * 2048, 8192, 1024, 2), id2, kk > 0);
                    if (MODE == 5) mma_commit(&bar2[1 + h]);
                }
                if (MODE == 5) mma_commit(&bar2[3]);
            } else if (MODE == 6) {   // MMA1 with A from TMEM (Q copied in), N=64
#pragma unroll
                for (int kk = 0; kk < 8; ++kk)
                    mma_ts(tmem + 128 + (it & 1) * 64, tmem + kk * 8,
                           smem_desc(sb + (kk >> 2) * 8192 + (kk & 3) * 32, 16, 1024, 2), id1, kk > 0);
            } else if (MODE == 7) {   // exact row task: MMA1 TS N=64 + 2 x MMA2 TS N=128 with commits
#pragma unroll
                for (int kk = 0; kk < 8; ++kk)
                    mma_ts(tmem + 128 + (it & 1) * 64, tmem + kk * 8,
                           smem_desc(sb + (kk >> 2) * 8192 + (kk & 3) * 32, 16, 1024, 2), id1, kk > 0);
                mma_commit(&bar2[0]);
#pragma unroll
                for (int h = 0; h < 2; ++h) {
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk)
                        mma_ts(tmem + 256 + h * 128, tmem + 128 + (it & 1) * 64 + kk * 8,
                               smem_desc(sb + h * 16384 + kk * 2048, 8192, 1024, 2), id2, kk > 0);
                    mma_commit(&bar2[1 + h]);
                }
            } else if (MODE == 8) {   // M=64 pair task: 2 x MMA1 (64x64xK128 SS) + 4 x MMA2 (64x128xK64 TS)
                const uint32_t i64a = idesc_bf16(64, 64, false, false), i64b = idesc_bf16(64, 128, false, true);
#pragma unroll
                for (int hh = 0; hh < 2; ++hh)
#pragma unroll
                    for (int kk = 0; kk < 8; ++kk)
                        mma_bf16(tmem + (uint32_t)(hh * 16 << 16) + (it & 1) * 64,
                                 smem_desc(sa + hh * 8192 + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024, 2),
                                 smem_desc(sb + (kk >> 2) * 8192 + (kk & 3) * 32, 16, 1024, 2), i64a, kk > 0);
#pragma unroll
                for (int hh = 0; hh < 2; ++hh)
#pragma unroll
                    for (int s = 0; s < 2; ++s)
#pragma unroll
                        for (int kk = 0; kk < 4; ++kk)
                            mma_ts(tmem + (uint32_t)(hh * 16 << 16) + 128 + s * 128, tmem + (uint32_t)(hh * 16 << 16) + (it & 1) * 64 + kk * 8,
                                   smem_desc(sb + s * 16384 + kk * 2048, 8192, 1024, 2), i64b, kk > 0);
            } else {   // big GEMM shape 128x256 K=64, both K-major
#pragma unroll
                for (int kk = 0; kk < 4; ++kk)
                    mma_bf16(tmem + (it & 1) * 256, smem_desc(sa + kk * 32, 16, 1024, 2),
                             smem_desc(sb + kk * 32, 16, 1024, 2), id3, kk > 0);
            }
        }
        mma_commit(&bar);
        mbar_wait(&bar, 0);
        long long t1 = clock64();
        out[blockIdx.x] = t1 - t0;
    }
    tc_fence_before();
    __syncthreads();
    if (threadIdx.x < 32) tmem_dealloc<512>(tmem);
}

template <int MODE>
void run(const char* name, double macs_per_iter) {
    long long* d;
    cudaMalloc(&d, 8 * 148);
    cudaFuncSetAttribute(probe<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000);
    const int iters = 2000;
    probe<MODE><<<148, 128, 100000>>>(d, iters);
    probe<MODE><<<148, 128, 100000>>>(d, iters);
    cudaError_t e = cudaDeviceSynchronize();
    long long c;
    cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
    printf("{\"mma\": \"%s\", \"err\": \"%s\", \"clk_per_iter\": %.1f, \"mac_per_clk\": %.0f}\n", name,
           cudaGetErrorString(e), (double)c / iters, macs_per_iter * iters / (double)c);
    cudaFree(d);
}

int main() {
    run<0>("row MMA1 128x64xK128 SS", 128.0 * 64 * 128);
    run<1>("row MMA2 half 128x128xK64 TS (A tmem, B MN-major)", 128.0 * 128 * 64);
    run<2>("row MMA2 half 128x128xK64 SS", 128.0 * 128 * 64);
    run<3>("gemm 128x256xK64 SS", 128.0 * 256 * 64);
    run<4>("row task (MMA1 + 2 x MMA2 half), no commits", 128.0 * 64 * 128 + 2 * 128.0 * 128 * 64);
    run<5>("row task with 4 commits", 128.0 * 64 * 128 + 2 * 128.0 * 128 * 64);
    run<6>("row MMA1 128x64xK128 TS (A tmem)", 128.0 * 64 * 128);
    run<7>("row task TS/TS exact with commits", 128.0 * 64 * 128 + 2 * 128.0 * 128 * 64);
    run<8>("M=64 pair task (2x MMA1 64x64x128 SS, 4x MMA2 64x128x64 TS)", 128.0 * 64 * 128 + 2 * 128.0 * 128 * 64);
    return 0;
}
