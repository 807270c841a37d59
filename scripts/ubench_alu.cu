// Per-SM instruction throughput probes (sm_100a): cvt.rn.bf16x2.f32 (F2FP),
// ex2.approx (MUFU), FFMA, st.shared.v4.  One CTA per SM, W warps, clock64
// around a long unrolled loop of independent ops.  Prints ops/clk/SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ubench_alu ubench_alu.cu
#include <cstdio>
#include <cuda_bf16.h>
#include <cstdint>

constexpr int kIters = 2048;

template <int OP>
__global__ void probe(float* out, long long* cyc, float seed) {
    float a[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) a[i] = seed * (threadIdx.x + i);
    uint32_t acc = 0;
    __shared__ __align__(16) uint32_t sm[8192];
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < kIters; ++it) {
#pragma unroll
        for (int i = 0; i < 16; i += 2) {
            if (OP == 0) {   // F2FP pack
                uint32_t r;
                asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(a[i]), "f"(a[i + 1]));
                acc ^= r;
                a[i] = __uint_as_float(__float_as_uint(a[i]) + 1);
            } else if (OP == 1) {   // MUFU ex2 (2 per step)
                float y0, y1;
                asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y0) : "f"(a[i]));
                asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y1) : "f"(a[i + 1]));
                a[i] = y0;
                a[i + 1] = y1;
            } else if (OP == 2) {   // FFMA (2 per step)
                a[i] = fmaf(a[i], 1.0001f, 0.5f);
                a[i + 1] = fmaf(a[i + 1], 1.0001f, 0.5f);
            } else if (OP == 3) {   // STS.128 (one per step), conflict-free
                uint32_t addr = static_cast<uint32_t>(__cvta_generic_to_shared(sm)) +
                                ((threadIdx.x * 16 + i * 1024) & 32767);
                asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" ::"r"(addr), "r"(acc), "r"(acc), "r"(acc),
                             "r"(acc)
                             : "memory");
                acc += 1;
            }
        }
    }
    long long t1 = clock64();
    float s = 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) s += a[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s + acc;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int OP>
void run(const char* name, int warps, double ops_per_step) {
    float* out;
    long long* cyc;
    cudaMalloc(&out, 148 * 1024 * 4);
    cudaMalloc(&cyc, 148 * 8);
    probe<OP><<<148, warps * 32>>>(out, cyc, 1.0001f);
    probe<OP><<<148, warps * 32>>>(out, cyc, 1.0001f);
    cudaDeviceSynchronize();
    long long c;
    cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    double ops = (double)kIters * 8 * ops_per_step * warps * 32;
    printf("{\"op\": \"%s\", \"warps\": %d, \"per_clk_per_sm\": %.2f}\n", name, warps, ops / (double)c);
    cudaFree(out);
    cudaFree(cyc);
}

int main() {
    for (int w : {4, 8, 16}) {
        run<0>("cvt.rn.bf16x2.f32 (pairs)", w, 1);
        run<1>("ex2.approx", w, 2);
        run<2>("ffma", w, 2);
        run<3>("st.shared.v4 (bytes/16)", w, 1);
    }
    return 0;
}
