// Probe: does tcgen05.cp.128x256b from a K-major SW128 smem tile give the TMEM
// A-operand layout the MMA expects?  Compares D = A(tmem, via cp) * B with
// D = A(smem) * B, and dumps the raw TMEM words of row 0..3.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_2602_12271_b200/csrc -o probe_utccp probe_utccp.cu -lcuda
#include <cstdio>
#include "mbx_sm100.cuh"

using namespace mbx::sm100;

__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, bool acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
        "r"(a), "l"(b), "r"(idesc), "r"((uint32_t)acc));
}

__device__ __forceinline__ float aval(int r, int k) { return (float)(((r * 7 + k * 3) % 17) - 8) * 0.125f; }
__device__ __forceinline__ float bval(int n, int k) { return (float)(((n * 5 + k * 11) % 13) - 6) * 0.25f; }

// K-major SW128 tile [rows][64 bf16]: element (r, k) at r*128 + (((k>>3) ^ (r&7))<<4) + (k&7)*2
__device__ __forceinline__ uint32_t sw128(int r, int k) { return r * 128 + ((((k >> 3) ^ (r & 7))) << 4) + (k & 7) * 2; }

__global__ void probe(float* out, uint32_t* raw) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t bar;
    __shared__ uint32_t slot;
    uint8_t* A = smem;            // [128][64] bf16, 16 KB
    uint8_t* B = smem + 16384;    // [64][64] bf16, 8 KB (N=64 rows, K=64)
    for (int i = threadIdx.x; i < 128 * 64; i += blockDim.x) {
        const int r = i / 64, k = i % 64;
        *reinterpret_cast<__nv_bfloat16*>(A + sw128(r, k)) = __float2bfloat16(aval(r, k));
    }
    for (int i = threadIdx.x; i < 64 * 64; i += blockDim.x) {
        const int n = i / 64, k = i % 64;
        *reinterpret_cast<__nv_bfloat16*>(B + sw128(n, k)) = __float2bfloat16(bval(n, k));
    }
    if (threadIdx.x < 32) tmem_alloc<512>(&slot);
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        fence_barrier_init();
    }
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = slot;
    const uint32_t idesc = idesc_bf16(128, 64, false, false);
    if (threadIdx.x == 0) {
        const uint32_t sa = smem_u32(A), sb = smem_u32(B);
        // reference: A from smem -> cols [0, 64)
        for (int kk = 0; kk < 4; ++kk)
            mma_bf16(tmem, smem_desc(sa + kk * 32, 16, 1024, 2), smem_desc(sb + kk * 32, 16, 1024, 2), idesc, kk > 0);
        // copy A into TMEM cols [256, 288): one 128x256b (K = 16) per K step
        for (int kk = 0; kk < 4; ++kk) {
            const uint64_t d = smem_desc(sa + kk * 32, 16, 1024, 2);
            asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;" ::"r"(tmem + 256 + kk * 8), "l"(d));
        }
        // A from TMEM -> cols [64, 128)
        for (int kk = 0; kk < 4; ++kk)
            mma_ts(tmem + 64, tmem + 256 + kk * 8, smem_desc(sb + kk * 32, 16, 1024, 2), idesc, kk > 0);
        mma_commit(&bar);
    }
    mbar_wait(&bar, 0);
    tc_fence_after();
    const int w = threadIdx.x >> 5;
    if (w < 4) {
        float d0[32], d1[32];
        const uint32_t lane_off = (uint32_t)(w * 32) << 16;
        for (int h = 0; h < 2; ++h) {
            tmem_ld32(tmem + lane_off + h * 32, d0);
            tmem_ld32(tmem + lane_off + 64 + h * 32, d1);
            const int r = threadIdx.x;
            for (int i = 0; i < 32; ++i) {
                out[(r * 64 + h * 32 + i) * 3 + 0] = d0[i];
                out[(r * 64 + h * 32 + i) * 3 + 1] = d1[i];
                float ref = 0.f;
                for (int k = 0; k < 64; ++k)
                    ref += __bfloat162float(__float2bfloat16(aval(r, k))) * __bfloat162float(__float2bfloat16(bval(h * 32 + i, k)));
                out[(r * 64 + h * 32 + i) * 3 + 2] = ref;
            }
        }
        float rw[32];
        tmem_ld32(tmem + lane_off + 256, rw);
        for (int i = 0; i < 32; ++i) raw[threadIdx.x * 32 + i] = __float_as_uint(rw[i]);
    }
    tc_fence_before();
    __syncthreads();
    if (threadIdx.x < 32) tmem_dealloc<512>(tmem);
}

int main() {
    float* d;
    uint32_t* rw;
    cudaMalloc(&d, 128 * 64 * 3 * 4);
    cudaMalloc(&rw, 128 * 32 * 4);
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 40000);
    probe<<<1, 128, 40000>>>(d, rw);
    cudaError_t e = cudaDeviceSynchronize();
    static float h[128 * 64 * 3];
    static uint32_t r[128 * 32];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    cudaMemcpy(r, rw, sizeof(r), cudaMemcpyDeviceToHost);
    double e_ss = 0, e_ts = 0;
    for (int i = 0; i < 128 * 64; ++i) {
        e_ss = fmax(e_ss, fabs(h[3 * i] - h[3 * i + 2]));
        e_ts = fmax(e_ts, fabs(h[3 * i + 1] - h[3 * i + 2]));
    }
    printf("{\"err\": \"%s\", \"max_abs_ss\": %g, \"max_abs_ts_via_cp\": %g}\n", cudaGetErrorString(e), e_ss, e_ts);
    for (int row = 0; row < 3; ++row) {
        printf("row %d raw:", row);
        for (int i = 0; i < 8; ++i) printf(" %08x", r[row * 32 + i]);
        printf("\n");
    }
    return 0;
}
