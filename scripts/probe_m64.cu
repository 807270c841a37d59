// Probe: TMEM placement of cta_group::1 M=64 MMAs.  Two M=64 SS MMAs (different
// A rows, same B) with D at TMEM lane offset 0 and 16; a TS MMA whose A comes
// from TMEM lanes written per-thread at offset 16.  Prints where each D row landed.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_2602_12271_b200/csrc -o probe_m64 probe_m64.cu -lcuda
#include <cstdio>
#include "mbx_sm100.cuh"

using namespace mbx::sm100;

__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, bool acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
        "r"(a), "l"(b), "r"(idesc), "r"((uint32_t)acc));
}
__device__ __forceinline__ uint32_t sw128(int r, int k) { return r * 128 + ((((k >> 3) ^ (r & 7))) << 4) + (k & 7) * 2; }

__global__ void probe(float* out) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t bar;
    __shared__ uint32_t slot;
    uint8_t* A0 = smem;           // [64 rows][16 K] : row r has value 1000*0 + r in column 0 only
    uint8_t* A1 = smem + 8192;    // second A: value 1000 + r
    uint8_t* B = smem + 16384;    // [N=16 rows][K=16]: identity-ish: B[n][k] = (k == 0) ? 1 : 0  -> D[r][n] = A[r][0]
    for (int i = threadIdx.x; i < 64 * 64; i += blockDim.x) {
        const int r = i / 64, k = i % 64;
        *reinterpret_cast<__nv_bfloat16*>(A0 + sw128(r, k)) = __float2bfloat16(k == 0 ? (float)r : 0.f);
        *reinterpret_cast<__nv_bfloat16*>(A1 + sw128(r, k)) = __float2bfloat16(k == 0 ? (float)(100 + r) : 0.f);
    }
    for (int i = threadIdx.x; i < 16 * 64; i += blockDim.x) {
        const int n = i / 64, k = i % 64;
        *reinterpret_cast<__nv_bfloat16*>(B + sw128(n, k)) = __float2bfloat16(k == 0 ? 1.f : 0.f);
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
    // TS operand: thread (lane L) writes A row value 200 + L in column pair 0 at TMEM cols [256, 264)
    {
        const int lane = threadIdx.x;   // 128 threads = all lanes
        uint32_t v[8];
        for (int i = 0; i < 8; ++i) v[i] = 0;
        __nv_bfloat162 h = __floats2bfloat162_rn((float)(200 + lane), 0.f);
        v[0] = *reinterpret_cast<uint32_t*>(&h);
        const uint32_t lane_off = (uint32_t)((threadIdx.x >> 5) * 32) << 16;
        asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(tmem + lane_off + 256),
                     "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]) : "memory");
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t id = idesc_bf16(64, 16, false, false);
    if (threadIdx.x == 0) {
        // SS M=64 into cols [0,16) lane offset 0, and cols [0,16) lane offset 16
        mma_bf16(tmem + 0, smem_desc(smem_u32(A0), 16, 1024, 2), smem_desc(smem_u32(B), 16, 1024, 2), id, false);
        mma_bf16(tmem + (16u << 16) + 0, smem_desc(smem_u32(A1), 16, 1024, 2), smem_desc(smem_u32(B), 16, 1024, 2), id,
                 false);
        // TS M=64: A from TMEM cols [256, 264) at lane offset 0 and 16 -> D cols [32,48) lane offsets 0 / 16
        mma_ts(tmem + 32, tmem + 256, smem_desc(smem_u32(B), 16, 1024, 2), id, false);
        mma_ts(tmem + (16u << 16) + 64, tmem + (16u << 16) + 256, smem_desc(smem_u32(B), 16, 1024, 2), id, false);
        mma_commit(&bar);
    }
    mbar_wait(&bar, 0);
    tc_fence_after();
    {
        float d[32];
        const uint32_t lane_off = (uint32_t)((threadIdx.x >> 5) * 32) << 16;
        tmem_ld32(tmem + lane_off, d);            // cols 0..31  (SS results in col 0)
        out[threadIdx.x * 4 + 0] = d[0];
        tmem_ld32(tmem + lane_off + 32, d);       // cols 32..63 (TS lane-offset-0 result in col 32)
        out[threadIdx.x * 4 + 1] = d[0];
        tmem_ld32(tmem + lane_off + 64, d);       // cols 64..95 (TS lane-offset-16 result in col 64)
        out[threadIdx.x * 4 + 2] = d[0];
    }
    tc_fence_before();
    __syncthreads();
    if (threadIdx.x < 32) tmem_dealloc<512>(tmem);
}

int main() {
    float* d;
    cudaMalloc(&d, 128 * 4 * 4);
    cudaMemset(d, 0, 128 * 16);
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 40000);
    probe<<<1, 128, 40000>>>(d);
    cudaError_t e = cudaDeviceSynchronize();
    float h[128 * 4];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    printf("err %s\nlane: SS(col0) TS0(col32) TS16(col64)\n", cudaGetErrorString(e));
    for (int l = 0; l < 128; ++l) printf("%3d: %6.0f %6.0f %6.0f\n", l, h[l * 4], h[l * 4 + 1], h[l * 4 + 2]);
    return 0;
}
