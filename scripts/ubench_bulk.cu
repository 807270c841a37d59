// Copy-engine throughput per SM from an L2-resident 8 MB source (all 148 SMs busy, one
// issuing thread, 4-slot smem ring): tensor boxes with 128 B SW128 lines vs 256 B
// unswizzled lines vs 1D cp.async.bulk copies -- to tell a per-line TMA limit from DRAM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_2602_12271_b200/csrc -o ubench_bulk ubench_bulk.cu -lcuda
#include <cstdio>
#include <cuda.h>
#include "mbx_sm100.cuh"

using namespace mbx::sm100;

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

// mode 0: tensor box (map, bx x by); mode 1: 1D bulk copy of `bytes`
__global__ void probe(const __grid_constant__ CUtensorMap map, const char* src, int mode, int bytes, int by,
                      int nrows, int iters, long long* out) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t full[4];
    if (threadIdx.x == 0) {
        for (int i = 0; i < 4; ++i) mbar_init(&full[i], 1);
        fence_barrier_init();
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        long long t0 = clock64();
        for (int it = 0; it < iters; ++it) {
            const int s = it & 3;
            if (it >= 4) mbar_wait(&full[s], ((it >> 2) - 1) & 1);
            mbar_expect_tx(&full[s], bytes);
            const int blk = (blockIdx.x * 13 + it * 7) % (nrows / by);
            if (mode == 0)
                tma_load_2d(smem + s * 32768, &map, &full[s], 0, blk * by);
            else
                bulk_load(smem + s * 32768, src + (size_t)blk * bytes, bytes, &full[s]);
        }
        for (int it = iters; it < iters + 4; ++it) mbar_wait(&full[it & 3], ((it >> 2) - 1) & 1);
        out[blockIdx.x] = clock64() - t0;
    }
}

int main() {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
    EncodeFn enc = (EncodeFn)p;
    const size_t total = 8 << 20;   // L2-resident
    char* buf;
    cudaMalloc(&buf, total);
    cudaMemset(buf, 1, total);
    long long* d;
    cudaMalloc(&d, 148 * 8);
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 32768 + 1024);
    struct Case { const char* name; int mode; int inner_b; int by; CUtensorMapSwizzle sw; };
    Case cases[] = {
        {"tensor 128 B lines SW128 x 52", 0, 128, 52, CU_TENSOR_MAP_SWIZZLE_128B},
        {"tensor 128 B lines SW128 x 128", 0, 128, 128, CU_TENSOR_MAP_SWIZZLE_128B},
        {"tensor 256 B lines none x 52", 0, 256, 52, CU_TENSOR_MAP_SWIZZLE_NONE},
        {"tensor 256 B lines none x 64", 0, 256, 64, CU_TENSOR_MAP_SWIZZLE_NONE},
        {"bulk 1D 6656 B (52 x 128 B)", 1, 128, 52, CU_TENSOR_MAP_SWIZZLE_NONE},
        {"bulk 1D 11520 B (90 x 128 B)", 1, 128, 90, CU_TENSOR_MAP_SWIZZLE_NONE},
        {"bulk 1D 16384 B", 1, 128, 128, CU_TENSOR_MAP_SWIZZLE_NONE},
    };
    for (auto& c : cases) {
        CUtensorMap m;
        const size_t rowb = c.mode == 0 && c.inner_b == 256 ? 256 : 128;
        const size_t nrows = total / rowb;
        cuuint64_t dims[2] = {rowb / 2, nrows};
        cuuint64_t strides[1] = {rowb};
        cuuint32_t box[2] = {(cuuint32_t)(c.inner_b / 2), (cuuint32_t)c.by};
        cuuint32_t es[2] = {1, 1};
        enc(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, c.sw,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        const int bytes = c.inner_b * c.by;
        const int iters = 3000;
        for (int rep = 0; rep < 2; ++rep)
            probe<<<148, 32, 4 * 32768 + 1024>>>(m, buf, c.mode, bytes, c.by, (int)nrows, iters, d);
        cudaError_t e = cudaDeviceSynchronize();
        long long h[148];
        cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
        long long mx = 0;
        for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
        const double sec = mx / 1.965e9;
        const double per_sm = (double)bytes * iters / sec / 1e9;
        printf("{\"case\": \"%s\", \"err\": \"%s\", \"GBps_per_sm\": %.1f, \"GBps_total\": %.0f, "
               "\"lines_128B_per_us_per_sm\": %.0f}\n",
               c.name, cudaGetErrorString(e), per_sm, per_sm * 148, per_sm * 1e3 / 128.0);
    }
    return 0;
}
