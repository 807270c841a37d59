// TMA throughput per SM (all 148 SMs busy): one thread streams box loads (or
// stores) through a 4-slot smem ring; reports GB/s per SM and aggregate for
// several box shapes.  Source tensor: 256 MB bf16, rows of 256 B (128 features).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_2602_12271_b200/csrc -o ubench_tma ubench_tma.cu -lcuda
#include <cstdio>
#include <cuda.h>
#include "mbx_sm100.cuh"

using namespace mbx::sm100;

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, const void* src, int c0, int c1) {
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                     reinterpret_cast<uint64_t>(map)),
                 "r"(smem_u32(src)), "r"(c0), "r"(c1)
                 : "memory");
}

// map: 2D (features_inner, rows); box (bx, by)
__global__ void tma_load_probe(const __grid_constant__ CUtensorMap map, int box_bytes, int bx, int by, int rows_total,
                               int iters, int store, long long* out) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t full[4];
    if (threadIdx.x == 0) {
        for (int i = 0; i < 4; ++i) mbar_init(&full[i], 1);
        fence_barrier_init();
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        const int slot_bytes = 32768;
        const int nbox_rows = rows_total / by;
        long long t0 = clock64();
        if (!store) {
            for (int it = 0; it < iters; ++it) {
                const int s = it & 3;
                if (it >= 4) mbar_wait(&full[s], ((it >> 2) - 1) & 1);
                mbar_expect_tx(&full[s], box_bytes);
                const int row = ((blockIdx.x * 7919 + it * 131) % nbox_rows) * by;
                tma_load_2d(smem + s * slot_bytes, &map, &full[s], 0, row);
            }
            for (int it = iters; it < iters + 4; ++it) mbar_wait(&full[it & 3], ((it >> 2) - 1) & 1);
        } else {
            for (int it = 0; it < iters; ++it) {
                const int s = it & 3;
                if (it >= 4) asm volatile("cp.async.bulk.wait_group.read 3;" ::: "memory");
                const int row = ((blockIdx.x * 7919 + it * 131) % nbox_rows) * by;
                tma_store_2d(&map, smem + s * slot_bytes, 0, row);
                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            }
            asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
        }
        long long t1 = clock64();
        out[blockIdx.x] = t1 - t0;
    }
}

int main() {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
    EncodeFn enc = (EncodeFn)p;
    const size_t rows = 1 << 20;   // 1M rows x 256 B = 256 MB
    void* buf;
    cudaMalloc(&buf, rows * 256);
    cudaMemset(buf, 0, rows * 256);
    long long* d;
    cudaMalloc(&d, 148 * 8);
    cudaFuncSetAttribute(tma_load_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 32768 + 1024);
    struct Case { const char* name; int bx; int by; CUtensorMapSwizzle sw; };
    Case cases[] = {
        {"64 feat (128 B rows) x 52 rows SW128", 64, 52, CU_TENSOR_MAP_SWIZZLE_128B},
        {"64 feat (128 B rows) x 128 rows SW128", 64, 128, CU_TENSOR_MAP_SWIZZLE_128B},
        {"128 feat (256 B rows) x 64 rows no swizzle", 128, 64, CU_TENSOR_MAP_SWIZZLE_NONE},
        {"128 feat (256 B rows) x 128 rows no swizzle", 128, 128, CU_TENSOR_MAP_SWIZZLE_NONE},
        {"64 feat x 32 rows SW128", 64, 32, CU_TENSOR_MAP_SWIZZLE_128B},
    };
    for (int store = 0; store < 2; ++store) {
        for (auto& c : cases) {
            CUtensorMap m;
            cuuint64_t dims[2] = {128, rows};
            cuuint64_t strides[1] = {256};
            cuuint32_t box[2] = {(cuuint32_t)c.bx, (cuuint32_t)c.by};
            cuuint32_t es[2] = {1, 1};
            CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, strides, box, es,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, c.sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            const int bb = c.bx * 2 * c.by;
            const int iters = 4000;
            tma_load_probe<<<148, 32, 4 * 32768 + 1024>>>(m, bb, c.bx, c.by, (int)rows, iters, store, d);
            tma_load_probe<<<148, 32, 4 * 32768 + 1024>>>(m, bb, c.bx, c.by, (int)rows, iters, store, d);
            cudaError_t e = cudaDeviceSynchronize();
            long long h[148];
            cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
            long long mx = 0;
            for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
            const double sec = mx / 1.965e9;
            const double per_sm = (double)bb * iters / sec / 1e9;
            printf("{\"op\": \"%s\", \"box\": \"%s\", \"enc\": %d, \"err\": \"%s\", \"GBps_per_sm\": %.1f, \"GBps_total\": %.0f, "
                   "\"rows_per_us_per_sm\": %.0f}\n",
                   store ? "store" : "load", c.name, (int)r, cudaGetErrorString(e), per_sm, per_sm * 148,
                   (double)c.by * iters / (sec * 1e6));
        }
    }
    return 0;
}
