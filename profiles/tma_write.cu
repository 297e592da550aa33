// tma_write.cu -- K3's write pattern (a warp writes 512 B of each row of an
// R-row tile, 4 warps per block, tiles launched piece row by piece row) with
// per-lane 16-B stores (STG) vs TMA 2D tile stores from shared memory
// (cp.async.bulk.tensor, UTMASTG): each warp stages 16 rows x 512 B and one
// lane stores the box.  4 GB = 40,000 rows x 100,000 B (configs[1] frames).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_write tma_write.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

constexpr int ROWS = 40000, PITCH = 100000, GROUPS = 196;

template <int RT>
__global__ void stg_tiles(char* p, uint32_t v) {
    const int lane = threadIdx.x & 31;
    const int g = blockIdx.x * 4 + (threadIdx.x >> 5);
    if (g >= GROUPS) return;
    const int r0 = blockIdx.y * RT;
    char* q = p + (size_t)r0 * PITCH + (size_t)g * 512 + lane * 16;
    for (int f = 0; f < RT && r0 + f < ROWS; ++f)
        *reinterpret_cast<uint4*>(q + (size_t)f * PITCH) = make_uint4(v, v, v, f);
}

// box = 128 u32 (512 B) x 16 rows per warp, double-buffered staging
template <int RT>
__global__ void tma_tiles(const __grid_constant__ CUtensorMap tm, uint32_t v) {
    extern __shared__ __align__(128) uint8_t sm[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int g = blockIdx.x * 4 + warp;
    if (g >= GROUPS) return;
    uint8_t* stage = sm + warp * 2 * 16 * 512;
    const int r0 = blockIdx.y * RT;
    int buf = 0;
    for (int f0 = 0; f0 < RT && r0 + f0 < ROWS; f0 += 16, buf ^= 1) {
        uint8_t* s = stage + buf * 16 * 512;
        if (f0 >= 32 && lane == 0)  // the store that used this buffer has read it
            asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
        __syncwarp();
#pragma unroll
        for (int f = 0; f < 16; ++f)
            *reinterpret_cast<uint4*>(s + f * 512 + lane * 16) = make_uint4(v, v, v, f0 + f);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) {
            const uint32_t sa = (uint32_t)__cvta_generic_to_shared(s);
            asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];"
                         ::"l"(&tm), "r"(g * 128), "r"(r0 + f0), "r"(sa) : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
    }
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
    const size_t bytes = (size_t)ROWS * PITCH;
    char* d;
    cudaMalloc(&d, bytes);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    EncodeFn enc = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
    CUtensorMap tm;
    cuuint64_t dims[2] = {PITCH / 4, ROWS};
    cuuint64_t strides[1] = {PITCH};
    cuuint32_t box[2] = {128, 16}, es[2] = {1, 1};
    CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, d, dims, strides, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                     CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode %d\n", (int)r);
    float ms;
    auto timeit = [&](const char* name, auto launch) {
        launch(1);
        cudaEventRecord(a);
        for (int k = 0; k < 10; ++k) launch(k);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        printf("%-28s %.3f ms  %.0f GB/s  (%s)\n", name, ms / 10, bytes / (ms / 10) / 1e6,
               cudaGetErrorString(cudaGetLastError()));
    };
    const int smem = 4 * 2 * 16 * 512;
    cudaFuncSetAttribute(tma_tiles<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(tma_tiles<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(tma_tiles<1024>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    timeit("stg 64-row tiles", [&](int k) { stg_tiles<64><<<dim3(49, (ROWS + 63) / 64), 128>>>(d, k); });
    timeit("tma 64-row tiles", [&](int k) { tma_tiles<64><<<dim3(49, (ROWS + 63) / 64), 128, smem>>>(tm, k); });
    timeit("stg 128-row tiles", [&](int k) { stg_tiles<128><<<dim3(49, (ROWS + 127) / 128), 128>>>(d, k); });
    timeit("tma 128-row tiles", [&](int k) { tma_tiles<128><<<dim3(49, (ROWS + 127) / 128), 128, smem>>>(tm, k); });
    timeit("stg 1024-row tiles", [&](int k) { stg_tiles<1024><<<dim3(49, (ROWS + 1023) / 1024), 128>>>(d, k); });
    timeit("tma 1024-row tiles", [&](int k) { tma_tiles<1024><<<dim3(49, (ROWS + 1023) / 1024), 128, smem>>>(tm, k); });
    timeit("memset", [&](int k) { cudaMemsetAsync(d, k, bytes); });
    // correctness spot check of the TMA path
    tma_tiles<64><<<dim3(49, (ROWS + 63) / 64), 128, smem>>>(tm, 7);
    uint32_t h[8];
    cudaMemcpy(h, d + (size_t)12345 * PITCH + 512 * 7, 32, cudaMemcpyDeviceToHost);
    printf("check row 12345 group 7: %u %u %u %u (expect 7 7 7 %u)\n", h[0], h[1], h[2], h[3], 12345 % 64);
    return 0;
}
