// walk_ceiling.cu -- write-pattern probe for the run-list walker (K3):
// C2-shaped output (40,000 rows of 100,000 B), every warp writing RB bytes of
// each row over a slice of L rows with 16-B stores (lanes 0-15 row r, lanes
// 16-31 row r+1 when RB = 256).  Blocks are ordered group-fastest, so the
// blocks running at once cover one band of slices.  Also: block-wide rows
// (the warps of a block side by side, bar.sync every 16 rows).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o walk_ceiling walk_ceiling.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

constexpr size_t kPitch = 100000;
constexpr int kRows = 40000;

template <int RB>
__global__ void wslice(char* p, int L, int groups, uint32_t v) {
    const int lane = threadIdx.x & 31;
    const int g = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
    if (g >= groups) return;
    const int r0 = blockIdx.y * L;
    const int r1 = min(kRows, r0 + L);
    constexpr int LPR = RB / 16;          // lanes per row
    constexpr int RPI = 32 / LPR;         // rows per instruction
    const int sub = lane / LPR;
    char* q = p + (size_t)g * RB + (lane % LPR) * 16;
    for (int r = r0 + sub; r < r1; r += RPI)
        *reinterpret_cast<uint4*>(q + (size_t)r * kPitch) = make_uint4(v, r, g, lane);
}

// block = W warps side by side (W*RB contiguous bytes per row), bar every 16 rows
template <int RB, int W>
__global__ void wblockrow(char* p, int L, int groups, uint32_t v) {
    const int lane = threadIdx.x & 31;
    const int g = blockIdx.x * W + threadIdx.x / 32;
    const int r0 = blockIdx.y * L;
    const int r1 = min(kRows, r0 + L);
    constexpr int LPR = RB / 16;
    constexpr int RPI = 32 / LPR;
    const int sub = lane / LPR;
    char* q = p + (size_t)g * RB + (lane % LPR) * 16;
    for (int rb = r0; rb < r1; rb += 16) {
        if (g < groups)
            for (int r = rb + sub; r < min(r1, rb + 16); r += RPI)
                *reinterpret_cast<uint4*>(q + (size_t)r * kPitch) = make_uint4(v, r, g, lane);
        __syncthreads();
    }
}

template <class F>
void timeit(const char* name, F f) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    f();
    cudaEventRecord(a);
    for (int i = 0; i < 5; ++i) f();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    ms /= 5;
    printf("%-48s %.3f ms  %.0f GB/s\n", name, ms, 4e9 / (ms * 1e-3) / 1e9);
}

int main() {
    char* d;
    cudaMalloc(&d, kPitch * kRows);
    char name[128];
    for (int L : {40000, 5008, 2048, 1024, 256, 64}) {
        const int ns = (kRows + L - 1) / L;
        {
            const int groups = kPitch / 256;
            snprintf(name, sizeof name, "wslice RB=256 L=%d (4 warps/block)", L);
            timeit(name, [&] { wslice<256><<<dim3((groups + 3) / 4, ns), 128>>>(d, L, groups, 1); });
        }
        {
            const int groups = kPitch / 512;
            snprintf(name, sizeof name, "wslice RB=512 L=%d (4 warps/block)", L);
            timeit(name, [&] { wslice<512><<<dim3((groups + 3) / 4, ns), 128>>>(d, L, groups, 1); });
        }
        {
            const int groups = kPitch / 256;
            snprintf(name, sizeof name, "wblockrow RB=256 x8 warps L=%d", L);
            timeit(name, [&] { wblockrow<256, 8><<<dim3((groups + 7) / 8, ns), 256>>>(d, L, groups, 1); });
        }
    }
    timeit("memset", [&] { cudaMemsetAsync(d, 1, kPitch * kRows); });
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
