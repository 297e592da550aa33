// write_ceiling.cu -- HBM write-only ceiling probe (reference point for K3):
// grid-stride 16-B stores, 32-B (v8) stores, and cudaMemsetAsync over 4 GB.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o write_ceiling write_ceiling.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__global__ void w16(uint4* p, size_t n, uint32_t v) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        p[i] = make_uint4(v, v, v, v);
}

// row-tiled like K3: warp writes 512 B of a row per frame, 16 frames per tile
__global__ void wrows(char* p, size_t pitch, int rows, int groups, uint32_t v) {
    const int lane = threadIdx.x & 31;
    const int g = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
    const int c = blockIdx.y;
    if (g >= groups) return;
    char* q = p + (size_t)c * 1024 * pitch + (size_t)g * 512 + lane * 16;
    for (int f = 0; f < 1024 && c * 1024 + f < rows; ++f)
        *reinterpret_cast<uint4*>(q + (size_t)f * pitch) = make_uint4(v, v, v, f);
}

// warp writes SEG bytes of each row (lane: SEG/32 bytes as 16-B stores), 1024 rows
template <int SEG>
__global__ void wseg(char* p, size_t pitch, int rows, int groups, uint32_t v) {
    const int lane = threadIdx.x & 31;
    const int g = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
    const int c = blockIdx.y;
    if (g >= groups) return;
    char* q = p + (size_t)c * 1024 * pitch + (size_t)g * SEG;
    for (int f = 0; f < 1024 && c * 1024 + f < rows; ++f) {
#pragma unroll
        for (int k = 0; k < SEG / 512; ++k)
            *reinterpret_cast<uint4*>(q + (size_t)f * pitch + k * 512 + lane * 16) = make_uint4(v, v, v, f);
    }
}

// block b writes its own contiguous range (whole rows), 16-B stores
__global__ void wblocked(char* p, size_t bytes, uint32_t v) {
    const size_t per = (bytes / gridDim.x) & ~(size_t)4095;
    char* q = p + (size_t)blockIdx.x * per;
    const size_t n = blockIdx.x + 1 == gridDim.x ? bytes - (size_t)blockIdx.x * per : per;
    for (size_t i = threadIdx.x * 16; i < n; i += blockDim.x * 16)
        *reinterpret_cast<uint4*>(q + i) = make_uint4(v, v, v, (uint32_t)i);
}

// K3-like tiles but a block covers RW contiguous bytes of each row (warps side by side)
template <int RW>
__global__ void wwide(char* p, size_t pitch, int rows, uint32_t v) {
    const int c = blockIdx.y;
    char* q = p + (size_t)c * 1024 * pitch + (size_t)blockIdx.x * RW;
    const int w = min(RW, (int)(pitch - (size_t)blockIdx.x * RW));
    for (int f = 0; f < 1024 && c * 1024 + f < rows; ++f)
        for (int i = threadIdx.x * 16; i < w; i += blockDim.x * 16)
            *reinterpret_cast<uint4*>(q + (size_t)f * pitch + i) = make_uint4(v, v, v, f);
}

// K3 tile pattern with RT rows per tile (warp = 512 B of a row, 4 warps per block)
template <int RT>
__global__ void wtile(char* p, size_t pitch, int rows, int groups, uint32_t v) {
    const int lane = threadIdx.x & 31;
    const int g = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
    const int c = blockIdx.y;
    if (g >= groups) return;
    char* q = p + (size_t)c * RT * pitch + (size_t)g * 512 + lane * 16;
    for (int f = 0; f < RT && c * RT + f < rows; ++f)
        *reinterpret_cast<uint4*>(q + (size_t)f * pitch) = make_uint4(v, v, v, f);
}

// fused-K2 pattern: one wave of 8-warp blocks, warp = 32 pixels (32 B of each
// row), per 32-row word every lane stores 8 u32 (lane = pixel quad q x row
// phase j: rows 4k + j, k = 0..7); ALU work between words simulates the scan
template <int SPIN>
__global__ void wk2(char* p, size_t pitch, int rows, int warps, uint32_t v) {
    const int lane = threadIdx.x & 31;
    const int w = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
    if (w >= warps) return;
    const int q = lane & 7, j = lane >> 3;
    char* base = p + (size_t)w * 32 + q * 4 + (size_t)j * pitch;
    uint32_t x = v + lane;
    for (int g = 0; g * 32 < rows; ++g) {
#pragma unroll
        for (int s = 0; s < SPIN; ++s) x = x * 1664525u + 1013904223u;
#pragma unroll
        for (int k = 0; k < 8; ++k)
            *reinterpret_cast<uint32_t*>(base + (size_t)(32 * g + 4 * k) * pitch) = x + k;
    }
    if (x == 0x12345678u) p[0] = 1;
}

// variants: MODE 1 = per lane 16 B of one row (2 x STG.128 per lane-word,
// rows l and l+... 32 B per row per warp); MODE 2 = block-cooperative: the 8
// warps of a block write 256 contiguous bytes of each row (warp w: rows
// 32g + 4w .. 4w+3, lane 8 B)
template <int MODE>
__global__ void wk2v(char* p, size_t pitch, int rows, int warps, uint32_t v) {
    const int lane = threadIdx.x & 31;
    const int wib = threadIdx.x / 32;
    const int w = blockIdx.x * (blockDim.x / 32) + wib;
    if (w >= warps) return;
    if (MODE == 1) {
        // lane l: rows 32g + l (16 B = pixels 0..15) -- half rows: lanes 0..15 pixels 0..15 of rows
        // 2k + (l>>4)?  simpler: lane l covers row 32g + (l>>1) + 16 * i, pixel half (l & 1)
        char* base = p + (size_t)w * 32 + (lane & 1) * 16;
        for (int g = 0; g * 32 < rows; ++g)
#pragma unroll
            for (int i = 0; i < 2; ++i)
                *reinterpret_cast<uint4*>(base + (size_t)(32 * g + 16 * i + (lane >> 1)) * pitch) =
                    make_uint4(v, g, i, lane);
    } else {
        const int b0 = blockIdx.x * 256;
        if (b0 + 8 * lane + 8 > 100000) return;
        char* base = p + (size_t)b0 + 8 * lane;
        for (int g = 0; g * 32 < rows; ++g)
#pragma unroll
            for (int k = 0; k < 4; ++k)
                *reinterpret_cast<uint2*>(base + (size_t)(32 * g + 4 * wib + k) * pitch) = make_uint2(v, g);
    }
}

template <int MODE>
void run_k2v(char* d, cudaEvent_t a, cudaEvent_t b) {
    const int warps = 100000 / 32;
    wk2v<MODE><<<(warps + 7) / 8, 256>>>(d, 100000, 40000, warps, 1);
    cudaEventRecord(a);
    for (int r = 0; r < 10; ++r) wk2v<MODE><<<(warps + 7) / 8, 256>>>(d, 100000, 40000, warps, r);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("wk2v mode %d: %.3f ms  %.0f GB/s\n", MODE, ms / 10, 4e9 / (ms / 10) / 1e6);
}

template <int SPIN>
void run_k2(char* d, cudaEvent_t a, cudaEvent_t b) {
    const int warps = 100000 / 32;
    wk2<SPIN><<<(warps + 7) / 8, 256>>>(d, 100000, 40000, warps, 1);
    cudaEventRecord(a);
    for (int r = 0; r < 10; ++r) wk2<SPIN><<<(warps + 7) / 8, 256>>>(d, 100000, 40000, warps, r);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("wk2 (fused-K2 pattern, spin %d): %.3f ms  %.0f GB/s\n", SPIN, ms / 10, 4e9 / (ms / 10) / 1e6);
}

template <int RT>
void run_tile(char* d, cudaEvent_t a, cudaEvent_t b) {
    dim3 grid((196 + 3) / 4, (40000 + RT - 1) / RT);
    wtile<RT><<<grid, 128>>>(d, 100000, 40000, 196, 1);
    cudaEventRecord(a);
    for (int r = 0; r < 10; ++r) wtile<RT><<<grid, 128>>>(d, 100000, 40000, 196, r);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("wtile %4d rows per tile: %.3f ms  %.0f GB/s\n", RT, ms / 10, 4e9 / (ms / 10) / 1e6);
}

// transposed launch order: chunk fastest (a wave covers few groups, many chunks)
__global__ void wtileT(char* p, size_t pitch, int rows, int groups, uint32_t v) {
    const int lane = threadIdx.x & 31;
    const int g = blockIdx.y * (blockDim.x / 32) + threadIdx.x / 32;
    const int c = blockIdx.x;
    if (g >= groups) return;
    char* q = p + (size_t)c * 1024 * pitch + (size_t)g * 512 + lane * 16;
    for (int f = 0; f < 1024 && c * 1024 + f < rows; ++f)
        *reinterpret_cast<uint4*>(q + (size_t)f * pitch) = make_uint4(v, v, v, f);
}

template <int SEG>
void run_seg(char* d, cudaEvent_t a, cudaEvent_t b, int wpb) {
    const int groups = 100000 / SEG;
    dim3 grid((groups + wpb - 1) / wpb, 40);
    wseg<SEG><<<grid, wpb * 32>>>(d, 100000, 40000, groups, 1);
    cudaEventRecord(a);
    for (int r = 0; r < 10; ++r) wseg<SEG><<<grid, wpb * 32>>>(d, 100000, 40000, groups, r);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double bytes = (double)groups * SEG * 40000;
    printf("wseg %5d B/row, %d warps/block: %.3f ms  %.0f GB/s\n", SEG, wpb, ms / 10, bytes / (ms / 10) / 1e6);
}

int main() {
    const size_t bytes = 40000ull * 100000ull;
    char* d;
    cudaMalloc(&d, bytes);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float ms;
    for (int blocks : {148 * 4, 148 * 8, 148 * 16, 148 * 32}) {
        w16<<<blocks, 512>>>((uint4*)d, bytes / 16, 1);
        cudaEventRecord(a);
        for (int r = 0; r < 10; ++r) w16<<<blocks, 512>>>((uint4*)d, bytes / 16, r);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        printf("w16 grid %5d x 512: %.3f ms  %.0f GB/s\n", blocks, ms / 10, bytes / (ms / 10) / 1e6);
    }
    cudaMemsetAsync(d, 1, bytes);
    cudaEventRecord(a);
    for (int r = 0; r < 10; ++r) cudaMemsetAsync(d, r, bytes);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("memset: %.3f ms  %.0f GB/s\n", ms / 10, bytes / (ms / 10) / 1e6);
    for (int wpb : {4, 8}) {
        dim3 grid((196 + wpb - 1) / wpb, 40);
        wrows<<<grid, wpb * 32>>>(d, 100000, 40000, 196, 1);
        cudaEventRecord(a);
        for (int r = 0; r < 10; ++r) wrows<<<grid, wpb * 32>>>(d, 100000, 40000, 196, r);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        printf("wrows (K3 pattern, %d warps/block): %.3f ms  %.0f GB/s\n", wpb, ms / 10, bytes / (ms / 10) / 1e6);
    }
    for (int wpb : {2, 4}) {
        run_seg<512>(d, a, b, wpb);
        run_seg<1024>(d, a, b, wpb);
        run_seg<2048>(d, a, b, wpb);
        run_seg<4096>(d, a, b, wpb);
    }
    run_k2v<1>(d, a, b);
    run_k2v<2>(d, a, b);
    run_k2<0>(d, a, b);
    run_k2<64>(d, a, b);
    run_k2<256>(d, a, b);
    run_tile<64>(d, a, b);
    run_tile<256>(d, a, b);
    run_tile<1024>(d, a, b);
    run_tile<4096>(d, a, b);
    {
        dim3 grid(40, 49);
        wtileT<<<grid, 128>>>(d, 100000, 40000, 196, 1);
        cudaEventRecord(a);
        for (int r = 0; r < 10; ++r) wtileT<<<grid, 128>>>(d, 100000, 40000, 196, r);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        printf("wtileT (chunk-fastest order): %.3f ms  %.0f GB/s\n", ms / 10, bytes / (ms / 10) / 1e6);
    }
    for (int blocks : {148, 296, 592, 1184}) {
        wblocked<<<blocks, 512>>>(d, bytes, 1);
        cudaEventRecord(a);
        for (int r = 0; r < 10; ++r) wblocked<<<blocks, 512>>>(d, bytes, r);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        printf("wblocked %5d blocks x 512: %.3f ms  %.0f GB/s\n", blocks, ms / 10, bytes / (ms / 10) / 1e6);
    }
    {
        dim3 grid((100000 + 8191) / 8192, 40);
        wwide<8192><<<grid, 512>>>(d, 100000, 40000, 1);
        cudaEventRecord(a);
        for (int r = 0; r < 10; ++r) wwide<8192><<<grid, 512>>>(d, 100000, 40000, r);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        printf("wwide 8192 B/row x 1024 rows per block: %.3f ms  %.0f GB/s\n", ms / 10, bytes / (ms / 10) / 1e6);
        dim3 grid2((100000 + 2047) / 2048, 40);
        wwide<2048><<<grid2, 128>>>(d, 100000, 40000, 1);
        cudaEventRecord(a);
        for (int r = 0; r < 10; ++r) wwide<2048><<<grid2, 128>>>(d, 100000, 40000, r);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        printf("wwide 2048 B/row x 1024 rows per block: %.3f ms  %.0f GB/s\n", ms / 10, bytes / (ms / 10) / 1e6);
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
