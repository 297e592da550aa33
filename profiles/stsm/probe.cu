// Empirical layout of stmatrix.sync.aligned.m16n8.x4.trans.shared.b8 (STSM.8.MT168.4)
#include <cstdio>
#include <cstdint>
__global__ void k(uint8_t* out, int mode) {
    __shared__ __align__(16) uint8_t sm[2048];
    for (int i = threadIdx.x; i < 2048; i += 32) sm[i] = 0xEE;
    __syncwarp();
    const int l = threadIdx.x;
    uint32_t r[4];
    for (int i = 0; i < 4; ++i) {
        uint32_t v = 0;
        for (int b = 0; b < 4; ++b) {
            const uint32_t val = mode == 0 ? (uint32_t)l : (uint32_t)(i * 4 + b);
            v |= val << (8 * b);
        }
        r[i] = v;
    }
    uint32_t a = (uint32_t)__cvta_generic_to_shared(sm + l * 64);
    asm volatile("stmatrix.sync.aligned.m16n8.x4.trans.shared.b8 [%0], {%1, %2, %3, %4};" :: "r"(a), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]));
    __syncwarp();
    for (int i = threadIdx.x; i < 2048; i += 32) out[i] = sm[i];
}
int main() {
    uint8_t* d; cudaMalloc(&d, 4096);
    uint8_t h[2][2048];
    for (int m = 0; m < 2; ++m) { k<<<1, 32>>>(d, m); cudaMemcpy(h[m], d, 2048, cudaMemcpyDeviceToHost); }
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
    for (int row = 0; row < 32; ++row) {
        printf("addr-lane %2d:", row);
        for (int c = 0; c < 64; ++c) {
            const int o = row * 64 + c;
            if (h[0][o] == 0xEE) continue;
            printf(" [%d]L%dR%dB%d", c, h[0][o], h[1][o] / 4, h[1][o] % 4);
        }
        printf("\n");
    }
}
