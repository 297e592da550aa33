// formats.cu -- SPK1 plane packing and the synthetic stream generator.
//
// k_pack / k_unpack restate pack_frame / unpack_frame (proj/src/io.cpp:52-76)
// on the device: one thread per plane byte (8 pixels).  k_bitrev_bytes turns
// an MSB-first raw dump (io.cpp:72) into the LSB-first layout in place.
//
// k_synth is benchmark/test input synthesis, not part of the reconstruction
// path: the integrate-and-fire recurrence of simulate_pixel
// (proj/src/simulator.cpp:41-68; threshold 1, subtractive reset, 1e-9 fire
// slack, rate sum in double so rounding does not accumulate) over seeded
// float32 rate fields with the shapes of BASELINE.json's configs.
#include "spk_common.cuh"
#include "spk_kernels.cuh"

namespace spk {

__global__ void k_pack(const uint8_t* bytes, int64_t npix, int64_t frames, uint8_t* planes,
                       size_t pitch) {
    const int64_t total = frames * (int64_t)pitch;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t n = i / (int64_t)pitch;
        const int64_t j = i - n * (int64_t)pitch;
        uint32_t b = 0;
        const uint8_t* src = bytes + n * npix;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const int64_t p = j * 8 + k;
            if (p < npix && src[p]) b |= 1u << k;
        }
        planes[i] = (uint8_t)b;  // pad bits and pad bytes are zero
    }
}

__global__ void k_unpack(const uint8_t* planes, size_t pitch, int64_t npix, int64_t frames,
                         uint8_t* bytes) {
    const int64_t row = (npix + 7) / 8;
    const int64_t total = frames * row;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t n = i / row;
        const int64_t j = i - n * row;
        const uint32_t b = planes[n * (int64_t)pitch + j];
        uint8_t* dst = bytes + n * npix;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const int64_t p = j * 8 + k;
            if (p < npix) dst[p] = (uint8_t)((b >> k) & 1u);
        }
    }
}

__global__ void k_bitrev_bytes(uint8_t* planes, size_t pitch, size_t row_bytes, int64_t frames) {
    const int64_t total = frames * (int64_t)row_bytes;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t n = i / (int64_t)row_bytes;
        const int64_t j = i - n * (int64_t)row_bytes;
        uint8_t* b = planes + n * (int64_t)pitch + j;
        *b = (uint8_t)(__brev((uint32_t)*b) >> 24);
    }
}

// ------------------------------------------------------------- synthesis ---
namespace {

__device__ __forceinline__ uint64_t mix64(uint64_t x) {  // splitmix64 finaliser
    x += 0x9e3779b97f4a7c15ull;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return x ^ (x >> 31);
}
__device__ __forceinline__ double u01(uint64_t h) { return (double)(h >> 11) * 0x1.0p-53; }
__device__ __forceinline__ double hash01(uint64_t seed, uint64_t a, uint64_t b) {
    return u01(mix64(mix64(seed ^ 0x5eedb0d1ull) ^ (a << 32 | (b & 0xffffffffull))));
}

constexpr float kTwoPi = 6.28318530717958647692f;

struct Scene2 {  // moving texture + occluding bar
    float amp[16], fx[16], fy[16], ph[16];
    float norm, bar_x0, bar_w, bar_i;
    __device__ void init(uint64_t seed) {
        float s = 0.f;
        for (int k = 0; k < 16; ++k) {
            amp[k] = 0.3f + (float)hash01(seed, 100 + k, 0);
            fx[k] = 0.004f + 0.06f * (float)hash01(seed, 200 + k, 0);
            fy[k] = 0.004f + 0.06f * (float)hash01(seed, 300 + k, 0);
            ph[k] = kTwoPi * (float)hash01(seed, 400 + k, 0);
            s += amp[k];
        }
        norm = 1.f / s;
        bar_x0 = 400.f * (float)hash01(seed, 500, 0);
        bar_w = 12.f + 20.f * (float)hash01(seed, 501, 0);
        bar_i = 0.01f + 0.1f * (float)hash01(seed, 502, 0);
    }
    __device__ float rate(int x, int y, int64_t n, int width) const {
        const float span = (float)width + bar_w;
        const float bx = fmodf(bar_x0 + 0.2f * (float)n, span) - bar_w;
        if ((float)x >= bx && (float)x < bx + bar_w) return bar_i;
        const float xs = (float)x - 0.05f * (float)n;  // texture translates +x
        float acc = 0.f;
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            float arg = fmodf(kTwoPi * (fx[k] * xs + fy[k] * (float)y) + ph[k], kTwoPi);
            acc += amp[k] * __sinf(arg);
        }
        const float u = 0.5f + 0.5f * acc * norm;  // [0, 1]
        return fminf(0.6f, fmaxf(0.01f, 0.01f + 0.59f * u));
    }
};

}  // namespace

__global__ void k_synth(int scene, uint64_t seed, int width, int height, int64_t frames,
                        int64_t frame0, double param, uint8_t* planes, size_t pitch) {
    const int lane = threadIdx.x & 31;
    const int64_t npix = (int64_t)width * height;
    const int64_t word = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (word * 32 >= npix) return;
    const int64_t p = word * 32 + lane;
    const bool valid = p < npix;
    const int x = valid ? (int)(p % width) : 0;
    const int y = valid ? (int)(p / width) : 0;

    // static rate (scenes 1, 5) or per-pixel parameters
    float q_static = 0.f;
    float base3 = 0.f;
    if (scene == 1) {  // smooth gradient + 8x8-block texture noise, I in [0.02, 0.5]
        const float g = 0.5f * ((width > 1 ? (float)x / (width - 1) : 0.f) +
                                (height > 1 ? (float)y / (height - 1) : 0.f));
        const float u = (float)hash01(seed, 1000 + (x >> 3), y >> 3);
        q_static = 0.02f + 0.48f * fminf(1.f, fmaxf(0.f, 0.55f * g + 0.45f * u));
    } else if (scene == 3) {  // log-uniform [0.005, 0.8] per 16x16 block
        const float u = (float)hash01(seed, 3000 + (x >> 4), y >> 4);
        base3 = expf(logf(0.005f) + u * (logf(0.8f) - logf(0.005f)));
    } else if (scene == 5) {  // 10% dark, 10% saturated, 80% mid
        const double c = hash01(seed, 5000 + x, y);
        const float u = (float)hash01(seed, 6000 + x, y);
        q_static = c < 0.1 ? 0.001f + 0.003f * u : c < 0.2 ? 1.0f : 0.01f + 0.49f * u;
    }
    Scene2 s2;
    if (scene == 2) s2.init(seed);

    const double residual = hash01(seed, 7000 + x, y);  // uniform [0, 1)
    const double eps = 1e-9;
    double rate_sum = 0.0;
    int64_t fired = 0;
    uint32_t* out = reinterpret_cast<uint32_t*>(planes + word * 4);
    const int64_t stop = frame0 + frames;
    for (int64_t n = 0; n < stop; ++n) {
        bool bit = false;
        if (valid) {
            if (scene == 0) {
                bit = hash01(seed ^ 0xabcdefull, (uint64_t)p, (uint64_t)n) < param;
            } else {
                float q = q_static;
                if (scene == 2) q = s2.rate(x, y, n, width);
                if (scene == 3)
                    q = fminf(1.f, base3 * (1.f + 0.3f * __sinf(kTwoPi * (float)(n % 5000) / 5000.f)));
                rate_sum += (double)q;
                const double status = residual + rate_sum - (double)fired;
                if (status >= 1.0 - eps) {
                    bit = true;
                    ++fired;
                }
            }
        }
        const uint32_t wbits = __ballot_sync(kFull, bit);
        if (n >= frame0 && lane == 0) out[(size_t)(n - frame0) * (pitch / 4)] = wbits;
    }
}

}  // namespace spk
