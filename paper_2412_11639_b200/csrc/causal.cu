// causal.cu -- TFI and TFP(L) baselines in one pass (sm_100a).
//
// Replaces reconstruct_row's TFP branch (proj/src/reconstruct.cpp:328-337)
// and TFI branch (338-354).  Both are causal, so no run lists: a warp owns 32
// pixels (one plane word), transposes each 32-frame block to per-pixel words
// (as K2 does), computes the 32 values of its pixel into a shared-memory tile
// [frame][pixel] and writes the tile back frame-major, one row per lane.
//
// TFI: frame n = 255/ISI of the latest completed interval (0 before the 2nd
// spike).  TFP: frame n = 255*count(bits in (n-L, n]) / min(L, n+1); the bit
// leaving the window comes from the word L frames back (reloaded and
// re-transposed, so any L works).  Per-value divisions are tabulated in shared
// memory (uint8: the integer round-half-away form of quantize, io.cpp:78-81).
#include "spk_common.cuh"
#include "spk_fsm.cuh"
#include "spk_kernels.cuh"

namespace spk {

namespace {

template <typename OUT>
__device__ __forceinline__ OUT ratio_val(uint32_t num, uint32_t den);  // 255*num/den
template <>
__device__ __forceinline__ uint8_t ratio_val<uint8_t>(uint32_t num, uint32_t den) {
    return (uint8_t)((510ull * num + den) / (2ull * den));
}
template <>
__device__ __forceinline__ float ratio_val<float>(uint32_t num, uint32_t den) {
    return (float)(255.0 * (double)num / (double)den);
}
template <>
__device__ __forceinline__ double ratio_val<double>(uint32_t num, uint32_t den) {
    return 255.0 * (double)num / (double)den;
}

__device__ __forceinline__ uint32_t ldw(const char* col, size_t pitch, int f, int frames) {
    return (f >= 0 && f < frames) ? __ldg(reinterpret_cast<const uint32_t*>(col + (size_t)f * pitch))
                                  : 0u;
}

}  // namespace

template <int METHOD, typename OUT>
__global__ void __launch_bounds__(kCausalWarps * 32) k_causal(CausalArgs a) {
    extern __shared__ __align__(16) unsigned char smem[];
    constexpr int ROW = 32 * (int)sizeof(OUT) + 16;  // padded: conflict-free 16-B row reads
    OUT* lut = reinterpret_cast<OUT*>(smem);
    const int lut_n = a.lut_n;
    const int L = a.window;
    for (int i = threadIdx.x; i < lut_n; i += blockDim.x) {
        if (METHOD == kTFI)
            lut[i] = i == 0 ? OUT(0) : ratio_val<OUT>(1u, (uint32_t)i);  // 255 / isi
        else
            lut[i] = ratio_val<OUT>((uint32_t)i, (uint32_t)L);  // 255 * cnt / L
    }
    __syncthreads();

    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const int64_t word = (int64_t)blockIdx.x * kCausalWarps + warp;
    if (word * 32 >= a.npix) return;  // warp-uniform
    const int64_t p = word * 32 + lane;
    const bool valid = p < a.npix;
    const int frames = a.frames;
    const int ngroups = (frames + 31) >> 5;
    const char* col = reinterpret_cast<const char*>(a.planes) + word * 4;
    const size_t pitch = a.pitch;
    const size_t lut_bytes = ((size_t)lut_n * sizeof(OUT) + 15) & ~(size_t)15;
    unsigned char* tile = smem + lut_bytes + (size_t)warp * 32 * ROW;

    const int q = L >> 5, r = L & 31;  // TFP: window in whole words + remainder
    const int64_t nvalid = min((int64_t)32, a.npix - word * 32);
    const bool vec_ok =
        nvalid == 32 &&
        ((reinterpret_cast<uintptr_t>(a.out) | (a.out_pitch * sizeof(OUT))) & 15) == 0;

    int last = -1;   // TFI: last spike frame
    OUT v = OUT(0);  // TFI: current value
    int cnt = 0;     // TFP: spikes in window
    uint32_t prev_old = 0;

    for (int g = 0; g < ngroups; ++g) {
        uint32_t w = transpose32(ldw(col, pitch, g * 32 + lane, frames), lane);
        uint32_t o = 0;
        if (METHOD == kTFP) {
            // words g-q-1 (prev_old) and g-q hold the frames leaving the window
            const uint32_t wo = transpose32(ldw(col, pitch, (g - q) * 32 + lane, frames), lane);
            o = r ? __funnelshift_r(prev_old, wo, 32 - r) : wo;
            prev_old = wo;
        }
        if (!valid) w = o = 0;
        const int base = g * 32;
#pragma unroll
        for (int b = 0; b < 32; ++b) {
            if (METHOD == kTFI) {
                if (w & (1u << b)) {
                    const int n = base + b;
                    if (last >= 0) {
                        const int isi = n - last;
                        v = isi < lut_n ? lut[isi] : ratio_val<OUT>(1u, (uint32_t)isi);
                    }
                    last = n;
                }
            } else {
                cnt += (int)((w >> b) & 1u) - (int)((o >> b) & 1u);
                const int n = base + b;
                if (n >= L - 1)
                    v = cnt < lut_n ? lut[cnt] : ratio_val<OUT>((uint32_t)cnt, (uint32_t)L);
                else
                    v = ratio_val<OUT>((uint32_t)cnt, (uint32_t)(n + 1));
            }
            *reinterpret_cast<OUT*>(tile + b * ROW + lane * sizeof(OUT)) = v;
        }
        __syncwarp();
        // lane i stores frame base+i of the warp's 32 pixels
        const int n = base + lane;
        if (n < frames) {
            const unsigned char* src = tile + lane * ROW;
            char* dst = reinterpret_cast<char*>(a.out) +
                        ((size_t)n * a.out_pitch + (size_t)word * 32) * sizeof(OUT);
            if (vec_ok) {
#pragma unroll
                for (int k = 0; k < 2 * (int)sizeof(OUT); ++k)
                    *reinterpret_cast<uint4*>(dst + 16 * k) =
                        *reinterpret_cast<const uint4*>(src + 16 * k);
            } else {
                for (int i = 0; i < nvalid; ++i)
                    reinterpret_cast<OUT*>(dst)[i] = reinterpret_cast<const OUT*>(src)[i];
            }
        }
        __syncwarp();
    }
}

template __global__ void k_causal<kTFI, uint8_t>(CausalArgs);
template __global__ void k_causal<kTFI, float>(CausalArgs);
template __global__ void k_causal<kTFI, double>(CausalArgs);
template __global__ void k_causal<kTFP, uint8_t>(CausalArgs);
template __global__ void k_causal<kTFP, float>(CausalArgs);
template __global__ void k_causal<kTFP, double>(CausalArgs);

}  // namespace spk
