// spk_common.cuh -- shared device helpers for the sm_100a reconstruction path.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace spk {

constexpr unsigned kFull = 0xffffffffu;

// Frames per table chunk: the expand kernel (K3) tiles time in chunks of
// kChunk frames and the segment kernel (K2) records, for every pixel and chunk
// boundary, which run covers that frame ("run table").
constexpr int kChunkLog2 = 10;
constexpr int kChunk = 1 << kChunkLog2;

// Sentinels of the streaming state machine.  Frames are < 2^29, so
//   t - kNoPair    < 0  -> unsigned compare fails the fast path,
//   idx - kNoIdx   in (2^29, 2^30]  -> gap - kNoPair < 0 -> fails as well.
constexpr int kNoPair = 1 << 30;   // pair rule has no value yet
constexpr int kNoIdx = -(1 << 29); // value has not occurred in the sub-run
constexpr int kNoSpike = -(1 << 29);

// 32x32 bit-matrix transpose across a warp.  On entry lane i holds row i
// (bit j = column j); on exit lane j holds column j (bit i = row i).
// Five butterfly stages of (funnel rotate, shuffle, bit-select): 15 issue
// slots per lane per 32x32 block.  Lane i's partner at stage s is i^s; the
// lower lane keeps the columns with (j & s) == 0 and receives the partner's
// same columns moved up by s, the upper lane the mirror image.
__device__ __forceinline__ uint32_t transpose32(uint32_t x, int lane) {
#pragma unroll
    for (int s = 16; s >= 1; s >>= 1) {
        const uint32_t m = s == 16 ? 0x0000ffffu
                         : s == 8  ? 0x00ff00ffu
                         : s == 4  ? 0x0f0f0f0fu
                         : s == 2  ? 0x33333333u
                                   : 0x55555555u;
        const bool lo = (lane & s) == 0;
        const uint32_t send = __funnelshift_r(x, x, lo ? s : 32 - s);
        const uint32_t y = __shfl_xor_sync(kFull, send, s);
        const uint32_t keep = lo ? m : ~m;
        x = (x & keep) | (y & ~keep);
    }
    return x;
}

// The reference's uint8 rule for a run value: round-half-away(255*N/span)
// (proj/src/io.cpp:78-81 applied to proj/src/reconstruct.cpp:124).  The
// exact rational is never within 1/(2*span) of a .5 boundary unless it is on
// it, so the integer form below equals the double path for every N <= span.
// Computed as floor of the double quotient: both operands are exact (< 2^53)
// and a non-integer quotient is >= 1/(2 span) >= 2^-30 from the next integer,
// far above the division's rounding error (<= 2^-45), so the floor is exact
// -- and much cheaper than a 64-bit integer division.
__host__ __device__ __forceinline__ uint32_t run_u8(uint32_t n, uint32_t span) {
    return (uint32_t)floor((510.0 * (double)n + (double)span) / (2.0 * (double)span));
}

__host__ __device__ __forceinline__ double run_f64(uint32_t n, uint32_t span) {
    return 255.0 * (double)n / (double)span;
}

template <typename T>
struct OutVal;
template <>
struct OutVal<uint8_t> {
    __device__ static uint8_t run(uint32_t n, uint32_t span) { return (uint8_t)run_u8(n, span); }
};
template <>
struct OutVal<float> {
    __device__ static float run(uint32_t n, uint32_t span) { return (float)run_f64(n, span); }
};
template <>
struct OutVal<double> {
    __device__ static double run(uint32_t n, uint32_t span) { return run_f64(n, span); }
};

// Read-only streaming load, bypassing L1 allocation (input planes are read
// once per warp; the 32-B sector is shared by the 8 warps of a 256-px group
// through L2).
__device__ __forceinline__ uint32_t ld_stream(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.global.nc.L1::no_allocate.b32 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
}

}  // namespace spk
