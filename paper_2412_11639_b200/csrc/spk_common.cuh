// spk_common.cuh -- shared device helpers for the sm_100a reconstruction path.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace spk {

constexpr unsigned kFull = 0xffffffffu;

// Bounds checks of the checked build (-DSPK_CHECKED, build.build_checked():
// compute-sanitizer is closed on the GPU pool, so the index invariants the
// kernels rely on are asserted in a separate build the GPU tests run).  A
// violated check traps the kernel (cudaErrorLaunchFailure).  Free otherwise.
#ifdef SPK_CHECKED
#define SPK_CHECK(cond)          \
    do {                         \
        if (!(cond)) __trap();   \
    } while (0)
#else
#define SPK_CHECK(cond) \
    do {                \
    } while (0)
#endif

// Frames per chunk: the expand kernel (K3) tiles time in chunks of kChunk
// frames, and K2c records every pixel's value at each chunk start.
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
// Five butterfly stages of shuffles.  Lane i's partner at stage s is i^s; the
// lower lane keeps the columns with (j & s) == 0 and receives the partner's
// same columns moved up by s, the upper lane the mirror image.
// Implementation with the per-lane constants computed once (hoisted out of
// the caller's loop): the two byte stages (s = 16, 8) are one PRMT each on
// the unrotated partner word, the three bit stages one funnel rotate and one
// 3-input bit-select (LOP3 0xE4) each -- 8 integer-ALU instructions per word
// instead of 20 with a lane-dependent mask per stage (K2 is bound by the
// integer ALU pipe).
struct Transpose32 {
    uint32_t sel16, sel8;        // PRMT selectors of the byte stages
    uint32_t keep4, keep2, keep1;  // bits this lane keeps at stages 4, 2, 1
    uint32_t rot4, rot2, rot1;     // rotate of the word this lane sends

    __device__ __forceinline__ void init(int lane) {
        const bool l16 = (lane & 16) == 0, l8 = (lane & 8) == 0;
        // lower lane: [x.b0, x.b1, y.b0, y.b1], upper: [y.b2, y.b3, x.b2, x.b3]
        sel16 = l16 ? 0x5410u : 0x3276u;
        // lower lane: [x.b0, y.b0, x.b2, y.b2], upper: [y.b1, x.b1, y.b3, x.b3]
        sel8 = l8 ? 0x6240u : 0x3715u;
        keep4 = (lane & 4) == 0 ? 0x0f0f0f0fu : 0xf0f0f0f0u;
        keep2 = (lane & 2) == 0 ? 0x33333333u : 0xccccccccu;
        keep1 = (lane & 1) == 0 ? 0x55555555u : 0xaaaaaaaau;
        rot4 = (lane & 4) == 0 ? 4u : 28u;
        rot2 = (lane & 2) == 0 ? 2u : 30u;
        rot1 = (lane & 1) == 0 ? 1u : 31u;
    }
    __device__ __forceinline__ static uint32_t bitsel(uint32_t x, uint32_t y, uint32_t keep) {
        uint32_t r;  // (x & keep) | (y & ~keep)
        asm("lop3.b32 %0, %1, %2, %3, 0xE4;" : "=r"(r) : "r"(x), "r"(y), "r"(keep));
        return r;
    }
    __device__ __forceinline__ uint32_t operator()(uint32_t x) const {
        x = __byte_perm(x, __shfl_xor_sync(kFull, x, 16), sel16);
        x = __byte_perm(x, __shfl_xor_sync(kFull, x, 8), sel8);
        x = bitsel(x, __shfl_xor_sync(kFull, __funnelshift_r(x, x, rot4), 4), keep4);
        x = bitsel(x, __shfl_xor_sync(kFull, __funnelshift_r(x, x, rot2), 2), keep2);
        x = bitsel(x, __shfl_xor_sync(kFull, __funnelshift_r(x, x, rot1), 1), keep1);
        return x;
    }
};

__device__ __forceinline__ uint32_t transpose32(uint32_t x, int lane) {
    Transpose32 t;  // loop-invariant: the compiler hoists init out of callers' loops
    t.init(lane);
    return t(x);
}

// The reference's uint8 rule for a run value: round-half-away(255*N/span)
// (proj/src/io.cpp:78-81 applied to proj/src/reconstruct.cpp:124).  The
// exact rational is never within 1/(2*span) of a .5 boundary unless it is on
// it, so the integer form below equals the double path for every N <= span.
// Computed as floor of the double quotient: both operands are exact (< 2^53)
// and a non-integer quotient is >= 1/(2 span) >= 2^-30 from the next integer,
// far above the division's rounding error (<= 2^-45), so the floor is exact
// -- and much cheaper than a 64-bit integer division.
//
// Fast path (every run of a stream below 2^22 frames): the quotient is at
// most 255 and num = 510 N + span < 2^31, so a float estimate num * rcp(den)
// (relative error < 2^-21) is within 1 of the exact quotient; one integer
// remainder corrects it.  ~12 instructions instead of a double division
// (K2c computes one value per run).  Host-tested against the integer rule.
__host__ __device__ __forceinline__ uint32_t run_u8(uint32_t n, uint32_t span) {
    if ((span - 1u < (1u << 22) - 1u) & (n <= span)) {
        const uint32_t num = 510u * n + span, den = 2u * span;
#ifdef __CUDA_ARCH__
        const float rc = __frcp_rn((float)den);
#else
        const float rc = 1.0f / (float)den;
#endif
        uint32_t q = (uint32_t)((float)num * rc);
        const int r = (int)(num - q * den);
        q += (uint32_t)(r >= (int)den) - (uint32_t)(r < 0);
        return q;
    }
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
