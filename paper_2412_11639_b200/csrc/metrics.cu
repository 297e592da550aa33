// metrics.cu -- quality metrics and the stability check on the device
// (SURVEY.md 8(f) row 4).
//
// K_te/mse  one block per frame: two_dimensional_entropy (proj/src/metrics.cpp:
//           12-43) and mse against a reference image (45-55).  The
//           256x256 (gray, rounded 3x3 mean) histogram is built in shared
//           memory in two halves of 128 gray levels (128 KB each, 32-bit
//           counts: a 1000x1000 frame has ~1M interior pixels); each half is
//           reduced to its -p*log2(p) sum in a fixed order, so the result is
//           deterministic (equal to the reference's sequential sum up to
//           double rounding).
// K_stab    one thread per pixel: stability_order (proj/src/stability.cpp:
//           61-128) -- the depth-first tree of interval streams, '-' first,
//           with the reference's pruning -- over the pixel's S1 kept in a
//           per-pixel global scratch region (a stack of one sequence per
//           depth; a child is never longer than its parent, so depth * |S1|
//           ints always suffice).
#include <cmath>

#include "spk_common.cuh"
#include "spk_kernels.cuh"

namespace spk {

namespace {

template <typename IN>
__device__ __forceinline__ int qv(IN v) {
    if constexpr (sizeof(IN) == 1) {
        return (int)v;
    } else {  // round(clamp(v, 0, 255)), metrics.cpp:18 (= quantize, io.cpp:78-81)
        return (int)round(fmin(fmax((double)v, 0.0), 255.0));
    }
}

template <typename IN>
__device__ __forceinline__ double dv(IN v) {
    return (double)v;
}

__device__ double block_sum(double x, double* red) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o; o >>= 1) x += __shfl_down_sync(kFull, x, o);
    __syncthreads();  // `red` may still be read from a previous call
    if (lane == 0) red[warp] = x;
    __syncthreads();
    double s = 0.0;
    if (threadIdx.x == 0)
        for (int i = 0; i < (int)(blockDim.x >> 5); ++i) s += red[i];
    return s;  // valid in thread 0
}

}  // namespace

template <typename IN>
__global__ void __launch_bounds__(kMetThreads) k_frame_metrics(MetArgs a) {
    extern __shared__ uint32_t hist[];  // kMetHalf bins
    __shared__ double red[kMetThreads / 32];
    const int64_t n = blockIdx.x;
    const int w = a.width, h = a.height;
    const IN* f = reinterpret_cast<const IN*>(a.frames) + n * (int64_t)a.pitch;
    if (a.mse != nullptr) {
        const int64_t r0 = n * a.ref_pitch;
        double acc = 0.0;
        for (int64_t i = threadIdx.x; i < (int64_t)w * h; i += blockDim.x) {
            const double rv = a.ref_type == SPK_OUT_U8
                                  ? (double)static_cast<const uint8_t*>(a.ref)[r0 + i]
                              : a.ref_type == SPK_OUT_F32
                                  ? (double)static_cast<const float*>(a.ref)[r0 + i]
                                  : static_cast<const double*>(a.ref)[r0 + i];
            const double d = dv(f[i]) - rv;
            acc += d * d;
        }
        const double s = block_sum(acc, red);
        if (threadIdx.x == 0) a.mse[n] = s / (double)((int64_t)w * h);
    }
    if (a.te == nullptr) return;
    const int iw = w - 2;
    const int64_t interior = (int64_t)iw * (h - 2);
    double te = 0.0;
    for (int half = 0; half < 2; ++half) {
        for (int i = threadIdx.x; i < kMetHalf; i += blockDim.x) hist[i] = 0u;
        __syncthreads();
        for (int64_t i = threadIdx.x; i < interior; i += blockDim.x) {
            const int x = 1 + (int)(i % iw), y = 1 + (int)(i / iw);
            const IN* c = f + (int64_t)y * w + x;
            const int g = qv(c[0]);
            if ((g >> 7) != half) continue;
            int sum = 0;
#pragma unroll
            for (int dy = -1; dy <= 1; ++dy)
#pragma unroll
                for (int dx = -1; dx <= 1; ++dx) sum += qv(c[(int64_t)dy * w + dx]);
            // lround(sum / 9.0): sum / 9 is never a tie, so floor((2 sum + 9) / 18)
            const int gbar = (2 * sum + 9) / 18;
            atomicAdd(&hist[(g & 127) * 256 + gbar], 1u);
        }
        __syncthreads();
        double acc = 0.0;
        const double tot = (double)interior;
        for (int i = threadIdx.x; i < kMetHalf; i += blockDim.x) {
            const uint32_t c = hist[i];
            if (c) {
                const double p = (double)c / tot;
                acc -= p * log2(p);
            }
        }
        te += block_sum(acc, red);  // thread 0: half 0 then half 1
        __syncthreads();
    }
    if (threadIdx.x == 0) a.te[n] = te;
}

template __global__ void k_frame_metrics<uint8_t>(MetArgs);
template __global__ void k_frame_metrics<float>(MetArgs);
template __global__ void k_frame_metrics<double>(MetArgs);

// ------------------------------------------------------------ stability --
// Spikes per pixel (the S1 length is this minus one).
__global__ void k_stab_count(StabArgs a) {
    const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= a.npix) return;
    const uint8_t* col = reinterpret_cast<const uint8_t*>(a.planes) + (p >> 3);
    const int bit = (int)(p & 7);
    uint32_t c = 0;
    for (int64_t n = 0; n < a.frames; ++n) c += (col[n * (int64_t)a.pitch] >> bit) & 1u;
    a.count[p] = c;
}

namespace {

struct StabLevel {
    int64_t off;  // first element in the pixel's region
    int32_t len;
    int32_t lo, hi;
    int32_t state;  // 0: not evaluated, 1: '-' child explored, 2: both explored
};

// interval_stream(seq, firing) (stability.cpp:93-106): gaps between
// successive occurrences of `firing`, written at dst; returns the count
__device__ int32_t gaps_of(const int32_t* seq, int32_t len, int32_t firing, int32_t* dst) {
    int32_t last = -1, m = 0;
    for (int32_t i = 0; i < len; ++i) {
        if (seq[i] != firing) continue;
        if (last >= 0) dst[m++] = i - last;
        last = i;
    }
    return m;
}

}  // namespace

// stability_order per pixel (stability.cpp:61-128), iterative: the reference's
// recursion order, pruning (`violation->depth <= depth` returns before
// anything else, so a pruned '+' child is skipped outright) and report.
__global__ void __launch_bounds__(128) k_stab(StabArgs a) {
    const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= a.nbatch) return;
    const int64_t p = a.pix0 + q;
    int32_t* reg = a.scratch + a.offs[q] - a.offs[0];
    // S1 of the pixel stream (pixel_stream, core.cpp:109-118: firing value 1)
    const uint8_t* col = reinterpret_cast<const uint8_t*>(a.planes) + (p >> 3);
    const int bit = (int)(p & 7);
    int32_t m = 0;
    int64_t last = -1;
    for (int64_t n = 0; n < a.frames; ++n) {
        if (!((col[n * (int64_t)a.pitch] >> bit) & 1u)) continue;
        if (last >= 0) reg[m++] = (int32_t)(n - last);
        last = n;
    }
    StabLevel L[kStabMaxDepth + 2];
    L[1] = StabLevel{0, m, 0, 0, 0};
    int k = 1;
    int vdepth = 0, deepest = 0, trunc = 0;
    int64_t vindex = 0;
    uint64_t path = 0, vpath = 0;  // bit j: branch from depth j+1 to j+2 ('+' = 1)
    const int maxd = a.max_depth;
    while (k >= 1) {
        StabLevel& c = L[k];
        const int32_t* seq = reg + c.off;
        if (c.state == 0) {
            if (vdepth && vdepth <= k) { --k; continue; }
            if (c.len == 0) {
                deepest = max(deepest, k);
                --k;
                continue;
            }
            // first_violation_index (stability.cpp:41-59) and min/max in one pass
            int32_t va = seq[0], vb = 0, lo = seq[0], hi = seq[0];
            bool hb = false;
            int32_t bad = -1;
            for (int32_t i = 1; i < c.len; ++i) {
                const int32_t x = seq[i];
                lo = min(lo, x);
                hi = max(hi, x);
                if (x == va || (hb && x == vb)) continue;
                if (!hb && abs(x - va) == 1) {
                    vb = x;
                    hb = true;
                    continue;
                }
                bad = i;
                break;
            }
            if (bad >= 0) {
                if (!vdepth || k < vdepth) {
                    vdepth = k;
                    vindex = bad;
                    vpath = path;
                }
                --k;
                continue;
            }
            deepest = max(deepest, k);
            if (lo == hi) { --k; continue; }
            if (k >= maxd) {
                trunc = 1;
                --k;
                continue;
            }
            c.lo = lo;
            c.hi = hi;
            c.state = 1;
            const int64_t off = c.off + c.len;
            L[k + 1] = StabLevel{off, gaps_of(seq, c.len, lo, reg + off), 0, 0, 0};
            path &= ~(1ull << (k - 1));
            ++k;
        } else if (c.state == 1) {
            c.state = 2;
            if (vdepth && vdepth <= k + 1) { --k; continue; }  // the '+' child returns at once
            const int64_t off = c.off + c.len;
            L[k + 1] = StabLevel{off, gaps_of(seq, c.len, c.hi, reg + off), 0, 0, 0};
            path |= 1ull << (k - 1);
            ++k;
        } else {
            --k;
        }
    }
    spk_stab_t r;
    r.depth = vdepth;
    r.verified_order = vdepth ? vdepth - 1 : (trunc ? maxd : deepest);
    r.absolute = vdepth ? 0 : !trunc;
    r.path_len = vdepth ? vdepth - 1 : 0;
    r.index = vdepth ? vindex : 0;
    r.path = vdepth > 1 ? vpath & ((1ull << (vdepth - 1)) - 1ull) : 0ull;
    a.out[p] = r;
}

}  // namespace spk
