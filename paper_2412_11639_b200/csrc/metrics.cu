// metrics.cu -- quality metrics and the stability check on the device
// (SURVEY.md 8(f) row 4).
//
// K_te/mse  one block per frame: two_dimensional_entropy (proj/src/metrics.cpp:
//           12-43) and mse against a reference image (45-55).  The
//           256x256 (gray, rounded 3x3 mean) histogram is built in 128 KB of
//           shared memory: at once with 16-bit counts when the frame has
//           fewer than 65,536 interior pixels, else in two halves of 128 gray
//           levels with 32-bit counts (a 1000x1000 frame has ~1M); the
//           -p*log2(p) terms are reduced in a fixed order, so the result is
//           deterministic (equal to the reference's sequential sum up to
//           double rounding).
// K_stab    one thread per pixel: stability_order (proj/src/stability.cpp:
//           61-128) -- the depth-first tree of interval streams, '-' first,
//           with the reference's pruning.  Only stable sequences (two values
//           differing by one) are explored further, so each level of the
//           pixel's depth-first stack is kept as one bit per element in a
//           per-pixel global scratch region; a child is never longer than
//           its parent, so depth * ceil(|S1| / 32) words always suffice.
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
    if (interior < 65536) {
        // every bin fits 16 bits: the whole 256x256 histogram at once, two
        // bins per 32-bit word
        for (int i = threadIdx.x; i < kMetHalf; i += blockDim.x) hist[i] = 0u;
        __syncthreads();
        for (int64_t i = threadIdx.x; i < interior; i += blockDim.x) {
            const int x = 1 + (int)(i % iw), y = 1 + (int)(i / iw);
            const IN* c = f + (int64_t)y * w + x;
            int sum = 0;
#pragma unroll
            for (int dy = -1; dy <= 1; ++dy)
#pragma unroll
                for (int dx = -1; dx <= 1; ++dx) sum += qv(c[(int64_t)dy * w + dx]);
            const int bin = qv(c[0]) * 256 + (2 * sum + 9) / 18;  // lround(sum / 9.0), no ties
            atomicAdd(&hist[bin >> 1], 1u << ((bin & 1) * 16));
        }
        __syncthreads();
        double acc = 0.0;
        const double tot = (double)interior;
        for (int i = threadIdx.x; i < kMetHalf; i += blockDim.x) {
            const uint32_t c2 = hist[i];
            if (c2) {
#pragma unroll
                for (int k = 0; k < 2; ++k) {
                    const uint32_t c = (c2 >> (16 * k)) & 0xffffu;
                    if (c) {
                        const double p = (double)c / tot;
                        acc -= p * log2(p);
                    }
                }
            }
        }
        te = block_sum(acc, red);
        if (threadIdx.x == 0) a.te[n] = te;
        return;
    }
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

// A stable sequence (stability.cpp:41-59: at most two values, differing by
// one) is stored as one bit per element: value = lo + (raw ^ flip), raw bit e
// at bit (e & 31) of word e >> 5.  Only stable sequences are ever explored
// further, so every level of the depth-first stack fits in |S1| bits.
struct StabLevel {
    int64_t off;  // first word in the pixel's region
    int32_t len;
    int32_t lo, hi;
    uint32_t flip;   // 0xffffffff when raw bit 1 stands for lo
    int32_t state;   // 0: not evaluated, 1: '-' child explored, 2: both explored
    int32_t bad;     // first_violation_index of the level (-1: stable)
};

// Appends the values of a sequence one by one, applying first_violation_index
// (a = first value, b = the first +-1 neighbour) and min/max, and writing the
// raw bits (value != a) to `dst` -- stops at the first violation.
struct SeqBuilder {
    uint32_t* dst;
    int32_t m = 0, a = 0, b = 0, lo = 0, hi = 0, bad = -1;
    bool hb = false;
    uint32_t acc = 0;
    __device__ bool push(int32_t v) {  // false once a violation was found
        uint32_t raw = 0;
        if (m == 0) {
            a = lo = hi = v;
        } else if (v == a) {
        } else if (hb && v == b) {
            raw = 1;
        } else if (!hb && abs(v - a) == 1) {
            b = v;
            hb = true;
            raw = 1;
            lo = min(lo, v);
            hi = max(hi, v);
        } else {
            bad = m;
            return false;
        }
        acc |= raw << (m & 31);
        if ((m & 31) == 31) {
            dst[m >> 5] = acc;
            acc = 0;
        }
        ++m;
        return true;
    }
    __device__ void finish(StabLevel& L) {
        if (bad < 0 && (m & 31)) dst[m >> 5] = acc;
        L.len = m;
        L.lo = lo;
        L.hi = hi;
        L.flip = hb && b < a ? 0xffffffffu : 0u;
        L.bad = bad;
        L.state = 0;
    }
};

// interval_stream(seq, firing) (stability.cpp:93-106) of a stored stable
// sequence: the gaps between successive elements equal to `firing` (hi_bit:
// the larger value), written as the next level
__device__ void child_of(const uint32_t* reg, const StabLevel& P, bool hi_bit, StabLevel& C) {
    SeqBuilder sb;
    sb.dst = const_cast<uint32_t*>(reg) + C.off;
    int32_t last = -1;
    const int32_t nw = (P.len + 31) >> 5;
    for (int32_t wi = 0; wi < nw; ++wi) {
        uint32_t w = reg[P.off + wi] ^ P.flip;  // bit 1 = the larger value
        if (!hi_bit) w = ~w;
        if (wi == nw - 1 && (P.len & 31)) w &= (1u << (P.len & 31)) - 1u;
        while (w) {
            const int32_t pos = wi * 32 + __ffs(w) - 1;
            w &= w - 1;
            if (last >= 0 && !sb.push(pos - last)) {
                sb.finish(C);
                return;
            }
            last = pos;
        }
    }
    sb.finish(C);
}

}  // namespace

// stability_order per pixel (stability.cpp:61-128), iterative: the reference's
// recursion order, pruning (`violation->depth <= depth` returns before
// anything else, so a pruned '+' child is skipped outright) and report.
__global__ void __launch_bounds__(128) k_stab(StabArgs a) {
    const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= a.nbatch) return;
    const int64_t p = a.pix0 + q;
    uint32_t* reg = reinterpret_cast<uint32_t*>(a.scratch) + (a.offs[q] - a.offs[0]);
    StabLevel L[kStabMaxDepth + 2];
    // level 1: S1 of the pixel stream (pixel_stream, core.cpp:109-118: firing value 1)
    {
        const uint8_t* col = reinterpret_cast<const uint8_t*>(a.planes) + (p >> 3);
        const int bit = (int)(p & 7);
        SeqBuilder sb;
        sb.dst = reg;
        int64_t last = -1;
        for (int64_t n = 0; n < a.frames; ++n) {
            if (!((col[n * (int64_t)a.pitch] >> bit) & 1u)) continue;
            if (last >= 0 && !sb.push((int32_t)(n - last))) break;
            last = n;
        }
        L[1].off = 0;
        sb.finish(L[1]);
    }
    int k = 1;
    int vdepth = 0, deepest = 0, trunc = 0;
    int64_t vindex = 0;
    uint64_t path = 0, vpath = 0;  // bit j: branch from depth j+1 to j+2 ('+' = 1)
    const int maxd = a.max_depth;
    while (k >= 1) {
        StabLevel& c = L[k];
        if (c.state == 0) {
            if (vdepth && vdepth <= k) { --k; continue; }
            if (c.len == 0 && c.bad < 0) {
                deepest = max(deepest, k);
                --k;
                continue;
            }
            if (c.bad >= 0) {
                if (!vdepth || k < vdepth) {
                    vdepth = k;
                    vindex = c.bad;
                    vpath = path;
                }
                --k;
                continue;
            }
            deepest = max(deepest, k);
            if (c.lo == c.hi) { --k; continue; }
            if (k >= maxd) {
                trunc = 1;
                --k;
                continue;
            }
            c.state = 1;
            L[k + 1].off = c.off + ((c.len + 31) >> 5);
            child_of(reg, c, false, L[k + 1]);  // '-': the smaller firing value
            path &= ~(1ull << (k - 1));
            ++k;
        } else if (c.state == 1) {
            c.state = 2;
            if (vdepth && vdepth <= k + 1) { --k; continue; }  // the '+' child returns at once
            L[k + 1].off = c.off + ((c.len + 31) >> 5);
            child_of(reg, c, true, L[k + 1]);
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
