// segment.cu -- K2: FSR / SSR segmentation of every pixel (sm_100a).
//
// Replaces the per-pixel scans of reconstruct_row (proj/src/reconstruct.cpp:
// 358-390) and the column->row gather of reconstruct_into (416-419).
//
// Mapping: one thread per pixel, one warp per 32-bit plane word (32
// consecutive pixels).  For every group of 32 frames lane i loads the warp's
// word from plane (32g + i); a 5-stage shuffle transpose turns the 32x32 bit
// block into one 32-frame word per pixel, and the lane walks its spikes with
// ffs.  Loads are issued one batch (kBatch groups = 256 frames) ahead.
//
// Output per pixel p: runs[p*cap + k] = {start, intervals} for k < cap,
// counts[p], last[p], and the run table tbl[c*npix + p] = index of the run
// covering frame c*kChunk (-1 before the first run).  The expand kernel (K3)
// turns these into frames.  Pixels whose run count exceeds `cap` are
// recomputed by k_fixup (direct column writes) after K3.
#include "spk_fsm.cuh"
#include "spk_kernels.cuh"

namespace spk {

namespace {

struct RunEmitter {
    spk_run_t* runs;  // this pixel's slice
    int32_t* tbl;     // tbl + p
    uint32_t* counts;
    int32_t* lastv;
    int64_t npix;
    int cap;
    int nchunks;
    int64_t p;

    __device__ __forceinline__ void table(int c0, int c1, int v) {
        for (int c = c0; c <= c1; ++c) tbl[(int64_t)c * npix] = v;
    }
    // run [rs, end) with `cnt` intervals, index idx
    __device__ void run(int rs, int cnt, int end, int idx) {
        if (idx < cap) runs[idx] = spk_run_t{(uint32_t)rs, (uint32_t)cnt};
        table((rs + kChunk - 1) >> kChunkLog2, (end - 1) >> kChunkLog2, idx);
    }
    __device__ void done(int first, int last, int nrun, int frames) {
        if (nrun == 0) {
            table(0, nchunks - 1, -1);
        } else {
            table(0, ((first + kChunk - 1) >> kChunkLog2) - 1, -1);  // lead [0, first)
            table((last + kChunk - 1) >> kChunkLog2, nchunks - 1, nrun - 1);  // tail
        }
        counts[p] = (uint32_t)nrun;
        lastv[p] = last;
        (void)frames;
    }
};

}  // namespace

template <int METHOD>
__global__ void __launch_bounds__(kSegThreads) k_segment(SegArgs a) {
    const int lane = threadIdx.x & 31;
    const int64_t word = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (word * 32 >= a.npix) return;  // warp-uniform
    const int64_t p = word * 32 + lane;
    const bool valid = p < a.npix;
    const int frames = a.frames;
    const int ngroups = (frames + 31) >> 5;
    const char* col = reinterpret_cast<const char*>(a.planes) + word * 4;
    const size_t pitch = a.pitch;

    Fsm<METHOD> fsm;
    fsm.init();
    RunEmitter em{a.runs + (valid ? p * a.cap : 0), a.tbl + (valid ? p : 0), a.counts, a.last,
                  a.npix, a.cap, a.nchunks, p};

    uint32_t nxt[kBatch];
#pragma unroll
    for (int j = 0; j < kBatch; ++j) {
        const int f = j * 32 + lane;
        nxt[j] = f < frames ? __ldg(reinterpret_cast<const uint32_t*>(col + (size_t)f * pitch)) : 0u;
    }
    for (int g0 = 0; g0 < ngroups; g0 += kBatch) {
        uint32_t cur[kBatch];
#pragma unroll
        for (int j = 0; j < kBatch; ++j) cur[j] = nxt[j];
        if (g0 + kBatch < ngroups) {
#pragma unroll
            for (int j = 0; j < kBatch; ++j) {
                const int f = (g0 + kBatch + j) * 32 + lane;
                nxt[j] = f < frames
                             ? __ldg(reinterpret_cast<const uint32_t*>(col + (size_t)f * pitch))
                             : 0u;
            }
        }
#pragma unroll
        for (int j = 0; j < kBatch; ++j) {
            if (g0 + j < ngroups) {
                uint32_t w = transpose32(cur[j], lane);
                if (!valid) w = 0;
                const int base = (g0 + j) * 32;
                while (w) {
                    const int b = __ffs(w) - 1;
                    w &= w - 1;
                    fsm.spike(base + b, em);
                }
            }
        }
    }
    if (valid) fsm.finish(frames, em);
}

template __global__ void k_segment<kFSR>(SegArgs);
template __global__ void k_segment<kSSR>(SegArgs);

// ---------------------------------------------------------------- fixup ----
// Pixels whose run list overflowed `cap`: rescan the pixel and write its
// frames directly (one byte/element per frame, column order).  Slow, exact,
// and only taken for pathological (e.g. pure-noise) pixels.
namespace {

template <typename OUT>
struct DirectEmitter {
    OUT* out;  // out + p
    size_t pitch;
    OUT carry;
    __device__ void fill(int a, int b, OUT v) {
        for (int n = a; n < b; ++n) out[(size_t)n * pitch] = v;
    }
    __device__ void run(int rs, int cnt, int end, int) {
        carry = OutVal<OUT>::run((uint32_t)cnt, (uint32_t)(end - rs));
        fill(rs, end, carry);
    }
    __device__ void done(int first, int last, int nrun, int frames) {
        if (nrun == 0) {
            fill(0, frames, OUT(0));
        } else {
            fill(0, first, OUT(0));
            fill(last, frames, carry);
        }
    }
};

}  // namespace

template <int METHOD, typename OUT>
__global__ void __launch_bounds__(128) k_fixup(SegArgs a, OUT* out, size_t out_pitch) {
    const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= a.npix) return;
    if (a.counts[p] <= (uint32_t)a.cap) return;
    Fsm<METHOD> fsm;
    fsm.init();
    DirectEmitter<OUT> em{out + p, out_pitch, OUT(0)};
    const uint8_t* col = reinterpret_cast<const uint8_t*>(a.planes) + (p >> 3);
    const int bit = (int)(p & 7);
    for (int n = 0; n < a.frames; ++n)
        if ((col[(size_t)n * a.pitch] >> bit) & 1) fsm.spike(n, em);
    fsm.finish(a.frames, em);
}

template __global__ void k_fixup<kFSR, uint8_t>(SegArgs, uint8_t*, size_t);
template __global__ void k_fixup<kSSR, uint8_t>(SegArgs, uint8_t*, size_t);
template __global__ void k_fixup<kFSR, float>(SegArgs, float*, size_t);
template __global__ void k_fixup<kSSR, float>(SegArgs, float*, size_t);
template __global__ void k_fixup<kFSR, double>(SegArgs, double*, size_t);
template __global__ void k_fixup<kSSR, double>(SegArgs, double*, size_t);

}  // namespace spk
