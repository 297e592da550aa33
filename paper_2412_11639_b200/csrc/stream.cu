// stream.cu -- the streaming form of FSR (PixelReconState, reconstruct.cpp:
// 230-290, reconstruct.hpp:46-67) for every pixel at once: frames arrive in
// blocks, each block is scanned with the automaton state carried from the
// previous one (K2 with an entry state), and the segments that close in the
// block come out as SegmentEvents (duration, intensity) -- the same sequence
// PixelReconState yields frame by frame (and fsr_events yields in batch):
//   * the degenerate lead [0, first spike) with intensity 0, when the first
//     spike arrives;
//   * every run, when the interval that breaks it arrives (duration = its
//     span, intensity = 255*N/span);
//   * at flush: the open run, then the tail [last spike, frames) carrying the
//     last intensity -- or, with no spike at all, one segment of all frames.
// Events of a push are grouped by pixel (exclusive prefix of per-pixel counts).
#include "spk_common.cuh"
#include "spk_fsm.cuh"
#include "spk_kernels.cuh"

namespace spk {

namespace {

// per pixel: the events of this block, counted (dst == nullptr) or written
struct EvSink {
    spk_event_t* dst;
    uint32_t n;
    __device__ void put(int64_t d, double v) {
        if (dst) dst[n] = spk_event_t{d, v};
        ++n;
    }
};

__device__ void block_events(const StreamArgs& a, int64_t p, EvSink& k) {
    Scan<kFSR> Ein, Eout;
    Ein.restore(a.state_in, a.npix, p);
    Eout.restore(a.state_out, a.npix, p);
    // lead: the stream's first spike arrived in this block
    if ((Ein.last == kNoSpike) & (Eout.last != kNoSpike)) {
        const uint32_t n = a.counts[p];
        const int first = n ? (int)a.runs[p * a.cap].start : Eout.last;  // the first run starts there
        const int64_t f = a.frame0 + first;
        if (f > 0) k.put(f, 0.0);
    }
    // closed runs: every listed run but the last, which is the one still open
    // (K2 lists the open run last); run k ends where run k+1 starts
    const int n = (int)min(a.counts[p], (uint32_t)a.cap);
    const int closed = Eout.lo < kLim ? n - 1 : n;
    for (int i = 0; i < closed; ++i) {
        const spk_run_t r = a.runs[p * a.cap + i];
        const int end = (int)a.runs[p * a.cap + i + 1].start;
        const int span = end - (int)r.start;
        const double v = run_f64(r.intervals, (uint32_t)span);
        k.put(span, v);
        if (k.dst) a.last_value[p] = v;
    }
}

}  // namespace

// K2 of a block leaves the run lists; count each pixel's events
__global__ void __launch_bounds__(128) k_stream_count(StreamArgs a) {
    const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= a.npix) return;
    EvSink k{nullptr, 0u};
    if (a.flush) {
        Scan<kFSR> X;
        X.restore(a.state_in, a.npix, p);
        if (a.frame0 > 0) k.n = X.last == kNoSpike ? 1u : (X.lo < kLim ? 2u : 1u);
    } else {
        block_events(a, p, k);
    }
    a.ecount[p] = k.n;
}

// write the events at the scanned offsets; keep each pixel's last intensity
__global__ void __launch_bounds__(128) k_stream_write(StreamArgs a) {
    const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= a.npix) return;
    EvSink k{a.events + a.eoffs[p], 0u};
    if (a.flush) {
        // a.frame0 = frames pushed so far; the state is relative to that frame
        Scan<kFSR> X;
        X.restore(a.state_in, a.npix, p);
        if (a.frame0 == 0) return;
        if (X.last == kNoSpike) {
            k.put(a.frame0, 0.0);
            return;
        }
        double carry = a.last_value[p];
        if (X.lo < kLim) {  // the open run: from its start to the last spike
            const int span = X.last - X.rs;
            carry = run_f64((uint32_t)X.cnt, (uint32_t)span);
            k.put(span, carry);
        }
        k.put(-(int64_t)X.last, carry);  // tail: frames after the last spike (X.last <= 0)
        return;
    }
    block_events(a, p, k);
}

__global__ void __launch_bounds__(256) k_max_u32(const uint32_t* v, int64_t n, uint32_t* out) {
    uint32_t m = 0u;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        m = max(m, v[i]);
    m = __reduce_max_sync(kFull, m);
    if ((threadIdx.x & 31) == 0) atomicMax(out, m);
}

// carry the end state into the next block's frames
__global__ void __launch_bounds__(256) k_stream_shift(int32_t* st, int64_t npix, int frames) {
    const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= npix) return;
    Scan<kFSR> X;
    X.restore(st, npix, p);
    if (X.last != kNoSpike) X.last -= frames;
    if (X.lo < kLim) X.rs -= frames;
    X.nrun = 0;
    X.save(st, npix, p);
}

}  // namespace spk
