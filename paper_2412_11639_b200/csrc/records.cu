// records.cu -- SPKR emission: every pixel's segments as
// the paper's 16-bit FPGA records, (duration << 8) | round(intensity), built
// straight from K2's run lists without expanding frames.
//
// Reference: the CLI's --emit-records loop (proj/tools/spikecam_main.cpp:
// 146-172) = per pixel segment_fsr / segment_ssr (reconstruct.cpp:198-211,
// build_segments 107-130) -> encode_events (codec.cpp:8-31) -> write_spkr
// (io.cpp:240-255).  Rounding: lround(255*N/span) equals run_u8 (the uint8
// frame rule); durations above 255 split into full 255-frame words first.
//
// Two passes, one thread per pixel: k_rec_count sizes every pixel's word
// list, an exclusive 64-bit scan places it, k_rec_write writes the file image
// (16-byte header, then per pixel a u32 count and its u16 words, little
// endian) directly in device memory.  Pixels whose run list overflowed K2's
// capacity are rescanned from the planes with the general automaton.
#include "spk_common.cuh"
#include "spk_fsm.cuh"
#include "spk_kernels.cuh"

namespace spk {

namespace {

struct WordCounter {
    uint32_t n = 0;
    __device__ void put(int d, uint32_t) { n += (uint32_t)((d + 254) / 255); }
};

struct WordWriter {
    uint16_t* dst;  // 2-byte aligned (every pixel block starts at an even offset)
    __device__ void put(int d, uint32_t q) {
        while (d > 255) {
            *dst++ = (uint16_t)(0xff00u | q);
            d -= 255;
        }
        *dst++ = (uint16_t)((uint32_t)d << 8 | q);
    }
};

// lead [0, first spike) at 0, one segment per run, tail [last, T) carrying the
// last run's value; no spike -> [0, T) at 0
template <class Sink>
__device__ void from_runs(const spk_run_t* rp, uint32_t n, int last, int frames, Sink& k) {
    if (frames == 0) return;
    if (last < 0) {
        k.put(frames, 0);
        return;
    }
    spk_run_t cur = n ? rp[0] : spk_run_t{(uint32_t)last, 0u};
    if (cur.start > 0) k.put((int)cur.start, 0);
    uint32_t q = 0;
    for (uint32_t i = 0; i < n; ++i) {
        const spk_run_t nx = i + 1 < n ? rp[i + 1] : spk_run_t{(uint32_t)last, 0u};
        const uint32_t span = nx.start - cur.start;
        q = run_u8(cur.intervals, span);
        k.put((int)span, q);
        cur = nx;
    }
    k.put(frames - last, q);
}

// the same segments from the general automaton (overflowed pixels)
template <class Sink>
struct FsmRecords {
    Sink* k;
    uint32_t q;
    __device__ void run(int rs, int cnt, int end, int idx) {
        if (idx == 0 && rs > 0) k->put(rs, 0);
        q = run_u8((uint32_t)cnt, (uint32_t)(end - rs));
        k->put(end - rs, q);
    }
    __device__ void done(int first, int last, int nrun, int frames) {
        if (frames == 0) return;
        if (last < 0) {
            k->put(frames, 0);
            return;
        }
        if (nrun == 0 && first > 0) k->put(first, 0);
        k->put(frames - last, q);
    }
};

template <int METHOD, class Sink>
__device__ void pixel_records(const SegArgs& a, int64_t p, Sink& k) {
    const uint32_t n = a.counts[p];
    if (n <= (uint32_t)a.cap) {
        from_runs(a.runs + p * a.cap, n, a.last[p], a.frames, k);
        return;
    }
    Fsm<METHOD> fsm;
    fsm.init();
    FsmRecords<Sink> em{&k, 0u};
    const uint8_t* col = reinterpret_cast<const uint8_t*>(a.planes) + (p >> 3);
    const int bit = (int)(p & 7);
    for (int f = 0; f < a.frames; ++f)
        if ((col[(size_t)f * a.pitch] >> bit) & 1) fsm.spike(f, em);
    fsm.finish(a.frames, em);
}

}  // namespace

template <int METHOD>
__global__ void __launch_bounds__(128) k_rec_count(RecArgs a) {
    const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= a.seg.npix) return;
    WordCounter c;
    pixel_records<METHOD>(a.seg, p, c);
    a.wc[p] = c.n;
}

template <int METHOD>
__global__ void __launch_bounds__(128) k_rec_write(RecArgs a) {
    const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (p == 0) {  // "SPKR", u16 W, u16 H, u32 fps, u32 frame count
        uint8_t* h = a.img;
        h[0] = 'S'; h[1] = 'P'; h[2] = 'K'; h[3] = 'R';
        h[4] = (uint8_t)a.width; h[5] = (uint8_t)(a.width >> 8);
        h[6] = (uint8_t)a.height; h[7] = (uint8_t)(a.height >> 8);
        for (int i = 0; i < 4; ++i) {
            h[8 + i] = (uint8_t)(a.fps >> (8 * i));
            h[12 + i] = (uint8_t)((uint32_t)a.seg.frames >> (8 * i));
        }
    }
    if (p >= a.seg.npix) return;
    uint16_t* w = reinterpret_cast<uint16_t*>(a.img + 16 + 4 * p + 2 * a.offs[p]);
    const uint32_t n = a.wc[p];
    w[0] = (uint16_t)(n & 0xffffu);
    w[1] = (uint16_t)(n >> 16);
    WordWriter k{w + 2};
    pixel_records<METHOD>(a.seg, p, k);
}

template __global__ void k_rec_count<kFSR>(RecArgs);
template __global__ void k_rec_count<kSSR>(RecArgs);
template __global__ void k_rec_write<kFSR>(RecArgs);
template __global__ void k_rec_write<kSSR>(RecArgs);

}  // namespace spk
