// spk_kernels.cuh -- kernel argument blocks and declarations shared by the
// kernel translation units and the C-ABI layer (capi.cu).
#pragma once

#include <cstddef>
#include <cstdint>

#include "spikecam_b200.h"

namespace spk {

using spk_run_t = ::spk_run;

constexpr int kSegThreads = 64;  // 2 warps: fine-grained blocks balance 148 SMs
constexpr int kBatch = 8;        // 32-frame groups per prefetch batch
constexpr int kExpThreads = 128;
constexpr int kFinThreads = 128;
constexpr int kCausalWarps = 2;  // warps per TFI/TFP block

struct SegArgs {
    const void* planes;
    size_t pitch;  // bytes between planes
    int64_t npix;
    int frames;
    int cap;  // runs per pixel in `runs`
    int nchunks;
    spk_run_t* runs;
    int32_t* tbl;
    uint32_t* counts;
    int32_t* last;
};

// K2b: run values + run table from the run lists
struct FinArgs {
    spk_run_t* runs;  // in: {start, intervals}; out (u8/f32): {start, value bits}
    double* vals;     // out (f64): value per run, same indexing as runs
    int32_t* tbl;     // out: [nchunks][npix] run covering frame c*kChunk, -1 = none
    const uint32_t* counts;
    const int32_t* last;
    int64_t npix;
    int frames;
    int cap;
    int nchunks;
};

struct ExpArgs {
    const double* vals;
    const spk_run_t* runs;
    const int32_t* tbl;
    const uint32_t* counts;
    const int32_t* last;
    int64_t npix;
    int frames;
    int cap;
    int chunk0;  // first chunk of this launch (blockIdx.y offset)
    void* out;
    size_t pitch;  // elements between frames
    int vec_ok;    // out base / pitch allow 16-B vector stores
};

struct CausalArgs {
    const void* planes;
    size_t pitch;
    int64_t npix;
    int frames;
    int window;  // TFP window
    void* out;
    size_t out_pitch;  // elements
    int lut_n;         // entries in the shared-memory value table
};

template <int METHOD>
__global__ void k_segment(SegArgs a);
template <int METHOD, typename OUT>
__global__ void k_fixup(SegArgs a, OUT* out, size_t out_pitch);
template <typename OUT>
__global__ void k_finalize(FinArgs a);
template <typename OUT>
__global__ void k_expand(ExpArgs a);
size_t expand_smem_bytes(int out_size);   // dynamic shared memory of k_expand<OUT>
int expand_pixels_per_lane(int out_size);
int expand_threads(int out_size);
template <int METHOD, typename OUT>
__global__ void k_causal(CausalArgs a);

__global__ void k_pack(const uint8_t* bytes, int64_t npix, int64_t frames, uint8_t* planes,
                       size_t pitch);
__global__ void k_unpack(const uint8_t* planes, size_t pitch, int64_t npix, int64_t frames,
                         uint8_t* bytes);
__global__ void k_bitrev_bytes(uint8_t* planes, size_t pitch, size_t row_bytes, int64_t frames);
__global__ void k_synth(int scene, uint64_t seed, int width, int height, int64_t frames,
                        int64_t frame0, double param, uint8_t* planes, size_t pitch);

}  // namespace spk
