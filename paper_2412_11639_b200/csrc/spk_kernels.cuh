// spk_kernels.cuh -- kernel argument blocks and declarations shared by the
// kernel translation units and the C-ABI layer (capi.cu).
#pragma once

#include <cstddef>
#include <cstdint>

#include <cuda.h>

#include "spikecam_b200.h"

namespace spk {

using spk_run_t = ::spk_run;
using spk_sync_t = ::spk_sync;
using spk_close_t = ::spk_close;
using spk_event_t = ::spk_event;
using spk_stab_t = ::spk_stab;

// K2 block = 8 warps = 256 pixels = one 32-byte sector of every plane row;
// the warps share each sector through L2, so they are kept within a drift
// bound (kDriftFsr / kDriftSsr groups) of each other (otherwise every 4-byte load pulls its own sector from
// DRAM on long streams)
#ifndef SPK_SEG_THREADS
#define SPK_SEG_THREADS 256
#endif
constexpr int kSegThreads = SPK_SEG_THREADS;
constexpr int kSegWarps = kSegThreads / 32;
// FSR on sensors that fit one wave: 11-warp blocks, two per SM.  400x250 is
// 3,125 warps on 148 SMs: 8-warp blocks put 24 warps on 95 SMs and 16 on the
// rest, 11-warp blocks at most 22 on every SM (C2 K2 0.83 -> 0.80 ms; SSR and
// many-wave sensors are slower with them: the blocks straddle 32-byte sectors).
constexpr int kSegWarpsWide = 11;
// max groups a warp may produce ahead of its block's slowest warp, per
// method (measured: FSR 48 vs 96 -- C5 K2 -3%, C3 -2%; 40, the smallest
// bound a warp cannot wait on itself with, vs 48 -- range-200k K2 1.82 ->
// 1.76 ms, C1 0.202 -> 0.200; SSR 160 vs 96 -- C3 SSR K2 -1%)
constexpr int kDriftFsr = 40;
#ifndef SPK_DRIFT_SSR
#define SPK_DRIFT_SSR 160
#endif
constexpr int kDriftSsr = SPK_DRIFT_SSR;
constexpr int kBatch = 8;        // 32-frame groups per prefetch batch
constexpr int kSsrSlotBytes = 2 * 32 * 16;  // SSR: per warp, [parity][lane] 16-byte slot records (shared memory)
constexpr int kSsrProbe = 64;    // SSR: words scanned in bulk mode before choosing the mode
#ifndef SPK_SSR_CB
#define SPK_SSR_CB 250
#endif
constexpr int kSsrBulkCost = SPK_SSR_CB;  // SSR mode choice: instructions per bulk pass (word or event) ...
constexpr int kSsrStepCost = 63;          // ... per spike-loop step ...
constexpr int kSsrWordCost = 15;          // ... and per spike-loop word
// transposed words buffered per lane (bounds lane drift); 32 keeps the rings
// at 32 KB per block, which leaves L1 room for the plane sectors the block's
// warps share (64: C3 K2 4.01 vs 3.82 ms)
constexpr int kRing = 32;
// A warp's own front is at most kRing + kBatch groups past its published
// lowest group, so a smaller bound would make it wait on itself (measured:
// a bound of 16 hangs).
static_assert(kDriftFsr >= kRing + kBatch && kDriftSsr >= kRing + kBatch,
              "the drift bound must exceed a warp's own ring span");
constexpr int kCausalWarps = 2;  // warps per TFI/TFP block

struct SegArgs {
    const void* planes;
    size_t pitch;  // bytes between planes
    int64_t npix;
    int frames;
    int cap;  // runs per pixel in `runs`
    int nchunks;
    spk_run_t* runs;
    uint32_t* counts;
    int32_t* last;
    int dense_runs = 0;  // host hint for K3: many runs per pixel expected (SSR lists)
    const int32_t* state_in = nullptr;  // time shards: automaton state at frame 0
    int32_t* state_out = nullptr;       //              state after the last frame
    // Several time shards in one launch (blockIdx.y = shard r, fresh state):
    // shard r covers frames [r*shard_frames, min(frames, (r+1)*shard_frames))
    // and writes its own runs / counts / last / state_out block (counts,
    // last: + r*npix; state_out: + r*17*npix).  shard_frames = 0: one shard.
    int shard_frames = 0;
    // run list placement: pixel p, shard r -> runs + r*run_shard_stride +
    // p*run_pix_stride + run_base (run_pix_stride 0: `cap`; run_shard_stride
    // -1: npix*cap); abs_frames: run starts in stream frames, not shard frames
    int64_t run_pix_stride = 0;
    int64_t run_shard_stride = -1;
    int run_base = 0;
    int abs_frames = 0;
    // re-scan of selected pixels (in-grid time split fallback): only lanes
    // with flags[p] != 0 store; warps without one exit.  seg_out: their
    // segment table becomes one segment [0, count) (nseg entries of 2 x u32)
    const uint8_t* flags = nullptr;
    uint32_t* seg_out = nullptr;
    int nseg = 0;
    // expand stage input in split form: the pixel's runs are the segments
    // seg_in[p*nseg + r] = {begin, end} of its row (runs + p*cap)
    const uint32_t* seg_in = nullptr;
};

// In-grid time split of one stream (capi.cu reconstruct_impl): shard r's
// speculative runs start kSplitGap slots into its region of the pixel's row
// (room for the resolved prefix runs placed in front of the synced run).
constexpr int kSplitGap = 64;
constexpr int kSplitMinFrames = 4096;    // shortest shard worth its resolve
constexpr int kSplitMinStream = 65536;  // shortest stream split by default
constexpr int kSplitMaxShards = 32;  // a pixel's segment table fits one warp

// ---- time shards (shard.cu): exact stitching of independently scanned
// frame ranges, see DESIGN.md "Time sharding".
struct ShardArgs {
    const void* planes;  // this shard's planes (frame 0 = shard start)
    size_t pitch;
    int64_t npix;
    int frames;                 // shard length
    const int32_t* entry;       // true automaton state at the shard start
    spk_run_t* prefix;          // true runs closed before the sync point
    int pcap;
    spk_sync_t* sync;
    int32_t* tstate;            // true end state when the scan ran through the shard
    // junction / stitch
    const spk_run_t* spec;      // speculative run list (fresh at the shard start)
    int scap;
    const uint32_t* scount;
    const int32_t* sstate;      // speculative end state
    const spk_run_t* fb;        // fallback: full re-scan from `entry` (or null)
    const uint32_t* fbcount;
    const int32_t* fbstate;
    int32_t* exit_state;        // true end state, frames relative to the next shard
    spk_close_t* entry_close;   // does the run open at the shard start close here?
    spk_close_t* tail_close;    // the run open at the end, closed at the stream end
    const spk_close_t* close;   // close of the run open at the end (from the right)
    spk_run_t* region;          // stitched true runs intersecting the shard
    int rcap;
    uint32_t* rcount;
    int32_t* rlast;             // end of the last region run (may lie past the shard)
    // In-grid time split (grid_sf > 0): one launch resolves shards 1..S-1
    // (blockIdx.y + 1) of a stream cut in grid_sf-frame shards; `planes`,
    // `frames` describe the whole stream; per shard r: entry = the
    // speculative end state of shard r-1 (sstate + (r-1)*17*npix, shifted to
    // shard r's frames), spec runs in the pixel rows (row = S*rstride
    // elements, shard r at r*rstride + kSplitGap, stream frames), scount /
    // sync / (prefix: npix*pcap) / tstate blocks + r*npix (*17 for states).
    int grid_sf = 0;
    int nshards = 0;
    int64_t rstride = 0;
    int total_frames = 0;
    int32_t* syncj = nullptr;  // index of the synced speculative run (-1: none)
};

// In-grid time split: the true run list per pixel is a sequence of segments
// of its row, one per shard (seg[p*S + r] = {begin, end}); the combine pass
// (k_split_combine) writes them, flags pixels whose shards need a full
// re-scan, and sets counts / last for the whole stream.
struct SplitArgs {
    int64_t npix;
    int nshards;
    int sf;                 // shard length (the last shard may be shorter)
    int frames;             // stream length
    int64_t rstride;        // row elements per shard region
    int scap;               // speculative capacity per shard (region - kSplitGap)
    int pcap;
    spk_run_t* runs;        // rows (npix x S*rstride)
    const uint32_t* scount; // [S][npix]
    const int32_t* sstate;  // [S][17][npix]
    const spk_run_t* prefix;  // [S][npix][pcap]
    const spk_sync_t* sync;   // [S][npix]
    const int32_t* syncj;     // [S][npix]
    const int32_t* tstate;    // [S][17][npix]
    uint32_t* seg;          // [npix][S] x {begin, end}
    uint32_t* counts;       // total true runs (or cap + 1: overflow -> k_fixup)
    int32_t* last;          // last spike (stream frames, -1: none)
    uint8_t* flags;         // 1: re-scan the whole stream (k_segment with flags)
    uint32_t* nflag;        // number of flagged pixels (one counter)
    int method;
};

// Geometry of the expand stage per output type: a warp owns a group of
// GP = 32*P consecutive pixels (P per lane) and walks one kChunk-frame chunk
// in sub-tiles of kSub frames (kBins sub-tiles per chunk).
#ifndef SPK_SUB
#define SPK_SUB 16
#endif
constexpr int kSub = SPK_SUB;
constexpr int kBins = kChunk / kSub;
constexpr int kPieceSubs = 64 / kSub;        // K3 tile height: 64 frames
constexpr int kPieces = kBins / kPieceSubs;  // K3 tiles per (group, chunk)
#ifndef SPK_PIECE_SPARSE  // (build-time overrides: A/B probes)
#define SPK_PIECE_SPARSE 2
#endif
constexpr int kPieceSparse = SPK_PIECE_SPARSE;  // changes per pixel per chunk up to which
                                             // K3 tiles are 64 frames high (else 128)
#ifndef SPK_PIECE_DENSITY
#define SPK_PIECE_DENSITY 12
#endif
constexpr int kPieceDensity = SPK_PIECE_DENSITY;            // ... up to which 128 frames high (else 256)
constexpr int kPieceDense = 48;              // ... above which K3 writes the chunk whole
#ifndef SPK_PIECE_MAXG
#define SPK_PIECE_MAXG 512
#endif
constexpr int kPieceMaxGroups = SPK_PIECE_MAXG;
constexpr int kWideGroups = 1024;  // K3: 8-warp blocks from this many groups per frame  // pieces only for narrow frames (few groups
                                             // per row: wide rows already keep the
                                             // concurrently written rows close)
template <typename OUT>
struct Geo;
template <>
struct Geo<uint8_t> {
    static constexpr int P = 16, WARPS = 4;  // (8 for wide sensors: k_expand<uint8_t, 8>)
};
template <>
struct Geo<float> {
    static constexpr int P = 8, WARPS = 2;
};
template <>
struct Geo<double> {
    static constexpr int P = 8, WARPS = 1;
};

// One value change of the frame-sorted change stream: frame offset in the
// chunk (fo), pixel in the group (pix) and the new value.
template <typename OUT>
struct Change;
template <>
struct Change<uint8_t> {  // (fo << 17) | (pix << 8) | value
    uint32_t w;
};
template <>
struct Change<float> {
    uint32_t key;  // (fo << 16) | pix
    uint32_t bits;
};
template <>
struct __align__(16) Change<double> {
    uint32_t key;
    uint32_t pad;
    double v;
};

// K2c: run lists -> value at every chunk start and the change stream sorted
// by (chunk, group, sub-tile)
struct FinArgs {
    const spk_run_t* runs;  // {start, intervals} per pixel (K2 output)
    const uint32_t* counts;
    const int32_t* last;
    int64_t npix;
    int frames;
    int cap;
    int nchunks;
    int ngroups;
    uint32_t* bins;        // [nchunks][ngroups][kBins] run starts per sub-tile (K2b)
    void* tblv;            // [nchunks][npix] OUT: value at frame c*kChunk (K2c)
    const uint32_t* offs;  // exclusive prefix of bins
    uint32_t* cursor;      // K2c: running copy of offs (claimed with atomics)
    void* stream;          // Change<OUT>[total] (K2c)
    int64_t stream_len = 0;  // its entries (checked build)
    // in-grid time split: runs of pixel p are the segments seg[p*nseg + r] =
    // {begin, end} of its row (runs + p*row); cap = row length.  null: one
    // contiguous list of min(counts[p], cap) runs.
    const uint32_t* seg = nullptr;
    int nseg = 0;
    int fin_seg = 64;  // K2c: runs per thread (fin_seg_for)
};
// K2c: runs per thread (a pixel's list spans cap / seg threads; even).  Few
// pixels want more threads in flight, many pixels fewer empty threads
// (measured, finalize: C2 400x250 0.350 -> 0.344 ms at 32; C3 1000x1000 1.04
// -> 0.96 ms at 128).
#ifdef SPK_FIN_SEG
inline int fin_seg_for(int64_t) { return SPK_FIN_SEG; }
#else
inline int fin_seg_for(int64_t npix) { return npix <= (1 << 18) ? 32 : npix < (3 << 18) ? 64 : 128; }
#endif
constexpr int kFinWarps = 16;     // K2b/K2c: warps per block (block = one pixel group)
constexpr int kFinWindow = 128;   // chunks per shared-memory window (32 KB of counters)

struct ExpArgs {
    const void* tblv;
    const uint32_t* bins;
    const uint32_t* offs;
    const void* stream;
    int64_t stream_len = 0;  // entries of `stream` (checked build)
    int64_t npix;
    int frames;
    int nchunks;
    int ngroups;
    int chunk0;  // first chunk of this launch (blockIdx.y offset)
    int pieces;  // tiles per (group, chunk): kPieces, or 1 (whole chunks)
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

// SPKR emission from K2's run lists (records.cu)
struct RecArgs {
    SegArgs seg;                  // runs / counts / last (+ planes for overflowed pixels)
    uint32_t* wc;                 // words per pixel (k_rec_count)
    const unsigned long long* offs;  // exclusive prefix of wc (k_rec_write)
    uint8_t* img;                 // SPKR file image (k_rec_write)
    int width, height;
    uint32_t fps;
};

// streaming FSR (stream.cu)
struct StreamArgs {
    int64_t npix;
    int64_t frame0;           // absolute frame of the block start (flush: frames pushed)
    int flush;
    const int32_t* state_in;  // state before the block (flush: the final state)
    const int32_t* state_out; // state after the block
    const spk_run_t* runs;    // the block's run lists (K2 with state_in)
    int cap;
    const uint32_t* counts;
    uint32_t* ecount;                 // events per pixel
    const unsigned long long* eoffs;  // exclusive prefix of ecount
    spk_event_t* events;
    double* last_value;       // per pixel: intensity of the last closed run
};
__global__ void k_stream_count(StreamArgs a);
__global__ void k_stream_write(StreamArgs a);
__global__ void k_stream_shift(int32_t* st, int64_t npix, int frames);
__global__ void k_max_u32(const uint32_t* v, int64_t n, uint32_t* out);

template <int METHOD, int WARPS = kSegWarps>
__global__ void k_segment(SegArgs a);
template <int METHOD>
__global__ void k_resolve(ShardArgs a);
template <int METHOD>
__global__ void k_junction(ShardArgs a);
template <int METHOD>
__global__ void k_split_combine(SplitArgs a);
__global__ void k_state_fresh(int32_t* st, int64_t npix);
__global__ void k_close_chain(const spk_close_t* entry_next, const spk_close_t* close_next,
                              int shard_len, int64_t npix, spk_close_t* close);
template <int METHOD>
__global__ void k_stitch(ShardArgs a);
template <int METHOD>
__global__ void k_rec_count(RecArgs a);
template <int METHOD>
__global__ void k_rec_write(RecArgs a);
template <int METHOD, typename OUT>
__global__ void k_fixup(SegArgs a, OUT* out, size_t out_pitch);
template <int GP, bool SPLIT>
__global__ void k_fin_bins(FinArgs a);
template <typename OUT, bool SPLIT>
__global__ void k_fin_scatter(FinArgs a);
template <typename OUT, int WARPS, bool TMA>
__global__ void k_expand(ExpArgs a, const __grid_constant__ CUtensorMap tmap);
size_t expand_smem_bytes(int out_size, int warps, bool tma);  // dynamic shared memory of k_expand
// exclusive scan of uint32 counts into T (uint32_t, or unsigned long long
// where totals may pass 2^32)
template <typename T>
__global__ void k_scan_blocks(const uint32_t* in, T* out, T* sums, int64_t n);
template <typename T>
__global__ void k_scan_sums(T* sums, int64_t nb);
template <typename T>
__global__ void k_scan_add(T* out, const T* sums, int64_t n, T* out2);
constexpr int kScanBlock = 1024;
template <int METHOD, typename OUT>
__global__ void k_causal(CausalArgs a);

// quality metrics / stability check (metrics.cu)
constexpr int kMetThreads = 512;
constexpr int kMetHalf = 128 * 256;  // histogram bins of one half (128 gray levels)
constexpr int kStabMaxDepth = 63;    // violation paths are 64-bit masks
struct MetArgs {
    const void* frames;  // [frames][pitch] elements
    int64_t pitch;
    const void* ref;     // [frames][ref_pitch] reference images (mse)
    int64_t ref_pitch;
    int ref_type;        // SPK_OUT_U8 / F32 / F64
    int width, height;
    double* te;   // per frame, or null
    double* mse;  // per frame, or null (then `ref` is unused)
};
struct StabArgs {
    const void* planes;
    size_t pitch;
    int64_t npix;
    int64_t frames;
    int max_depth;
    uint32_t* count;        // k_stab_count: spikes per pixel
    int64_t pix0, nbatch;   // k_stab: pixels [pix0, pix0 + nbatch)
    const int64_t* offs;    // per batch pixel: region start (ints, exclusive prefix)
    int32_t* scratch;       // the batch's regions (starting at offs[0])
    spk_stab_t* out;        // per pixel (all npix)
};
template <typename IN>
__global__ void k_frame_metrics(MetArgs a);
__global__ void k_stab_count(StabArgs a);
__global__ void k_stab(StabArgs a);

__global__ void k_pack(const uint8_t* bytes, int64_t npix, int64_t frames, uint8_t* planes,
                       size_t pitch);
__global__ void k_unpack(const uint8_t* planes, size_t pitch, int64_t npix, int64_t frames,
                         uint8_t* bytes);
__global__ void k_bitrev_bytes(uint8_t* planes, size_t pitch, size_t row_bytes, int64_t frames);
__global__ void k_synth(int scene, uint64_t seed, int width, int height, int64_t frames,
                        int64_t frame0, double param, uint8_t* planes, size_t pitch);

}  // namespace spk
