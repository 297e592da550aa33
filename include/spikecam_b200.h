/*
 * spikecam_b200.h -- C-ABI of the B200-native spike-camera reconstruction path.
 *
 * Plain C, no torch or CUDA types in the signatures (streams are passed as
 * `void*` holding a cudaStream_t, 0 = legacy default stream).  The library is
 * libspikecam_b200.so, built in-tree by __graft_entry__.build().
 *
 * Each entry point replaces one reference interface (paths relative to the
 * reference checkout, /root/reference):
 *
 *   spk_reconstruct_u8     reconstruct() (proj/src/reconstruct.cpp:441-471)
 *                          followed by quantize() (proj/src/io.cpp:78-81) -- the
 *                          uint8 frame the CLI writes per timestep
 *                          (proj/tools/spikecam_main.cpp:174-179)
 *   spk_reconstruct_f64    reconstruct() values, bit-exact doubles
 *                          (proj/include/spikecam/reconstruct.hpp:73-79)
 *   spk_reconstruct_f32    the same values rounded to float
 *   spk_segment            segment_fsr / segment_ssr run lists
 *                          (proj/src/reconstruct.cpp:107-130, 198-211)
 *   spk_pack_bytes         pack_frame (proj/src/io.cpp:52-64): SpikeVolume bytes
 *                          (proj/include/spikecam/core.hpp:32-33) -> SPK1 planes
 *   spk_unpack_planes      unpack_frame (proj/src/io.cpp:66-76), incl. msb_first
 *   spk_upload_planes      read_spk / read_raw payload ingest
 *                          (proj/src/io.cpp:185-223) into the pitched device layout
 *   spk_reconstruct_host   the host-buffer boundary of reconstruct(): host SPK1
 *                          payload in, host frames out
 *   spk_segment_host       segment_fsr / segment_ssr on a host payload
 *   spk_records[_host]     --emit-records: segment_* -> encode_events -> write_spkr
 *                          (proj/tools/spikecam_main.cpp:146-172) as one SPKR image
 *   spk_frame_metrics[_host]  two_dimensional_entropy / mse per frame
 *                          (proj/src/metrics.cpp:12-61; the CLI's compare)
 *   spk_stability[_host]   stability_order per pixel (proj/src/stability.cpp:
 *                          112-128; the CLI's verify-stability --in)
 *
 * Error behaviour mirrors the reference's exceptions: SPK_EINVAL where the
 * reference throws std::invalid_argument (bad method / window / geometry,
 * proj/src/reconstruct.cpp:177-186, proj/src/core.cpp:11-13), SPK_ECUDA /
 * SPK_ENOMEM for device failures (std::runtime_error in the C++ wrapper).
 * spk_last_error() returns the calling thread's last message.
 *
 * Device data layout:
 *   planes : T bit-planes, plane n at d_planes + n*plane_pitch; pixel
 *            p = y*W + x is bit (p & 7) of byte (p >> 3), LSB-first (SPK1).
 *            plane_pitch must be a multiple of 4 and >= 4*ceil(W*H/32).
 *   output : T frame planes, frame n at d_out + n*out_pitch elements, pixel p
 *            at element p (row-major W*H).  out_pitch >= W*H.
 */
#ifndef SPIKECAM_B200_H
#define SPIKECAM_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SPK_OK 0
#define SPK_EINVAL 1
#define SPK_ECUDA 2
#define SPK_ENOMEM 3

/* ReconMethod::kind (proj/include/spikecam/reconstruct.hpp:10-18) */
#define SPK_FSR 0
#define SPK_SSR 1
#define SPK_TFI 2
#define SPK_TFP 3

#define SPK_OUT_U8 0
#define SPK_OUT_F32 1
#define SPK_OUT_F64 2

typedef struct spk_geom {
    int32_t width;      /* W >= 1 */
    int32_t height;     /* H >= 1 */
    int64_t frames;     /* T >= 0, < 2^29 */
    size_t plane_pitch; /* bytes between consecutive bit-planes */
} spk_geom;

/* One stable run of one pixel: frames [start, next run's start) -- or
 * [start, last_spike) for the final run -- holding `intervals` intervals.
 * Value = 255 * intervals / span (proj/src/reconstruct.cpp:124). */
typedef struct spk_run {
    uint32_t start;
    uint32_t intervals;
} spk_run;

/* Time shards (exact stitching of independently scanned frame ranges):
 * per pixel, how the true automaton -- re-run from the true state at the
 * shard start -- met the speculative one (started fresh at the shard start).
 * npre >= 0: synced after `npre` true runs closed; the speculative run that
 * started at rs_spec is the true run that started at rs_true, holding `delta`
 * more intervals.  npre = -2: never synced, but every true run of the shard
 * is in the prefix list; npre = -1: needs the full re-scan. */
typedef struct spk_sync {
    int32_t rs_true;
    int32_t rs_spec;
    int32_t delta;
    int32_t npre;
} spk_sync;

/* Close of the run(s) that cross a shard boundary, relative to the shard the
 * record belongs to.  Run A is the run covering the boundary (the run open
 * there, or the run that will start at the last spike before it).
 * a_state: 0 = no such run; 1 = it closes at a_end with a_intervals intervals
 * in total; 2 (entry records only) = it runs on past the next boundary -- take
 * the next record's A.  When A closes at the last spike before the boundary,
 * run B starts there: b_kind 1 = b_intervals / b_end known, 2 = B runs on past
 * the next boundary (the next record's A), 0 = no such run. */
typedef struct spk_close {
    int32_t a_state;
    int32_t a_intervals;
    int32_t a_end;
    int32_t b_kind;
    int32_t b_intervals;
    int32_t b_end;
    int32_t pad0;
    int32_t pad1;
} spk_close;

/* ---- device-resident path (asynchronous on `stream`) -------------------- */
int spk_reconstruct_u8(const spk_geom* g, const void* d_planes, int method, int tfp_window,
                       uint8_t* d_out, size_t out_pitch, void* stream);
int spk_reconstruct_f32(const spk_geom* g, const void* d_planes, int method, int tfp_window,
                        float* d_out, size_t out_pitch, void* stream);
int spk_reconstruct_f64(const spk_geom* g, const void* d_planes, int method, int tfp_window,
                        double* d_out, size_t out_pitch, void* stream);

/* FSR / SSR runs of every pixel: pixel p's runs at d_runs[p*run_cap ...],
 * its run count in d_counts[p] (a count > run_cap means the list was
 * truncated), its last spike frame in d_last[p] (-1 if none). */
int spk_segment(const spk_geom* g, const void* d_planes, int method, spk_run* d_runs,
                int64_t run_cap, uint32_t* d_counts, int32_t* d_last, void* stream);

/* spk_segment with the automaton state carried across time shards: d_state_in
 * (nullable = stream start) is the state at frame 0 of these planes, d_state_out
 * (nullable) receives the state after the last frame.  State = 17 int32
 * fields per pixel, field-major (d_state[f * W*H + p]), frames relative to the
 * first plane (earlier spikes negative); see spk_shard_* below. */
int spk_segment_state(const spk_geom* g, const void* d_planes, int method, spk_run* d_runs,
                      int64_t run_cap, uint32_t* d_counts, int32_t* d_last,
                      const int32_t* d_state_in, int32_t* d_state_out, void* stream);

/* ---- time shards: exact reconstruction of one long stream cut in frame
 * ranges (BASELINE configs[4]).  Shard r is scanned on its own
 * (spk_segment_state from a fresh state: the speculative runs); then, in shard
 * order, spk_shard_resolve re-runs the start of shard r from the true entry
 * state until it agrees with the speculative automaton and spk_shard_junction
 * produces the true exit state (the next shard's entry) and whether the run
 * open at the entry closes inside the shard; spk_shard_close_chain carries the
 * close of boundary-crossing runs back; spk_shard_stitch writes each shard's
 * true run list, which spk_expand_runs_* turns into that shard's frames.
 * g->frames is the shard length throughout; state layout as spk_segment_state. */
/* Every shard's speculative scan in ONE launch: shard r = frames
 * [r*shard_frames, min(frames, (r+1)*shard_frames)) scanned from a fresh
 * state, exactly as spk_segment_state(shard r's geometry, ..., NULL, ...)
 * would; shard r writes d_runs + r*W*H*run_cap, d_counts / d_last + r*W*H and
 * (if d_state_out) d_state_out + r*17*W*H.  shard_frames: a multiple of 32. */
int spk_segment_shards(const spk_geom* g, const void* d_planes, int method, int64_t shard_frames,
                       spk_run* d_runs, int64_t run_cap, uint32_t* d_counts, int32_t* d_last,
                       int32_t* d_state_out, void* stream);
/* the automaton state at the start of a stream (entry of the first shard) */
int spk_state_fresh(int64_t npix, int32_t* d_state, void* stream);
int spk_shard_resolve(const spk_geom* g, const void* d_planes, int method, const int32_t* d_entry,
                      const spk_run* d_spec, int64_t spec_cap, const uint32_t* d_spec_counts,
                      const int32_t* d_spec_state, spk_run* d_prefix, int32_t prefix_cap,
                      spk_sync* d_sync, int32_t* d_tstate, void* stream);
int spk_shard_junction(const spk_geom* g, int method, const int32_t* d_entry, const spk_sync* d_sync,
                       const spk_run* d_prefix, int32_t prefix_cap, const int32_t* d_tstate,
                       const spk_run* d_spec, int64_t spec_cap, const uint32_t* d_spec_counts,
                       const int32_t* d_spec_state, const spk_run* d_fb, const uint32_t* d_fb_counts,
                       const int32_t* d_fb_state, int32_t* d_exit_state, spk_close* d_entry_close,
                       spk_close* d_tail_close, void* stream);
int spk_shard_close_chain(int64_t npix, const spk_close* d_entry_close_next,
                          const spk_close* d_close_next, int32_t shard_len, spk_close* d_close,
                          void* stream);
int spk_shard_stitch(const spk_geom* g, int method, const int32_t* d_entry, const spk_sync* d_sync,
                     const spk_run* d_prefix, int32_t prefix_cap, const int32_t* d_tstate,
                     const spk_run* d_spec, int64_t spec_cap, const uint32_t* d_spec_counts,
                     const int32_t* d_spec_state, const spk_run* d_fb, const uint32_t* d_fb_counts,
                     const int32_t* d_fb_state, const spk_close* d_close, spk_run* d_region,
                     int64_t region_cap, uint32_t* d_region_counts, int32_t* d_region_last,
                     void* stream);
/* Frames of one shard from its stitched run list (run starts may precede the
 * shard: such a run's change is placed at frame 0; values use the true span). */
int spk_expand_runs_u8(const spk_geom* g, const spk_run* d_runs, int64_t run_cap,
                       const uint32_t* d_counts, const int32_t* d_last, uint8_t* d_out,
                       size_t out_pitch, void* stream);
int spk_expand_runs_f32(const spk_geom* g, const spk_run* d_runs, int64_t run_cap,
                        const uint32_t* d_counts, const int32_t* d_last, float* d_out,
                        size_t out_pitch, void* stream);
int spk_expand_runs_f64(const spk_geom* g, const spk_run* d_runs, int64_t run_cap,
                        const uint32_t* d_counts, const int32_t* d_last, double* d_out,
                        size_t out_pitch, void* stream);

/* one byte per bit (frame-major n*W*H + p, nonzero = spike) <-> planes */
int spk_pack_bytes(const spk_geom* g, const uint8_t* d_bytes, void* d_planes, void* stream);
int spk_unpack_planes(const spk_geom* g, const void* d_planes, uint8_t* d_bytes, void* stream);

/* Host payload (planes `src_pitch` bytes apart; dense SPK1 payload:
 * src_pitch = ceil(W*H/8)) -> pitched device planes; msb_first reverses the
 * in-byte bit order of raw dumps (proj/src/io.cpp:72). */
int spk_upload_planes(const spk_geom* g, const void* h_payload, size_t src_pitch,
                      int msb_first, void* d_planes, void* stream);

/* ---- host-buffer boundary (synchronous) ---------------------------------- */
/* h_payload: dense SPK1 payload (T planes of ceil(W*H/8) bytes; g->plane_pitch
 * is ignored).  out_type SPK_OUT_U8/F32/F64; h_out frame-major with
 * out_pitch elements per frame.  Runs on the current CUDA device. */
int spk_reconstruct_host(const spk_geom* g, const void* h_payload, int method, int tfp_window,
                         int out_type, void* h_out, size_t out_pitch);

/* reconstruct() with `workers` GPUs (SURVEY.md 8(b) spk_reconstruct_sharded;
 * the reference's parallel split, proj/src/reconstruct.cpp:456-466, is a
 * pixel range per OpenMP thread, "identical for any worker count",
 * proj/include/spikecam/reconstruct.hpp:70-72): the pixels are cut into
 * nbands bands on 128-pixel boundaries and band i runs on CUDA device
 * devices[i] (a device may take several bands), each from its own host
 * thread: upload of its plane columns, reconstruction, download into its
 * columns of h_out.  Arguments otherwise as spk_reconstruct_host; the output
 * is identical for any band count.  Synchronous. */
int spk_reconstruct_host_multi(const spk_geom* g, const void* h_payload, int method, int tfp_window,
                               int out_type, void* h_out, size_t out_pitch, const int32_t* devices,
                               int32_t nbands);

/* Many volumes of one geometry through the host boundary, pipelined: the
 * upload and reconstruction of volume i+1 overlap the download of volume i
 * (two stream lanes), so a sequence is bound by the slower PCIe direction.
 * h_payloads[i] / h_outs[i] as in spk_reconstruct_host (pinned memory lets the
 * copies run asynchronously).  The ingest path of SURVEY.md 8(f) rank 2. */
int spk_reconstruct_host_batch(const spk_geom* g, int32_t count, const void* const* h_payloads,
                               int method, int tfp_window, int out_type, void* const* h_outs,
                               size_t out_pitch);

/* Device batch (BASELINE configs[3]: many independent streams of one
 * geometry): volume i = d_planes[i] -> d_outs[i] (out_type SPK_OUT_*, pitch
 * out_pitch elements), exactly as `count` spk_reconstruct_* calls.  The calls
 * are captured once into a CUDA graph over four forked branches (kernels of
 * different volumes overlap; no per-call launch gaps), cached per thread and
 * device by geometry, method and buffer addresses, and replayed on `stream`
 * by later calls with the same buffers.  Asynchronous. */
int spk_reconstruct_batch(const spk_geom* g, int32_t count, const void* const* d_planes, int method,
                          int tfp_window, int out_type, void* const* d_outs, size_t out_pitch,
                          void* stream);
/* drop this thread's cached batch graphs (waits for the device) */
int spk_batch_release(void);

/* Host boundary of segment_fsr / segment_ssr (proj/src/reconstruct.cpp:198-211):
 * dense SPK1 payload in, per-pixel run lists out (layout as spk_segment;
 * h_runs holds W*H*run_cap entries).  Synchronous. */
int spk_segment_host(const spk_geom* g, const void* h_payload, int method, spk_run* h_runs,
                     int64_t run_cap, uint32_t* h_counts, int32_t* h_last);

/* ---- segment records (SPKR) ------------------------------------------------ */
/* The CLI's --emit-records output (proj/tools/spikecam_main.cpp:146-172):
 * every pixel's FSR / SSR segments (lead, runs, tail) encoded as 16-bit
 * words (duration << 8 | lround(intensity), durations > 255 split;
 * proj/src/codec.cpp:8-19), laid out as the complete SPKR file image
 * (proj/src/io.cpp:240-255: "SPKR", u16 W, u16 H, u32 fps, u32 frames, then
 * per pixel a u32 word count and its words, little endian).
 * spk_records allocates *d_image from the device pool (stream-ordered on
 * `stream`; release with spk_free_device) and synchronises `stream` once to
 * learn the size.  W, H <= 65535. */
int spk_records(const spk_geom* g, const void* d_planes, int method, uint32_t fps, void** d_image,
                uint64_t* image_bytes, void* stream);
/* host payload in, malloc'd host image out (release with spk_free_host) */
int spk_records_host(const spk_geom* g, const void* h_payload, int method, uint32_t fps,
                     void** h_image, uint64_t* image_bytes);
int spk_free_device(void* d_ptr, void* stream);
void spk_free_host(void* h_ptr);

/* ---- streaming FSR (PixelReconState, proj/include/spikecam/reconstruct.hpp:
 * 46-67, for every pixel at once) --------------------------------------------
 * Frames arrive in blocks; each push scans its block with the automaton state
 * carried from the previous block and returns the segments that closed in it
 * as SegmentEvents -- the events PixelReconState::push_frame yields, in order,
 * grouped by pixel: pixel p's events are d_events[d_offsets[p] ..
 * d_offsets[p+1]) (W*H+1 offsets).  spk_stream_flush returns the still-open
 * spans (PixelReconState::flush) and ends the stream.  Both allocate
 * *d_events and *d_offsets from the device pool (release with
 * spk_free_device) and synchronise `stream` once. */
typedef struct spk_event {
    int64_t duration;
    double intensity;
} spk_event;
typedef struct spk_stream spk_stream;
int spk_stream_create(int32_t width, int32_t height, void* stream, spk_stream** out);
int spk_stream_push(spk_stream* st, const void* d_planes, size_t plane_pitch, int64_t frames,
                    spk_event** d_events, uint64_t** d_offsets, uint64_t* total, void* stream);
int spk_stream_flush(spk_stream* st, spk_event** d_events, uint64_t** d_offsets, uint64_t* total,
                     void* stream);
/* host boundary: dense SPK1 payload of the block in, malloc'd host events and
 * offsets out (release both with spk_free_host); synchronous */
int spk_stream_push_host(spk_stream* st, const void* h_payload, int64_t frames, spk_event** h_events,
                         uint64_t** h_offsets, uint64_t* total);
int spk_stream_flush_host(spk_stream* st, spk_event** h_events, uint64_t** h_offsets, uint64_t* total);
int64_t spk_stream_frames(const spk_stream* st);
int spk_stream_destroy(spk_stream* st);

/* ---- configuration / diagnostics ------------------------------------------ */
/* run-list capacity per pixel used by spk_reconstruct_*: 0 = automatic
 * (max(64, T/32)).  Pixels that overflow it are recomputed exactly by a
 * slower direct-write pass, so results never depend on this value. */
int spk_set_run_capacity(int64_t per_pixel);
/* device bytes the pitched plane layout needs per frame for W*H pixels */
size_t spk_plane_pitch(int32_t width, int32_t height);
/* kernels launched by this thread since the last call (and reset) */
int64_t spk_launch_count(int reset);
/* Per-phase device timing of this thread's next spk_reconstruct_* calls:
 * when enabled, CUDA events are recorded on the call's stream around the
 * segment kernel (K2), the run finalisation (K2b, scan, K2c), the expand
 * kernel (K3) and the overflow fixup (TFI/TFP: the single kernel is reported
 * as `expand`).  spk_last_timing waits for the last call's events and returns
 * milliseconds (negative if a phase did not run). */
int spk_set_timing(int enable);
int spk_last_timing(float* segment_ms, float* finalize_ms, float* expand_ms, float* fixup_ms);
/* The last timed FSR/SSR call's in-grid time split: the number of time shards
 * its scan ran as (1: none) and the pixels whose shards could not be stitched
 * from the one-launch resolve and were re-scanned whole. */
int spk_last_split(int32_t* shards, int64_t* flagged);
const char* spk_last_error(void);
/* number of visible CUDA devices (the C++ drop-in spreads `workers` bands
 * over them); -1 when the CUDA runtime reports an error */
int spk_device_count(void);
/* Workspaces come from the current device's default stream-ordered pool,
 * which keeps freed blocks cached for the next call (no host sync per
 * call).  This waits for the device and returns the cached blocks to the
 * driver -- e.g. before other processes share the GPU. */
int spk_release_memory(void);
int spk_version(void);

/* ---- quality metrics and the stability check ------- */
/* Per-frame metrics of a reconstruction on the device, replacing the
 * per-image loops of the CLI's `compare` (proj/tools/spikecam_main.cpp:
 * 263-299): d_te[n] = two_dimensional_entropy of frame n
 * (proj/src/metrics.cpp:12-43) and, when d_ref is given, d_mse[n] = mse of
 * frame n against reference image n (metrics.cpp:45-55; psnr is
 * 10*log10(255^2/mse), 57-61).  Frames are [g->frames][pitch] elements of
 * frame_type (SPK_OUT_U8: quantized values, as the entropy uses them;
 * SPK_OUT_F32 / SPK_OUT_F64: values, quantized for the entropy with
 * round(clamp(v, 0, 255))); reference images are [g->frames][ref_pitch]
 * elements of ref_type (uint8 for PGM images read back, or values).  Either
 * output may be null.  Entropy needs W, H >= 3 (SPK_EINVAL,
 * the reference's invalid_argument).  Sums are reduced in a fixed order:
 * deterministic, equal to the reference's sequential sums up to double
 * rounding (tests hold them to 1e-12 relative). */
int spk_frame_metrics(const spk_geom* g, const void* d_frames, int frame_type, size_t pitch,
                      const void* d_ref, int ref_type, size_t ref_pitch, double* d_te,
                      double* d_mse, void* stream);

/* stability_order (proj/src/stability.cpp:61-128) of one pixel stream:
 * depth of the shallowest zero-order violation (0: none; 1 = S1), its index
 * in that sequence, its '-'/'+' path (bit j = branch j+1 -> j+2, '+' = 1;
 * path_len = depth - 1 characters), verified_order and absolute. */
typedef struct spk_stab {
    int32_t depth;
    int32_t verified_order;
    int32_t absolute;
    int32_t path_len;
    int64_t index;
    uint64_t path;
} spk_stab;
/* stability_order of every pixel of a packed volume (the per-pixel loop of
 * `verify-stability --in`, spikecam_main.cpp:189-207), d_out[p] for p =
 * y*W + x.  max_depth in [1, 63] (SPK_EINVAL otherwise; the reference
 * rejects < 1).  Synchronous with respect to `stream` (it sizes per-pixel
 * scratch from the spike counts). */
int spk_stability(const spk_geom* g, const void* d_planes, int max_depth, spk_stab* d_out,
                  void* stream);

/* Host-buffer forms (upload, compute, download; synchronous): frames /
 * reference images as above in host memory, h_payload a dense SPK1 payload. */
int spk_frame_metrics_host(const spk_geom* g, const void* h_frames, int frame_type, size_t pitch,
                           const void* h_ref, int ref_type, size_t ref_pitch, double* h_te,
                           double* h_mse);
int spk_stability_host(const spk_geom* g, const void* h_payload, int max_depth, spk_stab* h_out);

/* ---- synthetic inputs (benchmark / test harness, not the hot path) -------- */
/* Integrate-and-fire streams (threshold 1, subtractive reset, uniform initial
 * residual; proj/src/simulator.cpp:41-68) of the BASELINE.json configs:
 * scene 1 static gradient+texture, 2 moving texture + bar, 3 large sensor
 * with slow illumination, 5 extreme dynamic range; 0 = uniform random bits
 * with probability `param` (noise).  frame0 offsets time (time shards). */
int spk_synth(int scene, uint64_t seed, const spk_geom* g, int64_t frame0, double param,
              void* d_planes, void* stream);

#ifdef __cplusplus
}
#endif
#endif
