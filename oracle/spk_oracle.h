/*
 * spk_oracle.h -- CPU restatement of the reference reconstruction path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product (paper_2412_11639_b200/,
 * include/, the CUDA library) links or calls this code.  It is used by
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg as the
 * checker for the CUDA path, never as the thing measured or shipped.
 *
 * Every function states the reference lines (paths relative to
 * /root/reference) whose behaviour it restates.  The restatement is pinned
 * against the reference itself: oracle/_ref/libspikecam_ref.so is compiled
 * from the reference sources (oracle/Makefile) and tests/test_oracle_pin.py
 * compares the two on seeded volumes; tests/golden/ holds the known-answer
 * vectors ported from proj/tests/*.cpp.
 */
#ifndef SPK_ORACLE_H
#define SPK_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { ORC_FSR = 0, ORC_SSR = 1, ORC_TFI = 2, ORC_TFP = 3 };

/* SPK1 payload framing (proj/src/io.cpp:48-76).  A plane holds
 * ceil(W*H/8) bytes; pixel p=y*W+x lives in byte p>>3, bit p&7 (LSB-first,
 * or bit 7-(p&7) for msb_first dumps, io.cpp:72).  `pitch` >= plane bytes is
 * the distance between consecutive planes (dense SPK1: pitch == plane bytes). */
size_t orc_plane_bytes(int width, int height);
void orc_pack(const uint8_t* bytes, int width, int height, long frames, uint8_t* planes,
              size_t pitch);
void orc_unpack(const uint8_t* planes, int width, int height, long frames, size_t pitch,
                int msb_first, uint8_t* bytes);

/* quantize (io.cpp:78-81): round-half-away(clamp(v, 0, 255)). */
uint8_t orc_quantize(double v);

/* One pixel's T-frame row (one byte per frame, nonzero = spike) to T doubles,
 * restating reconstruct_row (reconstruct.cpp:325-394) and, for SSR, the
 * two-pass fsr_runs_into / ssr_refine_into (reconstruct.cpp:40-99).
 * Returns 0, or -1 on a bad method / window. */
int orc_row_f64(const uint8_t* bits, long frames, int method, int window, double* out);

/* Whole (or a pixel range of a) packed volume.  Output is frame-major:
 * out[(n * out_pitch) + (p - pix_begin)] for p in [pix_begin, pix_end).
 * `threads` <= 0 means all OpenMP threads (only the pixel loop is parallel,
 * mirroring reconstruct.cpp:456-466; results do not depend on it). */
int orc_reconstruct_f64(const uint8_t* planes, int width, int height, long frames,
                        size_t pitch, int method, int window, long pix_begin, long pix_end,
                        double* out, size_t out_pitch, int threads);
int orc_reconstruct_u8(const uint8_t* planes, int width, int height, long frames,
                       size_t pitch, int method, int window, long pix_begin, long pix_end,
                       uint8_t* out, size_t out_pitch, int threads);

/* FSR/SSR segmentation of one pixel row as stable runs, restating
 * segment_fsr / segment_ssr + build_segments (reconstruct.cpp:107-130,
 * 198-211) but without the degenerate lead/tail entries: run k covers frames
 * [start[k], end[k]) and holds count[k] intervals.  Returns the number of
 * runs (<= cap are written), or -1 on a bad method. */
long orc_runs(const uint8_t* bits, long frames, int method, long* start, long* end,
              long* count, long cap);

/* PixelReconState::push_frame / flush (reconstruct.cpp:230-290): FSR event
 * stream (duration, intensity) of one row, any blocking.  Returns the number
 * of events (<= cap written). */
long orc_fsr_events(const uint8_t* bits, long frames, long* duration, double* intensity,
                    long cap);

/* 16-bit record codec (proj/src/codec.cpp:8-42). Returns words written or -1. */
long orc_encode(long duration, double intensity, uint16_t* words, long cap);

/* Quality metrics (proj/src/metrics.cpp:12-61): two_dimensional_entropy of a
 * W x H image (from its quantized uint8 values, or from doubles), NaN when
 * smaller than 3x3; mse of two n-value images. */
double orc_te_u8(const uint8_t* q, int width, int height);
double orc_te_f64(const double* values, int width, int height);
double orc_mse(const double* a, const double* b, long n);

/* stability_order (proj/src/stability.cpp:61-128) of one pixel row:
 * out[0] = depth of the first violation (0: none), out[1] = its index,
 * out[2] = verified_order, out[3] = absolute; `path` gets the violation's
 * '-'/'+' path.  Returns 0, or -1 for max_depth outside [1, 60]. */
int orc_stability(const uint8_t* bits, long frames, int max_depth, long* out, char* path,
                  long cap);

#ifdef __cplusplus
}
#endif
#endif
