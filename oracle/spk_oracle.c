/*
 * spk_oracle.c -- CPU restatement of the reference reconstruction path.
 *
 * TEST INFRASTRUCTURE ONLY (see spk_oracle.h).  Plain C11 + optional OpenMP.
 * Reference paths are relative to /root/reference.
 */
#include "spk_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#ifdef _OPENMP
#include <omp.h>
#endif

/* ---------------------------------------------------------------- framing */

size_t orc_plane_bytes(int width, int height) {
    /* frame_bytes, proj/src/io.cpp:48-50 */
    return ((size_t)width * (size_t)height + 7u) / 8u;
}

void orc_pack(const uint8_t* bytes, int width, int height, long frames, uint8_t* planes,
              size_t pitch) {
    /* pack_frame, proj/src/io.cpp:52-64: LSB-first, pad bits zero */
    const size_t npix = (size_t)width * (size_t)height;
    for (long n = 0; n < frames; ++n) {
        uint8_t* dst = planes + (size_t)n * pitch;
        memset(dst, 0, pitch);
        const uint8_t* src = bytes + (size_t)n * npix;
        for (size_t p = 0; p < npix; ++p) {
            if (src[p]) dst[p >> 3] |= (uint8_t)(1u << (p & 7u));
        }
    }
}

void orc_unpack(const uint8_t* planes, int width, int height, long frames, size_t pitch,
                int msb_first, uint8_t* bytes) {
    /* unpack_frame, proj/src/io.cpp:66-76 */
    const size_t npix = (size_t)width * (size_t)height;
    for (long n = 0; n < frames; ++n) {
        const uint8_t* src = planes + (size_t)n * pitch;
        uint8_t* dst = bytes + (size_t)n * npix;
        for (size_t p = 0; p < npix; ++p) {
            unsigned sh = msb_first ? 7u - (unsigned)(p & 7u) : (unsigned)(p & 7u);
            dst[p] = (uint8_t)((src[p >> 3] >> sh) & 1u);
        }
    }
}

uint8_t orc_quantize(double v) {
    /* quantize, proj/src/io.cpp:78-81: std::round(std::clamp(v, 0, 255)) */
    if (v < 0.0) v = 0.0;
    if (v > 255.0) v = 255.0;
    return (uint8_t)round(v);
}

/* ------------------------------------------------------- zero-order rule */

/* PairScanner, proj/src/reconstruct.cpp:17-36 (same rule as
 * PixelReconState::accept_interval 230-243): the first value is taken, then
 * the first value at distance exactly 1 completes the pair; anything else is
 * a violation.  The set only grows until reset. */
typedef struct {
    int first, second;
    int have_first, have_second;
} pair_rule;

static void pair_clear(pair_rule* r) { r->have_first = r->have_second = 0; }

static int pair_take(pair_rule* r, int t) {
    if (!r->have_first) {
        r->first = t;
        r->have_first = 1;
        return 1;
    }
    if (t == r->first) return 1;
    if (r->have_second) return t == r->second;
    if (t == r->first + 1 || t == r->first - 1) {
        r->second = t;
        r->have_second = 1;
        return 1;
    }
    return 0;
}

/* half-open S1 index range */
typedef struct {
    long a, b;
} span_t;

/* fsr_runs_into, reconstruct.cpp:40-53: cut S1 before each violating
 * interval; the violating interval seeds the next run. */
static long fsr_cut(const int* s1, long count, span_t* runs) {
    long nr = 0;
    if (count == 0) return 0;
    pair_rule r;
    pair_clear(&r);
    long from = 0;
    for (long i = 0; i < count; ++i) {
        if (!pair_take(&r, s1[i])) {
            runs[nr].a = from;
            runs[nr].b = i;
            ++nr;
            from = i;
            pair_clear(&r);
            pair_take(&r, s1[i]);
        }
    }
    runs[nr].a = from;
    runs[nr].b = count;
    return nr + 1;
}

/* ssr_refine_into, reconstruct.cpp:64-99: inside each first-order run, the
 * occurrence gaps (in S1 index units) of each of its <= 2 values are fed to
 * the same pair rule; the first rejected gap at index i ends the sub-run
 * [start, i) and a fresh sub-run (fresh per-value state) starts at i. */
static long ssr_cut(const int* s1, const span_t* runs, long nruns, span_t* out) {
    long no = 0;
    for (long k = 0; k < nruns; ++k) {
        long start = runs[k].a;
        const long stop = runs[k].b;
        while (start < stop) {
            int val[2];
            long prev[2];
            pair_rule gap[2];
            int nv = 0;
            long cut = stop;
            for (long i = start; i < stop; ++i) {
                const int v = s1[i];
                int slot = -1;
                for (int j = 0; j < nv; ++j)
                    if (val[j] == v) slot = j;
                if (slot < 0) {
                    slot = nv++;
                    val[slot] = v;
                    prev[slot] = -1;
                    pair_clear(&gap[slot]);
                }
                if (prev[slot] >= 0 && !pair_take(&gap[slot], (int)(i - prev[slot]))) {
                    cut = i;
                    break;
                }
                prev[slot] = i;
            }
            out[no].a = start;
            out[no].b = cut;
            ++no;
            start = cut;
        }
    }
    return no;
}

/* scratch for one row */
typedef struct {
    long cap;
    long* spikes;
    int* s1;
    span_t* runs;
    span_t* refined;
} row_scratch;

static int scratch_init(row_scratch* s, long frames) {
    long n = frames > 0 ? frames : 1;
    s->cap = n;
    s->spikes = (long*)malloc(sizeof(long) * (size_t)n);
    s->s1 = (int*)malloc(sizeof(int) * (size_t)n);
    s->runs = (span_t*)malloc(sizeof(span_t) * (size_t)(n + 1));
    s->refined = (span_t*)malloc(sizeof(span_t) * (size_t)(n + 1));
    return (s->spikes && s->s1 && s->runs && s->refined) ? 0 : -1;
}

static void scratch_free(row_scratch* s) {
    free(s->spikes);
    free(s->s1);
    free(s->runs);
    free(s->refined);
}

/* spike positions and S1 (spikes_and_intervals, reconstruct.cpp:132-139) */
static long gather_spikes(const uint8_t* bits, long frames, long* spikes) {
    long ns = 0;
    for (long n = 0; n < frames; ++n)
        if (bits[n]) spikes[ns++] = n;
    return ns;
}

/* stable runs (S1 ranges) of a row for FSR / SSR */
static long row_runs(const uint8_t* bits, long frames, int method, row_scratch* s,
                     long* ns_out, const span_t** runs_out) {
    const long ns = gather_spikes(bits, frames, s->spikes);
    *ns_out = ns;
    const long ni = ns > 0 ? ns - 1 : 0;
    for (long i = 0; i < ni; ++i) s->s1[i] = (int)(s->spikes[i + 1] - s->spikes[i]);
    long nr = fsr_cut(s->s1, ni, s->runs);
    if (method == ORC_SSR) {
        nr = ssr_cut(s->s1, s->runs, nr, s->refined);
        *runs_out = s->refined;
    } else {
        *runs_out = s->runs;
    }
    return nr;
}

static int row_f64(const uint8_t* bits, long frames, int method, int window, double* out,
                   row_scratch* s) {
    if (method == ORC_TFP) {
        /* reconstruct_row TFP branch, reconstruct.cpp:328-337 */
        if (window < 1) return -1;
        long count = 0;
        for (long n = 0; n < frames; ++n) {
            count += bits[n] != 0;
            if (n >= window) count -= bits[n - window] != 0;
            const long len = n + 1 < window ? n + 1 : window;
            out[n] = 255.0 * (double)count / (double)len;
        }
        return 0;
    }
    if (method == ORC_TFI) {
        /* TFI branch, reconstruct.cpp:338-354 */
        const long ns = gather_spikes(bits, frames, s->spikes);
        long next = 1;
        double value = 0.0;
        for (long n = 0; n < frames; ++n) {
            while (next < ns && s->spikes[next] <= n) {
                value = 255.0 / (double)(s->spikes[next] - s->spikes[next - 1]);
                ++next;
            }
            out[n] = value;
        }
        return 0;
    }
    if (method != ORC_FSR && method != ORC_SSR) return -1;
    /* FSR fused scan (358-377) and SSR (378-390) produce the same runs as
     * fsr_runs_into / ssr_refine_into; each run [a,b) of S1 fills frames
     * [s_a, s_b) with 255*(b-a)/(s_b-s_a).  Lead [0,s_0) is 0 (355-356), the
     * tail [s_last, T) carries the last run value (391-393). */
    long ns;
    const span_t* runs;
    const long nr = row_runs(bits, frames, method, s, &ns, &runs);
    const long lead = ns > 0 ? s->spikes[0] : frames;
    for (long n = 0; n < lead; ++n) out[n] = 0.0;
    double carry = 0.0;
    if (ns > 1) {
        for (long k = 0; k < nr; ++k) {
            const long a = runs[k].a, b = runs[k].b;
            carry = 255.0 * (double)(b - a) / (double)(s->spikes[b] - s->spikes[a]);
            for (long n = s->spikes[a]; n < s->spikes[b]; ++n) out[n] = carry;
        }
    }
    if (ns > 0)
        for (long n = s->spikes[ns - 1]; n < frames; ++n) out[n] = carry;
    return 0;
}

int orc_row_f64(const uint8_t* bits, long frames, int method, int window, double* out) {
    row_scratch s;
    if (scratch_init(&s, frames) != 0) {
        scratch_free(&s);
        return -1;
    }
    int rc = row_f64(bits, frames, method, window, out, &s);
    scratch_free(&s);
    return rc;
}

long orc_runs(const uint8_t* bits, long frames, int method, long* start, long* end,
              long* count, long cap) {
    if (method != ORC_FSR && method != ORC_SSR) return -1;
    row_scratch s;
    if (scratch_init(&s, frames) != 0) {
        scratch_free(&s);
        return -1;
    }
    long ns;
    const span_t* runs;
    long nr = row_runs(bits, frames, method, &s, &ns, &runs);
    if (ns < 2) nr = 0; /* build_segments: no interval, no run (reconstruct.cpp:112-115) */
    for (long k = 0; k < nr && k < cap; ++k) {
        start[k] = s.spikes[runs[k].a];
        end[k] = s.spikes[runs[k].b];
        count[k] = runs[k].b - runs[k].a;
    }
    scratch_free(&s);
    return nr;
}

/* --------------------------------------------------------- whole volume */

#define ORC_BLOCK 64 /* pixels per gather block (reference uses 256, 408) */

static int volume_rows(const uint8_t* planes, int width, int height, long frames, size_t pitch,
                       int method, int window, long pix_begin, long pix_end, void* out,
                       size_t out_pitch, int as_u8, int threads) {
    (void)height;
    (void)width;
    if (method < ORC_FSR || method > ORC_TFP) return -1;
    if (method == ORC_TFP && window < 1) return -1;
    const long nblocks = (pix_end - pix_begin + ORC_BLOCK - 1) / ORC_BLOCK;
    int failed = 0;
#ifdef _OPENMP
    int nt = threads > 0 ? threads : omp_get_max_threads();
#pragma omp parallel num_threads(nt) reduction(| : failed)
#endif
    {
        row_scratch s;
        uint8_t* bits = (uint8_t*)malloc((size_t)ORC_BLOCK * (size_t)(frames > 0 ? frames : 1));
        double* row = (double*)malloc(sizeof(double) * (size_t)(frames > 0 ? frames : 1));
        if (scratch_init(&s, frames) != 0 || !bits || !row) failed = 1;
#ifdef _OPENMP
#pragma omp for schedule(dynamic, 1)
#endif
        for (long blk = 0; blk < nblocks; ++blk) {
            if (failed) continue;
            const long p0 = pix_begin + blk * ORC_BLOCK;
            const long nb = (pix_end - p0) < ORC_BLOCK ? (pix_end - p0) : ORC_BLOCK;
            /* column -> row gather (reconstruct_into 416-419), from packed bits */
            for (long n = 0; n < frames; ++n) {
                const uint8_t* plane = planes + (size_t)n * pitch;
                for (long j = 0; j < nb; ++j) {
                    const long p = p0 + j;
                    bits[(size_t)j * (size_t)frames + (size_t)n] =
                        (uint8_t)((plane[p >> 3] >> (p & 7)) & 1);
                }
            }
            for (long j = 0; j < nb; ++j) {
                row_f64(bits + (size_t)j * (size_t)frames, frames, method, window, row, &s);
                const size_t col = (size_t)(p0 + j - pix_begin);
                if (as_u8) {
                    uint8_t* o = (uint8_t*)out;
                    for (long n = 0; n < frames; ++n)
                        o[(size_t)n * out_pitch + col] = orc_quantize(row[n]);
                } else {
                    double* o = (double*)out;
                    for (long n = 0; n < frames; ++n) o[(size_t)n * out_pitch + col] = row[n];
                }
            }
        }
        scratch_free(&s);
        free(bits);
        free(row);
    }
#ifndef _OPENMP
    (void)threads;
#endif
    return failed ? -1 : 0;
}

int orc_reconstruct_f64(const uint8_t* planes, int width, int height, long frames,
                        size_t pitch, int method, int window, long pix_begin, long pix_end,
                        double* out, size_t out_pitch, int threads) {
    return volume_rows(planes, width, height, frames, pitch, method, window, pix_begin,
                       pix_end, out, out_pitch, 0, threads);
}

int orc_reconstruct_u8(const uint8_t* planes, int width, int height, long frames,
                       size_t pitch, int method, int window, long pix_begin, long pix_end,
                       uint8_t* out, size_t out_pitch, int threads) {
    return volume_rows(planes, width, height, frames, pitch, method, window, pix_begin,
                       pix_end, out, out_pitch, 1, threads);
}

/* ------------------------------------------------------ streaming events */

long orc_fsr_events(const uint8_t* bits, long frames, long* duration, double* intensity,
                    long cap) {
    /* PixelReconState::push_frame / flush, reconstruct.cpp:245-290 */
    long ne = 0;
#define EMIT(d, v)                  \
    do {                            \
        if (ne < cap) {             \
            duration[ne] = (d);     \
            intensity[ne] = (v);    \
        }                           \
        ++ne;                       \
    } while (0)
    long last = -1, run_start = -1, sum = 0, cnt = 0;
    double last_val = 0.0;
    pair_rule r;
    pair_clear(&r);
    for (long n = 0; n < frames; ++n) {
        if (!bits[n]) continue;
        if (last < 0) {
            if (n > 0) EMIT(n, 0.0);
            last = run_start = n;
            continue;
        }
        const int t = (int)(n - last);
        const long prev = last;
        last = n;
        if (pair_take(&r, t)) {
            sum += t;
            ++cnt;
            continue;
        }
        const double v = 255.0 * (double)cnt / (double)sum;
        EMIT(prev - run_start, v);
        last_val = v;
        run_start = prev;
        pair_clear(&r);
        pair_take(&r, t);
        sum = t;
        cnt = 1;
    }
    if (frames > 0) {
        if (last < 0) {
            EMIT(frames, 0.0);
        } else {
            if (cnt > 0) {
                const double v = 255.0 * (double)cnt / (double)sum;
                EMIT(last - run_start, v);
                last_val = v;
            }
            EMIT(frames - last, last_val);
        }
    }
#undef EMIT
    return ne;
}

long orc_encode(long duration, double intensity, uint16_t* words, long cap) {
    /* encode_append, proj/src/codec.cpp:8-19: lround (ties away), split at 255 */
    if (duration < 1 || intensity < 0.0 || intensity > 255.0) return -1;
    const unsigned q = (unsigned)lround(intensity);
    long nw = 0;
    while (duration > 255) {
        if (nw < cap) words[nw] = (uint16_t)(255u << 8 | q);
        ++nw;
        duration -= 255;
    }
    if (nw < cap) words[nw] = (uint16_t)((unsigned)duration << 8 | q);
    return nw + 1;
}

/* ---- quality metrics and the stability check ---- */

double orc_te_u8(const uint8_t* q, int w, int h) {
    /* two_dimensional_entropy, proj/src/metrics.cpp:12-43, on the already
     * quantized image (q = round(clamp(v, 0, 255)), line 18): histogram of
     * (gray, lround(3x3 sum / 9)) over interior pixels, entropy summed over
     * bins in index order.  NaN for images smaller than 3x3 (line 13). */
    if (w < 3 || h < 3) return NAN;
    long* hist = (long*)calloc(256 * 256, sizeof(long));
    long total = 0;
    for (int y = 1; y < h - 1; ++y)
        for (int x = 1; x < w - 1; ++x) {
            long sum = 0;
            for (int dy = -1; dy <= 1; ++dy)
                for (int dx = -1; dx <= 1; ++dx) sum += q[(size_t)(y + dy) * w + (x + dx)];
            const int gbar = (int)lround((double)sum / 9.0);
            ++hist[(size_t)q[(size_t)y * w + x] * 256 + gbar];
            ++total;
        }
    double e = 0.0;
    for (int i = 0; i < 256 * 256; ++i) {
        if (!hist[i]) continue;
        const double p = (double)hist[i] / (double)total;
        e -= p * log2(p);
    }
    free(hist);
    return e;
}

double orc_te_f64(const double* v, int w, int h) {
    if (w < 3 || h < 3) return NAN;
    uint8_t* q = (uint8_t*)malloc((size_t)w * h);
    for (size_t i = 0; i < (size_t)w * h; ++i) q[i] = orc_quantize(v[i]);
    const double e = orc_te_u8(q, w, h);
    free(q);
    return e;
}

double orc_mse(const double* a, const double* b, long n) {
    /* mse, metrics.cpp:45-55: sequential sum of squared differences / n */
    double acc = 0.0;
    for (long i = 0; i < n; ++i) {
        const double d = a[i] - b[i];
        acc += d * d;
    }
    return acc / (double)n;
}

/* interval_stream(values, firing), proj/src/stability.cpp:93-106 */
static long gaps_of(const int* v, long n, int firing, int* out) {
    long last = -1, m = 0;
    for (long i = 0; i < n; ++i) {
        if (v[i] != firing) continue;
        if (last >= 0) out[m++] = (int)(i - last);
        last = i;
    }
    return m;
}

/* first_violation_index, stability.cpp:41-59 (-1: stable) */
static long first_violation(const int* v, long n) {
    int have_a = 0, have_b = 0, a = 0, b = 0;
    for (long i = 0; i < n; ++i) {
        const int x = v[i];
        if (!have_a) {
            a = x;
            have_a = 1;
        } else if (x == a || (have_b && x == b)) {
        } else if (!have_b && abs(x - a) == 1) {
            b = x;
            have_b = 1;
        } else {
            return i;
        }
    }
    return -1;
}

typedef struct {
    int max_depth, deepest_ok, truncated;
    int vdepth;  /* 0: no violation */
    long vindex;
    char vpath[64];
} orc_tree;

/* explore, stability.cpp:61-91: depth-first, '-' (smaller firing value) first */
static void explore(const int* seq, long n, int depth, char* path, orc_tree* st) {
    if (st->vdepth && st->vdepth <= depth) return;
    if (n == 0) {
        if (depth > st->deepest_ok) st->deepest_ok = depth;
        return;
    }
    const long bad = first_violation(seq, n);
    if (bad >= 0) {
        if (!st->vdepth || depth < st->vdepth) {
            st->vdepth = depth;
            st->vindex = bad;
            strcpy(st->vpath, path);
        }
        return;
    }
    if (depth > st->deepest_ok) st->deepest_ok = depth;
    int lo = seq[0], hi = seq[0];
    for (long i = 1; i < n; ++i) {
        if (seq[i] < lo) lo = seq[i];
        if (seq[i] > hi) hi = seq[i];
    }
    if (lo == hi) return;
    if (depth >= st->max_depth) {
        st->truncated = 1;
        return;
    }
    int* child = (int*)malloc((size_t)n * sizeof(int));
    for (int br = 0; br < 2; ++br) {
        const long m = gaps_of(seq, n, br ? hi : lo, child);
        const size_t k = strlen(path);
        path[k] = br ? '+' : '-';
        path[k + 1] = 0;
        explore(child, m, depth + 1, path, st);
        path[k] = 0;
    }
    free(child);
}

int orc_stability(const uint8_t* bits, long frames, int max_depth, long* out, char* path,
                  long cap) {
    /* stability_order, stability.cpp:112-128, of a pixel stream
     * (pixel_stream, core.cpp:109-118: firing value 1) */
    if (max_depth < 1 || max_depth > 60) return -1;
    int* s1 = (int*)malloc((size_t)(frames > 0 ? frames : 1) * sizeof(int));
    long m = 0, last = -1;
    for (long i = 0; i < frames; ++i) {
        if (!bits[i]) continue;
        if (last >= 0) s1[m++] = (int)(i - last);
        last = i;
    }
    orc_tree st;
    memset(&st, 0, sizeof st);
    st.max_depth = max_depth;
    char buf[64] = {0};
    explore(s1, m, 1, buf, &st);
    free(s1);
    out[0] = st.vdepth;
    out[1] = st.vdepth ? st.vindex : 0;
    out[2] = st.vdepth ? st.vdepth - 1 : (st.truncated ? max_depth : st.deepest_ok);
    out[3] = st.vdepth ? 0 : !st.truncated;
    if (cap > 0) {
        const char* p = st.vdepth ? st.vpath : "";
        const size_t k = strlen(p) < (size_t)(cap - 1) ? strlen(p) : (size_t)(cap - 1);
        memcpy(path, p, k);
        path[k] = 0;
    }
    return 0;
}
