// ref_shim.cpp -- extern "C" face of the UNMODIFIED reference library.
//
// TEST INFRASTRUCTURE ONLY.  oracle/Makefile compiles this file together with
// the reference sources where they lie (/root/reference/proj/src/*.cpp) into
// oracle/_ref/libspikecam_ref.so.  Nothing here re-implements reference
// logic: every entry point calls the reference's public API
// (proj/include/spikecam/*.hpp) and only converts buffers.  It is used to pin
// the C restatement (spk_oracle.c), to generate tests/golden fixtures, and as
// bench.py's CPU baseline ("kind": "reference").
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <exception>
#include <filesystem>
#include <string>
#include <vector>

#include "spikecam/codec.hpp"
#include "spikecam/core.hpp"
#include "spikecam/io.hpp"
#include "spikecam/metrics.hpp"
#include "spikecam/reconstruct.hpp"
#include "spikecam/simulator.hpp"
#include "spikecam/stability.hpp"

using namespace spikecam;

namespace {

thread_local std::string g_err;

ReconMethod method_of(int m, int window) {
    switch (m) {
        case 0: return ReconMethod::parse("fsr", window);
        case 1: return ReconMethod::parse("ssr", window);
        case 2: return ReconMethod::parse("tfi", window);
        case 3: return ReconMethod::parse("tfp", window);
    }
    return ReconMethod::parse("?", window);  // throws invalid_argument
}

// packed SPK1 planes (LSB-first, `pitch` bytes apart) -> one-byte-per-bit volume
SpikeVolume volume_of(const uint8_t* planes, size_t pitch, int w, int h, int t) {
    SpikeVolume v(w, h, t);
    auto raw = v.raw_mutable();
    const size_t npix = static_cast<size_t>(w) * h;
    for (int n = 0; n < t; ++n) {
        const uint8_t* src = planes + static_cast<size_t>(n) * pitch;
        uint8_t* dst = raw.data() + static_cast<size_t>(n) * npix;
        for (size_t p = 0; p < npix; ++p) dst[p] = (src[p >> 3] >> (p & 7)) & 1;
    }
    return v;
}

SpikeLikeStream stream_of(const uint8_t* bits, long frames) {
    std::vector<int> vals(static_cast<size_t>(frames));
    for (long n = 0; n < frames; ++n) vals[static_cast<size_t>(n)] = bits[n] ? 1 : 0;
    return SpikeLikeStream(std::move(vals), 1, 0);
}

template <class F>
long guarded(F&& f) {
    try {
        return f();
    } catch (const std::invalid_argument& e) {
        g_err = std::string("invalid_argument: ") + e.what();
        return -1;
    } catch (const std::out_of_range& e) {
        g_err = std::string("out_of_range: ") + e.what();
        return -1;
    } catch (const io_error& e) {
        g_err = std::string("io_error: ") + e.what();
        return -1;
    } catch (const std::exception& e) {
        g_err = std::string("error: ") + e.what();
        return -1;
    }
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// reconstruct(volume, method, workers, out) (reconstruct.cpp:448-471).
// out_f64: T*W*H doubles, frame-major; out_u8 (optional): the same values
// through round(clamp(v,0,255)) -- the quantize rule of io.cpp:78-81.
long ref_reconstruct(const uint8_t* planes, size_t pitch, int w, int h, int t, int method,
                     int window, int workers, double* out_f64, uint8_t* out_u8) {
    return guarded([&]() -> long {
        SpikeVolume v = volume_of(planes, pitch, w, h, t);
        std::vector<IntensityImage> images;
        reconstruct(v, method_of(method, window), workers, images);
        const size_t npix = static_cast<size_t>(w) * h;
        for (int n = 0; n < t; ++n) {
            const auto& vals = images[static_cast<size_t>(n)].values;
            if (out_f64) std::memcpy(out_f64 + n * npix, vals.data(), npix * sizeof(double));
            if (out_u8) {
                uint8_t* o = out_u8 + n * npix;
                for (size_t p = 0; p < npix; ++p)
                    o[p] = static_cast<uint8_t>(std::round(std::clamp(vals[p], 0.0, 255.0)));
            }
        }
        return 0;
    });
}

// reconstruct_serial (reconstruct.cpp:433-439)
long ref_reconstruct_serial(const uint8_t* planes, size_t pitch, int w, int h, int t,
                            int method, int window, double* out_f64) {
    return guarded([&]() -> long {
        SpikeVolume v = volume_of(planes, pitch, w, h, t);
        auto images = reconstruct_serial(v, method_of(method, window));
        const size_t npix = static_cast<size_t>(w) * h;
        for (int n = 0; n < t; ++n)
            std::memcpy(out_f64 + n * npix, images[static_cast<size_t>(n)].values.data(),
                        npix * sizeof(double));
        return 0;
    });
}

// bench (metrics.cpp:63-82): median frames/s of `repeats` reconstruct() calls.
double ref_bench_fps(const uint8_t* planes, size_t pitch, int w, int h, int t, int method,
                     int window, int repeats, int workers) {
    double fps = -1.0;
    guarded([&]() -> long {
        SpikeVolume v = volume_of(planes, pitch, w, h, t);
        fps = bench(v, method_of(method, window), repeats, workers).frames_per_second;
        return 0;
    });
    return fps;
}

// segment_fsr / segment_ssr (reconstruct.cpp:198-211) of one row, all
// segments including degenerate lead/tail.  Returns the count (<= cap written).
long ref_segments(const uint8_t* bits, long frames, int method, long* start, long* end,
                  long* nintervals, double* intensity, long cap) {
    return guarded([&]() -> long {
        SpikeLikeStream s = stream_of(bits, frames);
        std::vector<Segment> segs = method == 1 ? segment_ssr(s) : segment_fsr(s);
        long k = 0;
        for (const Segment& g : segs) {
            if (k < cap) {
                start[k] = g.start_frame;
                end[k] = g.end_frame;
                nintervals[k] = static_cast<long>(g.intervals.size());
                intensity[k] = g.intensity;
            }
            ++k;
        }
        return k;
    });
}

// reconstruct_pixel (reconstruct.cpp:292-316)
long ref_reconstruct_pixel(const uint8_t* bits, long frames, int method, int window,
                           double* out) {
    return guarded([&]() -> long {
        auto vals = reconstruct_pixel(stream_of(bits, frames), method_of(method, window));
        std::copy(vals.begin(), vals.end(), out);
        return static_cast<long>(vals.size());
    });
}

// PixelReconState fed in `block`-frame blocks, then flush (reconstruct.cpp:245-290)
long ref_stream_events(const uint8_t* bits, long frames, long block, long* duration,
                       double* intensity, long cap) {
    return guarded([&]() -> long {
        PixelReconState st;
        long k = 0;
        auto put = [&](const SegmentEvent& e) {
            if (k < cap) {
                duration[k] = e.duration;
                intensity[k] = e.intensity;
            }
            ++k;
        };
        long i = 0;
        while (i < frames) {
            long stop = std::min(frames, i + block);
            for (; i < stop; ++i)
                if (auto e = st.push_frame(bits[i] != 0)) put(*e);
        }
        for (const SegmentEvent& e : st.flush()) put(e);
        return k;
    });
}

// fsr_events (reconstruct.cpp:222-228)
long ref_fsr_events(const uint8_t* bits, long frames, long* duration, double* intensity,
                    long cap) {
    return guarded([&]() -> long {
        auto ev = fsr_events(stream_of(bits, frames));
        long k = 0;
        for (const SegmentEvent& e : ev) {
            if (k < cap) {
                duration[k] = e.duration;
                intensity[k] = e.intensity;
            }
            ++k;
        }
        return k;
    });
}

// simulate_pixel (simulator.cpp:41-68)
long ref_simulate_pixel(const double* rates, long frames, double threshold, double residual,
                        uint8_t* bits) {
    return guarded([&]() -> long {
        auto s = simulate_pixel(std::span<const double>(rates, static_cast<size_t>(frames)),
                                threshold, residual);
        for (long n = 0; n < frames; ++n) bits[n] = static_cast<uint8_t>(s.values[n]);
        return 0;
    });
}

uint64_t ref_pixel_seed(uint64_t seed, int x, int y) { return pixel_seed(seed, x, y); }

// write_spk / read_spk / read_raw (io.cpp:173-223) through files
long ref_write_spk(const uint8_t* planes, size_t pitch, int w, int h, int t, uint32_t fps,
                   const char* path) {
    return guarded([&]() -> long {
        write_spk(volume_of(planes, pitch, w, h, t), fps, path);
        return 0;
    });
}

// Reads an SPK1 (kind 0) or raw (kind 1 / 2 = msb-first) file; returns frames
// and writes the one-byte-per-bit volume into `bytes` (cap bytes).
long ref_read(const char* path, int kind, int w, int h, int* w_out, int* h_out,
              uint32_t* fps_out, uint8_t* bytes, size_t cap) {
    return guarded([&]() -> long {
        uint32_t fps = kDefaultFps;
        SpikeVolume v = kind == 0 ? [&] {
            auto pr = read_spk(path);
            fps = pr.second;
            return std::move(pr.first);
        }()
                                  : read_raw(path, w, h, kind == 2);
        *w_out = v.width();
        *h_out = v.height();
        *fps_out = fps;
        auto raw = v.raw();
        if (raw.size() <= cap) std::memcpy(bytes, raw.data(), raw.size());
        return v.frames();
    });
}

// write_image(..., pgm) (io.cpp:225-232): the reference's own quantize path
long ref_write_pgm(const double* values, int w, int h, const char* path) {
    return guarded([&]() -> long {
        IntensityImage img(w, h);
        std::copy(values, values + static_cast<size_t>(w) * h, img.values.begin());
        write_image(img, path, ImageFormat::pgm);
        return 0;
    });
}

// encode_events (codec.cpp:27-31)
long ref_encode_events(const long* duration, const double* intensity, long nev,
                       uint16_t* words, long cap) {
    return guarded([&]() -> long {
        std::vector<SegmentEvent> ev;
        for (long i = 0; i < nev; ++i) ev.push_back({duration[i], intensity[i]});
        auto out = encode_events(ev);
        for (size_t i = 0; i < out.size() && static_cast<long>(i) < cap; ++i) words[i] = out[i];
        return static_cast<long>(out.size());
    });
}

// The CLI's --emit-records loop (proj/tools/spikecam_main.cpp:146-172) on a
// packed volume: per pixel fsr_events / segment_ssr -> encode_events, then
// write_spkr to `path`.
long ref_emit_records(const uint8_t* planes, size_t pitch, int w, int h, int t, int method,
                      uint32_t fps, const char* path) {
    return guarded([&]() -> long {
        const SpikeVolume volume = volume_of(planes, pitch, w, h, t);
        RecordVolume rv;
        rv.width = w;
        rv.height = h;
        rv.fps = fps;
        rv.frame_count = static_cast<uint32_t>(t);
        rv.words.resize(static_cast<size_t>(w) * h);
        for (int y = 0; y < h; ++y) {
            for (int x = 0; x < w; ++x) {
                const SpikeLikeStream stream = pixel_stream(volume, x, y);
                std::vector<SegmentEvent> events;
                if (method == 0) {
                    events = fsr_events(stream);
                } else {
                    for (const Segment& sg : segment_ssr(stream)) events.push_back({sg.duration(), sg.intensity});
                }
                rv.pixel(x, y) = encode_events(events);
            }
        }
        write_spkr(rv, path);
        return 0;
    });
}

// ---- quality metrics and the stability check ----

// two_dimensional_entropy (metrics.cpp:12-43) of a W x H image of doubles;
// NaN on an error (message in ref_last_error).
double ref_te(const double* values, int w, int h) {
    double r = std::nan("");
    guarded([&]() -> long {
        IntensityImage im(w, h);
        std::copy(values, values + static_cast<size_t>(w) * h, im.values.begin());
        r = two_dimensional_entropy(im);
        return 0;
    });
    return r;
}

// mse / psnr (metrics.cpp:45-61) of two W x H images of doubles
double ref_mse(const double* a, const double* b, int w, int h) {
    double r = std::nan("");
    guarded([&]() -> long {
        IntensityImage x(w, h), y(w, h);
        std::copy(a, a + static_cast<size_t>(w) * h, x.values.begin());
        std::copy(b, b + static_cast<size_t>(w) * h, y.values.begin());
        r = mse(x, y);
        return 0;
    });
    return r;
}
double ref_psnr(const double* a, const double* b, int w, int h) {
    double r = std::nan("");
    guarded([&]() -> long {
        IntensityImage x(w, h), y(w, h);
        std::copy(a, a + static_cast<size_t>(w) * h, x.values.begin());
        std::copy(b, b + static_cast<size_t>(w) * h, y.values.begin());
        r = psnr(x, y);
        return 0;
    });
    return r;
}

// stability_order (stability.cpp:112-128) of one pixel row.  out[0] =
// violation depth (0: none), out[1] = violation index, out[2] =
// verified_order, out[3] = absolute; `path` receives the violation path
// ('-'/'+', NUL-terminated, cap bytes).  Returns 0 or -1.
long ref_stability(const uint8_t* bits, long frames, int depth, long* out, char* path,
                   long cap) {
    return guarded([&]() -> long {
        StabilityReport r = stability_order(stream_of(bits, frames), depth);
        out[0] = r.first_violation ? r.first_violation->depth : 0;
        out[1] = r.first_violation ? static_cast<long>(r.first_violation->index) : 0;
        out[2] = r.verified_order;
        out[3] = r.absolute ? 1 : 0;
        const std::string p = r.first_violation ? r.first_violation->path : std::string();
        if (cap > 0) {
            const size_t n = std::min(p.size(), static_cast<size_t>(cap - 1));
            std::memcpy(path, p.data(), n);
            path[n] = 0;
        }
        return 0;
    });
}

}  // extern "C"
