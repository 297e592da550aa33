// dropin_test.cpp -- exercises the C++ drop-in (include/spikecam/b200.hpp) the
// way the reference's own callers do.  Driven by tests/test_dropin.py:
//
//   dropin_test selftest             host-only checks (no GPU needed)
//   dropin_test gpucheck             self-consistency of the GPU-backed API
//   dropin_test rows IN OUT          per-stream API on the golden streams
//   dropin_test vol IN.spk OUTDIR    volume API on a golden SPK1 file
//   dropin_test records IN.spk DIR   the CLI's --emit-records loop + emit_records
//
// `rows` / `vol` only dump results; the Python side compares them with the
// reference's golden outputs (tests/golden/).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <functional>
#include <iterator>
#include <random>
#include <string>

// the reference's header names (include/spikecam/*.hpp forward to b200.hpp)
#include "spikecam/codec.hpp"
#include "spikecam/core.hpp"
#include "spikecam/io.hpp"
#include "spikecam/metrics.hpp"
#include "spikecam/reconstruct.hpp"
#include "spikecam/b200.hpp"  // the additions: EventStream, reconstruct_u8, PackedSpikes

using namespace spikecam;
namespace fs = std::filesystem;

static int g_fail = 0;
#define EXPECT(cond)                                                       \
    do {                                                                   \
        if (!(cond)) {                                                     \
            std::fprintf(stderr, "%s:%d: EXPECT(%s) failed\n", __FILE__,   \
                         __LINE__, #cond);                                 \
            ++g_fail;                                                      \
        }                                                                  \
    } while (0)

template <typename E>
static bool throws(const std::function<void()>& f) {
    try {
        f();
    } catch (const E&) {
        return true;
    } catch (...) {
        return false;
    }
    return false;
}

static SpikeVolume random_volume(int w, int h, int t, double p, unsigned seed) {
    SpikeVolume v(w, h, t);
    std::mt19937 rng(seed);
    std::bernoulli_distribution b(p);
    for (auto& x : v.raw_mutable()) x = b(rng) ? 1 : 0;
    return v;
}

// ------------------------------------------------------------ selftest ----
static void selftest(const fs::path& dir) {
    // core value rules (core.cpp:9-75)
    EXPECT(throws<std::invalid_argument>([] { SpikeVolume(0, 3, 4); }));
    EXPECT(throws<std::invalid_argument>([] { SpikeVolume(3, 3, -1); }));
    SpikeVolume v(5, 3, 4);
    EXPECT(v.raw().size() == 60u);
    v.set(4, 2, 3, true);
    EXPECT(v.at(4, 2, 3) && !v.at(3, 2, 3));
    EXPECT(v.raw()[3 * 15 + 2 * 5 + 4] == 1);
    EXPECT(throws<std::out_of_range>([&] { v.at(5, 0, 0); }));
    EXPECT(throws<std::out_of_range>([&] { v.set(0, 0, 4, true); }));
    EXPECT(throws<std::out_of_range>([&] { pixel_stream(v, 0, 3); }));
    EXPECT(pixel_stream(v, 4, 2).firing_positions() == std::vector<long>{3});
    EXPECT(throws<std::invalid_argument>([] { SpikeLikeStream({1, 0, 2}, 1, 0); }));
    EXPECT(throws<std::invalid_argument>([] { SpikeLikeStream({1, 1}, 1, 1); }));
    EXPECT(throws<std::invalid_argument>([] { SpikeLikeStream::from_values({1, 2, 3}); }));
    auto s = SpikeLikeStream::from_values({5, -1, 5});
    EXPECT(s.firing_value == 5 && s.resting_value == -1);
    EXPECT((s.firing_positions() == std::vector<long>{0, 2}));
    EXPECT(throws<std::invalid_argument>([] { IntervalStream({2, 0}); }));
    EXPECT(throws<std::invalid_argument>([] { Segment(3, 3, {}, 1.0); }));
    EXPECT(throws<std::invalid_argument>([] { Segment(0, 3, {}, 256.0); }));
    EXPECT(throws<std::invalid_argument>([] { IntensityImage(0, 1); }));
    EXPECT(throws<std::invalid_argument>([] { segment_intensity(Segment(0, 4, {}, 0.0)); }));
    EXPECT(segment_intensity(Segment(0, 10, IntervalStream({3, 3, 4}), 0.0)) == 255.0 * 3 / 10);

    // ReconMethod (reconstruct.cpp:177-196)
    EXPECT(ReconMethod::parse("ssr").kind == Method::ssr);
    EXPECT(ReconMethod::parse("tfp", 7).name() == "tfp-7");
    EXPECT(ReconMethod::parse("fsr").name() == "fsr");
    EXPECT(throws<std::invalid_argument>([] { ReconMethod::parse("tfp", 0); }));
    EXPECT(throws<std::invalid_argument>([] { ReconMethod::parse("nope"); }));

    // SPK1 round trip, odd pixel count (pad bits), and the header layout
    const SpikeVolume a = random_volume(13, 7, 37, 0.3, 5);
    write_spk(a, 1234, dir / "a.spk");
    auto [b, fps] = read_spk(dir / "a.spk");
    EXPECT(fps == 1234u && b == a);
    EXPECT(fs::file_size(dir / "a.spk") == 16u + 12u * 37u);
    const PackedSpikes pk = read_spk_packed(dir / "a.spk");
    EXPECT(pk.width == 13 && pk.height == 7 && pk.frames == 37u && pk.payload == pack(a).payload);
    {  // headerless dump, LSB and MSB bit order
        std::ofstream o(dir / "a.raw", std::ios::binary);
        o.write(reinterpret_cast<const char*>(pk.payload.data()), (std::streamsize)pk.payload.size());
    }
    EXPECT(read_raw(dir / "a.raw", 13, 7) == a);
    const SpikeVolume m = read_raw(dir / "a.raw", 13, 7, true);
    for (int n = 0; n < 37; ++n)
        for (int p = 0; p < 91; ++p) {
            const int q = (p & ~7) | (7 - (p & 7));  // bit reversed within its byte
            if (q < 91) EXPECT(m.at(p % 13, p / 13, n) == a.at(q % 13, q / 13, n));
        }
    EXPECT(throws<io_error>([&] { read_raw(dir / "a.raw", 10, 10); }));
    EXPECT(throws<io_error>([&] { read_spk(dir / "missing.spk"); }));
    {
        std::ofstream o(dir / "bad.spk", std::ios::binary);
        o << "SPK2xxxxxxxxxxxx";
    }
    EXPECT(throws<io_error>([&] { read_spk(dir / "bad.spk"); }));
    {  // truncated payload
        auto bytes = std::vector<char>(16 + 5);
        std::ifstream i(dir / "a.spk", std::ios::binary);
        i.read(bytes.data(), (std::streamsize)bytes.size());
        std::ofstream o(dir / "short.spk", std::ios::binary);
        o.write(bytes.data(), (std::streamsize)bytes.size());
    }
    EXPECT(throws<io_error>([&] { read_spk(dir / "short.spk"); }));

    // PGM: quantize() rounding (io.cpp:78-81) and read back
    IntensityImage img(4, 2);
    img.values = {0.0, 127.5, 127.49999, 254.5, 255.0, 0.5, -3.0, 300.0};
    write_image(img, dir / "q.pgm", ImageFormat::pgm);
    const IntensityImage r = read_image(dir / "q.pgm");
    EXPECT(r.width == 4 && r.height == 2);
    EXPECT((r.values == std::vector<double>{0, 128, 127, 255, 255, 1, 0, 255}));
    EXPECT(throws<io_error>([&] { write_image(img, dir / "q.png", ImageFormat::png); }));

    // codec (codec.cpp:8-41): word layout, splits past 255 frames, rounding, errors
    EXPECT((encode(3, 127.5) == std::vector<uint16_t>{static_cast<uint16_t>(3 << 8 | 128)}));
    const auto split = encode(600, 10.4);
    EXPECT((split == std::vector<uint16_t>{0xff0a, 0xff0a, static_cast<uint16_t>(90 << 8 | 10)}));
    EXPECT(duration_of(split[2]) == 90 && intensity_of(split[2]) == 10);
    EXPECT(decode(split).size() == 600u && decode(split)[599] == 10);
    EXPECT(throws<std::invalid_argument>([] { encode(0, 1.0); }));
    EXPECT(throws<std::invalid_argument>([] { encode(5, 255.5); }));
    EXPECT(throws<std::invalid_argument>([] { encode(5, -0.1); }));
    const std::vector<uint16_t> zero{0x0005};
    EXPECT(throws<std::runtime_error>([&] { decode(zero); }));
    const std::vector<SegmentEvent> evs{{2, 0.4}, {300, 254.6}};
    EXPECT((encode_events(evs) == std::vector<uint16_t>{0x0200, 0xffff, static_cast<uint16_t>(45 << 8 | 255)}));
    // SPKR (io.cpp:240-292): round trip, geometry check, truncation / trailing bytes
    RecordVolume rv;
    rv.width = 2;
    rv.height = 1;
    rv.frame_count = 7;
    rv.words = {{0x0701}, {0x0300, 0x0402}};
    write_spkr(rv, dir / "r.spkr");
    const RecordVolume back = read_spkr(dir / "r.spkr");
    EXPECT(back.width == 2 && back.height == 1 && back.fps == kDefaultFps && back.frame_count == 7);
    EXPECT(back.words == rv.words && back.pixel(1, 0).size() == 2u);
    RecordVolume bad = rv;
    bad.words.pop_back();
    EXPECT(throws<io_error>([&] { write_spkr(bad, dir / "bad.spkr"); }));
    {
        std::ifstream in(dir / "r.spkr", std::ios::binary);
        std::string bytes((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
        std::ofstream(dir / "trunc.spkr", std::ios::binary).write(bytes.data(), (std::streamsize)bytes.size() - 1);
        std::ofstream(dir / "trail.spkr", std::ios::binary).write((bytes + "x").data(), (std::streamsize)bytes.size() + 1);
    }
    EXPECT(throws<io_error>([&] { read_spkr(dir / "trunc.spkr"); }));
    EXPECT(throws<io_error>([&] { read_spkr(dir / "trail.spkr"); }));
    EXPECT(throws<io_error>([&] { read_spkr(dir / "q.pgm"); }));
    EXPECT(throws<std::invalid_argument>([&] { bench(SpikeVolume(2, 2, 2), ReconMethod::parse("fsr"), 2); }));
}

// ------------------------------------------------------------- records ----
// The CLI's --emit-records loop (spikecam_main.cpp:146-172) compiled against
// the drop-in (per pixel: pixel_stream -> fsr_events / segment_ssr ->
// encode_events -> write_spkr), and the whole-sensor GPU form emit_records;
// both files are compared with the reference's SPKR bytes by test_dropin.py.
static void records(const fs::path& spk, const fs::path& dir) {
    const auto [volume, fps] = read_spk(spk);
    for (const char* name : {"fsr", "ssr"}) {
        const ReconMethod method = ReconMethod::parse(name);
        RecordVolume rv;
        rv.width = volume.width();
        rv.height = volume.height();
        rv.fps = fps;
        rv.frame_count = static_cast<uint32_t>(volume.frames());
        rv.words.resize(static_cast<size_t>(rv.width) * rv.height);
        for (int y = 0; y < rv.height; ++y) {
            for (int x = 0; x < rv.width; ++x) {
                SpikeLikeStream stream = pixel_stream(volume, x, y);
                std::vector<SegmentEvent> events;
                if (method.kind == Method::fsr) {
                    events = fsr_events(stream);
                } else {
                    for (const Segment& sg : segment_ssr(stream)) events.push_back({sg.duration(), sg.intensity});
                }
                rv.pixel(x, y) = encode_events(events);
            }
        }
        write_spkr(rv, dir / (std::string(name) + "_loop.spkr"));
        const RecordVolume gpu = emit_records(volume, method, fps);
        write_spkr(gpu, dir / (std::string(name) + "_gpu.spkr"));
        EXPECT(gpu.words == rv.words);
        // decode of every pixel's words == its uint8 frames (codec.hpp:23-25)
        const auto u8 = reconstruct_u8(volume, method);
        bool eq = true;
        for (int p = 0; eq && p < rv.width * rv.height; ++p) {
            const auto d = decode(gpu.words[static_cast<size_t>(p)]);
            eq = d.size() == static_cast<size_t>(volume.frames());
            for (int n = 0; eq && n < volume.frames(); ++n) eq = d[static_cast<size_t>(n)] == u8[static_cast<size_t>(n)][static_cast<size_t>(p)];
        }
        EXPECT(eq);
    }
    EXPECT(throws<std::invalid_argument>([&] { emit_records(volume, ReconMethod::parse("tfi")); }));
    const BenchResult b = bench(volume, ReconMethod::parse("ssr"), 3, 1);
    EXPECT(b.method == "ssr" && b.repeats == 3 && b.frames == volume.frames() && b.frames_per_second > 0.0);
}

// ------------------------------------------------------------ gpucheck ----
static bool same_bits(double x, double y) { return std::memcmp(&x, &y, sizeof x) == 0; }

static void gpucheck() {
    // worked example of the paper / reconstruct.hpp:30-35: intervals 3,3,4,3 | 7,6,7
    std::vector<int> vals(40, 0);
    for (int f : {0, 3, 6, 10, 13, 20, 26, 33}) vals[f] = 1;
    const SpikeLikeStream ex(vals, 1, 0);
    const auto segs = segment_fsr(ex);
    EXPECT(segs.size() == 3u);
    if (segs.size() == 3u) {
        EXPECT(segs[0].start_frame == 0 && segs[0].end_frame == 13 && segs[0].intervals.size() == 4u);
        EXPECT(segs[1].start_frame == 13 && segs[1].end_frame == 33 && segs[1].intervals.size() == 3u);
        EXPECT((segs[1].intervals.intervals == std::vector<int>{7, 6, 7}));
        EXPECT(segs[2].degenerate() && segs[2].end_frame == 40);
        EXPECT(same_bits(segs[0].intensity, 255.0 * 4 / 13));
        EXPECT(same_bits(segs[2].intensity, 255.0 * 3 / 20));
        EXPECT(same_bits(segment_intensity(segs[1]), segs[1].intensity));
    }
    const auto ev = fsr_events(ex);
    EXPECT(ev.size() == 3u && ev[0].duration == 13 && ev[1].duration == 20 && ev[2].duration == 7);
    EXPECT(segment_fsr(SpikeLikeStream({}, 1, 0)).empty());
    const auto silent = segment_fsr(SpikeLikeStream(std::vector<int>(9, 0), 1, 0));
    EXPECT(silent.size() == 1u && silent[0].end_frame == 9 && silent[0].intensity == 0.0);
    // firing value other than 1 (SpikeLikeStream e1/e2)
    std::vector<int> alt(vals.size());
    for (size_t i = 0; i < vals.size(); ++i) alt[i] = vals[i] ? 7 : -2;
    const auto pix_alt = reconstruct_pixel(SpikeLikeStream(alt, 7, -2), ReconMethod::parse("fsr"));
    EXPECT(pix_alt == reconstruct_pixel(ex, ReconMethod::parse("fsr")));

    // volume API: identical for any worker count and buffer reuse
    // (test_reconstruct.cpp:250-267 property), per-pixel form == volume column
    const SpikeVolume vol = random_volume(11, 6, 300, 0.35, 9);
    for (const char* name : {"fsr", "ssr", "tfi", "tfp"}) {
        const ReconMethod m = ReconMethod::parse(name, 5);
        const auto base = reconstruct_serial(vol, m);
        EXPECT(base.size() == 300u && base[0].width == 11 && base[0].height == 6);
        for (int w : {0, 1, 3, 64}) {
            const auto o = reconstruct(vol, m, w);
            bool eq = o.size() == base.size();
            for (size_t n = 0; eq && n < o.size(); ++n)
                eq = std::memcmp(o[n].values.data(), base[n].values.data(), 66 * sizeof(double)) == 0;
            EXPECT(eq);
        }
        std::vector<IntensityImage> reuse(300, IntensityImage(11, 6, -1.0));
        const double* keep = reuse[0].values.data();
        reconstruct(vol, m, 2, reuse);
        EXPECT(reuse[0].values.data() == keep);  // same geometry -> buffers reused
        EXPECT(reuse[299].values == base[299].values);
        for (int p : {0, 17, 65}) {
            const auto col = reconstruct_pixel(pixel_stream(vol, p % 11, p / 11), m);
            bool eq = col.size() == 300u;
            for (int n = 0; eq && n < 300; ++n) eq = same_bits(col[n], base[n].at(p % 11, p / 11));
            EXPECT(eq);
        }
        // uint8 frames == quantize(values)
        const auto u8 = reconstruct_u8(vol, m);
        bool eq = u8.size() == 300u;
        for (size_t n = 0; eq && n < 300; ++n)
            for (size_t i = 0; i < 66; ++i)
                eq &= u8[n][i] == (uint8_t)std::round(std::clamp(base[n].values[i], 0.0, 255.0));
        EXPECT(eq);
    }
    // SSR refines FSR: every SSR segment lies inside one FSR segment
    for (int p = 0; p < 66; ++p) {
        const auto st = pixel_stream(vol, p % 11, p / 11);
        const auto f = segment_fsr(st), s = segment_ssr(st);
        EXPECT(s.size() >= f.size());
        size_t j = 0;
        for (const auto& seg : s) {
            while (j < f.size() && f[j].end_frame <= seg.start_frame) ++j;
            EXPECT(j < f.size() && f[j].start_frame <= seg.start_frame && seg.end_frame <= f[j].end_frame);
        }
    }
    // streaming form: PixelReconState events == fsr_events (reconstruct.hpp:46-50),
    // flush yields the open spans; EventStream gives the same per pixel in blocks
    {
        std::mt19937 rng(11);
        for (int trial = 0; trial < 12; ++trial) {
            const int t = 50 + trial * 37;
            std::vector<int> bits(t);
            std::bernoulli_distribution b(0.05 + 0.07 * (trial % 5));
            for (int& x : bits) x = b(rng) ? 1 : 0;
            if (trial == 0) std::fill(bits.begin(), bits.end(), 0);
            const SpikeLikeStream st(bits, 1, 0);
            PixelReconState ps;
            std::vector<SegmentEvent> got;
            for (int x : bits)
                if (auto e = ps.push_frame(x != 0)) got.push_back(*e);
            for (const auto& e : ps.flush()) got.push_back(e);
            EXPECT(ps.frames_seen() == t);
            EXPECT(got == fsr_events(st));
        }
        EventStream es(11, 6);
        std::vector<std::vector<SegmentEvent>> per(66);
        const PackedSpikes pk = pack(vol);
        const size_t fb = (66 + 7) / 8;
        for (long f0 = 0; f0 < 300; f0 += 70) {
            const long n = std::min<long>(70, 300 - f0);
            std::vector<uint8_t> blk(pk.payload.begin() + f0 * fb, pk.payload.begin() + (f0 + n) * fb);
            auto ev = es.push(blk, n);
            for (int p = 0; p < 66; ++p) per[p].insert(per[p].end(), ev[p].begin(), ev[p].end());
        }
        auto ev = es.flush();
        EXPECT(es.frames() == 300);
        for (int p = 0; p < 66; ++p) {
            per[p].insert(per[p].end(), ev[p].begin(), ev[p].end());
            EXPECT(per[p] == fsr_events(pixel_stream(vol, p % 11, p / 11)));
        }
    }
    // errors surface as the reference's exceptions
    EXPECT(throws<std::invalid_argument>([&] { reconstruct(vol, ReconMethod{Method::tfp, 0}); }));
    EXPECT(reconstruct(SpikeVolume(3, 2, 0), ReconMethod{}).empty());
}

// ---------------------------------------------------------------- rows ----
template <typename T>
static void put(std::ofstream& o, T v) {
    o.write(reinterpret_cast<const char*>(&v), sizeof v);
}

static void rows(const fs::path& in, const fs::path& out) {
    std::ifstream i(in, std::ios::binary);
    std::ofstream o(out, std::ios::binary);
    uint32_t ncase = 0;
    i.read(reinterpret_cast<char*>(&ncase), 4);
    for (uint32_t c = 0; c < ncase; ++c) {
        uint32_t t = 0;
        i.read(reinterpret_cast<char*>(&t), 4);
        std::vector<uint8_t> b(t);
        i.read(reinterpret_cast<char*>(b.data()), t);
        const SpikeLikeStream st(std::vector<int>(b.begin(), b.end()), 1, 0);
        for (auto* fn : {&segment_fsr, &segment_ssr}) {
            const auto segs = (*fn)(st);
            put<uint32_t>(o, (uint32_t)segs.size());
            for (const auto& s : segs) {
                put<int64_t>(o, s.start_frame);
                put<int64_t>(o, s.end_frame);
                put<int64_t>(o, (int64_t)s.intervals.size());
                put<double>(o, s.intensity);
            }
        }
        const std::pair<const char*, int> variants[] = {{"fsr", 32}, {"ssr", 32}, {"tfi", 32},
                                                        {"tfp", 32}, {"tfp", 7},  {"tfp", 1}};
        for (auto [name, win] : variants) {
            const auto pix = reconstruct_pixel(st, ReconMethod::parse(name, win));
            o.write(reinterpret_cast<const char*>(pix.data()), (std::streamsize)(pix.size() * 8));
        }
        const auto ev = fsr_events(st);
        put<uint32_t>(o, (uint32_t)ev.size());
        for (const auto& e : ev) {
            put<int64_t>(o, e.duration);
            put<double>(o, e.intensity);
        }
    }
}

// ----------------------------------------------------------------- vol ----
static void vol(const fs::path& spk, const fs::path& dir) {
    auto [v, fps] = read_spk(spk);
    (void)fps;
    const PackedSpikes pk = read_spk_packed(spk);
    const std::pair<const char*, int> variants[] = {{"fsr", 32}, {"ssr", 32}, {"tfi", 32},
                                                    {"tfp", 32}, {"tfp", 16}, {"tfp", 3}};
    for (auto [name, win] : variants) {
        const ReconMethod m = ReconMethod::parse(name, win);
        const std::string tag = std::string(name) + (std::string(name) == "tfp" ? std::to_string(win) : "");
        const auto imgs = reconstruct(v, m);  // SpikeVolume -> IntensityImage path
        std::ofstream f(dir / (tag + ".f64"), std::ios::binary);
        for (const auto& im : imgs)
            f.write(reinterpret_cast<const char*>(im.values.data()), (std::streamsize)(im.values.size() * 8));
        const auto u8 = reconstruct_u8(pk, m);  // packed file -> uint8 frames path
        std::ofstream g(dir / (tag + ".u8"), std::ios::binary);
        g.write(reinterpret_cast<const char*>(u8.data()), (std::streamsize)u8.size());
        if (imgs.size() > 1)
            write_image(imgs[imgs.size() / 2], dir / (tag + "_mid.pgm"), ImageFormat::pgm);
    }
}

// ------------------------------------------------------ metrics / stab ----
static void put_report(std::ofstream& o, const StabilityReport& r) {
    put<int32_t>(o, r.first_violation ? r.first_violation->depth : 0);
    put<int64_t>(o, r.first_violation ? (int64_t)r.first_violation->index : 0);
    put<int32_t>(o, r.verified_order);
    put<int32_t>(o, r.absolute ? 1 : 0);
    const std::string path = r.first_violation ? r.first_violation->path : std::string();
    put<uint32_t>(o, (uint32_t)path.size());
    o.write(path.data(), (std::streamsize)path.size());
}

static void stab_rows(const fs::path& in, const fs::path& out, int depth) {
    std::ifstream i(in, std::ios::binary);
    std::ofstream o(out, std::ios::binary);
    uint32_t ncase = 0;
    i.read(reinterpret_cast<char*>(&ncase), 4);
    for (uint32_t c = 0; c < ncase; ++c) {
        uint32_t t = 0;
        i.read(reinterpret_cast<char*>(&t), 4);
        std::vector<uint8_t> b(t);
        i.read(reinterpret_cast<char*>(b.data()), t);
        put_report(o, stability_order(SpikeLikeStream(std::vector<int>(b.begin(), b.end()), 1, 0), depth));
    }
}

// compare-style metrics of FSR frames against TFI frames, and the per-pixel
// stability of the volume (verify-stability --in)
static void metrics(const fs::path& spk, const fs::path& dir) {
    auto [v, fps] = read_spk(spk);
    (void)fps;
    const auto fsr = reconstruct(v, ReconMethod::parse("fsr"));
    const auto tfi = reconstruct(v, ReconMethod::parse("tfi"));
    std::vector<IntensityImage> ref;
    for (const auto& im : tfi) {  // reference images as PGM round trips them
        IntensityImage q(im.width, im.height);
        for (size_t k = 0; k < im.values.size(); ++k)
            q.values[k] = std::round(std::clamp(im.values[k], 0.0, 255.0));
        ref.push_back(std::move(q));
    }
    const auto te = two_dimensional_entropy(fsr);
    std::ofstream f(dir / "te.f64", std::ios::binary);
    f.write(reinterpret_cast<const char*>(te.data()), (std::streamsize)(te.size() * 8));
    std::ofstream g(dir / "single.f64", std::ios::binary);
    for (size_t n = 0; n < fsr.size(); n += 37) {
        put<double>(g, two_dimensional_entropy(fsr[n]));
        put<double>(g, mse(fsr[n], ref[n]));
        put<double>(g, psnr(fsr[n], ref[n]));
    }
    for (int depth : {4, 8}) {
        std::ofstream o(dir / ("stab_d" + std::to_string(depth) + ".bin"), std::ios::binary);
        for (const auto& r : stability_order(v, depth)) put_report(o, r);
    }
    EXPECT(throws<std::invalid_argument>([&] { two_dimensional_entropy(IntensityImage(2, 7)); }));
    EXPECT(throws<std::invalid_argument>([&] { mse(IntensityImage(3, 3), IntensityImage(3, 4)); }));
    EXPECT(throws<std::invalid_argument>([&] { stability_order(pixel_stream(v, 0, 0), 0); }));
    EXPECT(std::isinf(psnr(fsr[0], fsr[0])));
}

int main(int argc, char** argv) {
    const std::string mode = argc > 1 ? argv[1] : "";
    try {
        if (mode == "selftest" && argc == 3) {
            selftest(argv[2]);
        } else if (mode == "gpucheck") {
            gpucheck();
        } else if (mode == "rows" && argc == 4) {
            rows(argv[2], argv[3]);
        } else if (mode == "vol" && argc == 4) {
            vol(argv[2], argv[3]);
        } else if (mode == "stab" && argc == 5) {
            stab_rows(argv[2], argv[3], std::atoi(argv[4]));
        } else if (mode == "metrics" && argc == 4) {
            metrics(argv[2], argv[3]);
        } else if (mode == "records" && argc == 4) {
            records(argv[2], argv[3]);
        } else {
            std::fprintf(stderr, "usage: dropin_test selftest DIR | gpucheck | rows IN OUT | vol SPK DIR | "
                                 "stab IN OUT DEPTH | metrics SPK DIR | records SPK DIR\n");
            return 2;
        }
    } catch (const std::exception& e) {
        std::fprintf(stderr, "uncaught exception: %s\n", e.what());
        return 1;
    }
    if (g_fail) std::fprintf(stderr, "%d check(s) failed\n", g_fail);
    return g_fail ? 1 : 0;
}
