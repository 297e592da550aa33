// spikecam_b200.cpp -- the C++ drop-in (include/spikecam/b200.hpp) over the
// C-ABI of libspikecam_b200.so.  Reconstruction and segmentation are single
// calls into the GPU library (spk_reconstruct_host / spk_segment_host); what
// runs here is only the reference's container handling around them: value
// checks of core.cpp, SpikeVolume bytes <-> SPK1 bit packing (io.cpp:52-76),
// file headers (io.cpp:185-223) and turning run lists back into Segment
// objects.  A missing or failing GPU surfaces as std::runtime_error.
#include "spikecam/b200.hpp"

#include <algorithm>
#include <chrono>
#include <array>
#include <cmath>
#include <cstring>
#include <fstream>
#include <iterator>
#include <limits>
#include <set>

#include "spikecam_b200.h"

namespace spikecam {

namespace {

[[noreturn]] void raise(int rc) {
    const std::string msg = spk_last_error();
    if (rc == SPK_EINVAL) throw std::invalid_argument(msg);
    if (rc == SPK_ENOMEM) throw std::bad_alloc();
    throw std::runtime_error("spikecam_b200: " + msg);
}

inline void ck(int rc) {
    if (rc != SPK_OK) raise(rc);
}

size_t plane_bytes(int w, int h) { return (static_cast<size_t>(w) * h + 7) / 8; }

// byte b -> eight 0/1 bytes, bit i of b into byte i (LSB-first)
const std::array<uint64_t, 256>& spread_table(bool msb_first) {
    static const auto make = [](bool msb) {
        std::array<uint64_t, 256> t{};
        for (int b = 0; b < 256; ++b)
            for (int i = 0; i < 8; ++i)
                if ((b >> (msb ? 7 - i : i)) & 1) t[b] |= uint64_t{1} << (8 * i);
        return t;
    };
    static const std::array<uint64_t, 256> lsb = make(false), msb = make(true);
    return msb_first ? msb : lsb;
}

// eight bytes (any nonzero = spike) -> one LSB-first byte
inline uint8_t gather8(uint64_t v) {
    constexpr uint64_t k7f = 0x7f7f7f7f7f7f7f7fULL, k80 = 0x8080808080808080ULL;
    const uint64_t nz = (((v & k7f) + k7f) | v) & k80;  // high bit of each nonzero byte
    return static_cast<uint8_t>(((nz >> 7) * 0x0102040810204080ULL) >> 56);
}

// one frame of SpikeVolume bytes -> SPK1 plane (pack_frame, io.cpp:52-64)
void pack_plane(const uint8_t* src, size_t npix, uint8_t* dst) {
    const size_t full = npix / 8;
    for (size_t j = 0; j < full; ++j) {
        uint64_t v;
        std::memcpy(&v, src + 8 * j, 8);
        dst[j] = gather8(v);
    }
    if (npix % 8) {
        uint8_t b = 0;
        for (size_t p = full * 8; p < npix; ++p) b |= static_cast<uint8_t>((src[p] != 0) << (p % 8));
        dst[full] = b;
    }
}

// SPK1 plane -> SpikeVolume bytes (unpack_frame, io.cpp:66-76)
void unpack_plane(const uint8_t* src, size_t npix, bool msb_first, uint8_t* dst) {
    const auto& t = spread_table(msb_first);
    const size_t full = npix / 8;
    for (size_t j = 0; j < full; ++j) std::memcpy(dst + 8 * j, &t[src[j]], 8);
    for (size_t p = full * 8; p < npix; ++p) {
        const int shift = msb_first ? 7 - static_cast<int>(p % 8) : static_cast<int>(p % 8);
        dst[p] = (src[p / 8] >> shift) & 1;
    }
}

std::vector<uint8_t> read_file(const std::filesystem::path& path) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw io_error("cannot open " + path.string());
    std::vector<uint8_t> data((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
    if (in.bad()) throw io_error("read failure on " + path.string());
    return data;
}

void write_file(const std::filesystem::path& path, const uint8_t* data, size_t n) {
    std::ofstream out(path, std::ios::binary | std::ios::trunc);
    if (!out) throw io_error("cannot create " + path.string());
    out.write(reinterpret_cast<const char*>(data), static_cast<std::streamsize>(n));
    if (!out) throw io_error("write failure on " + path.string());
}

inline uint32_t le32(const uint8_t* p) {
    return uint32_t{p[0]} | uint32_t{p[1]} << 8 | uint32_t{p[2]} << 16 | uint32_t{p[3]} << 24;
}
inline void put_le(uint8_t* p, uint32_t v, int n) {
    for (int i = 0; i < n; ++i) p[i] = static_cast<uint8_t>(v >> (8 * i));
}

spk_geom geom(int w, int h, long frames) { return spk_geom{w, h, frames, 0}; }

// one pixel stream as a 1x1 SPK1 payload (bit n of byte n/8)
std::vector<uint8_t> stream_payload(const SpikeLikeStream& s) {
    std::vector<uint8_t> pay(s.size(), 0);
    for (size_t n = 0; n < s.size(); ++n) pay[n] = s.values[n] == s.firing_value ? 1 : 0;
    return pay;  // 1 pixel -> one byte per plane, bit 0
}

// workers > 1 with several visible CUDA devices: min(workers, devices)
// pixel bands, one per device (spk_reconstruct_host_multi); otherwise one
// call on the current device.  The result is the same for any worker count.
template <typename T>
std::vector<T> recon_host(const PackedSpikes& sp, ReconMethod m, int out_type, int workers = 1) {
    const size_t npix = static_cast<size_t>(sp.width) * sp.height;
    std::vector<T> out(npix * sp.frames);
    const spk_geom g = geom(sp.width, sp.height, sp.frames);
    if (sp.payload.size() != plane_bytes(sp.width, sp.height) * sp.frames)
        throw std::invalid_argument("PackedSpikes: payload size does not match the geometry");
    // one band per GPU, at most `workers` of them (narrow bands on one device
    // would only add copies: the single call already fills the GPU)
    const int nbands = std::min(std::max(workers, 1), std::max(1, spk_device_count()));
    if (nbands > 1) {
        std::vector<int32_t> devs(static_cast<size_t>(nbands));
        for (int i = 0; i < nbands; ++i) devs[static_cast<size_t>(i)] = i;
        ck(spk_reconstruct_host_multi(&g, sp.payload.data(), static_cast<int>(m.kind), m.tfp_window,
                                      out_type, out.data(), npix, devs.data(), nbands));
    } else {
        ck(spk_reconstruct_host(&g, sp.payload.data(), static_cast<int>(m.kind), m.tfp_window,
                                out_type, out.data(), npix));
    }
    return out;
}

void check_method(ReconMethod m) {
    if (m.kind == Method::tfp && m.tfp_window < 1)
        throw std::invalid_argument("tfp window must be >= 1");
}

// Segments of one stream from its GPU run list (build_segments semantics,
// reconstruct.cpp:106-130): degenerate lead [0, first spike) when the first
// spike is not frame 0, one segment per run, a degenerate tail from the last
// spike carrying the last run's value; no spike -> one segment [0, T).
std::vector<Segment> segments_of(const SpikeLikeStream& stream, Method kind) {
    std::vector<Segment> segs;
    const long T = static_cast<long>(stream.size());
    if (T == 0) return segs;
    const std::vector<long> spikes = stream.firing_positions();
    const std::vector<uint8_t> pay = stream_payload(stream);
    const spk_geom g = geom(1, 1, T);
    const int64_t cap = std::max<long>(1, static_cast<long>(spikes.size()));
    std::vector<spk_run> runs(static_cast<size_t>(cap));
    uint32_t count = 0;
    int32_t last = -1;
    ck(spk_segment_host(&g, pay.data(), kind == Method::fsr ? SPK_FSR : SPK_SSR, runs.data(), cap,
                        &count, &last));
    if (spikes.empty()) {
        segs.emplace_back(0, T, IntervalStream{}, 0.0);
        return segs;
    }
    if (last != spikes.back() || count > static_cast<uint32_t>(cap))
        throw std::runtime_error("spikecam_b200: inconsistent run list from the device");
    if (spikes.front() > 0) segs.emplace_back(0, spikes.front(), IntervalStream{}, 0.0);
    double carry = 0.0;
    size_t a = 0;  // spike index of the current run's first spike
    for (uint32_t k = 0; k < count; ++k) {
        const size_t b = a + runs[k].intervals;
        if (runs[k].intervals == 0 || b >= spikes.size() || spikes[a] != runs[k].start)
            throw std::runtime_error("spikecam_b200: inconsistent run list from the device");
        std::vector<int> iv(b - a);
        for (size_t i = a; i < b; ++i) iv[i - a] = static_cast<int>(spikes[i + 1] - spikes[i]);
        carry = 255.0 * static_cast<double>(b - a) / static_cast<double>(spikes[b] - spikes[a]);
        segs.emplace_back(spikes[a], spikes[b], IntervalStream(std::move(iv)), carry);
        a = b;
    }
    if (a != spikes.size() - 1)
        throw std::runtime_error("spikecam_b200: run list does not cover the stream");
    segs.emplace_back(spikes.back(), T, IntervalStream{}, carry);
    return segs;
}

}  // namespace

// ---------------------------------------------------------------- types ----
SpikeVolume::SpikeVolume(int width, int height, int frames)
    : width_(width), height_(height), frames_(frames) {
    if (width < 1 || height < 1 || frames < 0)
        throw std::invalid_argument("SpikeVolume: width/height must be >= 1, frames >= 0");
    bits_.assign(static_cast<size_t>(width) * height * frames, 0);
}

size_t SpikeVolume::index(int x, int y, int n) const {
    if (x < 0 || x >= width_ || y < 0 || y >= height_ || n < 0 || n >= frames_)
        throw std::out_of_range("SpikeVolume: index (" + std::to_string(x) + ", " +
                                std::to_string(y) + ", " + std::to_string(n) + ") out of bounds");
    return (static_cast<size_t>(n) * height_ + y) * width_ + x;
}

bool SpikeVolume::at(int x, int y, int n) const { return bits_[index(x, y, n)] != 0; }
void SpikeVolume::set(int x, int y, int n, bool v) { bits_[index(x, y, n)] = v ? 1 : 0; }

SpikeLikeStream::SpikeLikeStream(std::vector<int> vals, int e1, std::optional<int> e2)
    : values(std::move(vals)), firing_value(e1), resting_value(e2) {
    if (e2 && *e2 == e1)
        throw std::invalid_argument("SpikeLikeStream: firing and resting values must differ");
    for (int v : values)
        if (v != e1 && !(e2 && v == *e2))
            throw std::invalid_argument("SpikeLikeStream: element " + std::to_string(v) +
                                        " is neither the firing nor the resting value");
}

SpikeLikeStream SpikeLikeStream::from_values(std::vector<int> vals) {
    const std::set<int> seen(vals.begin(), vals.end());
    if (seen.size() > 2) throw std::invalid_argument("SpikeLikeStream: more than two distinct values");
    if (seen.empty()) return SpikeLikeStream({}, 1, 0);
    std::optional<int> rest;
    if (seen.size() == 2) rest = *seen.begin();
    return SpikeLikeStream(std::move(vals), *seen.rbegin(), rest);
}

std::vector<long> SpikeLikeStream::firing_positions() const {
    std::vector<long> pos;
    for (size_t i = 0; i < values.size(); ++i)
        if (values[i] == firing_value) pos.push_back(static_cast<long>(i));
    return pos;
}

IntervalStream::IntervalStream(std::vector<int> ivals) : intervals(std::move(ivals)) {
    for (int t : intervals)
        if (t < 1) throw std::invalid_argument("IntervalStream: intervals must be >= 1");
}

Segment::Segment(long start, long end, IntervalStream ivals, double inten)
    : start_frame(start), end_frame(end), intervals(std::move(ivals)), intensity(inten) {
    if (start >= end) throw std::invalid_argument("Segment: start_frame must precede end_frame");
    if (!(inten >= 0.0 && inten <= 255.0))
        throw std::invalid_argument("Segment: intensity out of [0, 255]");
}

IntensityImage::IntensityImage(int w, int h, double fill) : width(w), height(h) {
    if (w < 1 || h < 1) throw std::invalid_argument("IntensityImage: empty dimensions");
    values.assign(static_cast<size_t>(w) * h, fill);
}

SpikeLikeStream pixel_stream(const SpikeVolume& volume, int x, int y) {
    if (x < 0 || x >= volume.width() || y < 0 || y >= volume.height())
        throw std::out_of_range("pixel_stream: coordinates out of bounds");
    std::vector<int> vals(static_cast<size_t>(volume.frames()));
    for (int n = 0; n < volume.frames(); ++n) vals[n] = volume.at(x, y, n) ? 1 : 0;
    return SpikeLikeStream(std::move(vals), 1, 0);
}

// ------------------------------------------------------- reconstruction ----
ReconMethod ReconMethod::parse(const std::string& name, int window) {
    if (name == "fsr") return {Method::fsr};
    if (name == "ssr") return {Method::ssr};
    if (name == "tfi") return {Method::tfi};
    if (name == "tfp") {
        if (window < 1) throw std::invalid_argument("tfp window must be >= 1");
        return {Method::tfp, window};
    }
    throw std::invalid_argument("unknown reconstruction method: " + name);
}

std::string ReconMethod::name() const {
    switch (kind) {
        case Method::fsr: return "fsr";
        case Method::ssr: return "ssr";
        case Method::tfi: return "tfi";
        case Method::tfp: return "tfp-" + std::to_string(tfp_window);
    }
    return "?";
}

std::vector<Segment> segment_fsr(const SpikeLikeStream& stream) {
    return segments_of(stream, Method::fsr);
}

std::vector<Segment> segment_ssr(const SpikeLikeStream& stream) {
    return segments_of(stream, Method::ssr);
}

double segment_intensity(const Segment& segment) {
    if (segment.degenerate())
        throw std::invalid_argument("segment_intensity: degenerate segment has no interval");
    long sum = 0;
    for (int t : segment.intervals.intervals) sum += t;
    return 255.0 * static_cast<double>(segment.intervals.size()) / static_cast<double>(sum);
}

std::vector<SegmentEvent> fsr_events(const SpikeLikeStream& stream) {
    std::vector<SegmentEvent> ev;
    for (const Segment& s : segment_fsr(stream)) ev.push_back({s.duration(), s.intensity});
    return ev;
}

std::vector<double> reconstruct_pixel(const SpikeLikeStream& stream, ReconMethod method) {
    check_method(method);
    PackedSpikes sp;
    sp.width = sp.height = 1;
    sp.frames = static_cast<uint32_t>(stream.size());
    sp.payload = stream_payload(stream);
    return recon_host<double>(sp, method, SPK_OUT_F64);
}

void reconstruct(const SpikeVolume& volume, ReconMethod method, int workers,
                 std::vector<IntensityImage>& out) {
    // workers <= 0: the default (one GPU); the result does not depend on it
    check_method(method);
    const int W = volume.width(), H = volume.height();
    const size_t T = static_cast<size_t>(volume.frames());
    if (out.size() != T || (T > 0 && (out[0].width != W || out[0].height != H)))
        out.assign(T, IntensityImage(W, H));  // reuse rule of reconstruct.cpp:452-455
    if (T == 0) return;
    const std::vector<double> frames = recon_host<double>(pack(volume), method, SPK_OUT_F64, workers);
    const size_t npix = static_cast<size_t>(W) * H;
    for (size_t n = 0; n < T; ++n)
        std::copy_n(frames.begin() + n * npix, npix, out[n].values.begin());
}

std::vector<IntensityImage> reconstruct(const SpikeVolume& volume, ReconMethod method, int workers) {
    std::vector<IntensityImage> out;
    reconstruct(volume, method, workers, out);
    return out;
}

std::vector<IntensityImage> reconstruct_serial(const SpikeVolume& volume, ReconMethod method) {
    return reconstruct(volume, method, 1);
}

std::vector<std::vector<uint8_t>> reconstruct_u8(const SpikeVolume& volume, ReconMethod method) {
    const std::vector<uint8_t> flat = reconstruct_u8(pack(volume), method);
    const size_t npix = static_cast<size_t>(volume.width()) * volume.height();
    std::vector<std::vector<uint8_t>> frames(static_cast<size_t>(volume.frames()));
    for (size_t n = 0; n < frames.size(); ++n)
        frames[n].assign(flat.begin() + n * npix, flat.begin() + (n + 1) * npix);
    return frames;
}

std::vector<uint8_t> reconstruct_u8(const PackedSpikes& spikes, ReconMethod method) {
    check_method(method);
    return recon_host<uint8_t>(spikes, method, SPK_OUT_U8);
}

std::vector<double> reconstruct_f64(const PackedSpikes& spikes, ReconMethod method) {
    check_method(method);
    return recon_host<double>(spikes, method, SPK_OUT_F64);
}

PackedSpikes pack(const SpikeVolume& volume, uint32_t fps) {
    PackedSpikes sp;
    sp.width = volume.width();
    sp.height = volume.height();
    sp.fps = fps;
    sp.frames = static_cast<uint32_t>(volume.frames());
    const size_t npix = static_cast<size_t>(sp.width) * sp.height, fb = plane_bytes(sp.width, sp.height);
    sp.payload.assign(fb * sp.frames, 0);
    const uint8_t* raw = volume.raw().data();
    for (size_t n = 0; n < sp.frames; ++n) pack_plane(raw + n * npix, npix, sp.payload.data() + n * fb);
    return sp;
}

// ------------------------------------------------------------- streaming ----
namespace {

std::vector<std::vector<SegmentEvent>> take_events(spk_event* ev, uint64_t* offs, uint64_t total,
                                                   size_t npix) {
    std::vector<std::vector<SegmentEvent>> out(npix);
    for (size_t p = 0; p < npix; ++p)
        for (uint64_t i = offs[p]; i < offs[p + 1] && i < total; ++i)
            out[p].push_back(SegmentEvent{static_cast<long>(ev[i].duration), ev[i].intensity});
    spk_free_host(ev);
    spk_free_host(offs);
    return out;
}

spk_stream* make_stream(int w, int h) {
    spk_stream* st = nullptr;
    ck(spk_stream_create(w, h, nullptr, &st));
    return st;
}

}  // namespace

PixelReconState::PixelReconState() : stream_(make_stream(1, 1)) {}
PixelReconState::~PixelReconState() {
    if (stream_) spk_stream_destroy(static_cast<spk_stream*>(stream_));
}
PixelReconState::PixelReconState(PixelReconState&& o) noexcept
    : stream_(o.stream_), pending_(std::move(o.pending_)), frame_(o.frame_) {
    o.stream_ = nullptr;
}
PixelReconState& PixelReconState::operator=(PixelReconState&& o) noexcept {
    if (this != &o) {
        if (stream_) spk_stream_destroy(static_cast<spk_stream*>(stream_));
        stream_ = o.stream_;
        pending_ = std::move(o.pending_);
        frame_ = o.frame_;
        o.stream_ = nullptr;
    }
    return *this;
}

std::vector<SegmentEvent> PixelReconState::push_pending() {
    if (pending_.empty()) return {};
    spk_event* ev = nullptr;
    uint64_t* offs = nullptr;
    uint64_t total = 0;
    // one pixel: one payload byte per frame, the spike in bit 0
    ck(spk_stream_push_host(static_cast<spk_stream*>(stream_), pending_.data(),
                            static_cast<int64_t>(pending_.size()), &ev, &offs, &total));
    pending_.clear();
    return take_events(ev, offs, total, 1)[0];
}

std::optional<SegmentEvent> PixelReconState::push_frame(bool bit) {
    pending_.push_back(bit ? 1 : 0);
    ++frame_;
    if (!bit) return std::nullopt;  // a segment only closes at a spike
    std::vector<SegmentEvent> ev = push_pending();
    if (ev.empty()) return std::nullopt;
    return ev.back();
}

std::vector<SegmentEvent> PixelReconState::flush() {
    push_pending();
    spk_event* ev = nullptr;
    uint64_t* offs = nullptr;
    uint64_t total = 0;
    ck(spk_stream_flush_host(static_cast<spk_stream*>(stream_), &ev, &offs, &total));
    return take_events(ev, offs, total, 1)[0];
}

EventStream::EventStream(int width, int height)
    : stream_(make_stream(width, height)), width_(width), height_(height) {}
EventStream::~EventStream() {
    if (stream_) spk_stream_destroy(static_cast<spk_stream*>(stream_));
}

std::vector<std::vector<SegmentEvent>> EventStream::push(const std::vector<uint8_t>& payload, long frames) {
    if (payload.size() != plane_bytes(width_, height_) * static_cast<size_t>(frames))
        throw std::invalid_argument("EventStream::push: payload size does not match the frames");
    spk_event* ev = nullptr;
    uint64_t* offs = nullptr;
    uint64_t total = 0;
    ck(spk_stream_push_host(static_cast<spk_stream*>(stream_), payload.data(), frames, &ev, &offs, &total));
    return take_events(ev, offs, total, static_cast<size_t>(width_) * height_);
}

std::vector<std::vector<SegmentEvent>> EventStream::flush() {
    spk_event* ev = nullptr;
    uint64_t* offs = nullptr;
    uint64_t total = 0;
    ck(spk_stream_flush_host(static_cast<spk_stream*>(stream_), &ev, &offs, &total));
    return take_events(ev, offs, total, static_cast<size_t>(width_) * height_);
}

long EventStream::frames() const { return static_cast<long>(spk_stream_frames(static_cast<spk_stream*>(stream_))); }

// ------------------------------------------ metrics / stability (device) ----
namespace {

std::vector<double> metrics_of(const std::vector<IntensityImage>& images,
                               const std::vector<IntensityImage>* refs) {
    if (images.empty()) return {};
    const int w = images[0].width, h = images[0].height;
    const size_t npix = static_cast<size_t>(w) * h, t = images.size();
    std::vector<double> frames(npix * t), ref;
    for (size_t n = 0; n < t; ++n) {
        if (images[n].width != w || images[n].height != h)
            throw std::invalid_argument("two_dimensional_entropy: images differ in size");
        std::copy(images[n].values.begin(), images[n].values.end(), frames.begin() + n * npix);
    }
    if (refs) {
        ref.resize(npix * t);
        for (size_t n = 0; n < t; ++n)
            std::copy((*refs)[n].values.begin(), (*refs)[n].values.end(), ref.begin() + n * npix);
    }
    const spk_geom g = geom(w, h, static_cast<long>(t));
    std::vector<double> out(t);
    ck(spk_frame_metrics_host(&g, frames.data(), SPK_OUT_F64, npix, refs ? ref.data() : nullptr,
                              SPK_OUT_F64, npix, refs ? nullptr : out.data(),
                              refs ? out.data() : nullptr));
    return out;
}

StabilityReport report_of(const spk_stab& r) {
    StabilityReport rep;
    rep.verified_order = r.verified_order;
    rep.absolute = r.absolute != 0;
    if (r.depth > 0) {
        ViolationInfo v;
        v.depth = r.depth;
        v.index = static_cast<size_t>(r.index);
        for (int j = 0; j < r.path_len; ++j) v.path.push_back((r.path >> j) & 1 ? '+' : '-');
        rep.first_violation = std::move(v);
    }
    return rep;
}

void check_depth(int max_depth) {
    if (max_depth < 1) throw std::invalid_argument("stability_order: max_depth must be >= 1");
}

}  // namespace

double two_dimensional_entropy(const IntensityImage& image) {
    if (image.width < 3 || image.height < 3)
        throw std::invalid_argument("two_dimensional_entropy: image must be at least 3x3");
    return metrics_of({image}, nullptr)[0];
}

std::vector<double> two_dimensional_entropy(const std::vector<IntensityImage>& images) {
    if (!images.empty() && (images[0].width < 3 || images[0].height < 3))
        throw std::invalid_argument("two_dimensional_entropy: image must be at least 3x3");
    return metrics_of(images, nullptr);
}

double mse(const IntensityImage& image, const IntensityImage& reference) {
    if (image.width != reference.width || image.height != reference.height)
        throw std::invalid_argument("mse: dimension mismatch");
    const std::vector<IntensityImage> refs{reference};
    return metrics_of({image}, &refs)[0];
}

double psnr(const IntensityImage& image, const IntensityImage& reference) {
    const double m = mse(image, reference);
    if (m == 0.0) return std::numeric_limits<double>::infinity();
    return 10.0 * std::log10(255.0 * 255.0 / m);
}

StabilityReport stability_order(const SpikeLikeStream& stream, int max_depth) {
    check_depth(max_depth);
    const std::vector<uint8_t> pay = stream_payload(stream);
    const spk_geom g = geom(1, 1, static_cast<long>(stream.size()));
    spk_stab r{};
    ck(spk_stability_host(&g, pay.data(), max_depth, &r));
    return report_of(r);
}

std::vector<StabilityReport> stability_order(const SpikeVolume& volume, int max_depth) {
    check_depth(max_depth);
    const PackedSpikes sp = pack(volume);
    const spk_geom g = geom(volume.width(), volume.height(), volume.frames());
    std::vector<spk_stab> r(static_cast<size_t>(volume.width()) * volume.height());
    ck(spk_stability_host(&g, sp.payload.data(), max_depth, r.data()));
    std::vector<StabilityReport> out;
    out.reserve(r.size());
    for (const auto& x : r) out.push_back(report_of(x));
    return out;
}

// ------------------------------------------------------------------- io ----
PackedSpikes read_spk_packed(const std::filesystem::path& path) {
    std::vector<uint8_t> data = read_file(path);
    if (data.size() < 16 || std::memcmp(data.data(), "SPK1", 4) != 0)
        throw io_error("bad SPK1 magic in " + path.string());
    PackedSpikes sp;
    sp.width = data[4] | data[5] << 8;
    sp.height = data[6] | data[7] << 8;
    sp.fps = le32(data.data() + 8);
    sp.frames = le32(data.data() + 12);
    if (sp.width < 1 || sp.height < 1) throw io_error("empty geometry in " + path.string());
    const size_t expect = 16 + plane_bytes(sp.width, sp.height) * sp.frames;
    if (data.size() != expect)
        throw io_error("SPK1 length mismatch in " + path.string() + ": expected " +
                       std::to_string(expect) + " bytes, got " + std::to_string(data.size()));
    sp.payload.assign(data.begin() + 16, data.end());
    return sp;
}

std::pair<SpikeVolume, uint32_t> read_spk(const std::filesystem::path& path) {
    const PackedSpikes sp = read_spk_packed(path);
    SpikeVolume v(sp.width, sp.height, static_cast<int>(sp.frames));
    const size_t npix = static_cast<size_t>(sp.width) * sp.height, fb = plane_bytes(sp.width, sp.height);
    for (size_t n = 0; n < sp.frames; ++n)
        unpack_plane(sp.payload.data() + n * fb, npix, false, v.raw_mutable().data() + n * npix);
    return {std::move(v), sp.fps};
}

SpikeVolume read_raw(const std::filesystem::path& path, int width, int height, bool msb_first) {
    const std::vector<uint8_t> data = read_file(path);
    const size_t fb = plane_bytes(width, height);
    if (data.size() % fb != 0)
        throw io_error("raw file " + path.string() + " (" + std::to_string(data.size()) +
                       " bytes) is not a multiple of the " + std::to_string(fb) +
                       "-byte frame size for " + std::to_string(width) + "x" +
                       std::to_string(height) + "; check --width/--height");
    const int frames = static_cast<int>(data.size() / fb);
    SpikeVolume v(width, height, frames);
    const size_t npix = static_cast<size_t>(width) * height;
    for (int n = 0; n < frames; ++n)
        unpack_plane(data.data() + n * fb, npix, msb_first, v.raw_mutable().data() + n * npix);
    return v;
}

void write_spk(const SpikeVolume& volume, uint32_t fps, const std::filesystem::path& path) {
    const PackedSpikes sp = pack(volume, fps);
    std::vector<uint8_t> data(16 + sp.payload.size());
    std::memcpy(data.data(), "SPK1", 4);
    put_le(data.data() + 4, static_cast<uint32_t>(sp.width), 2);
    put_le(data.data() + 6, static_cast<uint32_t>(sp.height), 2);
    put_le(data.data() + 8, fps, 4);
    put_le(data.data() + 12, sp.frames, 4);
    std::copy(sp.payload.begin(), sp.payload.end(), data.begin() + 16);
    write_file(path, data.data(), data.size());
}

void write_image(const IntensityImage& image, const std::filesystem::path& path, ImageFormat format) {
    if (format != ImageFormat::pgm)
        throw io_error("png output is not built into spikecam_b200: " + path.string());
    const std::string head =
        "P5\n" + std::to_string(image.width) + " " + std::to_string(image.height) + "\n255\n";
    std::vector<uint8_t> data(head.begin(), head.end());
    data.reserve(head.size() + image.values.size());
    for (double v : image.values)  // quantize(), io.cpp:78-81
        data.push_back(static_cast<uint8_t>(std::round(std::clamp(v, 0.0, 255.0))));
    write_file(path, data.data(), data.size());
}

IntensityImage read_image(const std::filesystem::path& path) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw io_error("cannot open " + path.string());
    std::string magic;
    int w = 0, h = 0, maxval = 0;
    in >> magic >> w >> h >> maxval;
    if (magic != "P5" || maxval != 255 || w < 1 || h < 1)
        throw io_error("not an 8-bit P5 PGM: " + path.string());
    in.get();
    std::vector<uint8_t> px(static_cast<size_t>(w) * h);
    in.read(reinterpret_cast<char*>(px.data()), static_cast<std::streamsize>(px.size()));
    if (!in) throw io_error("truncated PGM payload: " + path.string());
    IntensityImage img(w, h);
    std::copy(px.begin(), px.end(), img.values.begin());
    return img;
}

// ----------------------------------------------------------------- SPKR ----
// write_spkr / read_spkr (io.cpp:240-292): same layout, checks and messages.
void write_spkr(const RecordVolume& records, const std::filesystem::path& path) {
    if (records.words.size() != static_cast<size_t>(records.width) * records.height)
        throw io_error("SPKR record table does not match geometry");
    size_t total = 16;
    for (const auto& w : records.words) total += 4 + 2 * w.size();
    std::vector<uint8_t> data(total);
    std::memcpy(data.data(), "SPKR", 4);
    put_le(data.data() + 4, static_cast<uint32_t>(records.width), 2);
    put_le(data.data() + 6, static_cast<uint32_t>(records.height), 2);
    put_le(data.data() + 8, records.fps, 4);
    put_le(data.data() + 12, records.frame_count, 4);
    size_t pos = 16;
    for (const auto& w : records.words) {
        put_le(data.data() + pos, static_cast<uint32_t>(w.size()), 4);
        pos += 4;
        for (uint16_t x : w) {
            put_le(data.data() + pos, x, 2);
            pos += 2;
        }
    }
    write_file(path, data.data(), data.size());
}

namespace {

RecordVolume parse_spkr(const uint8_t* data, size_t size, const std::string& name) {
    if (size < 16 || std::memcmp(data, "SPKR", 4) != 0) throw io_error("bad SPKR magic in " + name);
    RecordVolume rv;
    rv.width = data[4] | data[5] << 8;
    rv.height = data[6] | data[7] << 8;
    rv.fps = le32(data + 8);
    rv.frame_count = le32(data + 12);
    if (rv.width < 1 || rv.height < 1) throw io_error("empty geometry in " + name);
    const size_t pixels = static_cast<size_t>(rv.width) * rv.height;
    rv.words.resize(pixels);
    size_t pos = 16;
    for (size_t p = 0; p < pixels; ++p) {
        if (pos + 4 > size) throw io_error("truncated SPKR record table: " + name);
        const uint32_t count = le32(data + pos);
        pos += 4;
        if (pos + 2ull * count > size) throw io_error("truncated SPKR records: " + name);
        auto& w = rv.words[p];
        w.resize(count);
        for (uint32_t i = 0; i < count; ++i, pos += 2) w[i] = static_cast<uint16_t>(data[pos] | data[pos + 1] << 8);
    }
    if (pos != size) throw io_error("trailing bytes after SPKR records in " + name);
    return rv;
}

}  // namespace

RecordVolume read_spkr(const std::filesystem::path& path) {
    const std::vector<uint8_t> data = read_file(path);
    return parse_spkr(data.data(), data.size(), path.string());
}

RecordVolume emit_records(const SpikeVolume& volume, ReconMethod method, uint32_t fps) {
    if (method.kind != Method::fsr && method.kind != Method::ssr)
        throw std::invalid_argument("--emit-records needs method fsr or ssr");
    if (volume.width() > 65535 || volume.height() > 65535)
        throw std::invalid_argument("SPKR geometry is 16-bit: width/height must be <= 65535");
    const PackedSpikes sp = pack(volume, fps);
    const spk_geom g = geom(volume.width(), volume.height(), volume.frames());
    void* img = nullptr;
    uint64_t bytes = 0;
    ck(spk_records_host(&g, sp.payload.data(), static_cast<int>(method.kind), fps, &img, &bytes));
    try {
        RecordVolume rv = parse_spkr(static_cast<const uint8_t*>(img), static_cast<size_t>(bytes), "device image");
        spk_free_host(img);
        return rv;
    } catch (...) {
        spk_free_host(img);
        throw;
    }
}

// ---------------------------------------------------------------- codec ----
// encode_append / encode / encode_events / decode (codec.cpp:8-41): same
// rules and exceptions.
void encode_append(std::vector<uint16_t>& words, long duration, double intensity) {
    if (duration < 1) throw std::invalid_argument("encode: duration must be >= 1");
    if (!(intensity >= 0.0 && intensity <= 255.0)) throw std::invalid_argument("encode: intensity outside [0, 255]");
    const uint16_t q = static_cast<uint16_t>(std::lround(intensity));
    for (; duration > 255; duration -= 255) words.push_back(static_cast<uint16_t>(0xff00u | q));
    words.push_back(static_cast<uint16_t>(static_cast<uint16_t>(duration) << 8 | q));
}

std::vector<uint16_t> encode(long duration, double intensity) {
    std::vector<uint16_t> words;
    encode_append(words, duration, intensity);
    return words;
}

std::vector<uint16_t> encode_events(std::span<const SegmentEvent> events) {
    std::vector<uint16_t> words;
    for (const SegmentEvent& e : events) encode_append(words, e.duration, e.intensity);
    return words;
}

std::vector<uint8_t> decode(std::span<const uint16_t> words) {
    size_t n = 0;
    for (uint16_t w : words) {
        if (duration_of(w) == 0) throw std::runtime_error("decode: zero-duration record");
        n += static_cast<size_t>(duration_of(w));
    }
    std::vector<uint8_t> frames;
    frames.reserve(n);
    for (uint16_t w : words) frames.insert(frames.end(), static_cast<size_t>(duration_of(w)), static_cast<uint8_t>(intensity_of(w)));
    return frames;
}

// ---------------------------------------------------------------- bench ----
BenchResult bench(const SpikeVolume& volume, ReconMethod method, int repeats, int workers) {
    if (repeats < 3) throw std::invalid_argument("bench: repeats must be >= 3");
    std::vector<double> fps(static_cast<size_t>(repeats));
    std::vector<IntensityImage> images;  // reused across repeats, as the reference
    for (int r = 0; r < repeats; ++r) {
        const auto t0 = std::chrono::steady_clock::now();
        reconstruct(volume, method, workers, images);
        const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        fps[static_cast<size_t>(r)] = volume.frames() / std::max(s, 1e-12);
    }
    std::sort(fps.begin(), fps.end());
    const size_t h = static_cast<size_t>(repeats / 2);
    const double median = repeats % 2 ? fps[h] : 0.5 * (fps[h - 1] + fps[h]);
    return {method.name(), volume.width(), volume.height(), volume.frames(), workers, repeats, median};
}

}  // namespace spikecam
