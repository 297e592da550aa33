// spikecam/b200.hpp -- C++ drop-in for the reconstruction surface of the
// reference library (namespace spikecam, proj/include/spikecam/{core,
// reconstruct,io,codec,metrics}.hpp -- each of those names is also provided
// in include/spikecam/ and includes this header), implemented over the sm_100a C-ABI
// (include/spikecam_b200.h).  Same names, signatures, value semantics and
// exception classes as the reference, so its callers
// (proj/tools/spikecam_main.cpp:174,271, proj/src/metrics.cpp:71, the tests)
// compile against this header unchanged.  Every reconstruction runs on the
// GPU; there is no CPU code path for it.
//
// Also on the device: the quality metrics (metrics.hpp) and stability_order
// (stability.hpp), SURVEY.md 8(f) row 4.  Not provided: the simulator, the
// Lemma 1/2 helpers and the PNG writer -- outside the accelerated path.
#pragma once

#include <cstdint>
#include <filesystem>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace spikecam {

// ---------------------------------------------------------------- types ----
// W x H x T binary volume, frame-major, one byte per bit (core.hpp:15-49).
class SpikeVolume {
public:
    SpikeVolume(int width, int height, int frames);
    int width() const { return width_; }
    int height() const { return height_; }
    int frames() const { return frames_; }
    bool at(int x, int y, int n) const;
    void set(int x, int y, int n, bool v);
    std::span<const uint8_t> raw() const { return bits_; }
    std::span<uint8_t> raw_mutable() { return bits_; }
    bool operator==(const SpikeVolume&) const = default;

private:
    size_t index(int x, int y, int n) const;
    int width_, height_, frames_;
    std::vector<uint8_t> bits_;
};

// Integer sequence with firing value e1 and optional resting value e2 (core.hpp:54-69).
struct SpikeLikeStream {
    std::vector<int> values;
    int firing_value = 1;
    std::optional<int> resting_value;
    SpikeLikeStream() = default;
    SpikeLikeStream(std::vector<int> vals, int e1, std::optional<int> e2);
    static SpikeLikeStream from_values(std::vector<int> vals);
    size_t size() const { return values.size(); }
    std::vector<long> firing_positions() const;
};

struct IntervalStream {
    std::vector<int> intervals;
    IntervalStream() = default;
    explicit IntervalStream(std::vector<int> ivals);
    size_t size() const { return intervals.size(); }
    bool empty() const { return intervals.empty(); }
};

// Half-open frame span of one stable run (core.hpp:85-96); degenerate = no interval.
struct Segment {
    long start_frame = 0;
    long end_frame = 0;
    IntervalStream intervals;
    double intensity = 0.0;
    Segment() = default;
    Segment(long start, long end, IntervalStream ivals, double inten);
    bool degenerate() const { return intervals.empty(); }
    long duration() const { return end_frame - start_frame; }
};

struct IntensityImage {
    int width = 0;
    int height = 0;
    std::vector<double> values;  // row-major, [0, 255]
    IntensityImage() = default;
    IntensityImage(int w, int h, double fill = 0.0);
    double at(int x, int y) const { return values[static_cast<size_t>(y) * width + x]; }
    double& at(int x, int y) { return values[static_cast<size_t>(y) * width + x]; }
};

SpikeLikeStream pixel_stream(const SpikeVolume& volume, int x, int y);

// ------------------------------------------------------- reconstruction ----
enum class Method { fsr, ssr, tfi, tfp };

struct ReconMethod {
    Method kind = Method::fsr;
    int tfp_window = 32;
    static ReconMethod parse(const std::string& name, int window = 32);
    std::string name() const;
};

struct SegmentEvent {
    long duration = 0;
    double intensity = 0.0;
    bool operator==(const SegmentEvent&) const = default;
};

std::vector<Segment> segment_fsr(const SpikeLikeStream& stream);
std::vector<Segment> segment_ssr(const SpikeLikeStream& stream);
double segment_intensity(const Segment& segment);
std::vector<SegmentEvent> fsr_events(const SpikeLikeStream& stream);
std::vector<double> reconstruct_pixel(const SpikeLikeStream& stream, ReconMethod method);

// Per-pixel streaming form of FSR (reconstruct.hpp:46-67).  Same contract:
// push_frame returns the segment that closes at this frame, flush the still-
// open spans; the events equal fsr_events of the whole stream.  Backed by a
// one-pixel spk_stream: frames without a spike are buffered (no event can
// close there) and each spike pushes the buffered frames through the GPU, so
// this scalar form costs one device round trip per spike -- use EventStream
// for whole sensors.
class PixelReconState {
public:
    PixelReconState();
    ~PixelReconState();
    PixelReconState(const PixelReconState&) = delete;
    PixelReconState& operator=(const PixelReconState&) = delete;
    PixelReconState(PixelReconState&& o) noexcept;
    PixelReconState& operator=(PixelReconState&& o) noexcept;
    std::optional<SegmentEvent> push_frame(bool bit);
    std::vector<SegmentEvent> flush();
    long frames_seen() const { return frame_; }

private:
    std::vector<SegmentEvent> push_pending();
    void* stream_ = nullptr;  // spk_stream
    std::vector<uint8_t> pending_;
    long frame_ = 0;
};

// The same for every pixel of a sensor at once: frames arrive in blocks
// (SPK1 payloads); each push returns, per pixel (row-major), the segments
// that closed in the block.
class EventStream {
public:
    EventStream(int width, int height);
    ~EventStream();
    EventStream(const EventStream&) = delete;
    EventStream& operator=(const EventStream&) = delete;
    std::vector<std::vector<SegmentEvent>> push(const std::vector<uint8_t>& payload, long frames);
    std::vector<std::vector<SegmentEvent>> flush();
    long frames() const;

private:
    void* stream_ = nullptr;  // spk_stream
    int width_, height_;
};

// `workers` (the reference's CPU thread count) selects up to that many of the
// visible GPUs, one pixel band each (spk_reconstruct_host_multi); with one
// GPU, or workers <= 1, it is one call.  The result is identical for any
// worker count, as in the reference (reconstruct.hpp:70-72).
std::vector<IntensityImage> reconstruct(const SpikeVolume& volume, ReconMethod method,
                                        int workers = 0);
void reconstruct(const SpikeVolume& volume, ReconMethod method, int workers,
                 std::vector<IntensityImage>& out);
std::vector<IntensityImage> reconstruct_serial(const SpikeVolume& volume, ReconMethod method);

// uint8 frames straight from the GPU (the CLI's per-frame output, quantize()
// of io.cpp:78-81 applied on the device): frames[n][y*W + x].
std::vector<std::vector<uint8_t>> reconstruct_u8(const SpikeVolume& volume, ReconMethod method);

// ------------------------------------------ metrics / stability (device) ----
// metrics.hpp: two_dimensional_entropy (>= 3x3, else invalid_argument), mse
// (dimension mismatch -> invalid_argument), psnr (+inf for identical images).
// Each single-image call is one device round trip; the vector form does a
// whole sequence in one call.
double two_dimensional_entropy(const IntensityImage& image);
std::vector<double> two_dimensional_entropy(const std::vector<IntensityImage>& images);
double mse(const IntensityImage& image, const IntensityImage& reference);
double psnr(const IntensityImage& image, const IntensityImage& reference);

// stability.hpp: the shallowest zero-order violation of the interval tree
// ('-' = smaller firing value first), explored to max_depth (1..63 here).
struct ViolationInfo {
    std::string path;
    int depth = 0;     // 1 = S1
    size_t index = 0;  // first offending element in that sequence
};
struct StabilityReport {
    int verified_order = 0;
    bool absolute = false;
    std::optional<ViolationInfo> first_violation;
};
StabilityReport stability_order(const SpikeLikeStream& stream, int max_depth);
// every pixel of a volume at once, row-major (verify-stability --in)
std::vector<StabilityReport> stability_order(const SpikeVolume& volume, int max_depth);

// ------------------------------------------------------------------- io ----
struct io_error : std::runtime_error {
    using std::runtime_error::runtime_error;
};

inline constexpr uint32_t kDefaultFps = 20000;
inline constexpr int kDefaultRawWidth = 400;
inline constexpr int kDefaultRawHeight = 250;

void write_spk(const SpikeVolume& volume, uint32_t fps, const std::filesystem::path& path);
std::pair<SpikeVolume, uint32_t> read_spk(const std::filesystem::path& path);
SpikeVolume read_raw(const std::filesystem::path& path, int width = kDefaultRawWidth,
                     int height = kDefaultRawHeight, bool msb_first = false);

enum class ImageFormat { pgm, png };
// PGM only (PNG needs libpng, absent from this build): png -> io_error.
void write_image(const IntensityImage& image, const std::filesystem::path& path,
                 ImageFormat format);
// P5 PGM back into [0, 255] values (read_image, io.cpp:230-234, PGM branch).
IntensityImage read_image(const std::filesystem::path& path);

// SPKR container (io.hpp:44-60): "SPKR" magic, the SPK1 geometry header,
// then per pixel (row-major) a u32 word count and that many u16 words.
struct RecordVolume {
    int width = 0;
    int height = 0;
    uint32_t fps = kDefaultFps;
    uint32_t frame_count = 0;
    std::vector<std::vector<uint16_t>> words;  // per pixel, row-major
    std::vector<uint16_t>& pixel(int x, int y) { return words[static_cast<size_t>(y) * width + x]; }
    const std::vector<uint16_t>& pixel(int x, int y) const {
        return words[static_cast<size_t>(y) * width + x];
    }
};
void write_spkr(const RecordVolume& records, const std::filesystem::path& path);
RecordVolume read_spkr(const std::filesystem::path& path);

// ---------------------------------------------------------------- codec ----
// 16-bit records (codec.hpp:11-25): duration in the high byte, intensity
// (rounded, ties away from zero) in the low byte; durations > 255 split into
// full 255-frame words with the remainder last.
inline int duration_of(uint16_t word) { return word >> 8; }
inline int intensity_of(uint16_t word) { return word & 0xff; }
void encode_append(std::vector<uint16_t>& words, long duration, double intensity);
std::vector<uint16_t> encode(long duration, double intensity);
std::vector<uint16_t> encode_events(std::span<const SegmentEvent> events);
std::vector<uint8_t> decode(std::span<const uint16_t> words);

// The CLI's --emit-records loop (spikecam_main.cpp:146-172: per pixel
// fsr_events / segment_ssr -> encode_events) for every pixel at once on the
// GPU (spk_records_host); method fsr or ssr, else invalid_argument.
RecordVolume emit_records(const SpikeVolume& volume, ReconMethod method, uint32_t fps = kDefaultFps);

// -------------------------------------------------------------- metrics ----
struct MetricReport {
    double te = 0.0;  // two-dimensional entropy, bits
    std::optional<double> psnr;
    std::optional<double> mse;
    std::optional<double> throughput;  // frames / second
};
struct BenchResult {
    std::string method;
    int width = 0;
    int height = 0;
    int frames = 0;
    int workers = 0;
    int repeats = 0;
    double frames_per_second = 0.0;  // median over repeats
};
// metrics.cpp:63-82: `repeats` (>= 3) timed reconstruct() calls into one
// reused output, median frames/s -- here each call is the GPU path.
BenchResult bench(const SpikeVolume& volume, ReconMethod method, int repeats, int workers = 1);

// ------------------------------------------------ packed fast path (new) ----
// The SPK1 payload kept bit-packed: no byte-per-bit SpikeVolume in between.
// read_spk_packed + reconstruct_u8 is the CLI loop (spikecam_main.cpp:52,174-179)
// with the volume going file -> GPU -> uint8 frames.
struct PackedSpikes {
    int width = 0;
    int height = 0;
    uint32_t fps = kDefaultFps;
    uint32_t frames = 0;
    std::vector<uint8_t> payload;  // frames * ceil(W*H/8) bytes, LSB-first
};

PackedSpikes read_spk_packed(const std::filesystem::path& path);
PackedSpikes pack(const SpikeVolume& volume, uint32_t fps = kDefaultFps);
// frames * W*H bytes, frame-major, the reference's quantize() of each value.
std::vector<uint8_t> reconstruct_u8(const PackedSpikes& spikes, ReconMethod method);
// frames * W*H doubles, frame-major, bit-identical to reconstruct().
std::vector<double> reconstruct_f64(const PackedSpikes& spikes, ReconMethod method);

}  // namespace spikecam
