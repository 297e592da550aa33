// capi.cu -- the C-ABI of libspikecam_b200.so (declared in include/spikecam_b200.h).
//
// Validation mirrors the reference's exceptions (SPK_EINVAL where it throws
// std::invalid_argument), workspaces come from the device's stream-ordered
// memory pool (cudaMallocAsync: no host synchronisation, thread-safe across
// streams), and every kernel launch is counted for the benchmark's
// `gpu_launches` claim.  There is no CPU fallback: every path launches the
// sm_100a kernels or returns an error.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "spk_common.cuh"
#include "spk_fsm.cuh"
#include "spk_kernels.cuh"

using namespace spk;

namespace {

thread_local std::string g_err;
thread_local int64_t g_launches = 0;
thread_local bool g_timing = false;
thread_local cudaEvent_t g_ev[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};
thread_local int g_ev_used = 0;  // events recorded by the last call
// in-grid time split of the last timed call: shards and flagged pixels
// (copied into pinned memory behind the call; valid once its events are done)
thread_local int g_split_shards = 1;
thread_local uint32_t* g_split_flagged = nullptr;

// phase marker k (0..4) on stream s when timing is enabled: 0 before K2,
// 1 after K2, 2 after K2b/scan/K2c, 3 after K3, 4 after the fixup
int mark(int k, cudaStream_t s) {
    if (!g_timing) return SPK_OK;
    if (!g_ev[k]) {
        cudaError_t e = cudaEventCreate(&g_ev[k]);
        if (e != cudaSuccess) return SPK_ECUDA;
    }
    cudaEventRecord(g_ev[k], s);
    g_ev_used = k + 1;
    return SPK_OK;
}
std::atomic<int64_t> g_run_cap{0};

int fail(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

int cuda_fail(cudaError_t e, const char* what) {
    g_err = std::string(what) + ": " + cudaGetErrorString(e);
    cudaGetLastError();  // clear sticky-free errors
    return e == cudaErrorMemoryAllocation ? SPK_ENOMEM : SPK_ECUDA;
}

#define SPK_CK(call)                                         \
    do {                                                     \
        cudaError_t e_ = (call);                             \
        if (e_ != cudaSuccess) return cuda_fail(e_, #call);  \
    } while (0)

#define SPK_LAUNCHED(name)                                   \
    do {                                                     \
        ++g_launches;                                        \
        cudaError_t e_ = cudaGetLastError();                 \
        if (e_ != cudaSuccess) return cuda_fail(e_, name);   \
    } while (0)

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

int64_t npix_of(const spk_geom* g) { return (int64_t)g->width * (int64_t)g->height; }
size_t plane_bytes(const spk_geom* g) { return (size_t)((npix_of(g) + 7) / 8); }
size_t min_pitch(int64_t npix) { return (size_t)((npix + 31) / 32) * 4; }

// SpikeVolume / geometry rules (proj/src/core.cpp:11-13) + device layout rules
int check_geom(const spk_geom* g, bool check_pitch) {
    if (!g) return fail(SPK_EINVAL, "spk: null geometry");
    if (g->width < 1 || g->height < 1 || g->frames < 0)
        return fail(SPK_EINVAL, "SpikeVolume: width/height must be >= 1, frames >= 0");
    if (g->frames >= (int64_t)1 << 29)
        return fail(SPK_EINVAL, "spk: frames must be < 2^29");
    if (npix_of(g) >= (int64_t)1 << 31) return fail(SPK_EINVAL, "spk: W*H must be < 2^31");
    if (check_pitch && (g->plane_pitch % 4 != 0 || g->plane_pitch < min_pitch(npix_of(g))))
        return fail(SPK_EINVAL, "spk: plane_pitch must be a multiple of 4 and >= 4*ceil(W*H/32)");
    return SPK_OK;
}

// ReconMethod::parse rules (proj/src/reconstruct.cpp:177-186)
int check_method(int method, int window) {
    if (method < SPK_FSR || method > SPK_TFP)
        return fail(SPK_EINVAL, "unknown reconstruction method: " + std::to_string(method));
    if (method == SPK_TFP && window < 1) return fail(SPK_EINVAL, "tfp window must be >= 1");
    return SPK_OK;
}

int run_capacity(int64_t frames) {
    int64_t cap = g_run_cap.load();
    if (cap <= 0) cap = std::max<int64_t>(64, frames / 32);
    cap = std::min<int64_t>(cap, std::max<int64_t>(1, frames));
    return (int)cap;
}

void ensure_pool(int dev) {
    static std::atomic<uint64_t> done{0};
    if (dev < 0 || dev >= 64) return;
    const uint64_t bit = 1ull << dev;
    if (done.load() & bit) return;
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        uint64_t thr = UINT64_MAX;  // keep freed workspaces cached in the pool
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    done.fetch_or(bit);
}


// Test hook (tests/test_limits.py): SPK_TEST_PART_ENTRIES / SPK_TEST_GRID_Y
// lower the 2^32 change-stream limit and the 65535 grid.y limit so the splits
// run on small volumes.  Read once; unset in production.
int64_t test_limit(const char* name, int64_t dflt) {
    const char* v = std::getenv(name);
    return v && *v ? std::max<int64_t>(1, std::atoll(v)) : dflt;
}

// RAII stream-ordered scratch
struct Scratch {
    void* p = nullptr;
    cudaStream_t s;
    explicit Scratch(cudaStream_t st) : s(st) {}
    cudaError_t alloc(size_t bytes) { return cudaMallocAsync(&p, std::max<size_t>(bytes, 16), s); }
    ~Scratch() {
        if (p) cudaFreeAsync(p, s);
    }
};


// warps per K2 block: kSegWarpsWide when FSR fits one wave and those blocks
// leave fewer warps on the busiest SM (W * ceil(blocks / SMs)), else kSegWarps
int seg_warps_for(int method, int64_t nwords, unsigned shards) {
#ifdef SPK_SEG_WARPS_FIXED
    (void)method; (void)nwords; (void)shards;
    return kSegWarps;
#else
    if (method != SPK_FSR || shards != 1) return kSegWarps;
    static int sms = [] {
        int dev = 0, n = 148;
        if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        return std::max(n, 1);
    }();
    auto busiest = [&](int w, int per_sm) -> int64_t {  // -1: more than one wave
        const int64_t blocks = (nwords + w - 1) / w;
        return blocks <= (int64_t)sms * per_sm ? w * ((blocks + sms - 1) / sms) : -1;
    };
    const int64_t b8 = busiest(kSegWarps, 3), b11 = busiest(kSegWarpsWide, 2);
    return b8 > 0 && b11 > 0 && b11 < b8 ? kSegWarpsWide : kSegWarps;
#endif
}

int launch_segment(int method, const SegArgs& a, cudaStream_t s) {
    const int64_t nwords = (a.npix + 31) / 32;
    const unsigned shards = a.shard_frames > 0 ? (unsigned)((a.frames + a.shard_frames - 1) / a.shard_frames) : 1u;
    auto go = [&](auto kern, int warps) -> int {
        // the warps' rings (+ SSR: their parity-slot records)
        const size_t smem = (size_t)warps * (kRing * 32 * sizeof(uint32_t) + (method == SPK_SSR ? kSsrSlotBytes : 0));
        const unsigned blocks = (unsigned)((nwords + warps - 1) / warps);
        SPK_CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        kern<<<dim3(blocks, shards), warps * 32, smem, s>>>(a);
        return SPK_OK;
    };
    const int warps = a.flags != nullptr ? kSegWarps : seg_warps_for(method, nwords, shards);
    int rc = method == SPK_FSR ? (warps == kSegWarpsWide ? go(k_segment<kFSR, kSegWarpsWide>, warps)
                                                         : go(k_segment<kFSR, kSegWarps>, warps))
                               : go(k_segment<kSSR, kSegWarps>, kSegWarps);
    if (rc) return rc;
    SPK_LAUNCHED("k_segment");
    return SPK_OK;
}

// exclusive scan of n uint32 counts into T (three small launches)
template <typename T>
int launch_scan(const uint32_t* in, T* out, int64_t n, cudaStream_t s, T* out2 = nullptr) {
    const int64_t nb = (n + kScanBlock - 1) / kScanBlock;
    Scratch sums(s);
    SPK_CK(sums.alloc((size_t)nb * sizeof(T)));
    T* sp = static_cast<T*>(sums.p);
    k_scan_blocks<T><<<(unsigned)nb, kScanBlock, 0, s>>>(in, out, sp, n);
    SPK_LAUNCHED("k_scan_blocks");
    k_scan_sums<T><<<1, kScanBlock, 0, s>>>(sp, nb);
    SPK_LAUNCHED("k_scan_sums");
    k_scan_add<T><<<(unsigned)nb, kScanBlock, 0, s>>>(out, sp, n, out2);
    SPK_LAUNCHED("k_scan_add");
    return SPK_OK;
}

// TMA tile stores of K3: the frames as a 2-D uint32 tensor (W*H/4 columns,
// `frames` rows, `pitch_bytes` apart), box 128 columns (512 B) x `rows`.
// cuTensorMapEncodeTiled through the runtime's driver entry point.
// Opt-in (SPK_TMA=1): measured on B200 the same as the per-lane stores --
// K3 is bound by its change handling, not by the store path (C2 K3 0.726 vs
// 0.718 ms, C3 3.615 vs 3.625 ms; profiles/r02/walk_experiments.md).
bool tma_enabled() {
    const char* v = std::getenv("SPK_TMA");
    return v && *v && *v != '0';
}

bool encode_out_map(CUtensorMap* m, const void* out, int64_t npix, int64_t frames, size_t pitch_bytes,
                    int rows) {
    using Encode = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                                CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                                CUtensorMapFloatOOBfill);
    static Encode enc = []() -> Encode {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            return nullptr;
        return reinterpret_cast<Encode>(f);
    }();
    if (!enc || frames < 1 || npix < 4 || pitch_bytes % 16 != 0 || (reinterpret_cast<uintptr_t>(out) & 15))
        return false;
    const cuuint64_t dims[2] = {(cuuint64_t)(npix / 4), (cuuint64_t)frames};
    const cuuint64_t strides[1] = {(cuuint64_t)pitch_bytes};
    const cuuint32_t box[2] = {128u, (cuuint32_t)rows}, es[2] = {1u, 1u};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, const_cast<void*>(out), dims, strides, box, es,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// workspaces of the expand stage (allocated before K2, which fills `bins`)
template <typename OUT>
struct ExpandWork {
    Scratch tblv, bins, offs, cursor, stream;
    int ngroups = 0;
    int64_t nbins = 0;
    bool exact_stream = false;  // the change stream is allocated after the scan, at its exact length
    explicit ExpandWork(cudaStream_t s) : tblv(s), bins(s), offs(s), cursor(s), stream(s) {}
};

template <typename OUT>
int prepare_expand(SegArgs& sa, ExpandWork<OUT>& w, cudaStream_t s) {
    constexpr int GP = 32 * Geo<OUT>::P;
    w.ngroups = (int)((sa.npix + GP - 1) / GP);
    w.nbins = (int64_t)sa.nchunks * w.ngroups * kBins;
    SPK_CK(w.tblv.alloc((size_t)sa.nchunks * sa.npix * sizeof(OUT)));
    SPK_CK(w.bins.alloc((size_t)w.nbins * sizeof(uint32_t)));
    SPK_CK(w.offs.alloc((size_t)w.nbins * sizeof(uint32_t)));
    SPK_CK(w.cursor.alloc((size_t)w.nbins * sizeof(uint32_t)));
    // The change stream holds one entry per stored run: at most npix * cap,
    // usually far fewer (a 1M-frame static stream: 12.5 GB worst case, ~0.2 GB
    // of runs).  Large worst cases are allocated after the scan at the exact
    // length -- one 8-byte read-back and a stream synchronisation, ~20 us on
    // steps of several ms; small ones (and calls under stream capture, which
    // may not synchronise) take the bound.
    static const int64_t exact_from = test_limit("SPK_TEST_EXACT_STREAM", (int64_t)1 << 30);
    cudaStreamCaptureStatus cap_status = cudaStreamCaptureStatusNone;
    SPK_CK(cudaStreamIsCapturing(s, &cap_status));
    const size_t worst = (size_t)sa.npix * sa.cap * sizeof(Change<OUT>);
    w.exact_stream = (int64_t)worst >= exact_from && cap_status == cudaStreamCaptureStatusNone;
    if (!w.exact_stream) SPK_CK(w.stream.alloc(worst));
    // chunks before a pixel's first run keep value 0
    SPK_CK(cudaMemsetAsync(w.tblv.p, 0, (size_t)sa.nchunks * sa.npix * sizeof(OUT), s));
    return SPK_OK;
}

// K2b + scan + K2c + K3: run lists -> frames
template <typename OUT>
int launch_expand(const SegArgs& sa, ExpandWork<OUT>& w, OUT* out, size_t out_pitch,
                  cudaStream_t s) {
    constexpr int GP = 32 * Geo<OUT>::P;
    mark(1, s);
    FinArgs f;
    f.runs = sa.runs;
    f.counts = sa.counts;
    f.last = sa.last;
    f.npix = sa.npix;
    f.frames = sa.frames;
    f.cap = sa.cap;
    f.nchunks = sa.nchunks;
    f.ngroups = w.ngroups;
    f.bins = static_cast<uint32_t*>(w.bins.p);
    f.tblv = w.tblv.p;
    f.offs = static_cast<const uint32_t*>(w.offs.p);
    f.stream = w.stream.p;
    f.stream_len = sa.npix * sa.cap;
    f.seg = sa.seg_in;
    f.nseg = sa.nseg;
    // few groups (narrow sensors): split each group's pixels over 4 blocks
    const unsigned fsplit = w.ngroups < 1024 ? 4u : 1u;
    const dim3 fgrid((unsigned)w.ngroups, (unsigned)((sa.nchunks + kFinWindow - 1) / kFinWindow), fsplit);
    if (fsplit > 1) SPK_CK(cudaMemsetAsync(w.bins.p, 0, (size_t)w.nbins * sizeof(uint32_t), s));
    if (f.seg)
        k_fin_bins<GP, true><<<fgrid, kFinWarps * 32, 0, s>>>(f);
    else
        k_fin_bins<GP, false><<<fgrid, kFinWarps * 32, 0, s>>>(f);
    SPK_LAUNCHED("k_fin_bins");
    // the scan also writes the copy K2c claims slots from
    int rc = launch_scan(f.bins, static_cast<uint32_t*>(w.offs.p), w.nbins, s,
                         static_cast<uint32_t*>(w.cursor.p));
    if (rc) return rc;
    f.cursor = static_cast<uint32_t*>(w.cursor.p);
    if (w.exact_stream) {  // entries = last offset + last bin
        static thread_local uint32_t* h_tot = nullptr;
        if (!h_tot) SPK_CK(cudaMallocHost(&h_tot, 2 * sizeof(uint32_t)));
        SPK_CK(cudaMemcpyAsync(h_tot, f.offs + (w.nbins - 1), sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
        SPK_CK(cudaMemcpyAsync(h_tot + 1, f.bins + (w.nbins - 1), sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
        SPK_CK(cudaStreamSynchronize(s));
        const int64_t total = (int64_t)h_tot[0] + h_tot[1];
        SPK_CK(w.stream.alloc((size_t)std::max<int64_t>(total, 1) * sizeof(Change<OUT>)));
        f.stream = w.stream.p;
        f.stream_len = total;
    }
    // threads stride over a pixel's kFinSeg-run blocks (grid.y <= 64: a
    // 1M-frame list of one run per pixel is not 500 block rows of exits)
    f.fin_seg = fin_seg_for(sa.npix);
    const int nseg = (sa.cap + f.fin_seg - 1) / f.fin_seg;
    static const int maxy = (int)test_limit("SPK_TEST_GRID_Y", 64);
    const dim3 grid((unsigned)((sa.npix + 255) / 256), (unsigned)std::min(maxy, nseg));
    if (f.seg)
        k_fin_scatter<OUT, true><<<grid, 256, 0, s>>>(f);
    else
        k_fin_scatter<OUT, false><<<grid, 256, 0, s>>>(f);
    SPK_LAUNCHED("k_fin_scatter");
    mark(2, s);

    ExpArgs e;
    e.tblv = w.tblv.p;
    e.bins = static_cast<const uint32_t*>(w.bins.p);
    e.offs = f.offs;
    e.stream = w.stream.p;
    e.stream_len = f.stream_len;
    e.npix = sa.npix;
    e.frames = sa.frames;
    e.nchunks = sa.nchunks;
    e.ngroups = w.ngroups;
    e.out = out;
    e.pitch = out_pitch;
    e.vec_ok = ((reinterpret_cast<uintptr_t>(out) | (out_pitch * sizeof(OUT))) & 15) == 0;
    // uint8 frames of wide sensors (>= kWideGroups 512-pixel groups per frame,
    // e.g. 1000x1000): 8-warp blocks, 4 KB of each row per block (C3 K3 3.77
    // -> 3.63 ms; 400x250: 4 warps, 0.717 vs 0.762 ms)
    const bool wide = sizeof(OUT) == 1 && w.ngroups >= kWideGroups;
    const int warps = wide ? 2 * Geo<OUT>::WARPS : Geo<OUT>::WARPS;
    const unsigned bx = (unsigned)((w.ngroups + warps - 1) / warps);
    // uint8 frames can leave K3 as TMA tensor stores of whole sub-tiles (one
    // cp.async.bulk.tensor per kSub rows x 512 B; SPK_TMA=1): the write probe
    // (profiles/tma_write.cu) gives 7.3 TB/s for K3's 128-row tiles against
    // 6.5 with per-lane 16-B stores, but inside K3 the two measure the same.
    // Needs 16-B aligned rows and W*H a multiple of 4 (the map's uint32
    // columns end at the last pixel).
    CUtensorMap tmap;
    std::memset(&tmap, 0, sizeof(tmap));
    const bool tma = sizeof(OUT) == 1 && e.vec_ok && sa.npix % 4 == 0 && tma_enabled() &&
                     encode_out_map(&tmap, out, sa.npix, sa.frames, out_pitch * sizeof(OUT), kSub);
    // Narrow uint8 frames, FSR run lists: four 4-warp blocks per SM instead of
    // the five that fit (the request is padded to 54 KB; SSR's denser change
    // stream wants the five: C2 SSR K3 0.808 vs 0.842 ms).  K3 is bound by its DRAM write
    // pattern: fewer warps keep fewer rows open at a time (C2 K3 0.710 ->
    // 0.696 ms; three blocks 0.752; twice the warps, with half-size cells,
    // 0.768).  SPK_K3_PAD overrides the padding (probes).
    static const long k3_pad = [] { const char* v = std::getenv("SPK_K3_PAD"); return v ? std::atol(v) : -1L; }();
    size_t smem = expand_smem_bytes(sizeof(OUT), warps, tma);
    if (k3_pad >= 0)
        smem += (size_t)k3_pad;
    else if (sizeof(OUT) == 1 && !wide && !tma && !sa.dense_runs)
        smem = std::max<size_t>(smem, 54 * 1024);
    void (*kexp)(ExpArgs, const CUtensorMap) = k_expand<OUT, Geo<OUT>::WARPS, false>;
    if constexpr (sizeof(OUT) == 1) {
        if (tma)
            kexp = wide ? k_expand<OUT, 2 * Geo<OUT>::WARPS, true> : k_expand<OUT, Geo<OUT>::WARPS, true>;
        else if (wide)
            kexp = k_expand<OUT, 2 * Geo<OUT>::WARPS, false>;
    }
    if (smem > 48 * 1024)
        SPK_CK(cudaFuncSetAttribute(kexp, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    e.pieces = w.ngroups <= kPieceMaxGroups ? kPieces : 1;
    const int per_launch = 65535 / e.pieces;  // grid.y = chunks x pieces
    for (int c0 = 0; c0 < sa.nchunks; c0 += per_launch) {
        e.chunk0 = c0;
        const unsigned by = (unsigned)(std::min(per_launch, sa.nchunks - c0) * e.pieces);
        kexp<<<dim3(bx, by), warps * 32, smem, s>>>(e, tmap);
        SPK_LAUNCHED("k_expand");
    }
    return SPK_OK;
}

// The change stream of one expand is indexed with 32-bit offsets (scan of
// the bins, K2c slot claims, K3): its length, at most npix * cap, must stay
// below 2^32.  Larger (pixels x capacity) products are expanded in pixel
// parts, each a whole number of pixel groups with npix_part * cap < 2^32.
template <typename OUT>
int expand_parts(const SegArgs& sa, OUT* out, size_t out_pitch, cudaStream_t s) {
    constexpr int64_t GP = 32 * Geo<OUT>::P;
    static const int64_t entries = test_limit("SPK_TEST_PART_ENTRIES", (int64_t)UINT32_MAX);
    const int64_t limit = entries / std::max(sa.cap, 1);
    const int64_t part = std::max<int64_t>(GP, limit / GP * GP);
    for (int64_t p0 = 0; p0 < sa.npix; p0 += part) {
        SegArgs sub = sa;
        sub.npix = std::min(part, sa.npix - p0);
        sub.runs = sa.runs + p0 * sa.cap;
        sub.counts = sa.counts + p0;
        sub.last = sa.last + p0;
        if (sa.seg_in) sub.seg_in = sa.seg_in + p0 * 2 * sa.nseg;
        ExpandWork<OUT> w(s);
        int rc = prepare_expand<OUT>(sub, w, s);
        if (rc) return rc;
        if ((rc = launch_expand<OUT>(sub, w, out + p0, out_pitch, s))) return rc;
    }
    return SPK_OK;
}

template <typename OUT>
int launch_fixup(int method, const SegArgs& sa, OUT* out, size_t out_pitch, cudaStream_t s) {
    const unsigned blocks = (unsigned)((sa.npix + 127) / 128);
    if (method == SPK_FSR)
        k_fixup<kFSR, OUT><<<blocks, 128, 0, s>>>(sa, out, out_pitch);
    else
        k_fixup<kSSR, OUT><<<blocks, 128, 0, s>>>(sa, out, out_pitch);
    SPK_LAUNCHED("k_fixup");
    return SPK_OK;
}

template <typename OUT>
int launch_causal(const spk_geom* g, const void* planes, int method, int window, OUT* out,
                  size_t out_pitch, cudaStream_t s) {
    CausalArgs c;
    c.planes = planes;
    c.pitch = g->plane_pitch;
    c.npix = npix_of(g);
    c.frames = (int)g->frames;
    c.window = method == SPK_TFP ? window : 1;
    c.out = out;
    c.out_pitch = out_pitch;
    const int lut_cap = (int)(32768 / sizeof(OUT));
    if (method == SPK_TFI)
        c.lut_n = sizeof(OUT) == 1 ? 512 : 1024;
    else
        c.lut_n = window + 1 <= lut_cap ? window + 1 : 0;
    const size_t lut_bytes = ((size_t)c.lut_n * sizeof(OUT) + 15) & ~(size_t)15;
    const size_t smem = lut_bytes + (size_t)kCausalWarps * 32 * (32 * sizeof(OUT) + 16);
    const int64_t nwords = (c.npix + 31) / 32;
    const unsigned blocks = (unsigned)((nwords + kCausalWarps - 1) / kCausalWarps);
    auto go = [&](auto kern) -> int {
        if (smem > 48 * 1024)
            SPK_CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        kern<<<blocks, kCausalWarps * 32, smem, s>>>(c);
        SPK_LAUNCHED("k_causal");
        return SPK_OK;
    };
    return method == SPK_TFI ? go(k_causal<kTFI, OUT>) : go(k_causal<kTFP, OUT>);
}

// ------------------------------------------------------ in-grid time split --
// K2 is one wave of 8-warp blocks (a block = 256 pixels = one 32-B sector of
// every plane row) when the sensor has few pixels: 400x250 is 391 blocks on
// 148 SMs x 3, so some SMs hold three blocks and others two, and each warp's
// serial chain spans the whole stream.  Cutting the stream in S time shards
// scanned in ONE launch (S x more blocks, each 1/S as long) balances the SMs;
// the exact stitching (csrc/shard.cu) runs as one resolve launch and one
// combine pass.  Measured (K2 alone, profiles/shard_k2_probe.py): C2 0.966 ->
// 0.844 ms at S = 4, configs[4] 11.26 -> 9.26 ms at S = 16.
int split_shards(int method, int64_t npix, int64_t frames, int dev) {
    // test hook: SPK_SPLIT=S forces S shards (1 = off), read on every call
    const char* fv = std::getenv("SPK_SPLIT");
    if (fv && *fv) {
        const int64_t S = std::min<int64_t>(std::min<int64_t>(std::atoll(fv), (frames + 31) / 32),
                                            kSplitMaxShards);
        return S >= 2 ? (int)S : 1;
    }
    // FSR only: SSR's resolves sync late and cost more than the balance
    // gains (C2 SSR K2 5.54 vs 5.36 ms).  Long streams only: the resolve,
    // the combine and the segmented finalize cost ~0.16 ms at 400x250, about
    // what the balance saves on a 40,000-frame K2 (C2: 2.11 vs 2.07 ms) and
    // far less than on a 1,000,000-frame one (configs[4]: 24.2 vs 26.0 ms).
    if (method != SPK_FSR || frames < kSplitMinStream) return 1;
    int sms = 148, per_sm = 3;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const size_t smem = (size_t)kSegWarps * kRing * 32 * sizeof(uint32_t);
    if (method == SPK_FSR)
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_segment<kFSR>, kSegThreads, smem);
    else
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_segment<kSSR>, kSegThreads, smem);
    const int64_t blocks = (npix + kSegThreads - 1) / kSegThreads;
    const int64_t slots = (int64_t)sms * std::max(per_sm, 1);
    int64_t S = 6 * slots / std::max<int64_t>(blocks, 1);  // ~6 waves
    S = std::min<int64_t>(S, frames / kSplitMinFrames);
    S = std::min<int64_t>(S, kSplitMaxShards);
    return S >= 2 ? (int)S : 1;
}

template <typename OUT>
int reconstruct_split(const spk_geom* g, const void* planes, int method, int S, OUT* out,
                      size_t out_pitch, cudaStream_t s) {
    const int64_t npix = npix_of(g);
    const int frames = (int)g->frames;
    const int words = (frames + 31) / 32;
    const int sf = (words + S - 1) / S * 32;
    S = (frames + sf - 1) / sf;
    const int scap = std::max(64, sf / 32);
    const int64_t rstride = kSplitGap + scap;
    const int64_t row = (int64_t)S * rstride;
    if (row > INT_MAX) return fail(SPK_EINVAL, "spk: run list too long");
    constexpr int F = Scan<kSSR>::kFields;
    Scratch rows(s), scount(s), slast(s), sstate(s), prefix(s), sync(s), syncj(s), tstate(s), seg(s),
        counts(s), last(s), flags(s), nflag(s);
    SPK_CK(rows.alloc((size_t)npix * row * sizeof(spk_run_t)));
    SPK_CK(scount.alloc((size_t)S * npix * sizeof(uint32_t)));
    SPK_CK(slast.alloc((size_t)S * npix * sizeof(int32_t)));
    SPK_CK(sstate.alloc((size_t)S * F * npix * sizeof(int32_t)));
    SPK_CK(prefix.alloc((size_t)S * npix * kSplitGap * sizeof(spk_run_t)));
    SPK_CK(sync.alloc((size_t)S * npix * sizeof(spk_sync_t)));
    SPK_CK(syncj.alloc((size_t)S * npix * sizeof(int32_t)));
    SPK_CK(tstate.alloc((size_t)S * F * npix * sizeof(int32_t)));
    SPK_CK(seg.alloc((size_t)npix * S * 2 * sizeof(uint32_t)));
    SPK_CK(counts.alloc((size_t)npix * sizeof(uint32_t)));
    SPK_CK(last.alloc((size_t)npix * sizeof(int32_t)));
    SPK_CK(flags.alloc((size_t)npix));
    SPK_CK(nflag.alloc(sizeof(uint32_t)));
    SPK_CK(cudaMemsetAsync(nflag.p, 0, sizeof(uint32_t), s));

    mark(0, s);
    // 1. every shard's speculative scan, one launch
    SegArgs a;
    a.planes = planes;
    a.pitch = g->plane_pitch;
    a.npix = npix;
    a.frames = frames;
    a.cap = scap;
    a.nchunks = (frames + kChunk - 1) / kChunk;
    a.runs = static_cast<spk_run_t*>(rows.p);
    a.counts = static_cast<uint32_t*>(scount.p);
    a.last = static_cast<int32_t*>(slast.p);
    a.state_out = static_cast<int32_t*>(sstate.p);
    a.shard_frames = sf;
    a.run_pix_stride = row;
    a.run_shard_stride = rstride;
    a.run_base = kSplitGap;
    a.abs_frames = 1;
    int rc = launch_segment(method, a, s);
    if (rc) return rc;
    // 2. every boundary's resolve, one launch (shard r from shard r-1's
    //    speculative end state)
    ShardArgs h{};
    h.planes = planes;
    h.pitch = g->plane_pitch;
    h.npix = npix;
    h.frames = sf;
    h.prefix = static_cast<spk_run_t*>(prefix.p);
    h.pcap = kSplitGap;
    h.sync = static_cast<spk_sync_t*>(sync.p);
    h.tstate = static_cast<int32_t*>(tstate.p);
    h.spec = static_cast<spk_run_t*>(rows.p);
    h.scap = scap;
    h.scount = static_cast<uint32_t*>(scount.p);
    h.sstate = static_cast<int32_t*>(sstate.p);
    h.grid_sf = sf;
    h.nshards = S;
    h.rstride = rstride;
    h.total_frames = frames;
    h.syncj = static_cast<int32_t*>(syncj.p);
    {
        const int64_t threads = (npix + 31) / 32 * 32;
        const dim3 grid((unsigned)((threads + 63) / 64), (unsigned)(S - 1));
        if (method == SPK_FSR)
            k_resolve<kFSR><<<grid, 64, 0, s>>>(h);
        else
            k_resolve<kSSR><<<grid, 64, 0, s>>>(h);
        SPK_LAUNCHED("k_resolve");
    }
    // 3. the true run list per pixel as segments of its row
    SplitArgs c;
    c.npix = npix;
    c.nshards = S;
    c.sf = sf;
    c.frames = frames;
    c.rstride = rstride;
    c.scap = scap;
    c.pcap = kSplitGap;
    c.runs = static_cast<spk_run_t*>(rows.p);
    c.scount = static_cast<uint32_t*>(scount.p);
    c.sstate = static_cast<int32_t*>(sstate.p);
    c.prefix = static_cast<spk_run_t*>(prefix.p);
    c.sync = static_cast<spk_sync_t*>(sync.p);
    c.syncj = static_cast<const int32_t*>(syncj.p);
    c.tstate = static_cast<int32_t*>(tstate.p);
    c.seg = static_cast<uint32_t*>(seg.p);
    c.counts = static_cast<uint32_t*>(counts.p);
    c.last = static_cast<int32_t*>(last.p);
    c.flags = static_cast<uint8_t*>(flags.p);
    c.nflag = static_cast<uint32_t*>(nflag.p);
    c.method = method;
    {
        const unsigned blocks = (unsigned)((npix + 127) / 128);
        if (method == SPK_FSR)
            k_split_combine<kFSR><<<blocks, 128, 0, s>>>(c);
        else
            k_split_combine<kSSR><<<blocks, 128, 0, s>>>(c);
        SPK_LAUNCHED("k_split_combine");
    }
    // 4. flagged pixels (an entry that decides differently, a capacity
    //    overflow): whole-stream re-scan into their rows; warps without a
    //    flagged pixel exit at once
    SegArgs r;
    r.planes = planes;
    r.pitch = g->plane_pitch;
    r.npix = npix;
    r.frames = frames;
    r.cap = (int)row;
    r.nchunks = a.nchunks;
    r.runs = static_cast<spk_run_t*>(rows.p);
    r.counts = static_cast<uint32_t*>(counts.p);
    r.last = static_cast<int32_t*>(last.p);
    r.flags = static_cast<uint8_t*>(flags.p);
    r.seg_out = static_cast<uint32_t*>(seg.p);
    r.nseg = S;
    if ((rc = launch_segment(method, r, s))) return rc;
    if (g_timing) {
        if (!g_split_flagged) SPK_CK(cudaMallocHost(&g_split_flagged, sizeof(uint32_t)));
        SPK_CK(cudaMemcpyAsync(g_split_flagged, nflag.p, sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
        g_split_shards = S;
    }
    // 5. frames from the segmented lists; overflowed pixels by k_fixup
    SegArgs e = r;
    e.flags = nullptr;
    e.seg_out = nullptr;
    e.seg_in = static_cast<const uint32_t*>(seg.p);
    if ((rc = expand_parts<OUT>(e, out, out_pitch, s))) return rc;
    mark(3, s);
    rc = launch_fixup<OUT>(method, e, out, out_pitch, s);
    mark(4, s);
    return rc;
}

template <typename OUT>
int reconstruct_impl(const spk_geom* g, const void* planes, int method, int window, OUT* out,
                     size_t out_pitch, void* stream) {
    int rc = check_geom(g, true);
    if (rc) return rc;
    if ((rc = check_method(method, window))) return rc;
    const int64_t npix = npix_of(g);
    if (g->frames == 0) return SPK_OK;
    if (!planes || !out) return fail(SPK_EINVAL, "spk: null device buffer");
    if (out_pitch < (size_t)npix) return fail(SPK_EINVAL, "spk: out_pitch must be >= W*H");
    cudaStream_t s = as_stream(stream);
    g_ev_used = 0;
    g_split_shards = 1;
    if (method == SPK_TFI || method == SPK_TFP) {
        mark(0, s);
        mark(1, s);
        mark(2, s);
        rc = launch_causal<OUT>(g, planes, method, window, out, out_pitch, s);
        mark(3, s);
        return rc;
    }

    int dev = 0;
    SPK_CK(cudaGetDevice(&dev));
    ensure_pool(dev);
    if (g_run_cap.load() <= 0) {  // (a fixed run capacity is a test setting: one pass)
        const int S = split_shards(method, npix, g->frames, dev);
        if (S > 1) return reconstruct_split<OUT>(g, planes, method, S, out, out_pitch, s);
    }
    SegArgs a;
    a.planes = planes;
    a.pitch = g->plane_pitch;
    a.npix = npix;
    a.frames = (int)g->frames;
    a.cap = run_capacity(g->frames);
    a.nchunks = (int)((g->frames + kChunk - 1) / kChunk);
    Scratch runs(s), counts(s), last(s);
    SPK_CK(runs.alloc((size_t)npix * a.cap * sizeof(spk_run_t)));
    SPK_CK(counts.alloc((size_t)npix * sizeof(uint32_t)));
    SPK_CK(last.alloc((size_t)npix * sizeof(int32_t)));
    a.runs = static_cast<spk_run_t*>(runs.p);
    a.counts = static_cast<uint32_t*>(counts.p);
    a.last = static_cast<int32_t*>(last.p);

    // One pass: pipelining pixel parts of K2 with K3 was measured slower at
    // every size (K2 fills the SMs, so K3 of part k only runs in the gaps of
    // part k+1: C3 FSR 9.72 vs 9.34 ms, SSR 25.5 vs 24.5 ms).
    mark(0, s);
    a.dense_runs = method == SPK_SSR;
    if ((rc = launch_segment(method, a, s))) return rc;
    if ((rc = expand_parts<OUT>(a, out, out_pitch, s))) return rc;
    mark(3, s);
    rc = launch_fixup<OUT>(method, a, out, out_pitch, s);
    mark(4, s);
    return rc;
}

template <typename OUT>
int expand_runs_impl(const spk_geom* g, const spk_run* runs, int64_t cap, const uint32_t* counts,
                     const int32_t* last, OUT* out, size_t out_pitch, void* stream) {
    int rc = check_geom(g, false);
    if (rc) return rc;
    const int64_t npix = npix_of(g);
    if (g->frames == 0) return SPK_OK;
    if (cap < 1 || cap > INT_MAX) return fail(SPK_EINVAL, "spk_expand_runs: bad run_cap");
    if (!runs || !counts || !last || !out) return fail(SPK_EINVAL, "spk: null device buffer");
    if (out_pitch < (size_t)npix) return fail(SPK_EINVAL, "spk: out_pitch must be >= W*H");
    cudaStream_t s = as_stream(stream);
    int dev = 0;
    SPK_CK(cudaGetDevice(&dev));
    ensure_pool(dev);
    SegArgs a;
    a.planes = nullptr;
    a.pitch = 0;
    a.npix = npix;
    a.frames = (int)g->frames;
    a.cap = (int)cap;
    a.nchunks = (int)((g->frames + kChunk - 1) / kChunk);
    a.runs = const_cast<spk_run*>(runs);
    a.counts = const_cast<uint32_t*>(counts);
    a.last = const_cast<int32_t*>(last);
    return expand_parts<OUT>(a, out, out_pitch, s);
}

}  // namespace

extern "C" {

int spk_expand_runs_u8(const spk_geom* g, const spk_run* d_runs, int64_t run_cap,
                       const uint32_t* d_counts, const int32_t* d_last, uint8_t* d_out,
                       size_t out_pitch, void* stream) {
    return expand_runs_impl<uint8_t>(g, d_runs, run_cap, d_counts, d_last, d_out, out_pitch, stream);
}
int spk_expand_runs_f32(const spk_geom* g, const spk_run* d_runs, int64_t run_cap,
                        const uint32_t* d_counts, const int32_t* d_last, float* d_out,
                        size_t out_pitch, void* stream) {
    return expand_runs_impl<float>(g, d_runs, run_cap, d_counts, d_last, d_out, out_pitch, stream);
}
int spk_expand_runs_f64(const spk_geom* g, const spk_run* d_runs, int64_t run_cap,
                        const uint32_t* d_counts, const int32_t* d_last, double* d_out,
                        size_t out_pitch, void* stream) {
    return expand_runs_impl<double>(g, d_runs, run_cap, d_counts, d_last, d_out, out_pitch, stream);
}

int spk_reconstruct_u8(const spk_geom* g, const void* d_planes, int method, int tfp_window,
                       uint8_t* d_out, size_t out_pitch, void* stream) {
    return reconstruct_impl<uint8_t>(g, d_planes, method, tfp_window, d_out, out_pitch, stream);
}

int spk_reconstruct_f32(const spk_geom* g, const void* d_planes, int method, int tfp_window,
                        float* d_out, size_t out_pitch, void* stream) {
    return reconstruct_impl<float>(g, d_planes, method, tfp_window, d_out, out_pitch, stream);
}

int spk_reconstruct_f64(const spk_geom* g, const void* d_planes, int method, int tfp_window,
                        double* d_out, size_t out_pitch, void* stream) {
    return reconstruct_impl<double>(g, d_planes, method, tfp_window, d_out, out_pitch, stream);
}

int spk_segment(const spk_geom* g, const void* d_planes, int method, spk_run* d_runs,
                int64_t run_cap, uint32_t* d_counts, int32_t* d_last, void* stream) {
    int rc = check_geom(g, true);
    if (rc) return rc;
    if (method != SPK_FSR && method != SPK_SSR)
        return fail(SPK_EINVAL, "spk_segment: method must be fsr or ssr");
    if (run_cap < 1 || run_cap > INT_MAX) return fail(SPK_EINVAL, "spk_segment: bad run_cap");
    const int64_t npix = npix_of(g);
    cudaStream_t s = as_stream(stream);
    if (g->frames == 0) {
        SPK_CK(cudaMemsetAsync(d_counts, 0, (size_t)npix * sizeof(uint32_t), s));
        SPK_CK(cudaMemsetAsync(d_last, 0xff, (size_t)npix * sizeof(int32_t), s));
        return SPK_OK;
    }
    if (!d_planes || !d_runs || !d_counts || !d_last)
        return fail(SPK_EINVAL, "spk: null device buffer");
    int dev = 0;
    SPK_CK(cudaGetDevice(&dev));
    ensure_pool(dev);
    SegArgs a;
    a.planes = d_planes;
    a.pitch = g->plane_pitch;
    a.npix = npix;
    a.frames = (int)g->frames;
    a.cap = (int)run_cap;
    a.nchunks = (int)((g->frames + kChunk - 1) / kChunk);
    a.runs = d_runs;
    a.counts = d_counts;
    a.last = d_last;
    return launch_segment(method, a, s);
}

int spk_segment_state(const spk_geom* g, const void* d_planes, int method, spk_run* d_runs,
                      int64_t run_cap, uint32_t* d_counts, int32_t* d_last,
                      const int32_t* d_state_in, int32_t* d_state_out, void* stream) {
    int rc = check_geom(g, true);
    if (rc) return rc;
    if (method != SPK_FSR && method != SPK_SSR)
        return fail(SPK_EINVAL, "spk_segment: method must be fsr or ssr");
    if (run_cap < 1 || run_cap > INT_MAX) return fail(SPK_EINVAL, "spk_segment: bad run_cap");
    if (!d_runs || !d_counts || !d_last || (g->frames > 0 && !d_planes))
        return fail(SPK_EINVAL, "spk: null device buffer");
    int dev = 0;
    SPK_CK(cudaGetDevice(&dev));
    ensure_pool(dev);
    SegArgs a;
    a.planes = d_planes;
    a.pitch = g->plane_pitch;
    a.npix = npix_of(g);
    a.frames = (int)g->frames;
    a.cap = (int)run_cap;
    a.nchunks = (int)((g->frames + kChunk - 1) / kChunk);
    a.runs = d_runs;
    a.counts = d_counts;
    a.last = d_last;
    a.state_in = d_state_in;
    a.state_out = d_state_out;
    return launch_segment(method, a, as_stream(stream));
}

int spk_segment_shards(const spk_geom* g, const void* d_planes, int method, int64_t shard_frames,
                       spk_run* d_runs, int64_t run_cap, uint32_t* d_counts, int32_t* d_last,
                       int32_t* d_state_out, void* stream) {
    int rc = check_geom(g, true);
    if (rc) return rc;
    if (method != SPK_FSR && method != SPK_SSR)
        return fail(SPK_EINVAL, "spk_segment_shards: method must be fsr or ssr");
    if (run_cap < 1 || run_cap > INT_MAX) return fail(SPK_EINVAL, "spk_segment_shards: bad run_cap");
    if (shard_frames < 32 || shard_frames % 32 != 0 || shard_frames > INT_MAX)
        return fail(SPK_EINVAL, "spk_segment_shards: shard_frames must be a positive multiple of 32");
    if (g->frames == 0) return SPK_OK;
    if (!d_planes || !d_runs || !d_counts || !d_last) return fail(SPK_EINVAL, "spk: null device buffer");
    const int64_t shards = (g->frames + shard_frames - 1) / shard_frames;
    if (shards > 65535) return fail(SPK_EINVAL, "spk_segment_shards: more than 65535 shards");
    int dev = 0;
    SPK_CK(cudaGetDevice(&dev));
    ensure_pool(dev);
    SegArgs a;
    a.planes = d_planes;
    a.pitch = g->plane_pitch;
    a.npix = npix_of(g);
    a.frames = (int)g->frames;
    a.cap = (int)run_cap;
    a.nchunks = 0;
    a.runs = d_runs;
    a.counts = d_counts;
    a.last = d_last;
    a.state_out = d_state_out;
    a.shard_frames = (int)shard_frames;
    return launch_segment(method, a, as_stream(stream));
}

namespace {

ShardArgs shard_args(const spk_geom* g, const void* planes, const int32_t* entry, const spk_sync* sync,
                     const spk_run* prefix, int32_t pcap, const int32_t* tstate) {
    ShardArgs a{};
    a.planes = planes;
    a.pitch = g->plane_pitch;
    a.npix = npix_of(g);
    a.frames = (int)g->frames;
    a.entry = entry;
    a.prefix = const_cast<spk_run*>(prefix);
    a.pcap = pcap;
    a.sync = const_cast<spk_sync*>(sync);
    a.tstate = const_cast<int32_t*>(tstate);
    return a;
}

int check_shard(const spk_geom* g, int method, int32_t pcap) {
    int rc = check_geom(g, false);
    if (rc) return rc;
    if (method != SPK_FSR && method != SPK_SSR)
        return fail(SPK_EINVAL, "spk_shard: method must be fsr or ssr");
    if (pcap < 1) return fail(SPK_EINVAL, "spk_shard: prefix_cap must be >= 1");
    return SPK_OK;
}

}  // namespace

int spk_shard_resolve(const spk_geom* g, const void* d_planes, int method, const int32_t* d_entry,
                      const spk_run* d_spec, int64_t spec_cap, const uint32_t* d_spec_counts,
                      const int32_t* d_spec_state, spk_run* d_prefix, int32_t prefix_cap,
                      spk_sync* d_sync, int32_t* d_tstate, void* stream) {
    int rc = check_shard(g, method, prefix_cap);
    if (rc) return rc;
    if ((rc = check_geom(g, true))) return rc;
    if (!d_entry || !d_prefix || !d_sync || !d_tstate || (g->frames > 0 && !d_planes))
        return fail(SPK_EINVAL, "spk: null device buffer");
    if (!d_spec || !d_spec_counts || !d_spec_state || spec_cap < 1 || spec_cap > INT_MAX)
        return fail(SPK_EINVAL, "spk_shard_resolve: bad speculative lists");
    ShardArgs a = shard_args(g, d_planes, d_entry, d_sync, d_prefix, prefix_cap, d_tstate);
    a.spec = d_spec;
    a.scap = (int)spec_cap;
    a.scount = d_spec_counts;
    a.sstate = d_spec_state;
    const int64_t threads = (a.npix + 31) / 32 * 32;
    const unsigned blocks = (unsigned)((threads + 63) / 64);
    cudaStream_t s = as_stream(stream);
    if (method == SPK_FSR)
        k_resolve<kFSR><<<blocks, 64, 0, s>>>(a);
    else
        k_resolve<kSSR><<<blocks, 64, 0, s>>>(a);
    SPK_LAUNCHED("k_resolve");
    return SPK_OK;
}

int spk_shard_junction(const spk_geom* g, int method, const int32_t* d_entry, const spk_sync* d_sync,
                       const spk_run* d_prefix, int32_t prefix_cap, const int32_t* d_tstate,
                       const spk_run* d_spec, int64_t spec_cap, const uint32_t* d_spec_counts,
                       const int32_t* d_spec_state, const spk_run* d_fb, const uint32_t* d_fb_counts,
                       const int32_t* d_fb_state, int32_t* d_exit_state, spk_close* d_entry_close,
                       spk_close* d_tail_close, void* stream) {
    int rc = check_shard(g, method, prefix_cap);
    if (rc) return rc;
    if (spec_cap < 1 || spec_cap > INT_MAX) return fail(SPK_EINVAL, "spk_shard: bad spec_cap");
    if (!d_entry || !d_sync || !d_prefix || !d_tstate || !d_spec || !d_spec_counts || !d_spec_state ||
        !d_exit_state || !d_entry_close || !d_tail_close)
        return fail(SPK_EINVAL, "spk: null device buffer");
    ShardArgs a = shard_args(g, nullptr, d_entry, d_sync, d_prefix, prefix_cap, d_tstate);
    a.spec = d_spec;
    a.scap = (int)spec_cap;
    a.scount = d_spec_counts;
    a.sstate = d_spec_state;
    a.fb = d_fb;
    a.fbcount = d_fb_counts;
    a.fbstate = d_fb_state;
    a.exit_state = d_exit_state;
    a.entry_close = d_entry_close;
    a.tail_close = d_tail_close;
    const unsigned blocks = (unsigned)((a.npix + 127) / 128);
    cudaStream_t s = as_stream(stream);
    if (method == SPK_FSR)
        k_junction<kFSR><<<blocks, 128, 0, s>>>(a);
    else
        k_junction<kSSR><<<blocks, 128, 0, s>>>(a);
    SPK_LAUNCHED("k_junction");
    return SPK_OK;
}

int spk_state_fresh(int64_t npix, int32_t* d_state, void* stream) {
    if (npix < 1 || !d_state) return fail(SPK_EINVAL, "spk_state_fresh: bad arguments");
    k_state_fresh<<<(unsigned)((npix + 255) / 256), 256, 0, as_stream(stream)>>>(d_state, npix);
    SPK_LAUNCHED("k_state_fresh");
    return SPK_OK;
}

int spk_shard_close_chain(int64_t npix, const spk_close* d_entry_close_next,
                          const spk_close* d_close_next, int32_t shard_len, spk_close* d_close,
                          void* stream) {
    if (npix < 1 || !d_entry_close_next || !d_close_next || !d_close)
        return fail(SPK_EINVAL, "spk_shard_close_chain: bad arguments");
    k_close_chain<<<(unsigned)((npix + 255) / 256), 256, 0, as_stream(stream)>>>(
        d_entry_close_next, d_close_next, shard_len, npix, d_close);
    SPK_LAUNCHED("k_close_chain");
    return SPK_OK;
}

int spk_shard_stitch(const spk_geom* g, int method, const int32_t* d_entry, const spk_sync* d_sync,
                     const spk_run* d_prefix, int32_t prefix_cap, const int32_t* d_tstate,
                     const spk_run* d_spec, int64_t spec_cap, const uint32_t* d_spec_counts,
                     const int32_t* d_spec_state, const spk_run* d_fb, const uint32_t* d_fb_counts,
                     const int32_t* d_fb_state, const spk_close* d_close, spk_run* d_region,
                     int64_t region_cap, uint32_t* d_region_counts, int32_t* d_region_last,
                     void* stream) {
    int rc = check_shard(g, method, prefix_cap);
    if (rc) return rc;
    if (spec_cap < 1 || spec_cap > INT_MAX || region_cap < 1 || region_cap > INT_MAX)
        return fail(SPK_EINVAL, "spk_shard: bad capacity");
    if (!d_entry || !d_sync || !d_prefix || !d_tstate || !d_spec || !d_spec_counts || !d_spec_state ||
        !d_close || !d_region || !d_region_counts || !d_region_last)
        return fail(SPK_EINVAL, "spk: null device buffer");
    ShardArgs a = shard_args(g, nullptr, d_entry, d_sync, d_prefix, prefix_cap, d_tstate);
    a.spec = d_spec;
    a.scap = (int)spec_cap;
    a.scount = d_spec_counts;
    a.sstate = d_spec_state;
    a.fb = d_fb;
    a.fbcount = d_fb_counts;
    a.fbstate = d_fb_state;
    a.close = d_close;
    a.region = d_region;
    a.rcap = (int)region_cap;
    a.rcount = d_region_counts;
    a.rlast = d_region_last;
    const unsigned blocks = (unsigned)((a.npix + 127) / 128);
    cudaStream_t s = as_stream(stream);
    if (method == SPK_FSR)
        k_stitch<kFSR><<<blocks, 128, 0, s>>>(a);
    else
        k_stitch<kSSR><<<blocks, 128, 0, s>>>(a);
    SPK_LAUNCHED("k_stitch");
    return SPK_OK;
}

int spk_pack_bytes(const spk_geom* g, const uint8_t* d_bytes, void* d_planes, void* stream) {
    int rc = check_geom(g, true);
    if (rc) return rc;
    if (g->frames == 0) return SPK_OK;
    if (!d_bytes || !d_planes) return fail(SPK_EINVAL, "spk: null device buffer");
    const int64_t total = g->frames * (int64_t)g->plane_pitch;
    const unsigned blocks = (unsigned)std::min<int64_t>((total + 255) / 256, 148 * 64);
    k_pack<<<blocks, 256, 0, as_stream(stream)>>>(d_bytes, npix_of(g), g->frames,
                                                  static_cast<uint8_t*>(d_planes), g->plane_pitch);
    SPK_LAUNCHED("k_pack");
    return SPK_OK;
}

int spk_unpack_planes(const spk_geom* g, const void* d_planes, uint8_t* d_bytes, void* stream) {
    int rc = check_geom(g, true);
    if (rc) return rc;
    if (g->frames == 0) return SPK_OK;
    if (!d_bytes || !d_planes) return fail(SPK_EINVAL, "spk: null device buffer");
    const int64_t total = g->frames * (int64_t)plane_bytes(g);
    const unsigned blocks = (unsigned)std::min<int64_t>((total + 255) / 256, 148 * 64);
    k_unpack<<<blocks, 256, 0, as_stream(stream)>>>(static_cast<const uint8_t*>(d_planes),
                                                    g->plane_pitch, npix_of(g), g->frames, d_bytes);
    SPK_LAUNCHED("k_unpack");
    return SPK_OK;
}

int spk_upload_planes(const spk_geom* g, const void* h_payload, size_t src_pitch, int msb_first,
                      void* d_planes, void* stream) {
    int rc = check_geom(g, true);
    if (rc) return rc;
    if (g->frames == 0) return SPK_OK;
    const size_t row = plane_bytes(g);
    if (!h_payload || !d_planes || src_pitch < row)
        return fail(SPK_EINVAL, "spk_upload_planes: bad buffer or src_pitch");
    cudaStream_t s = as_stream(stream);
    if (g->plane_pitch > row)  // deterministic pad bytes
        SPK_CK(cudaMemsetAsync(d_planes, 0, g->plane_pitch * (size_t)g->frames, s));
    SPK_CK(cudaMemcpy2DAsync(d_planes, g->plane_pitch, h_payload, src_pitch, row,
                             (size_t)g->frames, cudaMemcpyHostToDevice, s));
    if (msb_first) {
        const int64_t total = g->frames * (int64_t)row;
        const unsigned blocks = (unsigned)std::min<int64_t>((total + 255) / 256, 148 * 64);
        k_bitrev_bytes<<<blocks, 256, 0, s>>>(static_cast<uint8_t*>(d_planes), g->plane_pitch, row,
                                              g->frames);
        SPK_LAUNCHED("k_bitrev_bytes");
    }
    return SPK_OK;
}

size_t spk_plane_pitch(int32_t width, int32_t height) {
    const int64_t npix = (int64_t)width * height;
    return (min_pitch(npix) + 15) & ~(size_t)15;  // 16-B rows: vector/TMA friendly
}

namespace {

// One pixel band (a bn x 1 volume) through the host boundary on the current
// device: its plane columns are read from a payload of src_pitch bytes per
// frame, its frames written to columns [0, bn) of h_out (out_pitch elements
// per frame).  Synchronous.
int spk_reconstruct_host_band(const spk_geom* bg, const uint8_t* h_payload, size_t src_pitch,
                              int method, int tfp_window, int out_type, uint8_t* h_out,
                              size_t out_pitch, int64_t bn) {
    spk_geom dg = *bg;
    dg.plane_pitch = spk_plane_pitch(bg->width, bg->height);
    const size_t esz = out_type == SPK_OUT_U8 ? 1 : out_type == SPK_OUT_F32 ? 4 : 8;
    int dev = 0;
    SPK_CK(cudaGetDevice(&dev));
    ensure_pool(dev);
    cudaStream_t s;
    SPK_CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    int rc = [&]() -> int {
        Scratch planes(s), out(s);
        SPK_CK(planes.alloc(dg.plane_pitch * (size_t)bg->frames));
        SPK_CK(out.alloc((size_t)bn * esz * (size_t)bg->frames));
        int r = spk_upload_planes(&dg, h_payload, src_pitch, 0, planes.p, s);
        if (r) return r;
        if (out_type == SPK_OUT_U8)
            r = spk_reconstruct_u8(&dg, planes.p, method, tfp_window, static_cast<uint8_t*>(out.p), (size_t)bn, s);
        else if (out_type == SPK_OUT_F32)
            r = spk_reconstruct_f32(&dg, planes.p, method, tfp_window, static_cast<float*>(out.p), (size_t)bn, s);
        else
            r = spk_reconstruct_f64(&dg, planes.p, method, tfp_window, static_cast<double*>(out.p), (size_t)bn, s);
        if (r) return r;
        SPK_CK(cudaMemcpy2DAsync(h_out, out_pitch * esz, out.p, (size_t)bn * esz, (size_t)bn * esz,
                                 (size_t)bg->frames, cudaMemcpyDeviceToHost, s));
        return SPK_OK;
    }();
    cudaError_t se = cudaStreamSynchronize(s);
    cudaStreamDestroy(s);
    if (rc) return rc;
    if (se != cudaSuccess) return cuda_fail(se, "cudaStreamSynchronize");
    return SPK_OK;
}

}  // namespace

int spk_reconstruct_host(const spk_geom* g, const void* h_payload, int method, int tfp_window,
                         int out_type, void* h_out, size_t out_pitch) {
    spk_geom dg = *g;
    dg.plane_pitch = spk_plane_pitch(g->width, g->height);
    int rc = check_geom(&dg, true);
    if (rc) return rc;
    if ((rc = check_method(method, tfp_window))) return rc;
    if (out_type < SPK_OUT_U8 || out_type > SPK_OUT_F64)
        return fail(SPK_EINVAL, "spk_reconstruct_host: bad out_type");
    const int64_t npix = npix_of(g);
    if (out_pitch < (size_t)npix) return fail(SPK_EINVAL, "spk: out_pitch must be >= W*H");
    if (g->frames == 0) return SPK_OK;
    if (!h_payload || !h_out) return fail(SPK_EINVAL, "spk: null host buffer");
    const size_t esz = out_type == SPK_OUT_U8 ? 1 : out_type == SPK_OUT_F32 ? 4 : 8;
    int dev = 0;
    SPK_CK(cudaGetDevice(&dev));
    ensure_pool(dev);
    cudaStream_t s;
    SPK_CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    rc = [&]() -> int {
        Scratch planes(s), out(s);
        SPK_CK(planes.alloc(dg.plane_pitch * (size_t)g->frames));
        SPK_CK(out.alloc(out_pitch * esz * (size_t)g->frames));
        int r = spk_upload_planes(&dg, h_payload, plane_bytes(g), 0, planes.p, s);
        if (r) return r;
        if (out_type == SPK_OUT_U8)
            r = spk_reconstruct_u8(&dg, planes.p, method, tfp_window, static_cast<uint8_t*>(out.p),
                                   out_pitch, s);
        else if (out_type == SPK_OUT_F32)
            r = spk_reconstruct_f32(&dg, planes.p, method, tfp_window, static_cast<float*>(out.p),
                                    out_pitch, s);
        else
            r = spk_reconstruct_f64(&dg, planes.p, method, tfp_window, static_cast<double*>(out.p),
                                    out_pitch, s);
        if (r) return r;
        SPK_CK(cudaMemcpyAsync(h_out, out.p, out_pitch * esz * (size_t)g->frames,
                               cudaMemcpyDeviceToHost, s));
        return SPK_OK;
    }();
    cudaError_t se = cudaStreamSynchronize(s);
    cudaStreamDestroy(s);
    if (rc) return rc;
    if (se != cudaSuccess) return cuda_fail(se, "cudaStreamSynchronize");
    return SPK_OK;
}

int spk_reconstruct_host_multi(const spk_geom* g, const void* h_payload, int method, int tfp_window,
                               int out_type, void* h_out, size_t out_pitch, const int32_t* devices,
                               int32_t nbands) {
    spk_geom dg = *g;
    dg.plane_pitch = spk_plane_pitch(g->width, g->height);
    int rc = check_geom(&dg, true);
    if (rc) return rc;
    if ((rc = check_method(method, tfp_window))) return rc;
    if (out_type < SPK_OUT_U8 || out_type > SPK_OUT_F64)
        return fail(SPK_EINVAL, "spk_reconstruct_host_multi: bad out_type");
    if (nbands < 1 || !devices) return fail(SPK_EINVAL, "spk_reconstruct_host_multi: no devices");
    const int64_t npix = npix_of(g);
    if (out_pitch < (size_t)npix) return fail(SPK_EINVAL, "spk: out_pitch must be >= W*H");
    if (g->frames == 0) return SPK_OK;
    if (!h_payload || !h_out) return fail(SPK_EINVAL, "spk: null host buffer");
    int ndev = 0;
    SPK_CK(cudaGetDeviceCount(&ndev));
    for (int i = 0; i < nbands; ++i)
        if (devices[i] < 0 || devices[i] >= ndev)
            return fail(SPK_EINVAL, "spk_reconstruct_host_multi: no such device");
    const size_t esz = out_type == SPK_OUT_U8 ? 1 : out_type == SPK_OUT_F32 ? 4 : 8;
    // pixel bands on 128-pixel boundaries (16-byte aligned plane columns and
    // output columns), one host thread and one device each; every band is an
    // independent (p1-p0) x 1 volume: pixels never interact
    const int64_t units = (npix + 127) / 128;
    struct Band {
        int rc = SPK_OK;
        std::string err;
        int64_t launches = 0;
    };
    std::vector<Band> res((size_t)nbands);
    std::vector<std::thread> th;
    for (int i = 0; i < nbands; ++i) {
        const int64_t p0 = std::min(npix, units * i / nbands * 128);
        const int64_t p1 = std::min(npix, units * (i + 1) / nbands * 128);
        if (p1 <= p0) continue;
        th.emplace_back([&, i, p0, p1]() {
            Band& b = res[(size_t)i];
            b.rc = [&]() -> int {
                SPK_CK(cudaSetDevice(devices[i]));
                spk_geom bg;
                bg.width = (int32_t)(p1 - p0);
                bg.height = 1;
                bg.frames = g->frames;
                bg.plane_pitch = 0;
                const int64_t bn = p1 - p0;
                return spk_reconstruct_host_band(&bg, static_cast<const uint8_t*>(h_payload) + p0 / 8,
                                                 plane_bytes(g), method, tfp_window, out_type,
                                                 static_cast<uint8_t*>(h_out) + p0 * esz, out_pitch, bn);
            }();
            if (b.rc) b.err = g_err;
            b.launches = g_launches;
        });
    }
    for (auto& t : th) t.join();
    for (const Band& b : res) {
        g_launches += b.launches;
        if (b.rc) return fail(b.rc, b.err);
    }
    return SPK_OK;
}

// ---- device batch: one CUDA graph of `count` reconstructions --------------
// configs[3] (64 independent streams): every call is a handful of short
// kernels, so a batch issued call by call leaves SM tails and launch gaps
// between them.  The batch is captured once into a CUDA graph -- the calls
// spread over kBatchBranches forked branches so kernels of different volumes
// overlap -- and the instantiated graph is cached (keyed by geometry, method
// and the buffer addresses) and replayed on later calls with the same
// buffers.  Measured (configs[3], profiles/c4_probe.py): FSR 14.4 -> 12.6 ms,
// SSR 32.7 -> 29.5 ms per batch of 64.
namespace {

constexpr int kBatchBranches = 4;
constexpr int kBatchCache = 4;

struct BatchGraph {
    std::vector<uint64_t> key;
    cudaGraphExec_t exec = nullptr;
};

struct BatchState {
    cudaStream_t origin = nullptr;  // capture origin
    cudaStream_t branch[kBatchBranches] = {};
    cudaEvent_t fork = nullptr, join[kBatchBranches] = {};
    std::vector<BatchGraph> cache;  // most recent last
};

BatchState& batch_state(int dev) {
    thread_local BatchState per_dev[64];
    BatchState& b = per_dev[dev & 63];
    if (!b.origin) {
        cudaStreamCreateWithFlags(&b.origin, cudaStreamNonBlocking);
        for (auto& x : b.branch) cudaStreamCreateWithFlags(&x, cudaStreamNonBlocking);
        cudaEventCreateWithFlags(&b.fork, cudaEventDisableTiming);
        for (auto& e : b.join) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
    }
    return b;
}

}  // namespace

int spk_reconstruct_batch(const spk_geom* g, int32_t count, const void* const* d_planes, int method,
                          int tfp_window, int out_type, void* const* d_outs, size_t out_pitch,
                          void* stream) {
    int rc = check_geom(g, true);
    if (rc) return rc;
    if ((rc = check_method(method, tfp_window))) return rc;
    if (out_type < SPK_OUT_U8 || out_type > SPK_OUT_F64)
        return fail(SPK_EINVAL, "spk_reconstruct_batch: bad out_type");
    if (out_pitch < (size_t)npix_of(g)) return fail(SPK_EINVAL, "spk: out_pitch must be >= W*H");
    if (count < 0 || (count > 0 && (!d_planes || !d_outs)))
        return fail(SPK_EINVAL, "spk_reconstruct_batch: bad volume list");
    if (g->frames == 0 || count == 0) return SPK_OK;
    for (int i = 0; i < count; ++i)
        if (!d_planes[i] || !d_outs[i]) return fail(SPK_EINVAL, "spk: null device buffer");
    int dev = 0;
    SPK_CK(cudaGetDevice(&dev));
    ensure_pool(dev);
    BatchState& b = batch_state(dev);
    std::vector<uint64_t> key = {(uint64_t)dev, (uint64_t)g->width, (uint64_t)g->height, (uint64_t)g->frames,
                                 (uint64_t)g->plane_pitch, (uint64_t)method, (uint64_t)tfp_window,
                                 (uint64_t)out_type, (uint64_t)out_pitch, (uint64_t)count,
                                 (uint64_t)g_run_cap.load()};
    for (int i = 0; i < count; ++i) {
        key.push_back(reinterpret_cast<uintptr_t>(d_planes[i]));
        key.push_back(reinterpret_cast<uintptr_t>(d_outs[i]));
    }
    cudaGraphExec_t exec = nullptr;
    for (size_t i = 0; i < b.cache.size(); ++i)
        if (b.cache[i].key == key) {
            exec = b.cache[i].exec;
            std::rotate(b.cache.begin() + i, b.cache.begin() + i + 1, b.cache.end());
            break;
        }
    if (!exec) {
        const bool timing = g_timing;
        g_timing = false;  // no timing events inside the graph
        SPK_CK(cudaStreamBeginCapture(b.origin, cudaStreamCaptureModeThreadLocal));
        rc = [&]() -> int {
            SPK_CK(cudaEventRecord(b.fork, b.origin));
            for (auto& x : b.branch) SPK_CK(cudaStreamWaitEvent(x, b.fork, 0));
            for (int i = 0; i < count; ++i) {
                cudaStream_t s = b.branch[i % kBatchBranches];
                int r;
                if (out_type == SPK_OUT_U8)
                    r = reconstruct_impl<uint8_t>(g, d_planes[i], method, tfp_window,
                                                  static_cast<uint8_t*>(d_outs[i]), out_pitch, s);
                else if (out_type == SPK_OUT_F32)
                    r = reconstruct_impl<float>(g, d_planes[i], method, tfp_window,
                                                static_cast<float*>(d_outs[i]), out_pitch, s);
                else
                    r = reconstruct_impl<double>(g, d_planes[i], method, tfp_window,
                                                 static_cast<double*>(d_outs[i]), out_pitch, s);
                if (r) return r;
            }
            for (int k = 0; k < kBatchBranches; ++k) {
                SPK_CK(cudaEventRecord(b.join[k], b.branch[k]));
                SPK_CK(cudaStreamWaitEvent(b.origin, b.join[k], 0));
            }
            return SPK_OK;
        }();
        g_timing = timing;
        cudaGraph_t graph = nullptr;
        const cudaError_t ee = cudaStreamEndCapture(b.origin, &graph);
        if (rc) {
            if (graph) cudaGraphDestroy(graph);
            return rc;
        }
        if (ee != cudaSuccess) return cuda_fail(ee, "spk_reconstruct_batch: capture");
        const cudaError_t ie = cudaGraphInstantiate(&exec, graph, 0);
        cudaGraphDestroy(graph);
        if (ie != cudaSuccess) return cuda_fail(ie, "spk_reconstruct_batch: instantiate");
        if ((int)b.cache.size() >= kBatchCache) {
            cudaGraphExecDestroy(b.cache.front().exec);
            b.cache.erase(b.cache.begin());
        }
        b.cache.push_back(BatchGraph{key, exec});
    }
    SPK_CK(cudaGraphLaunch(exec, as_stream(stream)));
    SPK_LAUNCHED("spk_reconstruct_batch graph");
    return SPK_OK;
}

int spk_batch_release(void) {
    int dev = 0;
    SPK_CK(cudaGetDevice(&dev));
    BatchState& b = batch_state(dev);
    SPK_CK(cudaDeviceSynchronize());
    for (auto& c : b.cache) cudaGraphExecDestroy(c.exec);
    b.cache.clear();
    return SPK_OK;
}

int spk_reconstruct_host_batch(const spk_geom* g, int32_t count, const void* const* h_payloads,
                               int method, int tfp_window, int out_type, void* const* h_outs,
                               size_t out_pitch) {
    spk_geom dg = *g;
    dg.plane_pitch = spk_plane_pitch(g->width, g->height);
    int rc = check_geom(&dg, true);
    if (rc) return rc;
    if ((rc = check_method(method, tfp_window))) return rc;
    if (out_type < SPK_OUT_U8 || out_type > SPK_OUT_F64)
        return fail(SPK_EINVAL, "spk_reconstruct_host_batch: bad out_type");
    const int64_t npix = npix_of(g);
    if (out_pitch < (size_t)npix) return fail(SPK_EINVAL, "spk: out_pitch must be >= W*H");
    if (count < 0 || (count > 0 && (!h_payloads || !h_outs)))
        return fail(SPK_EINVAL, "spk_reconstruct_host_batch: bad volume list");
    if (g->frames == 0 || count == 0) return SPK_OK;
    for (int i = 0; i < count; ++i)
        if (!h_payloads[i] || !h_outs[i]) return fail(SPK_EINVAL, "spk: null host buffer");
    const size_t esz = out_type == SPK_OUT_U8 ? 1 : out_type == SPK_OUT_F32 ? 4 : 8;
    int dev = 0;
    SPK_CK(cudaGetDevice(&dev));
    ensure_pool(dev);
    // Two lanes of (H2D, kernels, D2H), round robin: while volume i's frames
    // come back over PCIe, volume i+1 is uploaded and reconstructed.
    constexpr int kLanes = 2;
    cudaStream_t st[kLanes] = {nullptr, nullptr};
    for (auto& x : st) SPK_CK(cudaStreamCreateWithFlags(&x, cudaStreamNonBlocking));
    rc = [&]() -> int {
        Scratch planes0(st[0]), planes1(st[1]), out0(st[0]), out1(st[1]);
        Scratch* planes[kLanes] = {&planes0, &planes1};
        Scratch* outs[kLanes] = {&out0, &out1};
        for (int l = 0; l < kLanes && l < count; ++l) {
            SPK_CK(planes[l]->alloc(dg.plane_pitch * (size_t)g->frames));
            SPK_CK(outs[l]->alloc(out_pitch * esz * (size_t)g->frames));
        }
        for (int i = 0; i < count; ++i) {
            const int l = i % kLanes;
            cudaStream_t s = st[l];
            int r = spk_upload_planes(&dg, h_payloads[i], plane_bytes(g), 0, planes[l]->p, s);
            if (r) return r;
            if (out_type == SPK_OUT_U8)
                r = spk_reconstruct_u8(&dg, planes[l]->p, method, tfp_window,
                                       static_cast<uint8_t*>(outs[l]->p), out_pitch, s);
            else if (out_type == SPK_OUT_F32)
                r = spk_reconstruct_f32(&dg, planes[l]->p, method, tfp_window,
                                        static_cast<float*>(outs[l]->p), out_pitch, s);
            else
                r = spk_reconstruct_f64(&dg, planes[l]->p, method, tfp_window,
                                        static_cast<double*>(outs[l]->p), out_pitch, s);
            if (r) return r;
            SPK_CK(cudaMemcpyAsync(h_outs[i], outs[l]->p, out_pitch * esz * (size_t)g->frames,
                                   cudaMemcpyDeviceToHost, s));
        }
        return SPK_OK;
    }();
    cudaError_t se = cudaSuccess;
    for (auto& x : st) {
        const cudaError_t e = cudaStreamSynchronize(x);
        if (se == cudaSuccess) se = e;
        cudaStreamDestroy(x);
    }
    if (rc) return rc;
    if (se != cudaSuccess) return cuda_fail(se, "cudaStreamSynchronize");
    return SPK_OK;
}

int spk_segment_host(const spk_geom* g, const void* h_payload, int method, spk_run* h_runs,
                     int64_t run_cap, uint32_t* h_counts, int32_t* h_last) {
    spk_geom dg = *g;
    dg.plane_pitch = spk_plane_pitch(g->width, g->height);
    int rc = check_geom(&dg, true);
    if (rc) return rc;
    if (method != SPK_FSR && method != SPK_SSR)
        return fail(SPK_EINVAL, "spk_segment: method must be fsr or ssr");
    if (run_cap < 1 || run_cap > INT_MAX) return fail(SPK_EINVAL, "spk_segment: bad run_cap");
    const size_t npix = (size_t)npix_of(g);
    if (!h_counts || !h_last || (g->frames > 0 && (!h_payload || !h_runs)))
        return fail(SPK_EINVAL, "spk: null host buffer");
    if (g->frames == 0) {
        std::fill(h_counts, h_counts + npix, 0u);
        std::fill(h_last, h_last + npix, -1);
        return SPK_OK;
    }
    int dev = 0;
    SPK_CK(cudaGetDevice(&dev));
    ensure_pool(dev);
    cudaStream_t s;
    SPK_CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    rc = [&]() -> int {
        Scratch planes(s), runs(s), counts(s), last(s);
        SPK_CK(planes.alloc(dg.plane_pitch * (size_t)g->frames));
        SPK_CK(runs.alloc(npix * (size_t)run_cap * sizeof(spk_run)));
        SPK_CK(counts.alloc(npix * sizeof(uint32_t)));
        SPK_CK(last.alloc(npix * sizeof(int32_t)));
        int r = spk_upload_planes(&dg, h_payload, plane_bytes(g), 0, planes.p, s);
        if (r) return r;
        r = spk_segment(&dg, planes.p, method, static_cast<spk_run*>(runs.p), run_cap,
                        static_cast<uint32_t*>(counts.p), static_cast<int32_t*>(last.p), s);
        if (r) return r;
        SPK_CK(cudaMemcpyAsync(h_runs, runs.p, npix * (size_t)run_cap * sizeof(spk_run),
                               cudaMemcpyDeviceToHost, s));
        SPK_CK(cudaMemcpyAsync(h_counts, counts.p, npix * sizeof(uint32_t),
                               cudaMemcpyDeviceToHost, s));
        SPK_CK(cudaMemcpyAsync(h_last, last.p, npix * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
        return SPK_OK;
    }();
    cudaError_t se = cudaStreamSynchronize(s);
    cudaStreamDestroy(s);
    if (rc) return rc;
    if (se != cudaSuccess) return cuda_fail(se, "cudaStreamSynchronize");
    return SPK_OK;
}

int spk_records(const spk_geom* g, const void* d_planes, int method, uint32_t fps, void** d_image,
                uint64_t* image_bytes, void* stream) {
    int rc = check_geom(g, true);
    if (rc) return rc;
    if (method != SPK_FSR && method != SPK_SSR)
        return fail(SPK_EINVAL, "--emit-records needs method fsr or ssr");
    if (g->width > 65535 || g->height > 65535)
        return fail(SPK_EINVAL, "spk_records: SPKR geometry is 16-bit (W, H <= 65535)");
    if (!d_image || !image_bytes || (g->frames > 0 && !d_planes))
        return fail(SPK_EINVAL, "spk: null buffer");
    *d_image = nullptr;
    *image_bytes = 0;
    const int64_t npix = npix_of(g);
    cudaStream_t s = as_stream(stream);
    int dev = 0;
    SPK_CK(cudaGetDevice(&dev));
    ensure_pool(dev);
    const int cap = run_capacity(g->frames);
    Scratch runs(s), counts(s), last(s), wc(s), offs(s);
    SPK_CK(runs.alloc((size_t)npix * cap * sizeof(spk_run)));
    SPK_CK(counts.alloc((size_t)npix * sizeof(uint32_t)));
    SPK_CK(last.alloc((size_t)npix * sizeof(int32_t)));
    SPK_CK(wc.alloc((size_t)npix * sizeof(uint32_t)));
    SPK_CK(offs.alloc((size_t)npix * sizeof(unsigned long long)));
    RecArgs r;
    r.seg.planes = d_planes;
    r.seg.pitch = g->plane_pitch;
    r.seg.npix = npix;
    r.seg.frames = (int)g->frames;
    r.seg.cap = cap;
    r.seg.nchunks = (int)((g->frames + kChunk - 1) / kChunk);
    r.seg.runs = static_cast<spk_run*>(runs.p);
    r.seg.counts = static_cast<uint32_t*>(counts.p);
    r.seg.last = static_cast<int32_t*>(last.p);
    r.wc = static_cast<uint32_t*>(wc.p);
    r.offs = static_cast<unsigned long long*>(offs.p);
    r.img = nullptr;
    r.width = g->width;
    r.height = g->height;
    r.fps = fps;
    if (g->frames > 0) {
        if ((rc = launch_segment(method, r.seg, s))) return rc;
    } else {
        SPK_CK(cudaMemsetAsync(r.seg.counts, 0, (size_t)npix * sizeof(uint32_t), s));
        SPK_CK(cudaMemsetAsync(r.seg.last, 0xff, (size_t)npix * sizeof(int32_t), s));
    }
    const unsigned blocks = (unsigned)((npix + 127) / 128);
    if (method == SPK_FSR)
        k_rec_count<kFSR><<<blocks, 128, 0, s>>>(r);
    else
        k_rec_count<kSSR><<<blocks, 128, 0, s>>>(r);
    SPK_LAUNCHED("k_rec_count");
    if ((rc = launch_scan(r.wc, static_cast<unsigned long long*>(offs.p), npix, s))) return rc;
    // image size = header + per-pixel counts + all words (one small readback)
    unsigned long long tail[2] = {0, 0};
    uint32_t tail_wc = 0;
    SPK_CK(cudaMemcpyAsync(&tail[0], r.offs + (npix - 1), sizeof(unsigned long long),
                           cudaMemcpyDeviceToHost, s));
    SPK_CK(cudaMemcpyAsync(&tail_wc, r.wc + (npix - 1), sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
    SPK_CK(cudaStreamSynchronize(s));
    const uint64_t words = tail[0] + tail_wc;
    const uint64_t bytes = 16 + 4 * (uint64_t)npix + 2 * words;
    void* img = nullptr;
    SPK_CK(cudaMallocAsync(&img, bytes, s));
    r.img = static_cast<uint8_t*>(img);
    if (method == SPK_FSR)
        k_rec_write<kFSR><<<blocks, 128, 0, s>>>(r);
    else
        k_rec_write<kSSR><<<blocks, 128, 0, s>>>(r);
    ++g_launches;
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        cudaFreeAsync(img, s);
        return cuda_fail(e, "k_rec_write");
    }
    *d_image = img;
    *image_bytes = bytes;
    return SPK_OK;
}

int spk_records_host(const spk_geom* g, const void* h_payload, int method, uint32_t fps,
                     void** h_image, uint64_t* image_bytes) {
    spk_geom dg = *g;
    dg.plane_pitch = spk_plane_pitch(g->width, g->height);
    int rc = check_geom(&dg, true);
    if (rc) return rc;
    if (!h_image || !image_bytes || (g->frames > 0 && !h_payload))
        return fail(SPK_EINVAL, "spk: null host buffer");
    *h_image = nullptr;
    *image_bytes = 0;
    int dev = 0;
    SPK_CK(cudaGetDevice(&dev));
    ensure_pool(dev);
    cudaStream_t s;
    SPK_CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    void* host = nullptr;
    rc = [&]() -> int {
        Scratch planes(s), img(s);
        SPK_CK(planes.alloc(dg.plane_pitch * (size_t)std::max<int64_t>(1, g->frames)));
        int r = spk_upload_planes(&dg, h_payload, plane_bytes(g), 0, planes.p, s);
        if (r) return r;
        uint64_t bytes = 0;
        r = spk_records(&dg, planes.p, method, fps, &img.p, &bytes, s);
        if (r) return r;
        host = std::malloc(bytes);
        if (!host) return fail(SPK_ENOMEM, "spk_records_host: host allocation failed");
        SPK_CK(cudaMemcpyAsync(host, img.p, bytes, cudaMemcpyDeviceToHost, s));
        *image_bytes = bytes;
        return SPK_OK;
    }();
    cudaError_t se = cudaStreamSynchronize(s);
    cudaStreamDestroy(s);
    if (!rc && se != cudaSuccess) rc = cuda_fail(se, "cudaStreamSynchronize");
    if (rc) {
        std::free(host);
        *image_bytes = 0;
        return rc;
    }
    *h_image = host;
    return SPK_OK;
}

int spk_free_device(void* d_ptr, void* stream) {
    if (d_ptr) SPK_CK(cudaFreeAsync(d_ptr, as_stream(stream)));
    return SPK_OK;
}

void spk_free_host(void* h_ptr) { std::free(h_ptr); }

}  // extern "C"

struct spk_stream {
    int32_t width, height;
    int64_t npix;
    int64_t frames;      // pushed so far
    int32_t* state;      // automaton state, relative to frame `frames`
    double* last_value;  // per pixel: intensity of the last closed run
};

namespace {

// count -> scan -> allocate -> write the events of one push / the flush
int stream_events(spk_stream* st, StreamArgs& a, spk_event** d_events, uint64_t** d_offsets,
                  uint64_t* total, cudaStream_t s) {
    const int64_t npix = st->npix;
    Scratch ecount(s);
    SPK_CK(ecount.alloc((size_t)(npix + 1) * sizeof(uint32_t)));
    SPK_CK(cudaMemsetAsync(static_cast<uint32_t*>(ecount.p) + npix, 0, sizeof(uint32_t), s));
    void* offs = nullptr;
    SPK_CK(cudaMallocAsync(&offs, (size_t)(npix + 1) * sizeof(unsigned long long), s));
    a.ecount = static_cast<uint32_t*>(ecount.p);
    a.eoffs = static_cast<unsigned long long*>(offs);
    const unsigned blocks = (unsigned)((npix + 127) / 128);
    k_stream_count<<<blocks, 128, 0, s>>>(a);
    SPK_LAUNCHED("k_stream_count");
    int rc = launch_scan(a.ecount, static_cast<unsigned long long*>(offs), npix + 1, s);
    if (rc) {
        cudaFreeAsync(offs, s);
        return rc;
    }
    unsigned long long tot = 0;
    SPK_CK(cudaMemcpyAsync(&tot, static_cast<unsigned long long*>(offs) + npix, sizeof(tot),
                           cudaMemcpyDeviceToHost, s));
    SPK_CK(cudaStreamSynchronize(s));
    void* ev = nullptr;
    SPK_CK(cudaMallocAsync(&ev, std::max<size_t>(16, (size_t)tot * sizeof(spk_event)), s));
    a.events = static_cast<spk_event*>(ev);
    k_stream_write<<<blocks, 128, 0, s>>>(a);
    SPK_LAUNCHED("k_stream_write");
    *d_events = static_cast<spk_event*>(ev);
    *d_offsets = static_cast<uint64_t*>(offs);
    *total = tot;
    return SPK_OK;
}

}  // namespace

extern "C" {

int spk_stream_create(int32_t width, int32_t height, void* stream, spk_stream** out) {
    if (!out) return fail(SPK_EINVAL, "spk_stream_create: null handle");
    *out = nullptr;
    spk_geom g{width, height, 0, 0};
    int rc = check_geom(&g, false);
    if (rc) return rc;
    cudaStream_t s = as_stream(stream);
    spk_stream* st = new spk_stream{width, height, npix_of(&g), 0, nullptr, nullptr};
    const int64_t npix = st->npix;
    cudaError_t e = cudaMalloc(&st->state, (size_t)Scan<kFSR>::kFields * npix * sizeof(int32_t));
    if (e == cudaSuccess) e = cudaMalloc(&st->last_value, (size_t)npix * sizeof(double));
    if (e == cudaSuccess) e = cudaMemsetAsync(st->last_value, 0, (size_t)npix * sizeof(double), s);
    if (e != cudaSuccess) {
        cudaFree(st->state);
        cudaFree(st->last_value);
        delete st;
        return cuda_fail(e, "spk_stream_create");
    }
    k_state_fresh<<<(unsigned)((npix + 255) / 256), 256, 0, s>>>(st->state, npix);
    ++g_launches;
    if ((e = cudaGetLastError()) != cudaSuccess) {
        cudaFree(st->state);
        cudaFree(st->last_value);
        delete st;
        return cuda_fail(e, "k_state_fresh");
    }
    *out = st;
    return SPK_OK;
}

int spk_stream_push(spk_stream* st, const void* d_planes, size_t plane_pitch, int64_t frames,
                    spk_event** d_events, uint64_t** d_offsets, uint64_t* total, void* stream) {
    if (!st || !d_events || !d_offsets || !total) return fail(SPK_EINVAL, "spk_stream_push: null argument");
    spk_geom g{st->width, st->height, frames, plane_pitch};
    int rc = check_geom(&g, true);
    if (rc) return rc;
    if (st->frames + frames >= (int64_t)1 << 29) return fail(SPK_EINVAL, "spk_stream_push: frames must stay < 2^29");
    if (frames > 0 && !d_planes) return fail(SPK_EINVAL, "spk: null device buffer");
    cudaStream_t s = as_stream(stream);
    int dev = 0;
    SPK_CK(cudaGetDevice(&dev));
    ensure_pool(dev);
    const int64_t npix = st->npix;
    Scratch state_out(s), counts(s), last(s), mx(s);
    SPK_CK(state_out.alloc((size_t)Scan<kFSR>::kFields * npix * sizeof(int32_t)));
    SPK_CK(counts.alloc((size_t)npix * sizeof(uint32_t)));
    SPK_CK(last.alloc((size_t)npix * sizeof(int32_t)));
    SPK_CK(mx.alloc(sizeof(uint32_t)));
    // the block's run lists (capacity grown once if any pixel needs more)
    int cap = (int)std::max<int64_t>(64, frames / 32);
    Scratch runs(s);
    for (int attempt = 0; attempt < 2; ++attempt) {
        if (runs.p) {
            cudaFreeAsync(runs.p, s);
            runs.p = nullptr;
        }
        SPK_CK(runs.alloc((size_t)npix * cap * sizeof(spk_run)));
        if (frames > 0) {
            SegArgs a;
            a.planes = d_planes;
            a.pitch = plane_pitch;
            a.npix = npix;
            a.frames = (int)frames;
            a.cap = cap;
            a.nchunks = (int)((frames + kChunk - 1) / kChunk);
            a.runs = static_cast<spk_run*>(runs.p);
            a.counts = static_cast<uint32_t*>(counts.p);
            a.last = static_cast<int32_t*>(last.p);
            a.state_in = st->state;
            a.state_out = static_cast<int32_t*>(state_out.p);
            if ((rc = launch_segment(SPK_FSR, a, s))) return rc;
        } else {
            SPK_CK(cudaMemsetAsync(counts.p, 0, (size_t)npix * sizeof(uint32_t), s));
            SPK_CK(cudaMemcpyAsync(state_out.p, st->state, (size_t)Scan<kFSR>::kFields * npix * sizeof(int32_t),
                                   cudaMemcpyDeviceToDevice, s));
        }
        SPK_CK(cudaMemsetAsync(mx.p, 0, sizeof(uint32_t), s));
        k_max_u32<<<148, 256, 0, s>>>(static_cast<uint32_t*>(counts.p), npix, static_cast<uint32_t*>(mx.p));
        SPK_LAUNCHED("k_max_u32");
        uint32_t need = 0;
        SPK_CK(cudaMemcpyAsync(&need, mx.p, sizeof(need), cudaMemcpyDeviceToHost, s));
        SPK_CK(cudaStreamSynchronize(s));
        if (need <= (uint32_t)cap) break;
        cap = (int)need;
    }
    StreamArgs a{};
    a.npix = npix;
    a.frame0 = st->frames;
    a.flush = 0;
    a.state_in = st->state;
    a.state_out = static_cast<int32_t*>(state_out.p);
    a.runs = static_cast<spk_run*>(runs.p);
    a.cap = cap;
    a.counts = static_cast<uint32_t*>(counts.p);
    a.last_value = st->last_value;
    if ((rc = stream_events(st, a, d_events, d_offsets, total, s))) return rc;
    // the end state, in the next block's frames, becomes the stream's state
    k_stream_shift<<<(unsigned)((npix + 255) / 256), 256, 0, s>>>(static_cast<int32_t*>(state_out.p), npix,
                                                                 (int)frames);
    SPK_LAUNCHED("k_stream_shift");
    SPK_CK(cudaMemcpyAsync(st->state, state_out.p, (size_t)Scan<kFSR>::kFields * npix * sizeof(int32_t),
                           cudaMemcpyDeviceToDevice, s));
    st->frames += frames;
    return SPK_OK;
}

int spk_stream_flush(spk_stream* st, spk_event** d_events, uint64_t** d_offsets, uint64_t* total,
                     void* stream) {
    if (!st || !d_events || !d_offsets || !total) return fail(SPK_EINVAL, "spk_stream_flush: null argument");
    cudaStream_t s = as_stream(stream);
    StreamArgs a{};
    a.npix = st->npix;
    a.frame0 = st->frames;
    a.flush = 1;
    a.state_in = st->state;
    a.last_value = st->last_value;
    return stream_events(st, a, d_events, d_offsets, total, s);
}

namespace {

// device events / offsets of one stream call -> malloc'd host copies
int stream_to_host(spk_stream* st, spk_event* d_ev, uint64_t* d_offs, uint64_t tot, spk_event** h_events,
                   uint64_t** h_offsets, cudaStream_t s) {
    const size_t ob = (size_t)(st->npix + 1) * sizeof(uint64_t), eb = (size_t)tot * sizeof(spk_event);
    *h_offsets = static_cast<uint64_t*>(std::malloc(ob));
    *h_events = static_cast<spk_event*>(std::malloc(std::max<size_t>(eb, 16)));
    int rc = SPK_OK;
    if (!*h_offsets || !*h_events) rc = fail(SPK_ENOMEM, "spk_stream: host allocation failed");
    cudaError_t e = cudaSuccess;
    if (!rc) e = cudaMemcpyAsync(*h_offsets, d_offs, ob, cudaMemcpyDeviceToHost, s);
    if (!rc && e == cudaSuccess && eb) e = cudaMemcpyAsync(*h_events, d_ev, eb, cudaMemcpyDeviceToHost, s);
    cudaFreeAsync(d_ev, s);
    cudaFreeAsync(d_offs, s);
    const cudaError_t se = cudaStreamSynchronize(s);
    if (!rc && e != cudaSuccess) rc = cuda_fail(e, "spk_stream: copy to host");
    if (!rc && se != cudaSuccess) rc = cuda_fail(se, "cudaStreamSynchronize");
    if (rc) {
        std::free(*h_offsets);
        std::free(*h_events);
        *h_offsets = nullptr;
        *h_events = nullptr;
    }
    return rc;
}

}  // namespace

int spk_stream_push_host(spk_stream* st, const void* h_payload, int64_t frames, spk_event** h_events,
                         uint64_t** h_offsets, uint64_t* total) {
    if (!st || !h_events || !h_offsets || !total || (frames > 0 && !h_payload))
        return fail(SPK_EINVAL, "spk_stream_push_host: null argument");
    spk_geom g{st->width, st->height, frames, spk_plane_pitch(st->width, st->height)};
    int rc = check_geom(&g, true);
    if (rc) return rc;
    cudaStream_t s;
    SPK_CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    rc = [&]() -> int {
        Scratch planes(s);
        SPK_CK(planes.alloc(g.plane_pitch * (size_t)std::max<int64_t>(1, frames)));
        int r = spk_upload_planes(&g, h_payload, plane_bytes(&g), 0, planes.p, s);
        if (r) return r;
        spk_event* dev = nullptr;
        uint64_t* doffs = nullptr;
        r = spk_stream_push(st, planes.p, g.plane_pitch, frames, &dev, &doffs, total, s);
        if (r) return r;
        return stream_to_host(st, dev, doffs, *total, h_events, h_offsets, s);
    }();
    cudaStreamDestroy(s);
    return rc;
}

int spk_stream_flush_host(spk_stream* st, spk_event** h_events, uint64_t** h_offsets, uint64_t* total) {
    if (!st || !h_events || !h_offsets || !total) return fail(SPK_EINVAL, "spk_stream_flush_host: null argument");
    cudaStream_t s;
    SPK_CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    spk_event* dev = nullptr;
    uint64_t* doffs = nullptr;
    int rc = spk_stream_flush(st, &dev, &doffs, total, s);
    if (!rc) rc = stream_to_host(st, dev, doffs, *total, h_events, h_offsets, s);
    cudaStreamDestroy(s);
    return rc;
}

int64_t spk_stream_frames(const spk_stream* st) { return st ? st->frames : -1; }

int spk_stream_destroy(spk_stream* st) {
    if (!st) return SPK_OK;
    cudaFree(st->state);
    cudaFree(st->last_value);
    delete st;
    return SPK_OK;
}

int spk_set_run_capacity(int64_t per_pixel) {
    if (per_pixel < 0 || per_pixel > INT_MAX) return fail(SPK_EINVAL, "spk: bad run capacity");
    g_run_cap.store(per_pixel);
    return SPK_OK;
}

int64_t spk_launch_count(int reset) {
    const int64_t n = g_launches;
    if (reset) g_launches = 0;
    return n;
}

int spk_set_timing(int enable) {
    g_timing = enable != 0;
    return SPK_OK;
}

int spk_last_split(int32_t* shards, int64_t* flagged) {
    if (g_ev_used < 2) return fail(SPK_EINVAL, "spk_last_split: no timed call");
    SPK_CK(cudaEventSynchronize(g_ev[g_ev_used - 1]));
    if (shards) *shards = g_split_shards;
    if (flagged) *flagged = g_split_shards > 1 && g_split_flagged ? (int64_t)*g_split_flagged : 0;
    return SPK_OK;
}

int spk_last_timing(float* segment_ms, float* finalize_ms, float* expand_ms, float* fixup_ms) {
    float* outs[4] = {segment_ms, finalize_ms, expand_ms, fixup_ms};
    for (float* o : outs)
        if (o) *o = -1.f;
    if (g_ev_used < 2) return fail(SPK_EINVAL, "spk_last_timing: no timed call");
    SPK_CK(cudaEventSynchronize(g_ev[g_ev_used - 1]));
    for (int k = 0; k + 1 < g_ev_used; ++k) {
        float ms = 0.f;
        SPK_CK(cudaEventElapsedTime(&ms, g_ev[k], g_ev[k + 1]));
        if (outs[k]) *outs[k] = ms;
    }
    return SPK_OK;
}

const char* spk_last_error(void) { return g_err.c_str(); }

int spk_device_count(void) {
    int n = 0;
    return cudaGetDeviceCount(&n) == cudaSuccess ? n : -1;
}

int spk_release_memory(void) {
    int dev = 0;
    SPK_CK(cudaGetDevice(&dev));
    int rc = spk_batch_release();  // cached batch graphs hold their workspaces
    if (rc) return rc;
    SPK_CK(cudaDeviceGraphMemTrim(dev));
    cudaMemPool_t pool;
    SPK_CK(cudaDeviceGetDefaultMemPool(&pool, dev));
    SPK_CK(cudaMemPoolTrimTo(pool, 0));
    return SPK_OK;
}

int spk_version(void) { return 100; }

// ---- quality metrics and the stability check (metrics.cu) ----
int spk_frame_metrics(const spk_geom* g, const void* d_frames, int frame_type, size_t pitch,
                      const void* d_ref, int ref_type, size_t ref_pitch, double* d_te,
                      double* d_mse, void* stream) {
    int rc = check_geom(g, false);
    if (rc) return rc;
    if (frame_type != SPK_OUT_U8 && frame_type != SPK_OUT_F32 && frame_type != SPK_OUT_F64)
        return fail(SPK_EINVAL, "spk_frame_metrics: bad frame_type");
    if (d_te && (g->width < 3 || g->height < 3))
        return fail(SPK_EINVAL, "two_dimensional_entropy: image must be at least 3x3");
    if (d_mse && !d_ref) return fail(SPK_EINVAL, "spk_frame_metrics: mse needs reference images");
    if (d_mse && ref_type != SPK_OUT_U8 && ref_type != SPK_OUT_F32 && ref_type != SPK_OUT_F64)
        return fail(SPK_EINVAL, "spk_frame_metrics: bad ref_type");
    const int64_t npix = npix_of(g);
    if (g->frames == 0 || (!d_te && !d_mse)) return SPK_OK;
    if (!d_frames) return fail(SPK_EINVAL, "spk: null device buffer");
    if (pitch < (size_t)npix || (d_mse && ref_pitch < (size_t)npix))
        return fail(SPK_EINVAL, "spk_frame_metrics: pitch must be >= W*H");
    cudaStream_t s = as_stream(stream);
    MetArgs a;
    a.frames = d_frames;
    a.pitch = (int64_t)pitch;
    a.ref = d_ref;
    a.ref_pitch = (int64_t)ref_pitch;
    a.ref_type = ref_type;
    a.width = g->width;
    a.height = g->height;
    a.te = d_te;
    a.mse = d_mse;
    const size_t smem = d_te ? (size_t)kMetHalf * sizeof(uint32_t) : 0;
    auto go = [&](auto kern) -> int {
        SPK_CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)((size_t)kMetHalf * sizeof(uint32_t))));
        kern<<<(unsigned)g->frames, kMetThreads, smem, s>>>(a);
        SPK_LAUNCHED("k_frame_metrics");
        return SPK_OK;
    };
    return frame_type == SPK_OUT_U8    ? go(k_frame_metrics<uint8_t>)
           : frame_type == SPK_OUT_F32 ? go(k_frame_metrics<float>)
                                       : go(k_frame_metrics<double>);
}

int spk_stability(const spk_geom* g, const void* d_planes, int max_depth, spk_stab* d_out,
                  void* stream) {
    int rc = check_geom(g, true);
    if (rc) return rc;
    if (max_depth < 1 || max_depth > kStabMaxDepth)
        return fail(SPK_EINVAL, "stability_order: max_depth must be in [1, 63]");
    if (!d_out || (g->frames > 0 && !d_planes)) return fail(SPK_EINVAL, "spk: null device buffer");
    const int64_t npix = npix_of(g);
    cudaStream_t s = as_stream(stream);
    int dev = 0;
    SPK_CK(cudaGetDevice(&dev));
    ensure_pool(dev);
    Scratch cnt(s);
    SPK_CK(cnt.alloc((size_t)npix * sizeof(uint32_t)));
    StabArgs a;
    a.planes = d_planes;
    a.pitch = g->plane_pitch;
    a.npix = npix;
    a.frames = g->frames;
    a.max_depth = max_depth;
    a.count = static_cast<uint32_t*>(cnt.p);
    a.out = d_out;
    k_stab_count<<<(unsigned)((npix + 255) / 256), 256, 0, s>>>(a);
    SPK_LAUNCHED("k_stab_count");
    std::vector<uint32_t> hc((size_t)npix);
    SPK_CK(cudaMemcpyAsync(hc.data(), cnt.p, (size_t)npix * sizeof(uint32_t),
                           cudaMemcpyDeviceToHost, s));
    SPK_CK(cudaStreamSynchronize(s));
    // per-pixel stack of bit-packed sequences: a child is at most its
    // parent's length and the deepest level is max_depth, so max_depth *
    // ceil(|S1| / 32) words suffice
    constexpr int64_t kBudget = (int64_t)1 << 30;  // scratch words per batch (4 GB)
    for (int64_t p0 = 0; p0 < npix;) {
        std::vector<int64_t> offs;
        int64_t tot = 0, p1 = p0;
        while (p1 < npix) {
            const int64_t len = hc[(size_t)p1] > 1 ? (int64_t)hc[(size_t)p1] - 1 : 0;
            const int64_t need = (int64_t)max_depth * ((len + 31) / 32) + 1;
            if (p1 > p0 && tot + need > kBudget) break;
            offs.push_back(tot);
            tot += need;
            ++p1;
        }
        Scratch doffs(s), scr(s);
        SPK_CK(doffs.alloc(offs.size() * sizeof(int64_t)));
        SPK_CK(scr.alloc((size_t)tot * sizeof(int32_t)));
        SPK_CK(cudaMemcpyAsync(doffs.p, offs.data(), offs.size() * sizeof(int64_t),
                               cudaMemcpyHostToDevice, s));
        a.pix0 = p0;
        a.nbatch = p1 - p0;
        a.offs = static_cast<const int64_t*>(doffs.p);
        a.scratch = static_cast<int32_t*>(scr.p);
        k_stab<<<(unsigned)((a.nbatch + 127) / 128), 128, 0, s>>>(a);
        SPK_LAUNCHED("k_stab");
        SPK_CK(cudaStreamSynchronize(s));  // `offs` is pageable host memory
        p0 = p1;
    }
    return SPK_OK;
}

int spk_frame_metrics_host(const spk_geom* g, const void* h_frames, int frame_type, size_t pitch,
                           const void* h_ref, int ref_type, size_t ref_pitch, double* h_te,
                           double* h_mse) {
    int rc = check_geom(g, false);
    if (rc) return rc;
    if (frame_type != SPK_OUT_U8 && frame_type != SPK_OUT_F32 && frame_type != SPK_OUT_F64)
        return fail(SPK_EINVAL, "spk_frame_metrics: bad frame_type");
    const size_t esz = frame_type == SPK_OUT_U8 ? 1 : frame_type == SPK_OUT_F32 ? 4 : 8;
    const size_t npix = (size_t)npix_of(g), t = (size_t)g->frames;
    if (h_te && (g->width < 3 || g->height < 3))
        return fail(SPK_EINVAL, "two_dimensional_entropy: image must be at least 3x3");
    if (h_mse && !h_ref) return fail(SPK_EINVAL, "spk_frame_metrics: mse needs reference images");
    if (h_mse && ref_type != SPK_OUT_U8 && ref_type != SPK_OUT_F32 && ref_type != SPK_OUT_F64)
        return fail(SPK_EINVAL, "spk_frame_metrics: bad ref_type");
    const size_t rsz = ref_type == SPK_OUT_U8 ? 1 : ref_type == SPK_OUT_F32 ? 4 : 8;
    if (t == 0 || (!h_te && !h_mse)) return SPK_OK;
    if (!h_frames) return fail(SPK_EINVAL, "spk: null host buffer");
    if (pitch < npix || (h_mse && ref_pitch < npix))
        return fail(SPK_EINVAL, "spk_frame_metrics: pitch must be >= W*H");
    int dev = 0;
    SPK_CK(cudaGetDevice(&dev));
    ensure_pool(dev);
    cudaStream_t s;
    SPK_CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    rc = [&]() -> int {
        Scratch fr(s), rf(s), te(s), ms(s);
        SPK_CK(fr.alloc(pitch * esz * t));
        SPK_CK(cudaMemcpyAsync(fr.p, h_frames, pitch * esz * t, cudaMemcpyHostToDevice, s));
        if (h_mse) {
            SPK_CK(rf.alloc(ref_pitch * rsz * t));
            SPK_CK(cudaMemcpyAsync(rf.p, h_ref, ref_pitch * rsz * t, cudaMemcpyHostToDevice, s));
            SPK_CK(ms.alloc(t * sizeof(double)));
        }
        if (h_te) SPK_CK(te.alloc(t * sizeof(double)));
        int r = spk_frame_metrics(g, fr.p, frame_type, pitch, rf.p, ref_type,
                                  ref_pitch, h_te ? static_cast<double*>(te.p) : nullptr,
                                  h_mse ? static_cast<double*>(ms.p) : nullptr, s);
        if (r) return r;
        if (h_te) SPK_CK(cudaMemcpyAsync(h_te, te.p, t * sizeof(double), cudaMemcpyDeviceToHost, s));
        if (h_mse)
            SPK_CK(cudaMemcpyAsync(h_mse, ms.p, t * sizeof(double), cudaMemcpyDeviceToHost, s));
        return SPK_OK;
    }();
    cudaError_t se = cudaStreamSynchronize(s);
    cudaStreamDestroy(s);
    if (rc) return rc;
    if (se != cudaSuccess) return cuda_fail(se, "cudaStreamSynchronize");
    return SPK_OK;
}

int spk_stability_host(const spk_geom* g, const void* h_payload, int max_depth, spk_stab* h_out) {
    spk_geom dg = *g;
    dg.plane_pitch = spk_plane_pitch(g->width, g->height);
    int rc = check_geom(&dg, true);
    if (rc) return rc;
    if (max_depth < 1 || max_depth > kStabMaxDepth)
        return fail(SPK_EINVAL, "stability_order: max_depth must be in [1, 63]");
    if (!h_out || (g->frames > 0 && !h_payload)) return fail(SPK_EINVAL, "spk: null host buffer");
    const size_t npix = (size_t)npix_of(g);
    int dev = 0;
    SPK_CK(cudaGetDevice(&dev));
    ensure_pool(dev);
    cudaStream_t s;
    SPK_CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    rc = [&]() -> int {
        Scratch planes(s), out(s);
        SPK_CK(planes.alloc(dg.plane_pitch * (size_t)std::max<int64_t>(g->frames, 1)));
        SPK_CK(out.alloc(npix * sizeof(spk_stab)));
        if (g->frames > 0) {
            const int r = spk_upload_planes(&dg, h_payload, plane_bytes(g), 0, planes.p, s);
            if (r) return r;
        }
        const int r = spk_stability(&dg, planes.p, max_depth, static_cast<spk_stab*>(out.p), s);
        if (r) return r;
        SPK_CK(cudaMemcpyAsync(h_out, out.p, npix * sizeof(spk_stab), cudaMemcpyDeviceToHost, s));
        return SPK_OK;
    }();
    cudaError_t se = cudaStreamSynchronize(s);
    cudaStreamDestroy(s);
    if (rc) return rc;
    if (se != cudaSuccess) return cuda_fail(se, "cudaStreamSynchronize");
    return SPK_OK;
}

int spk_synth(int scene, uint64_t seed, const spk_geom* g, int64_t frame0, double param,
              void* d_planes, void* stream) {
    int rc = check_geom(g, true);
    if (rc) return rc;
    if (scene < 0 || scene > 5 || scene == 4) return fail(SPK_EINVAL, "spk_synth: bad scene");
    if (frame0 < 0) return fail(SPK_EINVAL, "spk_synth: frame0 < 0");
    if (g->frames == 0) return SPK_OK;
    if (!d_planes) return fail(SPK_EINVAL, "spk: null device buffer");
    cudaStream_t s = as_stream(stream);
    SPK_CK(cudaMemsetAsync(d_planes, 0, g->plane_pitch * (size_t)g->frames, s));
    const int64_t threads = (npix_of(g) + 31) / 32 * 32;
    k_synth<<<(unsigned)((threads + 127) / 128), 128, 0, s>>>(
        scene, seed, g->width, g->height, g->frames, frame0, param,
        static_cast<uint8_t*>(d_planes), g->plane_pitch);
    SPK_LAUNCHED("k_synth");
    return SPK_OK;
}

}  // extern "C"
