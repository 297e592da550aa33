// expand.cu -- K2b (run values + run table) and K3 (runs -> frame planes).
//
// Replaces the run fill loops of reconstruct_row (proj/src/reconstruct.cpp:
// 355-393), the row->column transpose of reconstruct_into (424-427) and, for
// uint8 output, quantize (proj/src/io.cpp:78-81).
//
// K2b k_finalize: one thread per pixel walks its run list once: the run value
// 255*N/span (reconstruct.cpp:124; f64 bit-exact, u8 via the exact
// round-half-away integer form) replaces the interval count in place (f64
// values go to a side array), and the run table tbl[c][p] = run covering
// frame c*kChunk (-1 = lead before the first run; the last run also covers
// the tail [last spike, T), reconstruct.cpp:391-393).
//
// K3 k_expand: every output value is piecewise constant in time per pixel.
// A lane owns P consecutive pixels of one kChunk-frame chunk and keeps their
// current values packed in registers: the steady state is one vector store
// per frame (16 B for u8: a warp writes 512 contiguous bytes of a frame row
// per instruction) and a pointer bump, with all lanes of a warp on the same
// frame so every store covers whole 128-B lines.  Value changes are not
// handled in the frame loop (a data-dependent branch there would serialise
// the warp at almost every frame of a moving scene).  Instead, per sub-tile
// of F frames, each lane first buckets its pixels' changes by frame into
// lane-private shared memory (phase A: per-pixel loops over the run lists,
// with the record loads prefetched two runs ahead), then walks the F frames
// and merges a frame's pending changes with one masked select (phase B).
#include <climits>
#include <type_traits>

#include "spk_common.cuh"
#include "spk_kernels.cuh"

namespace spk {

namespace {

template <typename OUT>
struct RunVal;  // value of run r of one pixel, as stored by k_finalize
template <>
struct RunVal<uint8_t> {
    using T = uint32_t;
    __device__ static T load(const spk_run_t* rp, const double*, int r) { return rp[r].intervals; }
    __device__ static uint32_t put(uint8_t v) { return v; }
};
template <>
struct RunVal<float> {
    using T = uint32_t;
    __device__ static T load(const spk_run_t* rp, const double*, int r) { return rp[r].intervals; }
    __device__ static uint32_t put(float v) { return __float_as_uint(v); }
};
template <>
struct RunVal<double> {
    using T = double;
    __device__ static T load(const spk_run_t*, const double* vp, int r) { return vp[r]; }
};

template <int N>
__device__ __forceinline__ void st_words(char* p, const uint32_t (&o)[N]) {
    if constexpr (N == 2) {
        asm volatile("st.global.v2.b32 [%0], {%1, %2};" ::"l"(p), "r"(o[0]), "r"(o[1]) : "memory");
    } else {
#pragma unroll
        for (int k = 0; k < N / 4; ++k)
            asm volatile("st.global.v4.b32 [%0], {%1, %2, %3, %4};" ::"l"(p + 16 * k),
                         "r"(o[4 * k]), "r"(o[4 * k + 1]), "r"(o[4 * k + 2]), "r"(o[4 * k + 3])
                         : "memory");
    }
}

}  // namespace

// ------------------------------------------------------------ K2b finalize --
template <typename OUT>
__global__ void __launch_bounds__(kFinThreads) k_finalize(FinArgs a) {
    const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= a.npix) return;
    const uint32_t n = a.counts[p];
    if (n > (uint32_t)a.cap) return;  // overflowed: k_fixup writes this pixel
    int32_t* tb = a.tbl + p;
    auto table = [&](int c0, int c1, int v) {
        for (int c = c0; c <= c1; ++c) tb[(int64_t)c * a.npix] = v;
    };
    if (n == 0) {
        table(0, a.nchunks - 1, -1);
        return;
    }
    spk_run_t* rp = a.runs + p * a.cap;
    double* vp = a.vals ? a.vals + p * a.cap : nullptr;
    const int lastp = a.last[p];
    spk_run_t cur = rp[0];
    table(0, (int)((cur.start + kChunk - 1) >> kChunkLog2) - 1, -1);  // lead
    for (int k = 0; k < (int)n; ++k) {
        const bool more = k + 1 < (int)n;
        const spk_run_t nx = more ? rp[k + 1] : spk_run_t{(uint32_t)lastp, 0u};
        const uint32_t span = nx.start - cur.start;
        const OUT v = OutVal<OUT>::run(cur.intervals, span);
        if constexpr (sizeof(OUT) == 8)
            vp[k] = v;
        else
            rp[k].intervals = RunVal<OUT>::put(v);
        const int c0 = (int)((cur.start + kChunk - 1) >> kChunkLog2);
        const int c1 = more ? (int)((nx.start - 1) >> kChunkLog2) : a.nchunks - 1;
        table(c0, c1, k);
        cur = nx;
    }
}

template __global__ void k_finalize<uint8_t>(FinArgs);
template __global__ void k_finalize<float>(FinArgs);
template __global__ void k_finalize<double>(FinArgs);

// -------------------------------------------------------------- K3 expand --
// Per output type: P pixels per lane, F frames per sub-tile, K-deep record
// ring per pixel.
template <typename OUT>
struct ExpGeo;
template <>
struct ExpGeo<uint8_t> {
    static constexpr int P = 8, F = 16, K = 4;
};
template <>
struct ExpGeo<float> {
    static constexpr int P = 8, F = 8, K = 4;
};
template <>
struct ExpGeo<double> {
    static constexpr int P = 8, F = 8, K = 4;
};

// Lane-private shared memory, interleaved by lane (element e of lane j is at
// slot e*32 + j) so that lanes touching the same element never share a bank.
//   ring[P][K]  upcoming runs of each pixel: {start, value} (u8/f32: 8 B,
//               f64: 16 B), refilled with cp.async as runs are consumed
//   cur[P]      index of the run each pixel is in (int), cnt[P] its run count
//   D[F][P]     values of pending changes, M[F] pixel mask per frame
template <typename OUT>
struct ExpSmem {
    static constexpr int P = ExpGeo<OUT>::P, F = ExpGeo<OUT>::F, K = ExpGeo<OUT>::K;
    static constexpr int RE = sizeof(OUT) == 8 ? 16 : 8;  // ring entry bytes
    static constexpr int ring = P * K * RE;
    static constexpr int cur = P * 4, cnt = P * 4;
    static constexpr int d = F * P * (int)sizeof(OUT);
    static constexpr int m = F * 4;
    static constexpr int per_lane = ring + cur + cnt + d + m;
    static constexpr int per_warp = 32 * per_lane;
};

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"((uint32_t)__cvta_generic_to_shared(smem)),
                 "l"(gmem)
                 : "memory");
}
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"((uint32_t)__cvta_generic_to_shared(smem)),
                 "l"(gmem)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

template <typename OUT>
__global__ void __launch_bounds__(kExpThreads) k_expand(ExpArgs a) {
    using G = ExpSmem<OUT>;
    constexpr int P = G::P, F = G::F, K = G::K;
    constexpr int NW = P * (int)sizeof(OUT) / 4;  // 32-bit words per lane-frame
    extern __shared__ __align__(16) unsigned char sm[];
    const int lane = threadIdx.x & 31;
    unsigned char* wbase = sm + (size_t)(threadIdx.x >> 5) * G::per_warp;
    // element accessors (interleaved by lane)
    unsigned char* ring_b = wbase;
    int* cur_b = reinterpret_cast<int*>(wbase + 32 * G::ring);
    int* cnt_b = reinterpret_cast<int*>(wbase + 32 * (G::ring + G::cur));
    unsigned char* d_b = wbase + 32 * (G::ring + G::cur + G::cnt);
    uint32_t* m_b = reinterpret_cast<uint32_t*>(wbase + 32 * (G::ring + G::cur + G::cnt + G::d));
    auto ring_at = [&](int i, int q) -> unsigned char* {  // entry for run q of pixel i
        return ring_b + ((size_t)((i * K + (q & (K - 1))) * 32 + lane)) * G::RE;
    };
    auto ring_start = [&](int i, int q) -> int { return *reinterpret_cast<const int*>(ring_at(i, q)); };
    auto CUR = [&](int i) -> int& { return cur_b[i * 32 + lane]; };
    auto CNT = [&](int i) -> int& { return cnt_b[i * 32 + lane]; };
    auto M = [&](int f) -> uint32_t& { return m_b[f * 32 + lane]; };

    const int64_t p0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * P;
    const int c = a.chunk0 + (int)blockIdx.y;
    const int f0 = c << kChunkLog2;
    if (p0 >= a.npix || f0 >= a.frames) return;  // lanes never exchange data
    const int f1 = min(a.frames, f0 + kChunk);
    const int np = (int)min((int64_t)P, a.npix - p0);

    // issue the copy of run q of pixel i into its ring slot
    auto fetch = [&](int i, int q) {
        const int64_t p = p0 + i;
        unsigned char* dst = ring_at(i, q);
        const spk_run_t* rp = a.runs + p * a.cap + q;
        if constexpr (sizeof(OUT) == 8) {
            cp_async4(dst, &rp->start);
            cp_async8(dst + 8, a.vals + p * a.cap + q);
        } else {
            cp_async8(dst, rp);
        }
    };

    uint32_t words[NW];
#pragma unroll
    for (int k = 0; k < NW; ++k) words[k] = 0u;
#pragma unroll
    for (int i = 0; i < P; ++i) {
        int r = -1, cnt = 0;
        if (i < np) {
            const int64_t p = p0 + i;
            const uint32_t n = a.counts[p];
            if (n > 0 && n <= (uint32_t)a.cap) {  // overflowed pixels: k_fixup
                cnt = (int)n;
                r = a.tbl[(int64_t)c * a.npix + p];
                if (r >= 0) {  // value at the chunk start
                    if constexpr (sizeof(OUT) == 1)
                        words[i >> 2] |= (a.runs[p * a.cap + r].intervals & 0xffu) << ((i & 3) * 8);
                    else if constexpr (sizeof(OUT) == 4)
                        words[i] = a.runs[p * a.cap + r].intervals;
                    else {
                        const unsigned long long b = __double_as_longlong(a.vals[p * a.cap + r]);
                        words[2 * i] = (uint32_t)b;
                        words[2 * i + 1] = (uint32_t)(b >> 32);
                    }
                }
                for (int q = r + 1; q < min(cnt, r + 1 + K); ++q) fetch(i, q);
            }
        }
        CUR(i) = r;
        CNT(i) = cnt;
    }
    cp_async_commit();
#pragma unroll
    for (int f = 0; f < F; ++f) M(f) = 0u;

    const size_t step = a.pitch * sizeof(OUT);
    char* ptr = reinterpret_cast<char*>(a.out) + ((size_t)f0 * a.pitch + (size_t)p0) * sizeof(OUT);
    const bool vec_ok = a.vec_ok && np == P;

    cp_async_wait<0>();
    // Ring safety: run q of a pixel is requested when run q-K is consumed.
    // After wait_group 1 at a phase-A start, every request older than the
    // previous phase A has landed, so consuming q is safe unless the pixel
    // consumed >= K runs over this and the previous phase A; then wait for
    // all requests.  Per-pixel 4-bit counters of consumed runs: nprev, ncur.
    uint32_t ncur = 0;
    for (int t0 = f0; t0 < f1; t0 += F) {
        const int t1 = min(f1, t0 + F);
        // phase A: bucket this sub-tile's changes by frame
        cp_async_wait<1>();
        uint32_t nprev = ncur;
        ncur = 0;
        // before reading a ring entry of pixel i: wait if it may still be in flight
        auto ensure = [&](int i) {
            if (((nprev >> (4 * i)) & 15u) + ((ncur >> (4 * i)) & 15u) >= (uint32_t)K) {
                asm volatile("cp.async.wait_all;" ::: "memory");
                nprev = ncur = 0;
            }
        };
        uint32_t todo = 0;
#pragma unroll
        for (int i = 0; i < P; ++i) {
            const int q = CUR(i) + 1;
            if (q < CNT(i)) {
                ensure(i);
                if (ring_start(i, q) < t1) todo |= 1u << i;
            }
        }
        while (todo) {
            const int i = __ffs(todo) - 1;
            const int q = CUR(i) + 1;  // run starting inside this sub-tile (entry ensured)
            const unsigned char* e = ring_at(i, q);
            const int fo = *reinterpret_cast<const int*>(e) - t0;
            if constexpr (sizeof(OUT) == 1)
                d_b[((fo * P + i) >> 2) * 128 + lane * 4 + (i & 3)] = (uint8_t)reinterpret_cast<const uint32_t*>(e)[1];
            else if constexpr (sizeof(OUT) == 4)
                reinterpret_cast<uint32_t*>(d_b)[(fo * P + i) * 32 + lane] = reinterpret_cast<const uint32_t*>(e)[1];
            else
                reinterpret_cast<double*>(d_b)[(fo * P + i) * 32 + lane] = *reinterpret_cast<const double*>(e + 8);
            M(fo) |= 1u << i;
            CUR(i) = q;
            ncur += 1u << (4 * i);
            const int cnt = CNT(i);
            if (q + K < cnt) fetch(i, q + K);  // refill the slot just consumed
            bool again = false;
            if (q + 1 < cnt) {
                ensure(i);
                again = ring_start(i, q + 1) < t1;
            }
            if (!again) todo &= todo - 1;
        }
        cp_async_commit();
        // phase B: frames in order, one store per frame, pending changes merged
        const int nf = t1 - t0;
#pragma unroll 4
        for (int fo = 0; fo < nf; ++fo) {
            const uint32_t m = M(fo);
            if (m) {
                M(fo) = 0u;
                if constexpr (sizeof(OUT) == 1) {
#pragma unroll
                    for (int k = 0; k < NW; ++k) {
                        const uint32_t dw = reinterpret_cast<const uint32_t*>(d_b)[(fo * NW + k) * 32 + lane];
                        const uint32_t nib = (m >> (4 * k)) & 0xfu;
                        const uint32_t bm = ((nib * 0x00204081u) & 0x01010101u) * 0xffu;
                        words[k] = (words[k] & ~bm) | (dw & bm);
                    }
                } else if constexpr (sizeof(OUT) == 4) {
#pragma unroll
                    for (int i = 0; i < P; ++i)
                        if (m & (1u << i)) words[i] = reinterpret_cast<const uint32_t*>(d_b)[(fo * P + i) * 32 + lane];
                } else {
#pragma unroll
                    for (int i = 0; i < P; ++i)
                        if (m & (1u << i)) {
                            const unsigned long long b = __double_as_longlong(
                                reinterpret_cast<const double*>(d_b)[(fo * P + i) * 32 + lane]);
                            words[2 * i] = (uint32_t)b;
                            words[2 * i + 1] = (uint32_t)(b >> 32);
                        }
                }
            }
            if (vec_ok) {
                st_words(ptr, words);
            } else {
                OUT* o = reinterpret_cast<OUT*>(ptr);
#pragma unroll
                for (int i = 0; i < P; ++i)
                    if (i < np) {
                        if constexpr (sizeof(OUT) == 1)
                            o[i] = (OUT)((words[i >> 2] >> ((i & 3) * 8)) & 0xffu);
                        else if constexpr (sizeof(OUT) == 4)
                            o[i] = __uint_as_float(words[i]);
                        else
                            o[i] = __longlong_as_double((long long)((unsigned long long)words[2 * i] |
                                                                    (unsigned long long)words[2 * i + 1] << 32));
                    }
            }
            ptr += step;
        }
    }
}

size_t expand_smem_bytes(int out_size) {
    const int per = out_size == 1 ? ExpSmem<uint8_t>::per_warp
                  : out_size == 4 ? ExpSmem<float>::per_warp
                                  : ExpSmem<double>::per_warp;
    return (size_t)per * (kExpThreads / 32);
}

int expand_pixels_per_lane(int out_size) {
    return out_size == 1 ? ExpGeo<uint8_t>::P : out_size == 4 ? ExpGeo<float>::P : ExpGeo<double>::P;
}

template __global__ void k_expand<uint8_t>(ExpArgs);
template __global__ void k_expand<float>(ExpArgs);
template __global__ void k_expand<double>(ExpArgs);

}  // namespace spk
