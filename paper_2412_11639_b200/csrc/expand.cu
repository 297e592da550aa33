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

// Lane-private shared memory, interleaved by lane so that lanes touching the
// same element never share a bank (element e of lane j at slot e*32 + j):
//   ring[P][K]  upcoming runs of each pixel, {start, value} (u8/f32: 8 B,
//               f64: 16 B), refilled with cp.async as runs are consumed
//   D[F]        per frame of the sub-tile: the lane's pending values (P * OUT)
//   B[F]        per frame: u8 -> byte mask of the pending pixels (8 B),
//               f32/f64 -> pixel bit mask (4 B)
template <typename OUT>
struct ExpSmem {
    static constexpr int P = ExpGeo<OUT>::P, F = ExpGeo<OUT>::F, K = ExpGeo<OUT>::K;
    static constexpr int RE = sizeof(OUT) == 8 ? 16 : 8;  // ring entry bytes
    static constexpr int DE = P * (int)sizeof(OUT);       // D element bytes
    static constexpr int BE = sizeof(OUT) == 1 ? 8 : 4;   // B element bytes
    static constexpr int ring = P * K * RE * 32;
    static constexpr int d = F * DE * 32;
    static constexpr int b = F * BE * 32;
    static constexpr int per_warp = ring + d + b;
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
    unsigned char* ring_b = wbase;
    unsigned char* d_b = wbase + G::ring;
    unsigned char* b_b = wbase + G::ring + G::d;
    auto ring_at = [&](int i, int q) -> unsigned char* {  // entry of run q of pixel i
        return ring_b + ((i * K + (q & (K - 1))) * 32 + lane) * G::RE;
    };
    auto d_at = [&](int fo) -> unsigned char* { return d_b + (fo * 32 + lane) * G::DE; };
    auto b_at = [&](int fo) -> unsigned char* { return b_b + (fo * 32 + lane) * G::BE; };

    const int64_t p0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * P;
    const int c = a.chunk0 + (int)blockIdx.y;
    const int f0 = c << kChunkLog2;
    if (p0 >= a.npix || f0 >= a.frames) return;  // lanes never exchange data
    const int f1 = min(a.frames, f0 + kChunk);
    const int np = (int)min((int64_t)P, a.npix - p0);

    const spk_run_t* runs0 = a.runs + p0 * a.cap;
    const double* vals0 = a.vals ? a.vals + p0 * a.cap : nullptr;
    auto fetch = [&](int i, int q) {  // request run q of pixel i into its ring slot
        unsigned char* dst = ring_at(i, q);
        const size_t off = (size_t)i * a.cap + q;
        if constexpr (sizeof(OUT) == 8) {
            cp_async4(dst, &runs0[off].start);
            cp_async8(dst + 8, vals0 + off);
        } else {
            cp_async8(dst, runs0 + off);
        }
    };

    int rr[P], cn[P], ns[P];  // current run, run count, start of the next run
    uint32_t words[NW];
#pragma unroll
    for (int k = 0; k < NW; ++k) words[k] = 0u;
#pragma unroll
    for (int i = 0; i < P; ++i) {
        rr[i] = -1;
        cn[i] = 0;
        ns[i] = INT_MAX;
        if (i < np) {
            const int64_t p = p0 + i;
            const uint32_t n = a.counts[p];
            if (n > 0 && n <= (uint32_t)a.cap) {  // overflowed pixels: k_fixup
                cn[i] = (int)n;
                const int r = a.tbl[(int64_t)c * a.npix + p];
                rr[i] = r;
                if (r >= 0) {  // value at the chunk start
                    const size_t off = (size_t)i * a.cap + r;
                    if constexpr (sizeof(OUT) == 1)
                        words[i >> 2] |= (runs0[off].intervals & 0xffu) << ((i & 3) * 8);
                    else if constexpr (sizeof(OUT) == 4)
                        words[i] = runs0[off].intervals;
                    else {
                        const unsigned long long b = __double_as_longlong(vals0[off]);
                        words[2 * i] = (uint32_t)b;
                        words[2 * i + 1] = (uint32_t)(b >> 32);
                    }
                }
                for (int q = r + 1; q < min((int)n, r + 1 + K); ++q) fetch(i, q);
            }
        }
    }
    cp_async_commit();
#pragma unroll
    for (int f = 0; f < F; ++f) {
        if constexpr (sizeof(OUT) == 1)
            *reinterpret_cast<uint2*>(b_at(f)) = make_uint2(0u, 0u);
        else
            *reinterpret_cast<uint32_t*>(b_at(f)) = 0u;
    }
    cp_async_wait<0>();
#pragma unroll
    for (int i = 0; i < P; ++i)
        if (rr[i] + 1 < cn[i]) ns[i] = *reinterpret_cast<const int*>(ring_at(i, rr[i] + 1));

    const size_t step = a.pitch * sizeof(OUT);
    char* ptr = reinterpret_cast<char*>(a.out) + ((size_t)f0 * a.pitch + (size_t)p0) * sizeof(OUT);
    const bool vec_ok = a.vec_ok && np == P;

    // Ring safety: run q of a pixel is requested when run q-K is consumed.
    // After wait_group 1 at a phase-A start, every request older than the
    // previous phase A has landed, so reading run q is safe unless the pixel
    // consumed >= K runs over this and the previous phase A (then wait for
    // all).  Per-pixel 4-bit counters of consumed runs: nprev, ncur.
    uint32_t ncur = 0;
    for (int t0 = f0; t0 < f1; t0 += F) {
        const int t1 = min(f1, t0 + F);
        // phase A: bucket this sub-tile's value changes by frame
        cp_async_wait<1>();
        uint32_t nprev = ncur;
        ncur = 0;
#pragma unroll
        for (int i = 0; i < P; ++i) {
            while (ns[i] < t1) {  // run q starts inside this sub-tile
                const int q = rr[i] + 1;
                const unsigned char* e = ring_at(i, q);
                const int fo = ns[i] - t0;
                if constexpr (sizeof(OUT) == 1) {
                    d_at(fo)[i] = (uint8_t)reinterpret_cast<const uint32_t*>(e)[1];
                    b_at(fo)[i] = 0xffu;
                } else if constexpr (sizeof(OUT) == 4) {
                    reinterpret_cast<uint32_t*>(d_at(fo))[i] = reinterpret_cast<const uint32_t*>(e)[1];
                    *reinterpret_cast<uint32_t*>(b_at(fo)) |= 1u << i;
                } else {
                    reinterpret_cast<double*>(d_at(fo))[i] = *reinterpret_cast<const double*>(e + 8);
                    *reinterpret_cast<uint32_t*>(b_at(fo)) |= 1u << i;
                }
                rr[i] = q;
                ncur += 1u << (4 * i);
                if (q + K < cn[i]) fetch(i, q + K);  // refill the slot just consumed
                if (q + 1 < cn[i]) {
                    if (((nprev >> (4 * i)) & 15u) + ((ncur >> (4 * i)) & 15u) >= (uint32_t)K) {
                        asm volatile("cp.async.wait_all;" ::: "memory");
                        nprev = ncur = 0;
                    }
                    ns[i] = *reinterpret_cast<const int*>(ring_at(i, q + 1));
                } else {
                    ns[i] = INT_MAX;
                }
            }
        }
        cp_async_commit();
        // phase B: frames in order, one store per frame, pending values merged
        const int nf = t1 - t0;
#pragma unroll 4
        for (int fo = 0; fo < nf; ++fo) {
            if constexpr (sizeof(OUT) == 1) {
                const uint2 dv = *reinterpret_cast<const uint2*>(d_at(fo));
                const uint2 bm = *reinterpret_cast<const uint2*>(b_at(fo));
                *reinterpret_cast<uint2*>(b_at(fo)) = make_uint2(0u, 0u);
                words[0] = (words[0] & ~bm.x) | (dv.x & bm.x);
                words[1] = (words[1] & ~bm.y) | (dv.y & bm.y);
            } else {
                const uint32_t m = *reinterpret_cast<const uint32_t*>(b_at(fo));
                if (m) {
                    *reinterpret_cast<uint32_t*>(b_at(fo)) = 0u;
                    const uint32_t* dw = reinterpret_cast<const uint32_t*>(d_at(fo));
#pragma unroll
                    for (int i = 0; i < P; ++i) {
                        const bool take = (m >> i) & 1u;
                        if constexpr (sizeof(OUT) == 4) {
                            words[i] = take ? dw[i] : words[i];
                        } else {
                            words[2 * i] = take ? dw[2 * i] : words[2 * i];
                            words[2 * i + 1] = take ? dw[2 * i + 1] : words[2 * i + 1];
                        }
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
