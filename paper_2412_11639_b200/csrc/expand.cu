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
// Geometry per output type: P pixels per lane (one 16-B store per frame for
// u8, 32/64 B for f32/f64) and F frames per sub-tile.
template <typename OUT>
struct ExpGeo;
template <>
struct ExpGeo<uint8_t> {
    static constexpr int P = 16, F = 32;
};
template <>
struct ExpGeo<float> {
    static constexpr int P = 8, F = 16;
};
template <>
struct ExpGeo<double> {
    static constexpr int P = 8, F = 8;
};

template <typename OUT>
__host__ __device__ constexpr int exp_smem_per_lane() {
    return ExpGeo<OUT>::F * (ExpGeo<OUT>::P * (int)sizeof(OUT) + 4);
}

template <typename OUT>
__global__ void __launch_bounds__(kExpThreads) k_expand(ExpArgs a) {
    constexpr int P = ExpGeo<OUT>::P;
    constexpr int F = ExpGeo<OUT>::F;
    constexpr int NW = P * (int)sizeof(OUT) / 4;  // 32-bit words per lane-frame
    using V = typename RunVal<OUT>::T;            // u8/f32: 32-bit word, f64: double
    using S = typename std::conditional<sizeof(OUT) == 1, uint8_t, V>::type;  // D element
    extern __shared__ __align__(16) unsigned char sm[];
    // lane-private scratch: D[F][P] pending values, M[F] pending-pixel masks
    unsigned char* mine = sm + (size_t)threadIdx.x * exp_smem_per_lane<OUT>();
    S* D = reinterpret_cast<S*>(mine);
    uint32_t* Mk = reinterpret_cast<uint32_t*>(mine + F * P * sizeof(OUT));

    const int64_t p0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * P;
    const int c = a.chunk0 + (int)blockIdx.y;
    const int f0 = c << kChunkLog2;
    if (p0 >= a.npix || f0 >= a.frames) return;  // no cross-lane traffic: lanes may leave
    const int f1 = min(a.frames, f0 + kChunk);
    const int np = (int)min((int64_t)P, a.npix - p0);

    int ridx[P], nst[P], nnst[P], rcnt[P];
    V val[P], nval[P], nnval[P];
#pragma unroll
    for (int i = 0; i < P; ++i) {
        val[i] = nval[i] = nnval[i] = V(0);
        nst[i] = nnst[i] = INT_MAX;
        ridx[i] = -1;
        rcnt[i] = 0;
        if (i < np) {
            const int64_t p = p0 + i;
            const uint32_t cnt = a.counts[p];
            if (cnt > 0 && cnt <= (uint32_t)a.cap) {  // overflowed pixels: k_fixup
                const spk_run_t* rp = a.runs + p * a.cap;
                const double* vp = a.vals ? a.vals + p * a.cap : nullptr;
                const int r = a.tbl[(int64_t)c * a.npix + p];
                rcnt[i] = (int)cnt;
                ridx[i] = r;
                if (r >= 0) val[i] = RunVal<OUT>::load(rp, vp, r);
                if (r + 1 < (int)cnt) {
                    nst[i] = (int)rp[r + 1].start;
                    nval[i] = RunVal<OUT>::load(rp, vp, r + 1);
                }
                if (r + 2 < (int)cnt) {
                    nnst[i] = (int)rp[r + 2].start;
                    nnval[i] = RunVal<OUT>::load(rp, vp, r + 2);
                }
            }
        }
    }
    // current values, packed as the lane's per-frame store
    uint32_t words[NW];
    if constexpr (sizeof(OUT) == 1) {
#pragma unroll
        for (int k = 0; k < NW; ++k)
            words[k] = (val[4 * k] & 0xffu) | (val[4 * k + 1] & 0xffu) << 8 |
                       (val[4 * k + 2] & 0xffu) << 16 | (val[4 * k + 3] & 0xffu) << 24;
    } else if constexpr (sizeof(OUT) == 4) {
#pragma unroll
        for (int k = 0; k < NW; ++k) words[k] = (uint32_t)val[k];
    } else {
#pragma unroll
        for (int k = 0; k < P; ++k) {
            const unsigned long long b = __double_as_longlong((double)val[k]);
            words[2 * k] = (uint32_t)b;
            words[2 * k + 1] = (uint32_t)(b >> 32);
        }
    }
#pragma unroll
    for (int f = 0; f < F; ++f) Mk[f] = 0u;

    const size_t step = a.pitch * sizeof(OUT);
    char* ptr = reinterpret_cast<char*>(a.out) + ((size_t)f0 * a.pitch + (size_t)p0) * sizeof(OUT);
    const bool vec_ok = a.vec_ok && np == P;

    for (int t0 = f0; t0 < f1; t0 += F) {
        const int t1 = min(f1, t0 + F);
        // phase A: bucket this sub-tile's value changes by frame
        bool more = true;
        while (more) {
            more = false;
#pragma unroll
            for (int i = 0; i < P; ++i) {
                if (nst[i] < t1) {
                    const int fo = nst[i] - t0;
                    D[fo * P + i] = (S)nval[i];
                    Mk[fo] |= 1u << i;
                    const int r = ++ridx[i];
                    nst[i] = nnst[i];
                    nval[i] = nnval[i];
                    nnst[i] = INT_MAX;
                    if (r + 2 < rcnt[i]) {  // prefetch two runs ahead
                        const int64_t p = p0 + i;
                        const spk_run_t* rp = a.runs + p * a.cap;
                        nnst[i] = (int)rp[r + 2].start;
                        nnval[i] =
                            RunVal<OUT>::load(rp, a.vals ? a.vals + p * a.cap : nullptr, r + 2);
                    }
                    more |= nst[i] < t1;
                }
            }
        }
        // phase B: frames in order, one store per frame, pending changes merged
        const int nf = t1 - t0;
#pragma unroll 4
        for (int fo = 0; fo < nf; ++fo) {
            const uint32_t m = Mk[fo];
            if (m) {
                Mk[fo] = 0u;
                if constexpr (sizeof(OUT) == 1) {
                    const uint4 d = *reinterpret_cast<const uint4*>(D + fo * P);
                    const uint32_t dw[4] = {d.x, d.y, d.z, d.w};
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        const uint32_t nib = (m >> (4 * k)) & 0xfu;
                        const uint32_t bm = ((nib * 0x00204081u) & 0x01010101u) * 0xffu;
                        words[k] = (words[k] & ~bm) | (dw[k] & bm);
                    }
                } else if constexpr (sizeof(OUT) == 4) {
#pragma unroll
                    for (int i = 0; i < P; ++i)
                        if (m & (1u << i)) words[i] = D[fo * P + i];
                } else {
#pragma unroll
                    for (int i = 0; i < P; ++i)
                        if (m & (1u << i)) {
                            const unsigned long long b = __double_as_longlong(D[fo * P + i]);
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
    const int per = out_size == 1 ? exp_smem_per_lane<uint8_t>()
                  : out_size == 4 ? exp_smem_per_lane<float>()
                                  : exp_smem_per_lane<double>();
    return (size_t)per * kExpThreads;
}

int expand_pixels_per_lane(int out_size) {
    return out_size == 1 ? ExpGeo<uint8_t>::P : out_size == 4 ? ExpGeo<float>::P : ExpGeo<double>::P;
}

template __global__ void k_expand<uint8_t>(ExpArgs);
template __global__ void k_expand<float>(ExpArgs);
template __global__ void k_expand<double>(ExpArgs);

}  // namespace spk
