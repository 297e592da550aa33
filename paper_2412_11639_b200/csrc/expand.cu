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
// A thread owns kExpPix consecutive pixels of one kChunk-frame chunk and keeps
// their current values packed in registers, so the steady state is one
// vector store per frame (8 B for u8) and a pointer bump.  The warp walks the
// frames in lockstep -- the next stop is the warp-wide minimum of the lanes'
// next change frames (REDUX) -- so every store instruction writes whole
// 128-B lines of one frame row (no partial-sector read-modify-write in L2).
// At a change a lane takes the value it preloaded for its pixel's next run
// and issues the load of the run after that, two runs ahead of use.
#include <climits>

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

template <typename OUT, int P>
struct Pack;  // P values -> the thread's per-frame store
template <>
struct Pack<uint8_t, 8> {
    static constexpr int N = 2;  // 32-bit words
    __device__ static void pack(const uint32_t (&v)[8], uint32_t (&o)[N]) {
        o[0] = v[0] | v[1] << 8 | v[2] << 16 | v[3] << 24;
        o[1] = v[4] | v[5] << 8 | v[6] << 16 | v[7] << 24;
    }
};
template <>
struct Pack<float, 8> {
    static constexpr int N = 8;
    __device__ static void pack(const uint32_t (&v)[8], uint32_t (&o)[N]) {
#pragma unroll
        for (int i = 0; i < 8; ++i) o[i] = v[i];
    }
};
template <>
struct Pack<double, 8> {
    static constexpr int N = 16;
    __device__ static void pack(const double (&v)[8], uint32_t (&o)[N]) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const unsigned long long b = __double_as_longlong(v[i]);
            o[2 * i] = (uint32_t)b;
            o[2 * i + 1] = (uint32_t)(b >> 32);
        }
    }
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
template <typename OUT>
__global__ void __launch_bounds__(kExpThreads) k_expand(ExpArgs a) {
    constexpr int P = kExpPix;
    using V = typename RunVal<OUT>::T;
    using PK = Pack<OUT, P>;
    const int64_t p0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * P;
    // whole warps out of range leave; partial warps keep every lane in the
    // lockstep loop (inactive lanes never change and never store)
    if (((int64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31)) * P >= a.npix) return;
    const int c = a.chunk0 + (int)blockIdx.y;
    const int f0 = c << kChunkLog2;
    if (f0 >= a.frames) return;  // uniform across the block
    const int f1 = min(a.frames, f0 + kChunk);
    const int np = (int)max((int64_t)0, min((int64_t)P, a.npix - p0));

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
    int nc = INT_MAX;
#pragma unroll
    for (int i = 0; i < P; ++i) nc = min(nc, nst[i]);

    uint32_t words[PK::N];
    PK::pack(val, words);
    const size_t step = a.pitch * sizeof(OUT);
    char* ptr = reinterpret_cast<char*>(a.out) + ((size_t)f0 * a.pitch + (size_t)p0) * sizeof(OUT);
    const bool vec_ok = a.vec_ok && np == P;
    int f = f0;
    for (;;) {
        const int stop = (int)__reduce_min_sync(kFull, (unsigned)min(nc, f1));
        if (vec_ok) {
#pragma unroll 4
            for (; f < stop; ++f, ptr += step) st_words(ptr, words);
        } else {
            for (; f < stop; ++f, ptr += step) {
                OUT* o = reinterpret_cast<OUT*>(ptr);
#pragma unroll
                for (int i = 0; i < P; ++i)
                    if (i < np) {
                        if constexpr (sizeof(OUT) == 8)
                            o[i] = val[i];
                        else if constexpr (sizeof(OUT) == 4)
                            o[i] = __uint_as_float(val[i]);
                        else
                            o[i] = (OUT)val[i];
                    }
            }
        }
        if (f >= f1) break;
        if (nc == f) {  // this lane has pixels whose next run starts at f
            nc = INT_MAX;
#pragma unroll
            for (int i = 0; i < P; ++i) {
                if (nst[i] == f) {
                    const int64_t p = p0 + i;
                    const int r = ++ridx[i];
                    val[i] = nval[i];
                    nst[i] = nnst[i];
                    nval[i] = nnval[i];
                    nnst[i] = INT_MAX;
                    if (r + 2 < rcnt[i]) {  // prefetch two runs ahead
                        const spk_run_t* rp = a.runs + p * a.cap;
                        nnst[i] = (int)rp[r + 2].start;
                        nnval[i] = RunVal<OUT>::load(rp, a.vals ? a.vals + p * a.cap : nullptr, r + 2);
                    }
                }
                nc = min(nc, nst[i]);
            }
            PK::pack(val, words);
        }
    }
}

template __global__ void k_expand<uint8_t>(ExpArgs);
template __global__ void k_expand<float>(ExpArgs);
template __global__ void k_expand<double>(ExpArgs);

}  // namespace spk
