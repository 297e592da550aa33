// expand.cu -- K3: stable runs -> frame planes (sm_100a).
//
// Replaces the run fill loops of reconstruct_row (proj/src/reconstruct.cpp:
// 355-393), the row->column transpose of reconstruct_into (424-427) and, for
// uint8 output, quantize (proj/src/io.cpp:78-81).
//
// Every output value is piecewise constant in time per pixel, so a thread owns
// 16 consecutive pixels of one kChunk-frame chunk and keeps their 16 current
// values packed in registers: the steady state is one 16-B store per frame
// (u8; 4 / 8 stores for f32 / f64) plus a pointer bump.  A warp writes 512
// contiguous bytes of a frame row per store.  Value changes come from the run
// lists: the run table gives each pixel's run at the chunk start, and the
// next run's start frame is the next change.  Run values are computed here
// from (intervals, span), exactly as reconstruct.cpp:124 (f64 bit-exact,
// integer form for u8).
#include <climits>

#include "spk_common.cuh"
#include "spk_kernels.cuh"

namespace spk {

namespace {

template <typename OUT>
struct Vec;
template <>
struct Vec<uint8_t> {
    static constexpr int N = 1;
    __device__ static void pack(const uint8_t (&v)[kExpPix], uint4 (&o)[N]) {
        uint32_t w[4];
#pragma unroll
        for (int k = 0; k < 4; ++k)
            w[k] = (uint32_t)v[4 * k] | (uint32_t)v[4 * k + 1] << 8 |
                   (uint32_t)v[4 * k + 2] << 16 | (uint32_t)v[4 * k + 3] << 24;
        o[0] = make_uint4(w[0], w[1], w[2], w[3]);
    }
};
template <>
struct Vec<float> {
    static constexpr int N = 4;
    __device__ static void pack(const float (&v)[kExpPix], uint4 (&o)[N]) {
#pragma unroll
        for (int k = 0; k < N; ++k)
            o[k] = make_uint4(__float_as_uint(v[4 * k]), __float_as_uint(v[4 * k + 1]),
                              __float_as_uint(v[4 * k + 2]), __float_as_uint(v[4 * k + 3]));
    }
};
template <>
struct Vec<double> {
    static constexpr int N = 8;
    __device__ static void pack(const double (&v)[kExpPix], uint4 (&o)[N]) {
#pragma unroll
        for (int k = 0; k < N; ++k) {
            const unsigned long long a = __double_as_longlong(v[2 * k]);
            const unsigned long long b = __double_as_longlong(v[2 * k + 1]);
            o[k] = make_uint4((uint32_t)a, (uint32_t)(a >> 32), (uint32_t)b, (uint32_t)(b >> 32));
        }
    }
};

__device__ __forceinline__ void st_v4(char* p, uint4 v) {
    asm volatile("st.global.v4.b32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(v.x), "r"(v.y),
                 "r"(v.z), "r"(v.w)
                 : "memory");
}

}  // namespace

template <typename OUT>
__global__ void __launch_bounds__(kExpThreads) k_expand(ExpArgs a) {
    constexpr int P = kExpPix;
    constexpr int NV = Vec<OUT>::N;
    const int64_t p0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * P;
    if (p0 >= a.npix) return;
    const int c = a.chunk0 + (int)blockIdx.y;
    const int f0 = c << kChunkLog2;
    if (f0 >= a.frames) return;
    const int f1 = min(a.frames, f0 + kChunk);
    const int np = (int)min((int64_t)P, a.npix - p0);

    int ridx[P], nst[P], rcnt[P];
    OUT val[P];
#pragma unroll
    for (int i = 0; i < P; ++i) {
        val[i] = OUT(0);
        nst[i] = INT_MAX;
        ridx[i] = -1;
        rcnt[i] = 0;
        if (i < np) {
            const int64_t p = p0 + i;
            const uint32_t cnt = a.counts[p];
            if (cnt > 0 && cnt <= (uint32_t)a.cap) {  // overflowed pixels: k_fixup
                rcnt[i] = (int)cnt;
                const spk_run_t* rp = a.runs + p * a.cap;
                const int r = a.tbl[(int64_t)c * a.npix + p];
                ridx[i] = r;
                if (r >= 0) {
                    const spk_run_t cur = rp[r];
                    const int nx = r + 1 < (int)cnt ? (int)rp[r + 1].start : INT_MAX;
                    const int end = nx == INT_MAX ? a.last[p] : nx;
                    val[i] = OutVal<OUT>::run(cur.intervals, (uint32_t)(end - (int)cur.start));
                    nst[i] = nx;
                } else {
                    nst[i] = (int)rp[0].start;
                }
            }
        }
    }
    int nc = INT_MAX;
#pragma unroll
    for (int i = 0; i < P; ++i) nc = min(nc, nst[i]);

    uint4 vec[NV];
    Vec<OUT>::pack(val, vec);
    const size_t step = a.pitch * sizeof(OUT);
    char* ptr = reinterpret_cast<char*>(a.out) + ((size_t)f0 * a.pitch + p0) * sizeof(OUT);
    const bool vec_ok = a.vec_ok && np == P;
    int f = f0;
    for (;;) {
        const int stop = min(nc, f1);
        if (vec_ok) {
#pragma unroll 4
            for (; f < stop; ++f, ptr += step) {
#pragma unroll
                for (int k = 0; k < NV; ++k) st_v4(ptr + 16 * k, vec[k]);
            }
        } else {
            for (; f < stop; ++f, ptr += step) {
                OUT* o = reinterpret_cast<OUT*>(ptr);
#pragma unroll
                for (int i = 0; i < P; ++i)
                    if (i < np) o[i] = val[i];
            }
        }
        if (f >= f1) break;
        // runs starting at frame f (starts strictly increase per pixel)
        nc = INT_MAX;
#pragma unroll
        for (int i = 0; i < P; ++i) {
            if (nst[i] == f) {
                const int64_t p = p0 + i;
                const spk_run_t* rp = a.runs + p * a.cap;
                const int r = ++ridx[i];
                const spk_run_t cur = rp[r];
                const int nx = r + 1 < rcnt[i] ? (int)rp[r + 1].start : INT_MAX;
                const int end = nx == INT_MAX ? a.last[p] : nx;
                val[i] = OutVal<OUT>::run(cur.intervals, (uint32_t)(end - (int)cur.start));
                nst[i] = nx;
            }
            nc = min(nc, nst[i]);
        }
        Vec<OUT>::pack(val, vec);
    }
}

template __global__ void k_expand<uint8_t>(ExpArgs);
template __global__ void k_expand<float>(ExpArgs);
template __global__ void k_expand<double>(ExpArgs);

}  // namespace spk
