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
// Per output type: P pixels per lane, F frames per sub-tile, K-deep run ring
// per pixel, WARPS per block.
template <typename OUT>
struct ExpGeo;
template <>
struct ExpGeo<uint8_t> {
    static constexpr int P = 8, F = 16, K = 4, WARPS = 2;
};
template <>
struct ExpGeo<float> {
    static constexpr int P = 8, F = 16, K = 4, WARPS = 2;
};
template <>
struct ExpGeo<double> {
    static constexpr int P = 8, F = 8, K = 4, WARPS = 2;
};

// Per-warp shared memory.  A warp owns S = 32*P pixel slots; slot
// s = i*32 + lane is pixel i of lane `lane` (pixel p0(lane) + i), so slot
// arrays are bank-interleaved by lane.
//   ring[K][S]  the next K runs of each slot, {start, value} (8 B; f64 16 B),
//               refilled with cp.async as runs are consumed
//   cur[S], cnt[S], nxt[S]  run the slot is in, its run count, the start
//               frame of its next run (INT_MAX = none)
//   D[F][32]    per frame and lane: the pending values of its P pixels
//   B[F][32]    per frame and lane: byte i = 0xff if pixel i changes there
template <typename OUT>
struct ExpSmem {
    static constexpr int P = ExpGeo<OUT>::P, F = ExpGeo<OUT>::F, K = ExpGeo<OUT>::K;
    static constexpr int S = 32 * P;
    static constexpr int RE = sizeof(OUT) == 8 ? 16 : 8;
    static constexpr int DE = P * (int)sizeof(OUT);
    static constexpr int ring = K * S * RE;
    static constexpr int cur = S * 4, cnt = S * 4, nxt = S * 4;
    static constexpr int d = F * 32 * DE;
    static constexpr int b = F * 32 * 8;
    static constexpr int queue = S * 2;
    static constexpr int per_warp = ring + cur + cnt + nxt + d + b + queue;
};

__device__ __forceinline__ void cp_async8(uint32_t saddr, const void* gmem) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(saddr), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async4(uint32_t saddr, const void* gmem) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(saddr), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

template <typename OUT>
__global__ void __launch_bounds__(ExpGeo<OUT>::WARPS * 32) k_expand(ExpArgs a) {
    using G = ExpSmem<OUT>;
    constexpr int P = G::P, F = G::F, K = G::K, S = G::S;
    constexpr int NW = P * (int)sizeof(OUT) / 4;  // 32-bit words per lane-frame
    extern __shared__ __align__(16) unsigned char sm[];
    const int lane = threadIdx.x & 31;
    unsigned char* wb = sm + (size_t)(threadIdx.x >> 5) * G::per_warp;
    unsigned char* ring = wb;
    int* CUR = reinterpret_cast<int*>(wb + G::ring);
    int* CNT = CUR + S;
    int* NXT = CNT + S;
    unsigned char* D = wb + G::ring + G::cur + G::cnt + G::nxt;
    unsigned char* B = D + G::d;
    uint16_t* Q = reinterpret_cast<uint16_t*>(B + G::b);
    const uint32_t ring_s = (uint32_t)__cvta_generic_to_shared(ring);

    // warp geometry: lane l owns pixels pw + l*P + i
    const int64_t pw = ((int64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31)) * P;
    const int64_t p0 = pw + (int64_t)lane * P;
    const int c = a.chunk0 + (int)blockIdx.y;
    const int f0 = c << kChunkLog2;
    if (pw >= a.npix || f0 >= a.frames) return;  // warp-uniform
    const int f1 = min(a.frames, f0 + kChunk);
    const int np = (int)max((int64_t)0, min((int64_t)P, a.npix - p0));

    auto entry = [&](int s, int q) -> unsigned char* { return ring + ((q & (K - 1)) * S + s) * G::RE; };
    auto fetch = [&](int s, int q) {  // request run q of slot s
        const int64_t p = pw + (int64_t)(s & 31) * P + (s >> 5);
        const size_t off = (size_t)p * a.cap + q;
        const uint32_t dst = ring_s + (uint32_t)(((q & (K - 1)) * S + s) * G::RE);
        if constexpr (sizeof(OUT) == 8) {
            cp_async4(dst, &a.runs[off].start);
            cp_async8(dst + 8, a.vals + off);
        } else {
            cp_async8(dst, a.runs + off);
        }
    };

    uint32_t words[NW];
#pragma unroll
    for (int k = 0; k < NW; ++k) words[k] = 0u;
#pragma unroll
    for (int i = 0; i < P; ++i) {
        const int s = i * 32 + lane;
        int r = -1, n = 0;
        if (i < np) {
            const int64_t p = p0 + i;
            const uint32_t cn = a.counts[p];
            if (cn > 0 && cn <= (uint32_t)a.cap) {  // overflowed pixels: k_fixup
                n = (int)cn;
                r = a.tbl[(int64_t)c * a.npix + p];
                if (r >= 0) {  // value at the chunk start
                    const size_t off = (size_t)p * a.cap + r;
                    if constexpr (sizeof(OUT) == 1)
                        words[i >> 2] |= (a.runs[off].intervals & 0xffu) << ((i & 3) * 8);
                    else if constexpr (sizeof(OUT) == 4)
                        words[i] = a.runs[off].intervals;
                    else {
                        const unsigned long long b = __double_as_longlong(a.vals[off]);
                        words[2 * i] = (uint32_t)b;
                        words[2 * i + 1] = (uint32_t)(b >> 32);
                    }
                }
                for (int q = r + 1; q < min(n, r + 1 + K); ++q) fetch(s, q);
            }
        }
        CUR[s] = r;
        CNT[s] = n;
    }
    cp_async_commit();
#pragma unroll
    for (int f = 0; f < F; ++f) *reinterpret_cast<uint2*>(B + (f * 32 + lane) * 8) = make_uint2(0u, 0u);
    cp_async_wait_all();
#pragma unroll
    for (int i = 0; i < P; ++i) {
        const int s = i * 32 + lane;
        const int q = CUR[s] + 1;
        NXT[s] = q < CNT[s] ? *reinterpret_cast<const int*>(entry(s, q)) : INT_MAX;
    }
    __syncwarp();

    const size_t step = a.pitch * sizeof(OUT);
    char* ptr = reinterpret_cast<char*>(a.out) + ((size_t)f0 * a.pitch + (size_t)p0) * sizeof(OUT);
    const bool vec_ok = a.vec_ok && np == P;

    for (int t0 = f0; t0 < f1; t0 += F) {
        const int t1 = min(f1, t0 + F);
        // ---- phase A (warp-cooperative): every value change of the warp's
        // pixels inside [t0, t1) goes to its owner's D/B bucket.  Pending slots
        // are compacted with ballots and spread over all 32 lanes; a round
        // consumes one run per pending slot.  The ring of a slot holds runs
        // requested at least K rounds (or one phase) ago; before reading an
        // entry requested in this phase, all lanes drain their copies.
        cp_async_wait_all();
        __syncwarp();
        for (int round = 1;; ++round) {
            if (round > 1 && (round - 1) % K == 0) {  // entries requested in this phase
                cp_async_wait_all();
                __syncwarp();
            }
            // own pending slots; a slot consumed last round (NXT < 0) first
            // learns its next start from the ring
            uint32_t own = 0;
#pragma unroll
            for (int i = 0; i < P; ++i) {
                const int s = i * 32 + lane;
                int v = NXT[s];
                if (v < 0) {
                    v = *reinterpret_cast<const int*>(entry(s, -v));
                    NXT[s] = v;
                }
                if (v < t1) own |= 1u << i;
            }
            // warp-exclusive prefix of the pending counts -> queue positions
            const int cnt_l = __popc(own);
            int incl = cnt_l;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const int y = __shfl_up_sync(kFull, incl, d);
                if (lane >= d) incl += y;
            }
            const int tot = __shfl_sync(kFull, incl, 31);
            if (tot == 0) break;
            int pos = incl - cnt_l;
            for (uint32_t m = own; m; m &= m - 1) Q[pos++] = (uint16_t)((__ffs(m) - 1) * 32 + lane);
            __syncwarp();
            for (int k = lane; k < tot; k += 32) {
                const int s = Q[k];
                const int i = s >> 5, col = s & 31;
                const int q = CUR[s] + 1;
                const unsigned char* e = entry(s, q);
                const int fo = *reinterpret_cast<const int*>(e) - t0;
                unsigned char* dcell = D + (fo * 32 + col) * G::DE;
                if constexpr (sizeof(OUT) == 8)
                    reinterpret_cast<double*>(dcell)[i] = *reinterpret_cast<const double*>(e + 8);
                else if constexpr (sizeof(OUT) == 4)
                    reinterpret_cast<uint32_t*>(dcell)[i] = reinterpret_cast<const uint32_t*>(e)[1];
                else
                    dcell[i] = (uint8_t)reinterpret_cast<const uint32_t*>(e)[1];
                B[(fo * 32 + col) * 8 + i] = 0xffu;
                CUR[s] = q;
                const int n = CNT[s];
                if (q + K < n) fetch(s, q + K);  // refill the slot just consumed
                NXT[s] = q + 1 < n ? -(q + 1) : INT_MAX;
            }
            __syncwarp();
        }
        cp_async_commit();
        // ---- phase B: frames in order, one store per frame, pending merged
        const int nf = t1 - t0;
        if constexpr (sizeof(OUT) == 1) {
            if (nf == F && vec_ok) {  // steady state: batch the bucket reads for ILP
                uint2 dv[F], bm[F];
#pragma unroll
                for (int fo = 0; fo < F; ++fo) {
                    dv[fo] = *reinterpret_cast<const uint2*>(D + (fo * 32 + lane) * G::DE);
                    bm[fo] = *reinterpret_cast<const uint2*>(B + (fo * 32 + lane) * 8);
                }
#pragma unroll
                for (int fo = 0; fo < F; ++fo)
                    *reinterpret_cast<uint2*>(B + (fo * 32 + lane) * 8) = make_uint2(0u, 0u);
#pragma unroll
                for (int fo = 0; fo < F; ++fo) {
                    words[0] = (words[0] & ~bm[fo].x) | (dv[fo].x & bm[fo].x);
                    words[1] = (words[1] & ~bm[fo].y) | (dv[fo].y & bm[fo].y);
                    st_words(ptr, words);
                    ptr += step;
                }
                continue;
            }
        }
#pragma unroll 4
        for (int fo = 0; fo < nf; ++fo) {
            const unsigned char* dcell = D + (fo * 32 + lane) * G::DE;
            uint2* bcell = reinterpret_cast<uint2*>(B + (fo * 32 + lane) * 8);
            const uint2 bm = *bcell;
            if constexpr (sizeof(OUT) == 1) {
                const uint2 dv = *reinterpret_cast<const uint2*>(dcell);
                *bcell = make_uint2(0u, 0u);
                words[0] = (words[0] & ~bm.x) | (dv.x & bm.x);
                words[1] = (words[1] & ~bm.y) | (dv.y & bm.y);
            } else {
                if (bm.x | bm.y) {
                    *bcell = make_uint2(0u, 0u);
                    const uint32_t* dw = reinterpret_cast<const uint32_t*>(dcell);
#pragma unroll
                    for (int i = 0; i < P; ++i) {
                        const bool take = ((i < 4 ? bm.x : bm.y) >> ((i & 3) * 8)) & 1u;
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
    return out_size == 1 ? (size_t)ExpSmem<uint8_t>::per_warp * ExpGeo<uint8_t>::WARPS
         : out_size == 4 ? (size_t)ExpSmem<float>::per_warp * ExpGeo<float>::WARPS
                         : (size_t)ExpSmem<double>::per_warp * ExpGeo<double>::WARPS;
}

int expand_threads(int out_size) {
    return 32 * (out_size == 1 ? ExpGeo<uint8_t>::WARPS
               : out_size == 4 ? ExpGeo<float>::WARPS
                               : ExpGeo<double>::WARPS);
}

int expand_pixels_per_lane(int out_size) {
    return out_size == 1 ? ExpGeo<uint8_t>::P : out_size == 4 ? ExpGeo<float>::P : ExpGeo<double>::P;
}

template __global__ void k_expand<uint8_t>(ExpArgs);
template __global__ void k_expand<float>(ExpArgs);
template __global__ void k_expand<double>(ExpArgs);

}  // namespace spk
