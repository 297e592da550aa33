// walk.cu -- K3 from K2's run lists: a tile-local sort replaces the global
// finalize pass (K2b histogram / scan / K2c scatter).
//
// Replaces the run fill loops of reconstruct_row (proj/src/reconstruct.cpp:
// 355-393), the row->column transpose of reconstruct_into (424-427) and, for
// uint8 output, quantize (proj/src/io.cpp:78-81).
//
// A pixel's output is piecewise constant in time: the value of run k holds
// from its start to the next run's start, the last run's value holds to the
// end of the stream, and frames before the first run are 0.
//
// k_hints (thread per pixel, one pass over the pixel's run list):
//   H[t][p] = runs of pixel p starting before frame t*kTileRows
//   V[t][p] = the value at that frame before any change there (run H-1's
//             value, 0 when H = 0)
//   so the changes of tile t are the runs k in [H[t], H[t+1]).
// k_walk: warp = one group of 32*P pixels (P per lane, a 512-byte row
//   segment for uint8) x one tile of kTileRows frames; warps are independent.
//   1. the tile's changes, sorted by sub-tile in shared memory: a histogram
//      of their sub-tiles (run starts), a scan, then every run becomes a
//      change (frame, pixel, value) placed by an atomic cursor;
//   2. per sub-tile of kSub frames (as the chunked expand): the sub-tile's
//      changes -> per-frame cells (value + pending bit mask), then every lane
//      walks the frames merging its cell and storing its P values per frame
//      (16 B for uint8: 512 contiguous bytes of a frame row per warp).
//   A tile with more changes than the list holds (noise-like pixels) writes
//   each pixel's column directly instead.
//
// Run values: 255*N/span (reconstruct.cpp:124) -- f64 bit-exact, f32 its
// rounding, u8 the exact round-half-away integer form (spk_common.cuh).
// Pixels whose list overflowed the capacity get arbitrary values here and are
// rewritten by k_fixup afterwards.
#include <climits>

#include "spk_common.cuh"
#include "spk_kernels.cuh"

namespace spk {

namespace {

__device__ __forceinline__ void st_v4(char* p, uint4 v) {
    asm volatile("st.global.v4.b32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
                 : "memory");
}

// Mask bit of pixel i of a lane: for uint8 output (4 pixels per 32-bit word)
// bit 8*(i&3) + (i>>2), so word w's byte mask is ((m >> w) & 0x01010101)*255;
// otherwise bit i.
template <typename OUT>
__device__ __forceinline__ uint32_t pend_bit(int i) {
    if constexpr (sizeof(OUT) == 1)
        return 1u << (8 * (i & 3) + (i >> 2));
    else
        return 1u << i;
}

// change key: frame offset in the tile (fo), pixel in the group (pix)
template <typename OUT>
__device__ __forceinline__ uint32_t change_fo(const Change<OUT>& c) {
    if constexpr (sizeof(OUT) == 1) return c.w >> 17; else return c.key >> 16;
}
template <typename OUT>
__device__ __forceinline__ uint32_t change_pix(const Change<OUT>& c) {
    if constexpr (sizeof(OUT) == 1) return (c.w >> 8) & 0x1ffu; else return c.key & 0xffffu;
}
template <typename OUT>
__device__ __forceinline__ Change<OUT> make_change(uint32_t fo, uint32_t pix, OUT v) {
    Change<OUT> c;
    if constexpr (sizeof(OUT) == 1) {
        c.w = fo << 17 | pix << 8 | (uint32_t)v;
    } else if constexpr (sizeof(OUT) == 4) {
        c.key = fo << 16 | pix;
        c.bits = __float_as_uint(v);
    } else {
        c.key = fo << 16 | pix;
        c.pad = 0;
        c.v = v;
    }
    return c;
}

}  // namespace

// ------------------------------------------------------------- k_hints --
template <typename OUT>
__global__ void __launch_bounds__(256) k_hints(WalkArgs a) {
    const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= a.npix) return;
    const int n = (int)min(a.counts[p], (uint32_t)a.cap);
    const spk_run_t* rp = a.runs + p * (int64_t)a.cap;
    const int ntiles = (a.frames + kTileRows - 1) / kTileRows;
    OUT* V = reinterpret_cast<OUT*>(a.tilev);
    const int lastp = a.last[p];
    int t = 0;        // next boundary to place
    OUT vprev = OUT(0);  // value of the run before run k
    for (int k0 = 0; k0 < n; k0 += 8) {
        spk_run_t r[9];  // eight runs and the next start in flight
#pragma unroll
        for (int j = 0; j <= 8; ++j)
            r[j] = k0 + j < n ? rp[k0 + j] : spk_run_t{(uint32_t)(k0 + j == n ? lastp : INT_MAX), 0u};
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            if (k0 + j >= n) break;
            const int st = (int)r[j].start;
            // boundaries up to this start: runs before k0 + j start before them
            while (t <= ntiles && t * kTileRows <= st) {
                a.hints[(int64_t)t * a.npix + p] = k0 + j;
                V[(int64_t)t * a.npix + p] = vprev;
                ++t;
            }
            vprev = OutVal<OUT>::run(r[j].intervals, r[j + 1].start - r[j].start);
        }
    }
    for (; t <= ntiles; ++t) {
        a.hints[(int64_t)t * a.npix + p] = n;
        V[(int64_t)t * a.npix + p] = vprev;
    }
}

template __global__ void k_hints<uint8_t>(WalkArgs);
template __global__ void k_hints<float>(WalkArgs);
template __global__ void k_hints<double>(WalkArgs);

// -------------------------------------------------------------- k_walk --
template <typename OUT>
struct WalkSmem {
    static constexpr int P = Geo<OUT>::P;
    static constexpr int GP = 32 * P;
    static constexpr int DE = P * (int)sizeof(OUT);  // D cell bytes
    static constexpr int cells = kSub * 32 * (DE + 4);
    static constexpr int CAP = 4 * GP;               // changes per warp tile
    static constexpr int kBinsT = kTileRows / kSub;  // sub-tiles per tile
    static constexpr int per_warp = cells + CAP * (int)sizeof(Change<OUT>) + 2 * kBinsT * 4;
};

size_t walk_smem_bytes(int out_size) {
    return out_size == 1 ? (size_t)WalkSmem<uint8_t>::per_warp * Geo<uint8_t>::WARPS
         : out_size == 4 ? (size_t)WalkSmem<float>::per_warp * Geo<float>::WARPS
                         : (size_t)WalkSmem<double>::per_warp * Geo<double>::WARPS;
}

template <typename OUT>
__global__ void __launch_bounds__(Geo<OUT>::WARPS * 32) k_walk(WalkArgs a) {
    using G = WalkSmem<OUT>;
    constexpr int P = G::P;
    constexpr int GP = G::GP;
    constexpr int NW = P * (int)sizeof(OUT) / 4;  // 32-bit words per lane-frame
    constexpr int NV = NW / 4;                     // 16-B vectors per lane-frame
    constexpr int NB = G::kBinsT;
    extern __shared__ __align__(16) unsigned char sm[];
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    unsigned char* D = sm + (size_t)warp * G::per_warp;
    uint32_t* B = reinterpret_cast<uint32_t*>(D + kSub * 32 * G::DE);
    Change<OUT>* list = reinterpret_cast<Change<OUT>*>(D + G::cells);
    uint32_t* boff = reinterpret_cast<uint32_t*>(list + G::CAP);  // [NB] offsets, then [NB] cursors
    uint32_t* bcur = boff + NB;

    const int64_t g = (int64_t)blockIdx.x * Geo<OUT>::WARPS + warp;
    const int tile = a.tile0 + (int)blockIdx.y;
    const int64_t npix = a.npix;
    const int64_t p0g = g * GP;
    if (p0g >= npix) return;  // warp-uniform; lanes only exchange via __syncwarp
    const int f0 = tile * kTileRows;
    const int f1 = min(a.frames, f0 + kTileRows);
    const int64_t p0 = p0g + (int64_t)lane * P;
    const int np = (int)max((int64_t)0, min((int64_t)P, npix - p0));
    const spk_run_t* runs = a.runs;
    const int64_t cap = a.cap;
    const int32_t* H0 = a.hints + (int64_t)tile * npix + p0;
    const int32_t* H1 = H0 + npix;
    const int32_t* HN = a.hints + (int64_t)((a.frames + kTileRows - 1) / kTileRows) * npix + p0;  // run counts

    // ---- values at the tile start, change counts
    uint32_t words[NW];
#pragma unroll
    for (int k = 0; k < NW; ++k) words[k] = 0u;
    const OUT* tv = reinterpret_cast<const OUT*>(a.tilev) + (int64_t)tile * npix + p0;
#pragma unroll
    for (int i = 0; i < P; ++i) {
        if (i < np) {
            const OUT v = tv[i];
            if constexpr (sizeof(OUT) == 1)
                words[i >> 2] |= (uint32_t)v << ((i & 3) * 8);
            else if constexpr (sizeof(OUT) == 4)
                words[i] = __float_as_uint(v);
            else {
                const unsigned long long b = __double_as_longlong(v);
                words[2 * i] = (uint32_t)b;
                words[2 * i + 1] = (uint32_t)(b >> 32);
            }
        }
    }
    int h0[P], h1[P];
    int mine = 0;
#pragma unroll
    for (int i = 0; i < P; ++i) {
        h0[i] = i < np ? H0[i] : 0;
        h1[i] = i < np ? H1[i] : 0;
        mine += h1[i] - h0[i];
    }
    const int total = (int)__reduce_add_sync(kFull, (unsigned)mine);

    const size_t step = a.pitch * sizeof(OUT);
    char* ptr0 = reinterpret_cast<char*>(a.out) + ((size_t)f0 * a.pitch + (size_t)p0) * sizeof(OUT);
    const bool vec_ok = a.vec_ok && np == P;

    if (total > G::CAP) {
        // ---- too many changes (noise-like pixels): each lane writes its pixels' columns
#pragma unroll 1
        for (int i = 0; i < np; ++i) {
            const int64_t p = p0 + i;
            const spk_run_t* rp = runs + p * cap;
            const int n = HN[i];
            OUT v = tv[i];
            int fr = f0;
            OUT* col = reinterpret_cast<OUT*>(reinterpret_cast<char*>(a.out) + (size_t)p * sizeof(OUT));
            for (int k = h0[i]; k <= h1[i]; ++k) {
                const int until = k < h1[i] ? (int)rp[k].start : f1;
                for (; fr < until; ++fr) col[(size_t)fr * a.pitch] = v;
                if (k < h1[i]) {
                    const int end = k + 1 < n ? (int)rp[k + 1].start : a.last[p];
                    v = OutVal<OUT>::run(rp[k].intervals, (uint32_t)(end - (int)rp[k].start));
                }
            }
        }
        return;
    }

    // ---- the tile's changes sorted by sub-tile: histogram, scan, placement
    for (int i = lane; i < 2 * NB; i += 32) boff[i] = 0u;
    __syncwarp();
#pragma unroll
    for (int i = 0; i < P; ++i) {
        const spk_run_t* rp = runs + (p0 + i) * cap;
        for (int k = h0[i]; k < h1[i]; ++k) atomicAdd(&boff[((int)__ldg(&rp[k].start) - f0) / kSub], 1u);
    }
    __syncwarp();
    {
        // exclusive scan of the NB (<= 32) bin counts
        const uint32_t c = lane < NB ? boff[lane] : 0u;
        uint32_t inc = c;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const uint32_t y = __shfl_up_sync(kFull, inc, d);
            if (lane >= d) inc += y;
        }
        __syncwarp();
        if (lane < NB) {
            boff[lane] = inc - c;
            bcur[lane] = inc - c;
        }
        __syncwarp();
    }
#pragma unroll
    for (int i = 0; i < P; ++i) {
        const int64_t p = p0 + i;
        const spk_run_t* rp = runs + p * cap;
        const int n = HN[i];
        for (int k = h0[i]; k < h1[i]; ++k) {
            const spk_run_t r = rp[k];
            const int end = k + 1 < n ? (int)rp[k + 1].start : a.last[p];
            const OUT v = OutVal<OUT>::run(r.intervals, (uint32_t)(end - (int)r.start));
            const uint32_t fo = (uint32_t)((int)r.start - f0);
            const uint32_t pos = atomicAdd(&bcur[fo / kSub], 1u);
            list[pos] = make_change<OUT>(fo, (uint32_t)(lane * P + i), v);
        }
    }
#pragma unroll
    for (int f = 0; f < kSub; ++f) B[f * 32 + lane] = 0u;
    __syncwarp();

    auto bucket = [&](const Change<OUT>& ch, int sub) {
        const uint32_t fo = change_fo<OUT>(ch), pix = change_pix<OUT>(ch);
        const int fs = (int)fo - sub * kSub;  // frame within the sub-tile
        const int own = (int)(pix / P), i = (int)(pix % P);
        unsigned char* dcell = D + (fs * 32 + own) * G::DE;
        if constexpr (sizeof(OUT) == 1)
            dcell[i] = (uint8_t)ch.w;
        else if constexpr (sizeof(OUT) == 4)
            reinterpret_cast<uint32_t*>(dcell)[i] = ch.bits;
        else
            reinterpret_cast<double*>(dcell)[i] = ch.v;
        atomicOr(&B[fs * 32 + own], pend_bit<OUT>(i));
    };

    char* ptr = ptr0;
    for (int sub = 0; sub < NB; ++sub) {
        const int t0 = f0 + sub * kSub;
        if (t0 >= f1) break;
        // ---- phase A: this sub-tile's changes -> owners' buckets
        const uint32_t off = boff[sub];
        const uint32_t n = (sub + 1 < NB ? boff[sub + 1] : (uint32_t)total) - off;
        for (uint32_t k = lane; k < n; k += 32) bucket(list[off + k], sub);
        __syncwarp();
        // ---- phase B: frames in order, one store per frame
        const int nf = min(kSub, f1 - t0);
#pragma unroll 4
        for (int fs = 0; fs < nf; ++fs) {
            const uint32_t bm = B[fs * 32 + lane];
            if constexpr (sizeof(OUT) == 1) {  // branch-free: a clear mask keeps every byte
                B[fs * 32 + lane] = 0u;
                const uint4 dv = *reinterpret_cast<const uint4*>(D + (fs * 32 + lane) * G::DE);
                const uint32_t m0 = (bm & 0x01010101u) * 0xffu, m1 = ((bm >> 1) & 0x01010101u) * 0xffu;
                const uint32_t m2 = ((bm >> 2) & 0x01010101u) * 0xffu, m3 = ((bm >> 3) & 0x01010101u) * 0xffu;
                words[0] = (words[0] & ~m0) | (dv.x & m0);
                words[1] = (words[1] & ~m1) | (dv.y & m1);
                words[2] = (words[2] & ~m2) | (dv.z & m2);
                words[3] = (words[3] & ~m3) | (dv.w & m3);
            } else if (bm) {
                B[fs * 32 + lane] = 0u;
                const uint32_t* dw = reinterpret_cast<const uint32_t*>(D + (fs * 32 + lane) * G::DE);
#pragma unroll
                for (int i = 0; i < P; ++i) {
                    const bool take = (bm >> i) & 1u;
                    if constexpr (sizeof(OUT) == 4) {
                        words[i] = take ? dw[i] : words[i];
                    } else {
                        words[2 * i] = take ? dw[2 * i] : words[2 * i];
                        words[2 * i + 1] = take ? dw[2 * i + 1] : words[2 * i + 1];
                    }
                }
            }
            if (vec_ok) {
#pragma unroll
                for (int k = 0; k < NV; ++k)
                    st_v4(ptr + 16 * k, make_uint4(words[4 * k], words[4 * k + 1], words[4 * k + 2],
                                                   words[4 * k + 3]));
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
        __syncwarp();  // bucket clears done before the next phase A refills them
    }
}

template __global__ void k_walk<uint8_t>(WalkArgs);
template __global__ void k_walk<float>(WalkArgs);
template __global__ void k_walk<double>(WalkArgs);

}  // namespace spk
