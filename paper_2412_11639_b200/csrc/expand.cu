// expand.cu -- K2b/K2c (run values, chunk-start values, frame-sorted change
// stream) and K3 (change stream -> frame planes).
//
// Replaces the run fill loops of reconstruct_row (proj/src/reconstruct.cpp:
// 355-393), the row->column transpose of reconstruct_into (424-427) and, for
// uint8 output, quantize (proj/src/io.cpp:78-81).
//
// Output values are piecewise constant in time per pixel; they change only at
// run starts.  The expand kernel should therefore do one thing per frame --
// store the packed current values of its pixels -- and touch only the changes
// otherwise.  To make the changes cheap to find, they are sorted by time once:
//
//   K2b k_fin_bins    run starts per (chunk, pixel group, sub-tile) -> bins
//   scan              exclusive prefix of bins -> offs
//   K2c k_fin_scatter the value at every chunk start (tblv; chunks before the
//       first run stay 0) and the change stream: every run start as (frame
//       offset, pixel, value), grouped by (chunk, group, sub-tile).  Run
//       values are 255*N/span (reconstruct.cpp:124): f64 bit-exact, u8 via
//       the exact round-half-away integer form.
//   (K2b/K2c: block = pixel group x chunk window, warp = one pixel, 32 runs
//   per coalesced load, shared-memory counters.)
//   K3  k_expand      one warp per (group, chunk, 64-frame piece): per sub-tile of kSub
//       frames, the warp reads that sub-tile's changes (contiguous, coalesced)
//       into per-frame value/mask buckets in shared memory, then every lane
//       walks the frames merging its bucket and storing its P values per frame
//       (16 B for u8: a warp writes 512 contiguous bytes of a frame row).
#include <climits>

#include <cuda.h>

#include "spk_common.cuh"

#ifndef SPK_TMA_BUFS
#define SPK_TMA_BUFS 1  // staging buffers per warp (1: 10 KB per warp, 5 blocks per SM)
#endif
#include "spk_kernels.cuh"

namespace spk {

namespace {

__device__ __forceinline__ void st_v4(char* p, uint4 v) {
    asm volatile("st.global.v4.b32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
                 "r"(v.w)
                 : "memory");
}

}  // namespace

// --------------------------------------------------- K2b histogram / K2c --
// Both passes: block = one pixel group (GP pixels) x one window of
// kFinWindow chunks; warp = one pixel at a time, reading its run list 32 runs
// per load (lane k <- run b+k, coalesced).  The per-window counters live in
// shared memory, so no global atomics.

// K2b: run starts per (chunk, group, sub-tile)
template <int GP, bool SPLIT>
__global__ void __launch_bounds__(kFinWarps * 32, 2) k_fin_bins(FinArgs a) {
    __shared__ uint32_t hist[kFinWindow * kBins];
    const int g = blockIdx.x;
    const int cw0 = blockIdx.y * kFinWindow;
    const int cw1 = min(a.nchunks, cw0 + kFinWindow);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    // blockIdx.z: this block's share of the group's pixels (gridDim.z > 1
    // for sensors with few groups: more blocks in flight; the shares' counts
    // meet in global memory, zeroed beforehand)
    const int share = GP / (int)gridDim.z;
    const int pl0 = (int)blockIdx.z * share, pl1 = pl0 + share;
    for (int i = threadIdx.x; i < (cw1 - cw0) * kBins; i += blockDim.x) hist[i] = 0;
    __syncthreads();
    auto bin_start = [&](uint32_t sv) {
        const int st = (int)sv;
        const int c = st >> kChunkLog2;
        if (sv != 0xffffffffu && c >= cw0 && c < cw1)
            atomicAdd(&hist[(c - cw0) * kBins + ((st & (kChunk - 1)) / kSub)], 1u);
    };
    if constexpr (!SPLIT) {
        // One contiguous list per pixel.  The warp's pixels are pl0 + warp +
        // j * kFinWarps: lane j loads the count of pixel j (one round trip
        // for all of them instead of one per pixel), counts a short list
        // (<= kShortList runs: static pixels hold one or two) by itself, and
        // the longer lists are read by the whole warp, 128 runs per pass
        // (lane k <- runs b + 32u + k).  K2b on a static 400x250 scene was
        // 21 us of dependent count -> runs round trips.
        static_assert(GP <= 32 * kFinWarps, "a warp's pixels fit one lane each");
        constexpr int kShortList = 4;
        const int npx = max(0, (share - warp + kFinWarps - 1) / kFinWarps);
        int myn = 0;
        const int64_t pj = (int64_t)g * GP + pl0 + warp + (int64_t)lane * kFinWarps;
        if (lane < npx && pj < a.npix) myn = (int)min(a.counts[pj], (uint32_t)a.cap);
        if (myn > 0 && myn <= kShortList) {
            const spk_run_t* rp = a.runs + pj * a.cap;
            uint32_t sv[kShortList];
#pragma unroll
            for (int k = 0; k < kShortList; ++k)
                sv[k] = k < myn ? (uint32_t)max((int)rp[k].start, 0) : 0xffffffffu;
#pragma unroll
            for (int k = 0; k < kShortList; ++k) bin_start(sv[k]);
        }
        uint32_t todo = __ballot_sync(kFull, myn > kShortList);
        while (todo) {  // warp-uniform
            const int j = __ffs(todo) - 1;
            todo &= todo - 1;
            const int n = __shfl_sync(kFull, myn, j);
            const spk_run_t* rp = a.runs + ((int64_t)g * GP + pl0 + warp + (int64_t)j * kFinWarps) * a.cap;
            for (int b = 0; b < n; b += 128) {
                uint32_t sv[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int k = b + 32 * u + lane;
                    // a run started before frame 0 (time shards) changes the value at frame 0
                    sv[u] = k < n ? (uint32_t)max((int)rp[k].start, 0) : 0xffffffffu;
                }
#pragma unroll
                for (int u = 0; u < 4; ++u) bin_start(sv[u]);
            }
        }
    } else {
    for (int pl = pl0 + warp; pl < pl1; pl += kFinWarps) {
        const int64_t p = (int64_t)g * GP + pl;
        if (p >= a.npix) break;
        const spk_run_t* rp = a.runs + p * a.cap;
        const int n = (int)min(a.counts[p], (uint32_t)a.cap);
        {
        // in-grid time split: the row's segments, 32-slot blocks of them four
        // per pass; lane r holds segment r (begin, end, first block index)
        const uint32_t* sg = a.seg + p * a.nseg * 2;
        int sb = 0, se = 0, nb = 0;
        if (lane < a.nseg) {
            sb = (int)__ldg(sg + 2 * lane);
            se = (int)__ldg(sg + 2 * lane + 1);
            nb = (se - sb + 31) >> 5;
        }
        int inc = nb;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const int y = __shfl_up_sync(kFull, inc, d);
            if (lane >= d) inc += y;
        }
        const int bs = inc - nb;  // first block of segment `lane`
        const int blocks = __shfl_sync(kFull, inc, 31);
        for (int q0 = 0; q0 < blocks; q0 += 4) {
            uint32_t sv[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int q = q0 + u;  // warp-uniform block index
                // the last non-empty segment starting at or before block q
                const uint32_t m = __ballot_sync(kFull, (lane < a.nseg) & (bs <= q) & (nb > 0));
                const int rr = m ? 31 - __clz(m) : 0;
                const int k = __shfl_sync(kFull, sb, rr) + 32 * (q - __shfl_sync(kFull, bs, rr)) + lane;
                const int e = __shfl_sync(kFull, se, rr);
                sv[u] = (q < blocks) & (k < e) ? (uint32_t)max((int)rp[k].start, 0) : 0xffffffffu;
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) bin_start(sv[u]);
        }
        }
    }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < (cw1 - cw0) * kBins; i += blockDim.x) {
        const int c = cw0 + i / kBins;
        uint32_t* b = &a.bins[((int64_t)c * a.ngroups + g) * kBins + (i % kBins)];
        if (gridDim.z == 1)
            *b = hist[i];
        else if (hist[i])
            atomicAdd(b, hist[i]);
    }
}

template __global__ void k_fin_bins<512, false>(FinArgs);
template __global__ void k_fin_bins<256, false>(FinArgs);
template __global__ void k_fin_bins<512, true>(FinArgs);
template __global__ void k_fin_bins<256, true>(FinArgs);

template <typename OUT>
__device__ __forceinline__ Change<OUT> make_change(uint32_t fo, uint32_t pl, OUT val) {
    Change<OUT> ch;
    if constexpr (sizeof(OUT) == 1) {
        ch.w = fo << 17 | pl << 8 | (uint32_t)val;
    } else if constexpr (sizeof(OUT) == 4) {
        ch.key = fo << 16 | pl;
        ch.bits = __float_as_uint(val);
    } else {
        ch.key = fo << 16 | pl;
        ch.pad = 0;
        ch.v = val;
    }
    return ch;
}

// K2c: the change stream and the value at every chunk start.  Thread = one
// pixel, free-running (no block synchronisation): runs are read 8 at a time
// (run k's value needs run k+1's start, or the last spike for the final run),
// their stream slots are claimed with 8 independent atomics on a copy of the
// scanned histogram, then the 8 changes are stored -- one memory round trip
// per 8 runs.
#ifndef SPK_K2C_MINB
#define SPK_K2C_MINB 4  // uint8 lists: 64 registers, more warps in flight (C2 finalize 0.411 -> 0.398 ms)
#endif
#ifndef SPK_K2C_B
#define SPK_K2C_B 4
#endif
template <typename OUT, bool SPLIT>
__global__ void __launch_bounds__(256, sizeof(OUT) == 1 && !SPLIT ? SPK_K2C_MINB : 1) k_fin_scatter(FinArgs a) {
    constexpr int GP = 32 * Geo<OUT>::P;
    constexpr int B = SPK_K2C_B;
    const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= a.npix) return;
    const int g = (int)(p / GP);
    const uint32_t pl = (uint32_t)(p % GP);
    const uint32_t cnt = a.counts[p];
    const bool over = cnt > (uint32_t)a.cap;  // k_fixup rewrites it: values don't matter
    // blockIdx.y: this thread's block of a.fin_seg list slots (runs are
    // independent here -- a value needs only the next run's start -- so a
    // pixel's list is spread over several threads: enough loads and atomics
    // in flight even for sensors with few pixels)
    // (split lists: the same numbering over the row's segments in order)
    // blocks of a.fin_seg list entries, strided over gridDim.y (a long list
    // with few runs per pixel does not launch a block row per capacity block)
    const int n = (int)min(cnt, (uint32_t)a.cap);
    if ((int)blockIdx.y * a.fin_seg >= n) return;
    const spk_run_t* rp = a.runs + p * a.cap;
    const uint32_t lastp = (uint32_t)a.last[p];
    Change<OUT>* stp = reinterpret_cast<Change<OUT>*>(a.stream);
    OUT* tb = reinterpret_cast<OUT*>(a.tblv);
    const int64_t total_frames = (int64_t)a.nchunks << kChunkLog2;
    // the runs of [b, e) (slots of one list segment), `nxt` = the start of the
    // run after e (the next segment's first run, or the last spike when the
    // segment ends the list: `fin`)
    auto range = [&](int b, int e, uint32_t nxt, bool fin) {
        for (int k0 = b; k0 < e; k0 += B) {
            spk_run_t r[B + 1];
#pragma unroll
            for (int j = 0; j <= B; ++j)
                r[j] = k0 + j < e ? rp[k0 + j] : spk_run_t{k0 + j == e ? nxt : 0x7fffffffu, 0u};
            uint32_t pos[B];
#pragma unroll
            for (int j = 0; j < B; ++j) {
                if (k0 + j < e) {
                    const int st = max((int)r[j].start, 0);  // see K2b: starts before frame 0
                    const int c = st >> kChunkLog2;
                    const int bi = (st & (kChunk - 1)) / kSub;
                    SPK_CHECK(c < a.nchunks);
                    pos[j] = atomicAdd(&a.cursor[((int64_t)c * a.ngroups + g) * kBins + bi], 1u);
                    SPK_CHECK((int64_t)pos[j] < a.stream_len);
                }
            }
#pragma unroll
            for (int j = 0; j < B; ++j) {
                if (k0 + j < e) {
                    const int st = max((int)r[j].start, 0);
                    const uint32_t fo = (uint32_t)(st & (kChunk - 1));
                    const OUT val = over ? OUT(0) : OutVal<OUT>::run(r[j].intervals, r[j + 1].start - r[j].start);
                    stp[pos[j]] = make_change<OUT>(fo, pl, val);
                    if (!over) {  // chunk starts in [start, next start); the last run covers the tail
                        const int64_t hi = (fin & (k0 + j + 1 == e)) ? total_frames : (int64_t)(int)r[j + 1].start;
                        for (int64_t cc = ((int64_t)st + kChunk - 1) >> kChunkLog2; cc <= (hi - 1) >> kChunkLog2; ++cc)
                            tb[cc * a.npix + p] = val;
                    }
                }
            }
        }
    };
    // 16-byte run loads: the list base and every batch start (a multiple of B) are 16-byte aligned
#ifndef SPK_K2C_VEC
#define SPK_K2C_VEC 1
#endif
    const bool vec = (SPK_K2C_VEC != 0) & (B % 2 == 0) & ((a.cap & 1) == 0) &
                     ((reinterpret_cast<uintptr_t>(a.runs) & 15) == 0);
    for (int kb = (int)blockIdx.y * a.fin_seg; kb < n; kb += (int)gridDim.y * a.fin_seg) {
    const int ke = min(n, kb + a.fin_seg);
    if constexpr (!SPLIT) {  // one contiguous list
        // Software pipeline: the loads of batch k0 + B are issued before the
        // atomics and stores of batch k0 (the thread is bound by the latency
        // of its run loads: ncu long-scoreboard at their first use).  Batch
        // slots past the list hold the sentinel run {next start, 0}.
        auto load_batch = [&](int k0, spk_run_t (&r)[B]) {
            if (vec) {
                // (every per-lane load is its own 128-byte line: two runs per 16-byte load)
#pragma unroll
                for (int j = 0; j < B; j += 2) {
                    if (k0 + j + 1 < n) {
                        const uint4 v = *reinterpret_cast<const uint4*>(rp + k0 + j);
                        r[j] = spk_run_t{v.x, v.y};
                        r[j + 1] = spk_run_t{v.z, v.w};
                    } else {
                        r[j] = k0 + j < n ? rp[k0 + j] : spk_run_t{k0 + j == n ? lastp : 0x7fffffffu, 0u};
                        r[j + 1] = spk_run_t{k0 + j + 1 == n ? lastp : 0x7fffffffu, 0u};
                    }
                }
            } else {
#pragma unroll
                for (int j = 0; j < B; ++j)
                    r[j] = k0 + j < n ? rp[k0 + j] : spk_run_t{k0 + j == n ? lastp : 0x7fffffffu, 0u};
            }
        };
        spk_run_t r[B + 1], nx[B];
        load_batch(kb, nx);
        for (int k0 = kb; k0 < ke; k0 += B) {
#pragma unroll
            for (int j = 0; j < B; ++j) r[j] = nx[j];
            load_batch(k0 + B, nx);  // (past ke: sentinels or the next thread's runs, only nx[0].start is used)
            r[B] = nx[0];
            uint32_t pos[B];
#pragma unroll
            for (int j = 0; j < B; ++j) {
                if (k0 + j < ke) {
                    const int st = max((int)r[j].start, 0);  // see K2b: starts before frame 0
                    const int c = st >> kChunkLog2;
                    const int bi = (st & (kChunk - 1)) / kSub;
                    SPK_CHECK(c < a.nchunks);
                    pos[j] = atomicAdd(&a.cursor[((int64_t)c * a.ngroups + g) * kBins + bi], 1u);
                    SPK_CHECK((int64_t)pos[j] < a.stream_len);
                }
            }
#pragma unroll
            for (int j = 0; j < B; ++j) {
                if (k0 + j < ke) {
                    const int st = max((int)r[j].start, 0);
                    const uint32_t fo = (uint32_t)(st & (kChunk - 1));
                    const OUT val = over ? OUT(0) : OutVal<OUT>::run(r[j].intervals, r[j + 1].start - r[j].start);
                    stp[pos[j]] = make_change<OUT>(fo, pl, val);
                    if (!over) {  // chunk starts in [start, next start); the last run covers the tail
                        // (frames < 2^29: 32-bit arithmetic; most runs cover no chunk start)
                        const int hi = k0 + j + 1 < n ? (int)r[j + 1].start : (int)total_frames;
                        for (int cc = (st + kChunk - 1) >> kChunkLog2; cc <= (hi - 1) >> kChunkLog2; ++cc)
                            tb[(int64_t)cc * a.npix + p] = val;
                    }
                }
            }
        }
        continue;
    }
    // in-grid time split: list entries [kb, ke) over the row's segments
    const uint32_t* sg = a.seg + p * a.nseg * 2;
    int vo = 0;  // list index of segment r's first run
    for (int r = 0; r < a.nseg && vo < ke; ++r) {
        const int b = (int)__ldg(sg + 2 * r), e = (int)__ldg(sg + 2 * r + 1);
        const int len = e - b;
        if (vo + len > kb) {
            const int lo = b + max(kb - vo, 0), hi = b + min(ke - vo, len);
            uint32_t nxt = lastp;
            bool fin = true;
            if (hi < e) {
                nxt = rp[hi].start;
                fin = false;
            } else {
                for (int q = r + 1; q < a.nseg; ++q) {
                    const int qb = (int)__ldg(sg + 2 * q);
                    if ((int)__ldg(sg + 2 * q + 1) > qb) {
                        nxt = rp[qb].start;
                        fin = false;
                        break;
                    }
                }
            }
            range(lo, hi, nxt, fin);
        }
        vo += len;
    }
    }
}

template __global__ void k_fin_scatter<uint8_t, false>(FinArgs);
template __global__ void k_fin_scatter<float, false>(FinArgs);
template __global__ void k_fin_scatter<double, false>(FinArgs);
template __global__ void k_fin_scatter<uint8_t, true>(FinArgs);
template __global__ void k_fin_scatter<float, true>(FinArgs);
template __global__ void k_fin_scatter<double, true>(FinArgs);

// -------------------------------------------------------------- K3 expand --
// Per-warp shared memory: for each frame of the sub-tile and each lane, the
// pending values of its P pixels (D, P values) and a bit mask of the pending
// pixels (B, one 32-bit word: bit i = pixel i changes at this frame).  Only
// the masks are read for every frame; D cells are read when a mask is set.
template <typename OUT>
struct ExpSmem {
    static constexpr int P = Geo<OUT>::P;
    static constexpr int DE = P * (int)sizeof(OUT);  // D cell bytes
    static constexpr int BE = 4;                       // B cell bytes
    static constexpr int per_warp = kSub * 32 * (DE + BE);
    // TMA stores (uint8): two D buffers -- the merged frames are written back
    // into the cells, and the sub-tile leaves as one tensor store -- + B
    static constexpr int per_warp_tma = SPK_TMA_BUFS * kSub * 32 * DE + kSub * 32 * BE;
};

size_t expand_smem_bytes(int out_size, int warps, bool tma) {
    if (tma) return (size_t)warps * ExpSmem<uint8_t>::per_warp_tma;
    return (size_t)warps * (out_size == 1 ? ExpSmem<uint8_t>::per_warp
                          : out_size == 4 ? ExpSmem<float>::per_warp
                                          : ExpSmem<double>::per_warp);
}

// each byte of x -> 0xff if its top bit is set, else 0 (PRMT with sign
// replication; __byte_perm ignores the selector's replicate bit)
__device__ __forceinline__ uint32_t sign_bytes(uint32_t x) {
    uint32_t r;
    asm("prmt.b32 %0, %1, 0, 0xBA98;" : "=r"(r) : "r"(x));
    return r;
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

template <typename OUT, int WARPS, bool TMA>
__global__ void __launch_bounds__(WARPS * 32) k_expand(ExpArgs a, const __grid_constant__ CUtensorMap tmap) {
    using G = ExpSmem<OUT>;
    static_assert(!TMA || sizeof(OUT) == 1, "TMA tile stores: uint8 frames");
    constexpr int P = G::P;
    constexpr int GP = 32 * P;
    constexpr int NW = P * (int)sizeof(OUT) / 4;  // 32-bit words per lane-frame
    constexpr int NV = NW / 4;                     // 16-B vectors per lane-frame
    constexpr int DBYTES = kSub * 32 * G::DE;      // one D buffer: kSub rows x 32 lanes
    extern __shared__ __align__(128) unsigned char sm[];
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    unsigned char* const D0 = sm + (size_t)warp * (TMA ? G::per_warp_tma : G::per_warp);
    unsigned char* D = D0;  // (TMA: the buffer of the current sub-tile, D0 or D0 + DBYTES)
    uint32_t* B = reinterpret_cast<uint32_t*>(D0 + (TMA ? SPK_TMA_BUFS : 1) * DBYTES);

    const int g = blockIdx.x * WARPS + warp;
    // tile = (group, chunk, piece of kPieceSubs sub-tiles): blocks of one
    // piece row run together, so the rows being written at any time stay
    // within a narrow band of frames (DRAM page locality: 64-row tiles write
    // at 6.8 TB/s in the probe, 1024-row tiles at 5.7)
    const int c = a.chunk0 + (int)blockIdx.y / a.pieces;
    const int sub0 = ((int)blockIdx.y % a.pieces) * kPieceSubs;
    if (g >= a.ngroups) return;  // warp-uniform; lanes only exchange via __syncwarp
    const int fc = c << kChunkLog2;       // chunk start
    const int f0 = fc + sub0 * kSub;      // piece start
    const int f1 = min(a.frames, fc + kChunk);
    if (f0 >= f1) return;
    const int64_t p0 = (int64_t)g * GP + (int64_t)lane * P;
    const int np = (int)max((int64_t)0, min((int64_t)P, a.npix - p0));

    // values at the chunk start
    uint32_t words[NW];
    const OUT* tb = reinterpret_cast<const OUT*>(a.tblv) + (int64_t)c * a.npix + p0;
#pragma unroll
    for (int k = 0; k < NW; ++k) words[k] = 0u;
    if (np == P && ((reinterpret_cast<uintptr_t>(tb) & 15) == 0)) {
#pragma unroll
        for (int k = 0; k < NV; ++k) {
            const uint4 w4 = reinterpret_cast<const uint4*>(tb)[k];
            words[4 * k] = w4.x;
            words[4 * k + 1] = w4.y;
            words[4 * k + 2] = w4.z;
            words[4 * k + 3] = w4.w;
        }
    } else {
#pragma unroll
        for (int i = 0; i < P; ++i) {
            if (i < np) {
                if constexpr (sizeof(OUT) == 1)
                    words[i >> 2] |= (uint32_t)tb[i] << ((i & 3) * 8);
                else if constexpr (sizeof(OUT) == 4)
                    words[i] = __float_as_uint(tb[i]);
                else {
                    const unsigned long long b = __double_as_longlong(tb[i]);
                    words[2 * i] = (uint32_t)b;
                    words[2 * i + 1] = (uint32_t)(b >> 32);
                }
            }
        }
    }
    // the chunk's kBins (offset, count) pairs: lane l holds bins l and l+32
    const int64_t b0 = ((int64_t)c * a.ngroups + g) * kBins;
    const uint32_t off_lo = a.offs[b0 + lane], off_hi = a.offs[b0 + 32 + lane];
    const uint32_t cnt_lo = a.bins[b0 + lane], cnt_hi = a.bins[b0 + 32 + lane];
    const Change<OUT>* st = reinterpret_cast<const Change<OUT>*>(a.stream);
    SPK_CHECK((int64_t)(off_hi + cnt_hi) <= a.stream_len);
    // Dense tiles (many changes per pixel in the chunk) are written whole by
    // the piece-0 warp: the piece prefix would re-read too many changes.
    // Tile height by the tile's change density: the denser, the longer the
    // prefix a piece re-reads, so pieces merge (64 -> 128 frames) and dense
    // tiles are written whole; the merged-away pieces exit at once.
    const uint32_t tile_changes = __shfl_sync(kFull, off_hi + cnt_hi, 31) - __shfl_sync(kFull, off_lo, 0);
    const int span = a.pieces == 1 ? kBins
                   : tile_changes <= (uint32_t)(kPieceSparse * GP) ? kPieceSubs
                   : tile_changes <= (uint32_t)(kPieceDensity * GP) ? 2 * kPieceSubs
                   : tile_changes <= (uint32_t)(kPieceDense * GP) ? 4 * kPieceSubs
                                                                  : kBins;
    if (sub0 % span) return;  // warp-uniform
    const int sub1 = min(sub0 + span, kBins);
    if (sub0 > 0) {
        // values at the piece start: the chunk-start values updated by the
        // latest change of each pixel in the sub-tiles before the piece (one
        // contiguous range of the stream; a shared-memory max over
        // (frame offset, index) per pixel picks it)
        uint32_t* K = reinterpret_cast<uint32_t*>(D);
        for (int i = lane; i < GP; i += 32) K[i] = 0u;
        __syncwarp();
        const uint32_t pb = __shfl_sync(kFull, off_lo, 0);
        const uint32_t pe = __shfl_sync(kFull, sub0 < 32 ? off_lo : off_hi, sub0 & 31);
        // uint8: the key carries the value itself ((frame + 1) << 8 | value),
        // so the winner needs no second load; wider values keep the index.
        // Four changes per lane per pass (independent loads in flight).
        auto take = [&](const Change<OUT>& ch, uint32_t k) {
            if constexpr (sizeof(OUT) == 1) {
                const uint32_t fo = ch.w >> 17, pix = (ch.w >> 8) & 0x1ffu;
                SPK_CHECK(fo < (uint32_t)(sub0 * kSub));  // a change of an earlier sub-tile
                atomicMax(&K[pix], (fo + 1u) << 8 | (ch.w & 0xffu));
            } else {
                const uint32_t fo = ch.key >> 16, pix = ch.key & 0xffffu;
                atomicMax(&K[pix], (fo + 1u) << 20 | k);  // k < 2^20: at most 512 x 1024 changes
            }
        };
        const uint32_t np_ = pe - pb;
        uint32_t k = lane;
        for (; k + 96 < np_; k += 128) {
            Change<OUT> c4[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) c4[u] = st[pb + k + 32 * u];
#pragma unroll
            for (int u = 0; u < 4; ++u) take(c4[u], k + 32 * u);
        }
        for (; k < np_; k += 32) take(st[pb + k], k);
        __syncwarp();
#pragma unroll
        for (int i = 0; i < P; ++i) {
            const uint32_t key = K[lane * P + i];
            if (key) {
                if constexpr (sizeof(OUT) == 1) {
                    const int sh = (i & 3) * 8;
                    words[i >> 2] = (words[i >> 2] & ~(0xffu << sh)) | ((key & 0xffu) << sh);
                } else if constexpr (sizeof(OUT) == 4) {
                    const Change<OUT> ch = st[pb + (key & 0xfffffu)];
                    words[i] = ch.bits;
                } else {
                    const Change<OUT> ch = st[pb + (key & 0xfffffu)];
                    const unsigned long long bits = __double_as_longlong(ch.v);
                    words[2 * i] = (uint32_t)bits;
                    words[2 * i + 1] = (uint32_t)(bits >> 32);
                }
            }
        }
        __syncwarp();  // K (in D) is reused for the buckets below
    }
#pragma unroll
    for (int f = 0; f < kSub; ++f) B[f * 32 + lane] = 0u;

    const size_t step = a.pitch * sizeof(OUT);
    char* ptr = reinterpret_cast<char*>(a.out) + ((size_t)f0 * a.pitch + (size_t)p0) * sizeof(OUT);
    const bool vec_ok = a.vec_ok && np == P;

    auto bin_of = [&](int sub, uint32_t& off, uint32_t& n) {
        off = __shfl_sync(kFull, sub < 32 ? off_lo : off_hi, sub & 31);
        n = __shfl_sync(kFull, sub < 32 ? cnt_lo : cnt_hi, sub & 31);
    };
    // changes of the current sub-tile prefetched into registers (R per lane),
    // loaded while the previous sub-tile's frames are being stored
    constexpr int R = sizeof(OUT) == 8 ? 2 : 4;
    uint32_t off, n;
    bin_of(sub0, off, n);
    Change<OUT> pre[R];
#pragma unroll
    for (int i = 0; i < R; ++i)
        if ((uint32_t)(lane + 32 * i) < n) pre[i] = st[off + lane + 32 * i];

    auto bucket = [&](const Change<OUT>& ch, int sub) {
        uint32_t fo, pix;
        if constexpr (sizeof(OUT) == 1) {
            fo = ch.w >> 17;
            pix = (ch.w >> 8) & 0x1ffu;
        } else {
            fo = ch.key >> 16;
            pix = ch.key & 0xffffu;
        }
        const int fs = (int)fo - sub * kSub;  // frame within the sub-tile
        SPK_CHECK((fs >= 0) & (fs < kSub) & (pix < (uint32_t)GP));
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

    int tma_pending = 0;  // TMA: tile stores issued (the buffer alternates)
    for (int sub = sub0; sub < sub1; ++sub) {
        const int t0 = fc + sub * kSub;
        if (t0 >= f1) break;
        if constexpr (TMA) {
            D = D0 + (tma_pending % SPK_TMA_BUFS) * DBYTES;
            if (tma_pending >= SPK_TMA_BUFS && lane == 0) {  // the store that last read this buffer is done reading
                if (SPK_TMA_BUFS == 1)
                    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
                else
                    asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
            }
            __syncwarp();
        }
        // ---- phase A: this sub-tile's changes -> owners' buckets
        uint32_t noff = 0, nn = 0;
        if (sub + 1 < sub1) bin_of(sub + 1, noff, nn);
#pragma unroll
        for (int i = 0; i < R; ++i)
            if ((uint32_t)(lane + 32 * i) < n) bucket(pre[i], sub);
        for (uint32_t k = lane + 32 * R; k < n; k += 32) bucket(st[off + k], sub);
        __syncwarp();
        off = noff;
        n = nn;
#pragma unroll
        for (int i = 0; i < R; ++i)
            if ((uint32_t)(lane + 32 * i) < n) pre[i] = st[off + lane + 32 * i];
        // ---- phase B: frames in order, one store per frame
        const int nf = min(kSub, f1 - t0);
#pragma unroll 4
        for (int fs = 0; fs < nf; ++fs) {
            const uint32_t bm = B[fs * 32 + lane];
            if constexpr (sizeof(OUT) == 1) {  // branch-free: a clear mask keeps every byte
                B[fs * 32 + lane] = 0u;
                const uint4 dv = *reinterpret_cast<const uint4*>(D + (fs * 32 + lane) * G::DE);
                // word w's pending bits sit at 8b + w: shifted to the byte
                // sign bits, one PRMT replicates each into its byte
                const uint32_t m0 = sign_bytes(bm << 7), m1 = sign_bytes(bm << 6);
                const uint32_t m2 = sign_bytes(bm << 5), m3 = sign_bytes(bm << 4);
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
            if constexpr (TMA) {  // the merged frame back into its cell (row fs of the tile)
                *reinterpret_cast<uint4*>(D + (fs * 32 + lane) * G::DE) =
                    make_uint4(words[0], words[1], words[2], words[3]);
            } else if (vec_ok) {
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
        if constexpr (TMA) {
            // the sub-tile (kSub rows x 512 B) as one tensor store; rows past
            // the stream end and columns past the last pixel are clipped
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
            if (lane == 0) {
                const uint32_t sa = (uint32_t)__cvta_generic_to_shared(D);
                asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];"
                             ::"l"(&tmap), "r"(g * (GP / 4)), "r"(t0), "r"(sa) : "memory");
                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            }
            ++tma_pending;
        }
        __syncwarp();  // bucket clears done before the next phase A refills them
    }
    if constexpr (TMA) {
        if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        __syncwarp();
    }
}

template __global__ void k_expand<uint8_t, Geo<uint8_t>::WARPS, false>(ExpArgs, const __grid_constant__ CUtensorMap);
template __global__ void k_expand<uint8_t, 2 * Geo<uint8_t>::WARPS, false>(ExpArgs, const __grid_constant__ CUtensorMap);
template __global__ void k_expand<uint8_t, Geo<uint8_t>::WARPS, true>(ExpArgs, const __grid_constant__ CUtensorMap);
template __global__ void k_expand<uint8_t, 2 * Geo<uint8_t>::WARPS, true>(ExpArgs, const __grid_constant__ CUtensorMap);
template __global__ void k_expand<float, Geo<float>::WARPS, false>(ExpArgs, const __grid_constant__ CUtensorMap);
template __global__ void k_expand<double, Geo<double>::WARPS, false>(ExpArgs, const __grid_constant__ CUtensorMap);

// ----------------------------------------------------------------- scan --
// Exclusive prefix sum of uint32 counts (three launches: block scans, scan
// of block sums, add-back).
template <typename T>
__global__ void __launch_bounds__(kScanBlock) k_scan_blocks(const uint32_t* in, T* out, T* sums,
                                                            int64_t n) {
    __shared__ T ws[kScanBlock / 32];
    const int64_t i = (int64_t)blockIdx.x * kScanBlock + threadIdx.x;
    const T x = i < n ? (T)in[i] : T(0);
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    T incl = x;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const T y = __shfl_up_sync(kFull, incl, d);
        if (lane >= d) incl += y;
    }
    if (lane == 31) ws[w] = incl;
    __syncthreads();
    if (w == 0) {
        const T s = ws[lane];
        T si = s;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const T y = __shfl_up_sync(kFull, si, d);
            if (lane >= d) si += y;
        }
        ws[lane] = si - s;
        if (lane == 31) sums[blockIdx.x] = si;
    }
    __syncthreads();
    if (i < n) out[i] = incl - x + ws[w];
}

template <typename T>
__global__ void __launch_bounds__(kScanBlock) k_scan_sums(T* sums, int64_t nb) {
    __shared__ T ws[kScanBlock / 32];
    __shared__ T carry;
    if (threadIdx.x == 0) carry = T(0);
    __syncthreads();
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int64_t base = 0; base < nb; base += kScanBlock) {
        const int64_t i = base + threadIdx.x;
        const T x = i < nb ? sums[i] : T(0);
        T incl = x;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const T y = __shfl_up_sync(kFull, incl, d);
            if (lane >= d) incl += y;
        }
        if (lane == 31) ws[w] = incl;
        __syncthreads();
        if (w == 0) {
            const T s = ws[lane];
            T si = s;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const T y = __shfl_up_sync(kFull, si, d);
                if (lane >= d) si += y;
            }
            ws[lane] = si - s;
        }
        __syncthreads();
        const T c0 = carry;
        if (i < nb) sums[i] = c0 + incl - x + ws[w];
        __syncthreads();
        if (threadIdx.x == kScanBlock - 1) carry = c0 + incl + ws[w];
        __syncthreads();
    }
}

template <typename T>
__global__ void __launch_bounds__(kScanBlock) k_scan_add(T* out, const T* sums, int64_t n, T* out2) {
    const int64_t i = (int64_t)blockIdx.x * kScanBlock + threadIdx.x;
    if (i < n) {
        const T v = out[i] + sums[blockIdx.x];
        out[i] = v;
        if (out2) out2[i] = v;  // a second copy (K2c's running slot cursors)
    }
}

template __global__ void k_scan_blocks<uint32_t>(const uint32_t*, uint32_t*, uint32_t*, int64_t);
template __global__ void k_scan_sums<uint32_t>(uint32_t*, int64_t);
template __global__ void k_scan_add<uint32_t>(uint32_t*, const uint32_t*, int64_t, uint32_t*);
template __global__ void k_scan_blocks<unsigned long long>(const uint32_t*, unsigned long long*,
                                                           unsigned long long*, int64_t);
template __global__ void k_scan_sums<unsigned long long>(unsigned long long*, int64_t);
template __global__ void k_scan_add<unsigned long long>(unsigned long long*, const unsigned long long*,
                                                        int64_t, unsigned long long*);

}  // namespace spk
