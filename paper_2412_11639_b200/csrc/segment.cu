// segment.cu -- K2: FSR / SSR segmentation of every pixel (sm_100a).
//
// Replaces the per-pixel scans of reconstruct_row (proj/src/reconstruct.cpp:
// 358-390) and the column->row gather of reconstruct_into (416-419).
//
// Mapping: one thread per pixel, one warp per 32-bit plane word (32
// consecutive pixels), 8 warps per block (one 32-byte sector of every plane
// row, shared through L2 under a drift throttle).  For every group of 32
// frames lane i loads the warp's word from plane 32g + (31 - i); a 5-stage
// shuffle transpose (Transpose32) turns the 32x32 bit block into one 32-frame
// word per pixel with the earliest frame in bit 31, kept in a per-warp ring
// in shared memory.  FSR: every lane walks its own pixel kWin (3) words per
// iteration (fsr_batch: bit-parallel acceptance up to the next event, one
// exact automaton step for the event); SSR: bulk (ssr_flags) or word-lockstep
// spike mode per warp.  Plane loads run one batch (kBatch groups = 256
// frames) ahead of the scan.
//
// Output per pixel p: runs[p*cap + k] = {start frame, intervals} (k < cap),
// counts[p] (may exceed cap: overflow) and last[p] (last spike, -1 if none).
// K2b/K2c (expand.cu) turn them into values and a frame-sorted change stream
// for K3; overflowed pixels are rewritten exactly by k_fixup after K3.
#include <type_traits>

#ifndef SPK_SSR_REPS
#define SPK_SSR_REPS 2  // SSR bulk mode: words (or events) per pass of its loop head (with the smaller spike loop: C3 SSR K2 12.12 ms at 2, 12.28 at 3, 12.45 at 1, 13.0 at 4)
#endif

#ifndef SPK_SSR_SPIKE_UNROLL
#define SPK_SSR_SPIKE_UNROLL 2  // (8: the SSR kernel is 98 KB of code; 2: C3 SSR K2 13.45 -> 12.27 ms, fewer instruction-cache stalls)
#endif
#ifndef SPK_SSR_SLEEP_NS
#define SPK_SSR_SLEEP_NS 256
#endif
#ifndef SPK_SSR_SLOTS_SMEM
#define SPK_SSR_SLOTS_SMEM 1  // SSR spike loop: parity slots in shared memory (Scan::step_mem)
#endif

#include "spk_fsm.cuh"
#include "spk_kernels.cuh"

namespace spk {

constexpr int kSpikeUnroll = SPK_SSR_SPIKE_UNROLL;  // SSR spike loop: words of a batch unrolled

namespace {

// predicated 8-byte store of a closed run: no branch in the scan loop
__device__ __forceinline__ void st_run_if(bool pred, spk_run_t* addr, int rs, int cnt) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %0, 0;\n\t"
        "@p st.global.v2.u32 [%1], {%2, %3};\n\t}" ::"r"((uint32_t)pred),
        "l"(addr), "r"(rs), "r"(cnt)
        : "memory");
}

}  // namespace

template <int METHOD, int WARPS>
__global__ void __launch_bounds__(WARPS * 32) k_segment(SegArgs a) {
    // transposed words of each warp: ring of kRing 32-frame words per lane
    extern __shared__ uint32_t seg_smem[];
    __shared__ int prog[WARPS];  // per warp: earliest group still to be read
    const int lane = threadIdx.x & 31;
    const int wid = threadIdx.x >> 5;
    const int64_t word = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t p = word * 32 + lane;
    // re-scan mode (a.flags): only flagged pixels are scanned and stored
    const bool valid = p < a.npix && (a.flags == nullptr || a.flags[p] != 0);
    const bool busy = __any_sync(kFull, valid);
    if (lane == 0) prog[wid] = busy ? 0 : 0x7fffffff;  // idle warps never hold others back
    __syncthreads();
    if (!busy) return;  // warp-uniform
    uint32_t(*rg)[32] = reinterpret_cast<uint32_t(*)[32]>(seg_smem + (size_t)wid * kRing * 32);
    volatile int* vprog = prog;
    // stay within the drift bound of the block's slowest warp (L2 sector sharing)
    auto throttle = [&](int front) {
        for (;;) {
            int mn = 0x7fffffff;
#pragma unroll
            for (int i = 0; i < WARPS; ++i) mn = min(mn, vprog[i]);
            if (front - mn <= (METHOD == kFSR ? kDriftFsr : kDriftSsr)) break;
            __nanosleep(METHOD == kFSR ? 256 : SPK_SSR_SLEEP_NS);
        }
    };
    const size_t pitch = a.pitch;
    // time shard of this block (a.shard_frames > 0: blockIdx.y = shard)
    const int sf0 = a.shard_frames > 0 ? (int)blockIdx.y * a.shard_frames : 0;
    const int frames = a.shard_frames > 0 ? min(a.shard_frames, a.frames - sf0) : a.frames;
    const int64_t sh = blockIdx.y;  // 0 unless sharded
    const int ngroups = (frames + 31) >> 5;
    // lane i loads frame 32g + (31 - i): after the transpose bit 31 is the
    // group's first frame, so spikes come out in time order with clz
    const char* col = reinterpret_cast<const char*>(a.planes) + (size_t)sf0 * pitch + word * 4;
    const int rev = 31 - lane;
    const int64_t pstride = a.run_pix_stride > 0 ? a.run_pix_stride : a.cap;
    const int64_t sstride = a.run_shard_stride >= 0 ? a.run_shard_stride : a.npix * a.cap;
    spk_run_t* rp = a.runs + sh * sstride + (valid ? p * pstride : 0) + a.run_base;
    const int fbase = a.abs_frames ? sf0 : 0;  // stored run starts: shard or stream frames
    const int capm1 = a.cap - 1;

    Scan<METHOD> sc;
    sc.init();
    if (a.state_in != nullptr && valid) {  // time shard: continue from a carried state
        sc.restore(a.state_in, a.npix, p);
        sc.nrun = 0;
    }
    int nrun = 0;
    // runs beyond the capacity are counted (overflow -> k_fixup) but not stored.
    // The stored pair lives in its own registers (written only on an emit), so
    // the automaton's next update does not wait for the store to read them.
    int o_rs = 0, o_cnt = 0;
    // `wp` = rp + nrun while nrun < cap (a running store pointer: no 64-bit
    // address arithmetic per emit); past the capacity nothing is stored
    spk_run_t* wp = rp;
    auto emit = [&](bool e, int rs, int cnt) {
        SPK_CHECK(!e | (rs >= -(1 << 29)));  // a run start is a frame (time shards: may precede 0)
        o_rs = e ? rs + fbase : o_rs;
        o_cnt = e ? cnt : o_cnt;
        st_run_if(e & (nrun <= capm1), wp, o_rs, o_cnt);
        wp += (int)e;
        nrun += (int)e;
    };

    // The same for the SSR spike loop (integer-pipe bound): the store reads
    // the step's own copies of (rs, cnt) -- no selects into o_rs / o_cnt --
    // and the frame offset is added on the FMA pipe.
    auto emit_now = [&](bool e, int rs, int cnt) {
        st_run_if(e & (nrun <= capm1), wp, fadd(rs, fbase), cnt);
        wp += (int)e;
        nrun += (int)e;
    };

    // Producer (warp-uniform): kBatch groups per refill, loads one batch ahead.
    // The loads walk a running pointer (one 64-bit add per group instead of a
    // 64-bit multiply-add per load); a batch's ring slots never wrap
    // (kBatch divides kRing and `produced` is a multiple of kBatch).
    static_assert(kRing % kBatch == 0, "a batch must not wrap the ring");
    const size_t gstride = (size_t)32 * pitch;  // bytes between a lane's rows of consecutive groups
    const char* lp = col + (size_t)rev * pitch;  // this lane's row of the next group to load
    int lf = rev;                                // its frame
    uint32_t nxt[kBatch];
    int produced = 0;  // groups transposed into the ring
    // (SSR keeps per-load addressing: its spike loop schedules better with
    // the pointer state out of the registers -- SSR K2 5.94 vs 6.54 ms)
    auto load_batch = [&]() {
        const bool full = lf + 32 * (kBatch - 1) < frames;  // warp-uniform (lf - rev is)
#pragma unroll
        for (int j = 0; j < kBatch; ++j) {
            if constexpr (METHOD == kFSR) {
                // (a batch wholly inside the stream needs no per-row check)
                nxt[j] = full || lf < frames ? __ldg(reinterpret_cast<const uint32_t*>(lp)) : 0u;
                lp += gstride;
                lf += 32;
            } else {
                const int f = (produced + j) * 32 + rev;
                nxt[j] = f < frames ? __ldg(reinterpret_cast<const uint32_t*>(col + (size_t)f * pitch)) : 0u;
            }
        }
    };
    load_batch();
    Transpose32 tp;
    tp.init(lane);
    // `lowest`: this warp's earliest group still to be read (published for the
    // other warps of the block), then the next batch's loads wait for them
    auto produce = [&](int lowest) {
        if (lane == 0) vprog[wid] = lowest;
        uint32_t* slot = &rg[produced & (kRing - 1)][lane];
#pragma unroll
        for (int j = 0; j < kBatch; ++j) {
            const uint32_t t = tp(nxt[j]);  // every lane shuffles
            slot[32 * j] = valid ? t : 0u;
        }
        produced += kBatch;
        // the drift bound is checked every other batch (the block's warps
        // stay within the bound + kBatch groups)
        if ((produced & kBatch) == 0) throttle(produced);
        load_batch();
        __syncwarp();
    };

    if constexpr (METHOD == kSSR) {
        // SSR, two consumers over the same ring and automaton:
        //  * bulk: every lane walks its own pixel word by word at its own pace,
        //    one bit-parallel two-level test (ssr_flags: acceptance up to the
        //    next event) and at most one exact step per iteration -- fast when
        //    events are sparse (static scenes: whole words per iteration);
        //  * spike: the warp in lockstep over words, one exact step per spike
        //    -- cheaper when events come every few spikes (moving scenes).
        // The first kSsrProbe words run in bulk mode while counting events;
        // the warp then keeps the mode that fits its event rate.
        int wi = -1;  // word of this lane (its ring slot may be reused)
        uint32_t So = 0u, S = 0u;
        int prevlast = kNoSpike;
        int events = 0, nspk = 0;  // this lane's exact steps / spikes so far (the mode choice below)
        auto bulk = [&](int limit) {
            for (;;) {
                const bool more = wi + 1 < limit;
                if (__any_sync(kFull, (S == 0u) & more & (wi + 1 >= produced))) {
                    const int lowest = (int)__reduce_min_sync(kFull, (unsigned)(more ? wi + 1 : 0x7fffffff));
                    if (produced < ngroups && produced + kBatch <= lowest + kRing) produce(lowest);
                }
                if (!__any_sync(kFull, (S != 0u) | more)) break;
                // SPK_SSR_REPS words (or events) per pass of the loop head
#pragma unroll
                for (int rep = 0; rep < SPK_SSR_REPS; ++rep) {
                    if ((S == 0u) & (wi + 1 < produced) & (wi + 1 < limit)) {
                        ++wi;
                        So = S = rg[wi & (kRing - 1)][lane];
                        prevlast = sc.last;
                        nspk += __popc(So);
                    }
                    if (S) {
                        const int base = wi * 32;
                        uint32_t Cs, Cl;
                        const uint32_t V = ssr_flags(sc, So, S, base, prevlast, Cs, Cl);
                        const uint32_t A = S & ~bit_shr_clamp(0xffffffffu, 0u, V ? (uint32_t)__clz(V) : 32u);
                        ssr_accept(sc, A, Cs, Cl, base);
                        S &= ~A;
                        if (S) {
                            const int c = __clz(S);
                            S ^= 0x80000000u >> c;
                            int rs, cnt;
                            const bool e = sc.step(base + c, rs, cnt);
                            emit(e, rs, cnt);
                            ++events;
                        }
                    }
                }
            }
        };
        // (short streams: an eighth of the stream, at least 16 words -- a 64-word
        // probe is half of a 4,000-frame stream spent in what may be the slower mode)
#ifndef SPK_SSR_PROBE_DIV
#define SPK_SSR_PROBE_DIV 8
#endif
        const int probe = min(ngroups, min(kSsrProbe, max(16, ngroups / SPK_SSR_PROBE_DIV)));
        bulk(probe);
        // Mode for the rest of the stream, from the probe's busiest lanes:
        // bulk mode pays a pass (~kSsrBulkCost instructions) per word and per
        // event of its busiest lane, the spike loop a step (~kSsrStepCost)
        // per spike of the busiest lane plus a per-word overhead.  Bright
        // pixels with few events stay in bulk mode, dim or eventful ones
        // take the spike loop.
        const int emax = (int)__reduce_max_sync(kFull, (unsigned)events);
        const int smax = (int)__reduce_max_sync(kFull, (unsigned)nspk);
        if (kSsrBulkCost * (probe + emax) <= kSsrStepCost * smax + kSsrWordCost * probe) {
            bulk(ngroups);
        } else {  // lanes all stand at word `probe`
            // the frame fields of the state matter only for a saved state;
            // without one the parity slots move to shared memory (step_mem:
            // [parity][lane] 16-byte records behind the block's rings)
            char* const slots = reinterpret_cast<char*>(seg_smem + (size_t)WARPS * kRing * 32) +
                                (size_t)wid * kSsrSlotBytes + lane * 16;
            auto slot = [&](int k) -> int4& { return *reinterpret_cast<int4*>(slots + (k << 9)); };
            auto run_spikes = [&](auto frames) {
                constexpr bool FR = decltype(frames)::value;
                if constexpr (!FR && SPK_SSR_SLOTS_SMEM) sc.store_slots(slot);
                auto spikes = [&](int g) {
                    uint32_t w = rg[g & (kRing - 1)][lane];
                    // the word is shifted past each spike (one funnel shift on
                    // the integer pipe; the frame bookkeeping on the FMA pipe)
                    int pos = g * 32;  // frame of bit 31 of w
                    while (w) {
                        const int c = __clz(w);
                        const int n = fadd(pos, c);
                        const int c1 = fadd(c, 1);
                        w = bit_shl_clamp(w, (uint32_t)c1);
                        pos = fadd(pos, c1);
                        int rs, cnt;
                        bool e;
                        if constexpr (!FR && SPK_SSR_SLOTS_SMEM) {
                            e = sc.step_mem(n, slot, rs, cnt);
                            emit_now(e, rs, cnt);
                        } else {
                            e = sc.template step<FR>(n, rs, cnt);
                            emit(e, rs, cnt);
                        }
                    }
                };
                int g = probe;
                for (; g < produced && g < ngroups; ++g) spikes(g);  // words already in the ring
                for (int g0 = g; g0 < ngroups; g0 += kBatch) {
                    produce(g0);
#pragma unroll (kSpikeUnroll)
                    for (int j = 0; j < kBatch; ++j)
                        if (g0 + j < ngroups) spikes(g0 + j);
                }
            };
            if (a.state_out != nullptr)
                run_spikes(std::true_type{});
            else
                run_spikes(std::false_type{});
        }
    } else {
    // FSR consumers: every lane walks its own pixel through the words at its
    // own pace -- a window of kWin words per iteration, stopping at the first
    // event (fsr_batch) -- so a lane with many breaks does not hold the others
    // back word by word; the ring bounds how far lanes may drift apart.
    // After an iteration in which no lane met an event, the warp tries kQuiet
    // words at once (fsr_quiet: the test alone, no selection across words);
    // lanes whose window holds an event take the event window in the same
    // iteration.  Moving scenes rarely have such an iteration, static scenes
    // and long quiet stretches almost always.
    static_assert(kQuiet + kBatch <= kRing, "a quiet window must fit the ring beside a batch");
    // window of kWin words per iteration (fsr_batch): 3 measured best on
    // moving scenes (C2 K2 0.843 ms vs 0.876 at 4, 0.869 at 2), within 2% of
    // 4 on static and long streams
    constexpr int kWin = SPK_WIN;
    int wi = 0;    // first word of this lane's window
    int cpos = 0;  // frames of word wi already consumed
    bool quiet = false;  // warp-uniform: the last iteration had no event
    // Groups past the end are produced as zero words, so a window never
    // needs a bounds check.
    for (;;) {
        const bool more = wi < ngroups;
        const bool ready = wi + kWin <= produced;
        // refill only when a lane is starved (or, when quiet, short of a quiet
        // window), and only into slots no lane can still read (lowest = the
        // earliest window start)
        if (__any_sync(kFull, more & (quiet ? wi + kQuiet > produced : !ready))) {
            const int lowest = (int)__reduce_min_sync(kFull, (unsigned)(more ? wi : 0x7fffffff));
            if (produced < ngroups + kQuiet - 1 && produced + kBatch <= lowest + kRing) produce(lowest);
        }
        if (!__any_sync(kFull, more)) break;
        bool tookq = false;
        if (quiet && __all_sync(kFull, !more | (wi + kQuiet <= produced))) {
            if (more) {
                tookq = fsr_quiet<kQuiet>(sc, [&](int k) { return rg[(wi + k) & (kRing - 1)][lane]; },
                                          wi * 32, cpos);
                wi += tookq ? kQuiet : 0;
            }
        }
        bool ev = false;
        if (more & !tookq & (wi + kWin <= produced)) {
            const int k = fsr_batch<kWin>(sc, [&](int j) { return rg[(wi + j) & (kRing - 1)][lane]; },
                                         wi * 32, cpos, emit);
            ev = k < kWin;
            wi += k;
        }
        quiet = !__any_sync(kFull, ev);
    }
    }
    if (lane == 0) vprog[wid] = 0x7fffffff;  // done: never hold the others back
    if (valid) {
        if (a.state_out != nullptr) sc.save(a.state_out + sh * Scan<METHOD>::kFields * a.npix, a.npix, p);
        int rs, cnt;
        const bool e = sc.tail(rs, cnt);
        emit(e, rs, cnt);
        a.counts[sh * a.npix + p] = (uint32_t)nrun;
        a.last[sh * a.npix + p] = sc.last == kNoSpike ? -1 : sc.last + fbase;
        if (a.seg_out != nullptr) {  // re-scan: the whole list is segment 0
            uint32_t* sg = a.seg_out + p * 2 * a.nseg;
            const uint32_t nk = (uint32_t)min(nrun, a.cap);
            for (int r = 0; r < a.nseg; ++r) {  // [0, n), then empty segments at n
                sg[2 * r] = r == 0 ? 0u : nk;
                sg[2 * r + 1] = nk;
            }
        }
    }
}

template __global__ void k_segment<kFSR, kSegWarps>(SegArgs);
template __global__ void k_segment<kSSR, kSegWarps>(SegArgs);
template __global__ void k_segment<kFSR, kSegWarpsWide>(SegArgs);

// ---------------------------------------------------------------- fixup ----
// Pixels whose run list overflowed `cap`: rescan the pixel and write its
// frames directly (one byte/element per frame, column order).  Slow, exact,
// and only taken for pathological (e.g. pure-noise) pixels.
namespace {

template <typename OUT>
struct DirectEmitter {
    OUT* out;  // out + p
    size_t pitch;
    OUT carry;
    __device__ void fill(int a, int b, OUT v) {
        for (int n = a; n < b; ++n) out[(size_t)n * pitch] = v;
    }
    __device__ void run(int rs, int cnt, int end, int) {
        carry = OutVal<OUT>::run((uint32_t)cnt, (uint32_t)(end - rs));
        fill(rs, end, carry);
    }
    __device__ void done(int first, int last, int nrun, int frames) {
        if (nrun == 0) {
            fill(0, frames, OUT(0));
        } else {
            fill(0, first, OUT(0));
            fill(last, frames, carry);
        }
    }
};

}  // namespace

template <int METHOD, typename OUT>
__global__ void __launch_bounds__(128) k_fixup(SegArgs a, OUT* out, size_t out_pitch) {
    const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= a.npix) return;
    if (a.counts[p] <= (uint32_t)a.cap) return;
    Fsm<METHOD> fsm;
    fsm.init();
    DirectEmitter<OUT> em{out + p, out_pitch, OUT(0)};
    const uint8_t* col = reinterpret_cast<const uint8_t*>(a.planes) + (p >> 3);
    const int bit = (int)(p & 7);
    for (int n = 0; n < a.frames; ++n)
        if ((col[(size_t)n * a.pitch] >> bit) & 1) fsm.spike(n, em);
    fsm.finish(a.frames, em);
}

template __global__ void k_fixup<kFSR, uint8_t>(SegArgs, uint8_t*, size_t);
template __global__ void k_fixup<kSSR, uint8_t>(SegArgs, uint8_t*, size_t);
template __global__ void k_fixup<kFSR, float>(SegArgs, float*, size_t);
template __global__ void k_fixup<kSSR, float>(SegArgs, float*, size_t);
template __global__ void k_fixup<kFSR, double>(SegArgs, double*, size_t);
template __global__ void k_fixup<kSSR, double>(SegArgs, double*, size_t);

}  // namespace spk
