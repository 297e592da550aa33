// spk_fsm.cuh -- per-pixel streaming FSR / SSR stability state machine.
//
// One instance per pixel, fed the pixel's spike frames in increasing order.
// It reproduces the reference's batch segmentation exactly:
//   FSR  = fsr_runs_into            (proj/src/reconstruct.cpp:40-53)
//   SSR  = fsr_runs_into followed by ssr_refine_into (reconstruct.cpp:64-99)
// and emits every closed run as (start frame, interval count, end frame) to an
// Emitter.  Runs tile [first spike, last spike) with no gap (a run closed at a
// violating interval ends at that interval's opening spike, which starts the
// next run -- reconstruct.cpp:366-371).
//
// The zero-order rule (PairScanner, reconstruct.cpp:17-36) is kept as
// (lo, hw): accepted values are [lo, lo + hw] with hw in {0, 1}; "empty" is
// lo = kNoPair.  The common case -- the interval is already in the pair --
// is a single unsigned compare `(t - lo) <= hw`; everything else (first
// spikes, pair completion, violations) goes to the general slow path.
//
// SSR keeps one second-level state per value of the current FSR pair, indexed
// by value (slot A = lo, slot B = lo + 1) instead of first-occurrence order as
// in ssr_refine_into's Level2[2]; the two are the same states relabelled, and
// the relabelling is applied when the pair completes downwards (lo -> lo-1).
// A second-level violation closes the sub-run, resets only the second-level
// states (the FSR pair continues), and the violating interval reopens its
// slot -- exactly ssr_refine_into's restart at `broke` (reconstruct.cpp:95-96).
#pragma once

#include "spk_common.cuh"

// host+device so the state machine can also be unit-tested on the CPU
// (tests/native/fsm_host.cu); the product only runs it on the GPU.
#define SPK_HD __host__ __device__ __forceinline__

namespace spk {

// K2 is bound by the integer ALU pipe (ncu: 78% FSR, 92% SSR) while the FMA
// pipe idles (~12%): additions in the per-spike automaton are issued as
// IMAD with a multiplier the compiler cannot see (a constant-bank 1), which
// runs on the FMA pipe instead of IADD3 on the ALU pipe.
static __constant__ int kFmaOne = 1;
static __constant__ int kFmaNeg = -1;
SPK_HD int fadd(int a, int b) {  // a + b
#ifdef __CUDA_ARCH__
    int r;
    asm("mad.lo.s32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(kFmaOne), "r"(b));
    return r;
#else
    return a + b;
#endif
}
// the same with the multiplier in a register of the caller (Scan keeps 1 and
// -1 loaded once: inside the scan loop the constant-bank load sat on the
// step's critical path)
SPK_HD int fmad(int a, int m, int b) {  // a * m + b, m = 1 or -1
#ifdef __CUDA_ARCH__
    int r;
    asm("mad.lo.s32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(m), "r"(b));
    return r;
#else
    return a * m + b;
#endif
}
SPK_HD int fsub(int a, int b) {  // a - b
#ifdef __CUDA_ARCH__
    int r;
    asm("mad.lo.s32 %0, %1, %2, %3;" : "=r"(r) : "r"(b), "r"(kFmaNeg), "r"(a));
    return r;
#else
    return a - b;
#endif
}

// k ? a : b for an integer k in {0, 1}, as b + k * (a - b): two IMADs on the
// FMA pipe instead of a SEL on the (saturated) integer ALU pipe.
SPK_HD int fsel(int k, int a, int b) {
#if defined(__CUDA_ARCH__) && !defined(SPK_FSEL_SEL)
    int r;
    asm("mad.lo.s32 %0, %1, %2, %3;" : "=r"(r) : "r"(k), "r"(fsub(a, b)), "r"(b));
    return r;
#else
    return k ? a : b;
#endif
}

enum { kFSR = 0, kSSR = 1, kTFI = 2, kTFP = 3 };

template <int METHOD>
struct Fsm {
    int last;   // last spike frame (kNoSpike before the first spike)
    int first;  // first spike frame
    int rs;     // start frame of the open (sub-)run
    int cnt;    // intervals in the open (sub-)run
    int lo;     // FSR pair: accepted [lo, lo + hw]
    uint32_t hw;
    int nrun;   // runs emitted so far
    // SSR second level (unused for FSR; the compiler drops them)
    int ii;           // S1 index of the next interval
    int lA, lB;       // S1 index of the value's last occurrence in the sub-run
    int gAlo, gBlo;   // pair rule over that value's occurrence gaps
    uint32_t gAhw, gBhw;

    SPK_HD void init() {
        last = kNoSpike;
        first = 0;
        rs = 0;
        cnt = 0;
        lo = kNoPair;
        hw = 0;
        nrun = 0;
        ii = 0;
        lA = lB = kNoIdx;
        gAlo = gBlo = kNoPair;
        gAhw = gBhw = 0;
    }

    SPK_HD void ssr_reset_to(int k) {
        // fresh second-level states; the current interval (value lo + k) is
        // the first occurrence of its value in the new sub-run
        lA = k == 0 ? ii : kNoIdx;
        lB = k == 1 ? ii : kNoIdx;
        gAlo = gBlo = kNoPair;
        gAhw = gBhw = 0;
    }

    // pair rule on one second-level slot; returns false on a violation
    SPK_HD static bool gap_take(int& l, int& glo, uint32_t& ghw, int idx) {
        if (l == kNoIdx) {
            l = idx;
            return true;
        }
        const int gap = idx - l;
        if (glo == kNoPair) {
            glo = gap;
            ghw = 0;
            l = idx;
            return true;
        }
        const int gd = gap - glo;
        if (gd == 0 || (ghw && gd == 1)) {
            l = idx;
            return true;
        }
        if (!ghw && (gd == 1 || gd == -1)) {
            if (gd == -1) glo = gap;
            ghw = 1;
            l = idx;
            return true;
        }
        return false;
    }

    template <class E>
    SPK_HD void slow(int n, E& em) {
        if (last == kNoSpike) {  // first spike: lead [0, n) stays 0
            first = rs = last = n;
            return;
        }
        const int t = n - last;
        if (lo == kNoPair) {  // first interval fixes the pair's first value
            lo = t;
            hw = 0;
            cnt = 1;
            if (METHOD == kSSR) {
                ssr_reset_to(0);
                ++ii;
            }
            last = n;
            return;
        }
        const int d = t - lo;
        bool ok = d == 0 || (hw && d == 1);
        if (!ok && !hw && (d == 1 || d == -1)) {  // pair completes
            hw = 1;
            if (d == -1) {
                lo = t;
                if (METHOD == kSSR) {  // old value lo is now slot B
                    int tl = lA, tg = gAlo;
                    uint32_t th = gAhw;
                    lA = lB; gAlo = gBlo; gAhw = gBhw;
                    lB = tl; gBlo = tg; gBhw = th;
                }
            }
            ok = true;
        }
        if (!ok) {  // first-order violation: close the run at `last`
            em.run(rs, cnt, last, nrun);
            ++nrun;
            rs = last;
            lo = t;
            hw = 0;
            cnt = 1;
            if (METHOD == kSSR) {
                ssr_reset_to(0);
                ++ii;
            }
            last = n;
            return;
        }
        if (METHOD == kSSR) {
            const int k = t - lo;
            const bool gok = k == 0 ? gap_take(lA, gAlo, gAhw, ii) : gap_take(lB, gBlo, gBhw, ii);
            if (!gok) {  // second-order violation: close the sub-run at `last`
                em.run(rs, cnt, last, nrun);
                ++nrun;
                rs = last;
                cnt = 0;
                ssr_reset_to(k);
            }
            ++ii;
        }
        ++cnt;
        last = n;
    }

    // one spike at frame n (frames strictly increasing)
    template <class E>
    SPK_HD void spike(int n, E& em) {
        const int t = n - last;
        const int d = t - lo;
        if ((uint32_t)d > hw) {
            slow(n, em);
            return;
        }
        if (METHOD == kSSR) {
            const int l = d ? lB : lA;
            const int glo = d ? gBlo : gAlo;
            const uint32_t ghw = d ? gBhw : gAhw;
            if ((uint32_t)((ii - l) - glo) > ghw) {
                slow(n, em);
                return;
            }
            if (d) lB = ii; else lA = ii;
            ++ii;
        }
        ++cnt;
        last = n;
    }

    // end of stream: close the open run; the tail [last, T) carries its value
    template <class E>
    SPK_HD void finish(int frames, E& em) {
        if (lo != kNoPair) {
            em.run(rs, cnt, last, nrun);
            ++nrun;
        }
        em.done(first, last == kNoSpike ? -1 : last, nrun, frames);
    }
};

// ---------------------------------------------------------------------------
// Scan<METHOD>: the same automaton as Fsm, written branch-free for the warp
// scan of K2.  A warp advances all 32 pixels one spike per iteration; any
// data-dependent branch (pair completion, violation, first occurrence...)
// would serialise the lanes that take it, and with runs every few dozen
// spikes some lane takes one in most iterations.  Every case is therefore a
// select, and a closed run is a single predicated 8-byte store of
// (start frame, intervals); its end is the next run's start (or the pixel's
// last spike) and its value is computed later by K2c (expand.cu).
//
// Encodings (frames < 2^29):
//   lo >= kLim          no interval yet (kNoPair initially; after the first
//                        spike lo = t >= 2^29 because last = kNoSpike)
//   SSR slots are indexed by value parity (the pair {lo, lo+1} has one odd
//   and one even value), so a completing pair never relabels a slot; a slot
//   whose last occurrence precedes the sub-run start `sub0` is empty, so a
//   violation resets both slots by moving sub0 only; glo >= kLim = no gap yet.
constexpr int kLim = 1 << 29;

// FSR quiet windows: words accepted at once by fsr_quiet (segment kernel)
#ifndef SPK_QUIET
#define SPK_QUIET 8
#endif
constexpr int kQuiet = SPK_QUIET;
// FSR event windows: words tested per iteration (fsr_batch, segment kernel)
#ifndef SPK_WIN
#define SPK_WIN 3
#endif

template <int METHOD>
struct Scan {
    int last, lo, rs, cnt, nrun;
    uint32_t hw;
    int ii, sub0;         // SSR: S1 index of the next interval, sub-run start
    int l0, l1, g0, g1;   // SSR: per parity slot: last index, gap pair low
    uint32_t h0, h1;      //      gap pair width (0/1)
    int fl0, fl1;         // SSR: frame of each slot's last occurrence
    int sf;               // SSR: frame of the spike closing interval sub0

    SPK_HD void init() {
        last = kNoSpike;
        lo = kNoPair;
        rs = cnt = nrun = 0;
        hw = 0;
        ii = sub0 = 0;
        l0 = l1 = kNoIdx;
        g0 = g1 = kNoPair;
        h0 = h1 = 0;
        fl0 = fl1 = sf = kNoSpike;
    }

    // returns true when the run (rs, cnt) closed before this spike.  Written
    // with bitwise logic only (no && / ||), so the compiler emits selects,
    // not divergent branches.  FRAMES = false skips the frame fields fl0,
    // fl1, sf (read only by the bulk test ssr_flags and saved states): the
    // SSR spike loop uses it when neither follows.
    template <bool FRAMES = true>
    SPK_HD bool step(int n, int& out_rs, int& out_cnt) {
        // One compare for "in the pair or completing it": a pair of width w
        // accepts d in {0, w} and, while w = 0, completes on d = +-1 --
        // together (unsigned)(d + 1 - w) <= 2 - w (the scan is bound by the
        // integer pipe: compares and selects; the additions go to the FMA
        // pipe).  C2 FSR K2 0.771 -> 0.761 ms, C3 2.79 -> 2.73 ms.
        const int t = fsub(n, last);
        const int d = fsub(t, lo);
        const int c1 = fsub(1, (int)hw);
        const bool fbrk = (uint32_t)fadd(d, c1) > (uint32_t)fadd(c1, 1);
        const bool ext = (!fbrk) & ((uint32_t)d > hw);
        bool brk = fbrk;
        bool emit = fbrk & (lo < kLim);
        if (METHOD == kSSR) {
            // parity-slot selects on the FMA pipe (the SSR scan saturates the ALU pipe)
            const int ki = t & 1, kn = ki ^ 1;
            const int l = fsel(ki, l1, l0);
            const int glo = fsel(ki, g1, g0);
            const uint32_t ghw = (uint32_t)fsel(ki, (int)h1, (int)h0);
            const bool stale = l < sub0;
            const int gap = fsub(ii, l);
            const int gd = fsub(gap, glo);
            const bool gnone = glo >= kLim;
            const bool gempty = stale | gnone;
            const bool gin = (!gempty) & ((uint32_t)gd <= ghw);
            const bool gext = (!gempty) & (!gin) & (ghw == 0u) & ((uint32_t)fadd(gd, 1) <= 2u);
            const bool sbrk = (!fbrk) & (!gempty) & (!gin) & (!gext);
            brk = fbrk | sbrk;
            emit = emit | sbrk;
            const bool fresh = stale | brk;
            const int keep = gext ? min(glo, gap) : glo;
            const int nglo = fresh ? kNoPair : (gnone ? gap : keep);
            const uint32_t nghw = (fresh | gnone) ? 0u : (ghw | (uint32_t)gext);
            l0 = fsel(kn, ii, l0);
            l1 = fsel(ki, ii, l1);
            if (FRAMES) {
                fl0 = fsel(kn, n, fl0);
                fl1 = fsel(ki, n, fl1);
            }
            g0 = fsel(kn, nglo, g0);
            g1 = fsel(ki, nglo, g1);
            h0 = (uint32_t)fsel(kn, (int)nghw, (int)h0);
            h1 = (uint32_t)fsel(ki, (int)nghw, (int)h1);
            sub0 = brk ? ii : sub0;
            if (FRAMES) sf = brk ? n : sf;
            ii = fadd(ii, 1);
        }
        out_rs = rs;
        out_cnt = cnt;
        const int lext = ext ? min(lo, t) : lo;
        lo = fbrk ? t : lext;
        hw = fbrk ? 0u : (hw | (uint32_t)ext);
        rs = brk ? last : rs;
        cnt = brk ? 1 : fadd(cnt, 1);
        last = n;
        return emit;
    }

    // SSR: the same step with the two parity slots in memory instead of
    // registers -- slot(k) is the {last index, gap pair low, gap pair width,
    // -} record of parity k (K2's spike loop keeps them in shared memory:
    // one 16-byte load and one 16-byte store replace the 18 FMA-pipe
    // multiply-adds that select and write back l/g/h by parity; the scan is
    // issue-bound).  Only the slot of this interval's parity is read and
    // written, as in step().  The frame fields (fl0, fl1, sf) are not kept:
    // for loops that neither save the state nor return to the bulk test.
    // store_slots / load_slots move the register slots in and out.
    template <class SLOT>
    SPK_HD bool step_mem(int n, SLOT&& slot, int& out_rs, int& out_cnt) {
        static_assert(METHOD == kSSR, "parity slots are SSR state");
        // The loop this runs in is bound by the integer pipe (compares,
        // selects), so the pair tests are folded: a pair of width w accepts
        // d in {0, w} and, while w = 0, completes on d = +-1 -- together
        // (unsigned)(d + 1 - w) <= 2 - w, one compare; the additions go to
        // the FMA pipe.  Same decisions as step() for every 32-bit d.
        const int t = fsub(n, last);
        const int d = fsub(t, lo);
        const int c1 = fsub(1, (int)hw);
        const bool fbrk = (uint32_t)fadd(d, c1) > (uint32_t)fadd(c1, 1);
        const bool ext = (!fbrk) & ((uint32_t)d > hw);
        int4& sl = slot(t & 1);
        const int4 s = sl;
        const int l = s.x, glo = s.y;
        const uint32_t ghw = (uint32_t)s.z;
        const bool stale = l < sub0;
        const int gap = fsub(ii, l);
        const int gd = fsub(gap, glo);
        const bool gnone = glo >= kLim;
        const bool gempty = stale | gnone;
        const int e1 = fsub(1, (int)ghw);
        const bool gbad = (uint32_t)fadd(gd, e1) > (uint32_t)fadd(e1, 1);
        const bool gext = (!gempty) & (!gbad) & ((uint32_t)gd > ghw);
        const bool sbrk = (!fbrk) & (!gempty) & gbad;
        const bool brk = fbrk | sbrk;
        // (no interval yet, lo >= kLim, is a first-order break that emits nothing)
        const bool emit = brk & (lo < kLim);
        const bool fresh = stale | brk;
        const int keep = gext ? min(glo, gap) : glo;
        const int nglo = fresh ? kNoPair : (gnone ? gap : keep);
        // (selects on the predicates themselves: no predicate -> integer moves)
        const uint32_t nghw = (fresh | gnone) ? 0u : (gext ? 1u : ghw);
        sl = make_int4(ii, nglo, (int)nghw, 0);
        sub0 = brk ? ii : sub0;
        ii = fadd(ii, 1);
        out_rs = rs;
        out_cnt = cnt;
        const int lext = ext ? min(lo, t) : lo;
        lo = fbrk ? t : lext;
        hw = fbrk ? 0u : (ext ? 1u : hw);
        rs = brk ? last : rs;
        cnt = brk ? 1 : fadd(cnt, 1);
        last = n;
        return emit;
    }
    template <class SLOT>
    SPK_HD void store_slots(SLOT&& slot) const {
        slot(0) = make_int4(l0, g0, (int)h0, 0);
        slot(1) = make_int4(l1, g1, (int)h1, 0);
    }
    template <class SLOT>
    SPK_HD void load_slots(SLOT&& slot) {
        const int4 a = slot(0), b = slot(1);
        l0 = a.x; g0 = a.y; h0 = (uint32_t)a.z;
        l1 = b.x; g1 = b.y; h1 = (uint32_t)b.z;
    }

    // open run at end of stream (valid when at least one interval was seen)
    SPK_HD bool tail(int& out_rs, int& out_cnt) const {
        out_rs = rs;
        out_cnt = cnt;
        return lo < kLim;
    }

    // ---- state carried across time shards (SoA: field f of pixel p at
    // st[f * stride + p]; frames relative to the shard's first frame)
    static constexpr int kFields = 17;
    SPK_HD void save(int32_t* st, int64_t stride, int64_t p) const {
        const int32_t v[kFields] = {last, lo, rs, cnt, nrun, (int32_t)hw, ii, sub0,
                                    l0, l1, g0, g1, (int32_t)h0, (int32_t)h1, fl0, fl1, sf};
        for (int f = 0; f < kFields; ++f) st[f * stride + p] = v[f];
    }
    SPK_HD void restore(const int32_t* st, int64_t stride, int64_t p) {
        last = st[0 * stride + p];
        lo = st[1 * stride + p];
        rs = st[2 * stride + p];
        cnt = st[3 * stride + p];
        nrun = st[4 * stride + p];
        hw = (uint32_t)st[5 * stride + p];
        ii = st[6 * stride + p];
        sub0 = st[7 * stride + p];
        l0 = st[8 * stride + p];
        l1 = st[9 * stride + p];
        g0 = st[10 * stride + p];
        g1 = st[11 * stride + p];
        h0 = (uint32_t)st[12 * stride + p];
        h1 = (uint32_t)st[13 * stride + p];
        fl0 = st[14 * stride + p];
        fl1 = st[15 * stride + p];
        sf = st[16 * stride + p];
    }

    // Same future: from here on both automata take identical decisions on any
    // spike sequence (only the open run's bookkeeping rs / cnt may differ).
    // Requires an interval in both (rs is the open run's start only then).
    // FSR: the pair and the last spike; SSR also each parity slot's state,
    // relative to the interval index: empty (stale), or (gap base, gap pair).
    SPK_HD bool same_future(const Scan& o) const {
        if ((lo >= kLim) | (o.lo >= kLim)) return false;
        if ((lo != o.lo) | (hw != o.hw) | (last != o.last)) return false;
        if (METHOD == kSSR) {
            auto slot_eq = [&](int la, int ga, uint32_t ha, int lb, int gb, uint32_t hb) {
                const bool sa = la < sub0, sb = lb < o.sub0;
                if (sa != sb) return false;
                if (sa) return true;
                if (ii - la != o.ii - lb) return false;
                const bool na = ga >= kLim, nb = gb >= kLim;
                if (na != nb) return false;
                return na || ((ga == gb) & (ha == hb));
            };
            return slot_eq(l0, g0, h0, o.l0, o.g0, o.h0) && slot_eq(l1, g1, h1, o.l1, o.g1, o.h1);
        }
        return true;
    }
};

// ---- bit helpers usable on host and device (the host build backs the CPU tests)
SPK_HD int bit_clz(uint32_t x) {
#ifdef __CUDA_ARCH__
    return __clz(x);
#else
    return x ? __builtin_clz(x) : 32;
#endif
}
SPK_HD int bit_ffs(uint32_t x) {
#ifdef __CUDA_ARCH__
    return __ffs(x);
#else
    return __builtin_ffs((int)x);
#endif
}
SPK_HD int bit_popc(uint32_t x) {
#ifdef __CUDA_ARCH__
    return __popc(x);
#else
    return __builtin_popcount(x);
#endif
}
// cond ? a : b without a branch
SPK_HD uint32_t bit_sel(bool cond, uint32_t a, uint32_t b) {
    return b ^ ((a ^ b) & (0u - (uint32_t)cond));
}
// cond ? a : b as one SEL (the compiler would branch around a costly a)
SPK_HD int bit_selp(bool cond, int a, int b) {
#ifdef __CUDA_ARCH__
    int r;
    asm("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %1, 0;\n\tselp.b32 %0, %2, %3, q;\n\t}"
        : "=r"(r) : "r"((uint32_t)cond), "r"(a), "r"(b));
    return r;
#else
    return cond ? a : b;
#endif
}
// index of the highest set bit, -1 for 0 (FLO)
SPK_HD int bit_flo(uint32_t x) {
#ifdef __CUDA_ARCH__
    int r;
    asm("bfind.u32 %0, %1;" : "=r"(r) : "r"(x));
    return r;
#else
    return x ? 31 - __builtin_clz(x) : -1;
#endif
}
// x << min(s, 32) (s = 0xffffffff, i.e. -1, also gives 0)
SPK_HD uint32_t bit_shl_clamp(uint32_t x, uint32_t s) {
#ifdef __CUDA_ARCH__
    return __funnelshift_lc(0u, x, s);
#else
    return s >= 32u ? 0u : x << s;
#endif
}
// x >> min(s, 32)
SPK_HD uint32_t bit_shr_clamp(uint32_t x, uint32_t, uint32_t s) {
#ifdef __CUDA_ARCH__
    return __funnelshift_rc(x, 0u, s);
#else
    return s >= 32u ? 0u : x >> s;
#endif
}

// FSR over one 32-frame word (bit 31 = first frame), accepting spikes in
// bulk.  While the open run's pair is [lo, lo+hw], a spike is in the run iff
// its gap to the previous spike lies in the pair.  Bit-parallel over the word,
// the FIRST violating spike is the first one flagged by
//   * no spike exactly lo (or, hw = 1, lo+1) frames earlier:  ~(S>>lo | S>>(lo+1))
//   * a spike exactly 1 frame earlier while lo >= 2:          S & S>>1
//   * for the word's first spike, its gap to `last` directly.
// Proof sketch: a flagged spike is a violation (its real predecessor is at a
// flagged distance).  Conversely let c be the first violation, p its real
// predecessor.  A gap c-p > lo+hw leaves frames c-lo, c-lo-hw empty -> flagged.
// A gap c-p < lo escapes the first test only through a spike k at c-lo or
// c-lo-1 before p; every accepted gap (and the gap that opened the current
// state) is >= lo, so p-k >= lo, forcing c-p = 1 and c-k = lo+1 -- caught by
// the second test.  Everything before the first flagged spike is accepted at
// once (cnt += popc, last = latest accepted); the flagged spike -- a pair
// completion or a break -- goes through the exact per-spike automaton, then
// the bulk test resumes with the updated pair.  A word costs one iteration per
// event instead of one per spike.  FsrWord holds one word; iterate() does one
// bulk test plus at most one event, so a caller can interleave words freely.
struct FsrWord {
    uint32_t So, S;  // spikes of the word / not yet consumed
    uint32_t G1;     // spikes with a spike one frame earlier
    uint32_t fb;     // the word's first spike
    int f, base;     // its offset, the word's first frame

    SPK_HD void load(uint32_t w, int b) {
        So = S = w;
        base = b;
        G1 = So & (So >> 1);
        f = bit_clz(So | 1u);
        fb = So ? (0x80000000u >> f) : 0u;
    }

    template <class SC, class EMIT>
    SPK_HD void iterate(SC& sc, EMIT&& emit) {
        // ---- bulk: the first violation among the remaining spikes (selects only)
        const int lo = sc.lo;
        const uint32_t hw = sc.hw;
        const uint32_t Q = bit_shr_clamp(So, 0u, (uint32_t)lo) |
                           bit_sel(hw != 0u, bit_shr_clamp(So, 0u, (uint32_t)lo + 1u), 0u);
        const int d0 = base + f - sc.last;
        const bool bad0 = ((S & fb) != 0u) & ((uint32_t)(d0 - lo) > hw);
        const uint32_t V = (S & ~(Q | fb)) | bit_sel(lo >= 2, S & G1, 0u) | bit_sel(bad0, fb, 0u);
        const uint32_t p = V ? (uint32_t)bit_clz(V) : 32u;
        const uint32_t A = S & ~bit_shr_clamp(0xffffffffu, 0u, p);
        sc.cnt += bit_popc(A);
        sc.last = A ? base + 32 - bit_ffs(A) : sc.last;
        S &= ~A;
        if (!S) return;
        // ---- the violating spike through the exact automaton
        const int c = bit_clz(S);
        S ^= 0x80000000u >> c;
        int rs, cnt;
        const bool e = sc.step(base + c, rs, cnt);
        emit(e, rs, cnt);
    }
};

// FSR over a window of N consecutive words (frames base0 .. base0+32N-1; the
// first `cpos` frames of word 0 already consumed).  The FsrWord test is run on
// all N words at once -- independent given the open run's pair, so they
// overlap in the pipeline -- with each word's first remaining spike checked
// against the last spike before it (in an earlier word of the window, or
// sc.last).  The first word holding a violation decides: everything before
// the violating spike is accepted in bulk and the spike itself goes through
// the exact automaton.  Returns the number of words fully consumed (N when no
// word of the window violates) and leaves `cpos` = frames consumed in the new
// first word.  Words past the end of the stream must be passed as 0.
// word(j) returns word j of the window.
template <int N, class SC, class WORD, class EMIT>
SPK_HD int fsr_batch(SC& sc, WORD&& word, int base0, int& cpos, EMIT&& emit) {
    const int lo = sc.lo;
    const uint32_t hw = sc.hw;
    const uint32_t sh1 = (uint32_t)lo, sh2 = (uint32_t)lo + hw;
    const uint32_t sa = lo >= 2 ? 1u : 32u;
    int pv = sc.last + lo;
    uint32_t R[N], V[N], c[N];
    int PV[N];
#pragma unroll
    for (int j = 0; j < N; ++j) {
        const uint32_t w = word(j);
        const uint32_t r = j == 0 ? w & bit_shr_clamp(0xffffffffu, 0u, (uint32_t)cpos) : w;
        const int base = base0 + 32 * j;
        PV[j] = pv;
        const uint32_t Q = bit_shr_clamp(w, 0u, sh1) | bit_shr_clamp(w, 0u, sh2);
        const int hi = bit_flo(r);
        const uint32_t fb = bit_shl_clamp(1u, (uint32_t)hi);
        const uint32_t bad0 = (uint32_t)(base + 31 - hi - pv) > hw ? fb : 0u;
        V[j] = (r & ~(Q | fb)) | (r & w & bit_shr_clamp(w, 0u, sa)) | bad0;
        pv = bit_selp(r != 0u, base + lo + 32 - bit_ffs(r), pv);
        R[j] = r;
        c[j] = (uint32_t)bit_popc(r);
    }
    // first word with a violation (N: none), as a chain of selects from the
    // last word down (no bit scan over a flag word)
    int k = N;
#pragma unroll
    for (int j = N - 1; j >= 0; --j) k = V[j] != 0u ? j : k;
    const bool ev = k < N;
    const int kk = ev ? k : N - 1;
    uint32_t Vk = V[0], rk = R[0], before = 0u;
    int prevk = PV[0];
#pragma unroll
    for (int j = 1; j < N; ++j) {
        const bool sj = kk >= j;
        Vk = sj ? V[j] : Vk;
        rk = sj ? R[j] : rk;
        prevk = sj ? PV[j] : prevk;
        before += sj ? c[j - 1] : 0u;
    }
    prevk -= lo;
    const int basek = base0 + 32 * kk;
    const int p = bit_clz(Vk);
    const uint32_t A = rk & ~bit_shr_clamp(0xffffffffu, 0u, (uint32_t)p);
    sc.cnt += (int)(before + (uint32_t)bit_popc(A));
    sc.last = bit_selp(A != 0u, basek + 32 - bit_ffs(A), prevk);
    cpos = ev ? p + 1 : 0;
    if (ev) {
        int rs, cnt;
        const bool e = sc.step(basek + p, rs, cnt);
        emit(e, rs, cnt);
    }
    return ev ? kk : N;
}

// FSR over N consecutive words when the window holds no event at all: the
// fsr_batch test on every word (each word's first remaining spike against
// the last spike before it), OR-ed.  With no violation anywhere the whole
// window is accepted at once (cnt += spikes, last = the latest spike,
// cpos = 0) and true is returned; otherwise nothing changes and the caller
// takes the exact fsr_batch path.  No selection across words is needed, so
// a quiet window costs about half a window test per word (static scenes,
// long streams).  word(k) returns word k of the window; words past the end
// of the stream must read as 0.
//
// Per word ~20 instructions and no branch: the first spike as FLO (fb = its
// bit, 0 for an empty word), the adjacency test as one clamped shift (by 32
// when lo < 2: off), the last spike as FFS with a select.
template <int N, class SC, class WORD>
SPK_HD bool fsr_quiet(SC& sc, WORD&& word, int base0, int& cpos) {
    const int lo = sc.lo;
    const uint32_t hw = sc.hw;
    const uint32_t sh1 = (uint32_t)lo, sh2 = (uint32_t)lo + hw;
    const uint32_t sa = lo >= 2 ? 1u : 32u;
    int pv = sc.last + lo;  // last spike before the word under test, plus lo
    uint32_t bad = 0u, n = 0u;
#pragma unroll
    for (int k = 0; k < N; ++k) {
        const uint32_t w = word(k);
        const uint32_t r = k == 0 ? w & bit_shr_clamp(0xffffffffu, 0u, (uint32_t)cpos) : w;
        const int base = base0 + 32 * k;
        const uint32_t Q = bit_shr_clamp(w, 0u, sh1) | bit_shr_clamp(w, 0u, sh2);
        const int hi = bit_flo(r);                // r's first spike is frame base + 31 - hi
        const uint32_t fb = bit_shl_clamp(1u, (uint32_t)hi);  // its bit (0: no spike)
        const uint32_t bad0 = (uint32_t)(base + 31 - hi - pv) > hw ? fb : 0u;
        bad |= (r & ~(Q | fb)) | (r & w & bit_shr_clamp(w, 0u, sa)) | bad0;
        n += (uint32_t)bit_popc(r);
        // r's last spike (lowest set bit) is frame base + 32 - ffs(r)
        pv = bit_selp(r != 0u, base + lo + 32 - bit_ffs(r), pv);
    }
    if (bad) return false;
    sc.cnt += (int)n;
    sc.last = pv - lo;
    cpos = 0;
    return true;
}

// FSR: the remaining spikes S of word So (first frame in bit 31, frames
// base..base+31) that the automaton would flag -- its next event is the first
// one; everything before it is accepted as-is (fsr_accept).  Same test as
// FsrWord::iterate.
template <class SC>
SPK_HD uint32_t fsr_flags(const SC& sc, uint32_t So, uint32_t S, int base) {
    const int lo = sc.lo;
    const uint32_t hw = sc.hw;
    // (a single pair shifts by lo twice: OR-idempotent; the adjacency shift
    // is clamped to 32 -- off -- when lo < 2)
    const uint32_t Q = bit_shr_clamp(So, 0u, (uint32_t)lo) | bit_shr_clamp(So, 0u, (uint32_t)lo + hw);
    const int hi = bit_flo(So);  // So's first spike: frame base + 31 - hi
    const uint32_t fb = bit_shl_clamp(1u, (uint32_t)hi);
    const uint32_t sa = lo >= 2 ? 1u : 32u;
    const uint32_t bad0 = (uint32_t)(base + 31 - hi - sc.last - lo) > hw ? (S & fb) : 0u;
    return (S & ~(Q | fb)) | (S & So & bit_shr_clamp(So, 0u, sa)) | bad0;
}

template <class SC>
SPK_HD void fsr_accept(SC& sc, uint32_t A, int base) {
    sc.cnt += bit_popc(A);
    sc.last = bit_selp(A != 0u, base + 32 - bit_ffs(A), sc.last);
}

// ---- SSR in bulk ----------------------------------------------------------
// Inside an FSR run with pair [lo, lo+hw] every accepted interval is short
// (lo) or long (lo+1).  SSR's second level is the pair rule over each value's
// occurrence gaps (interval-index distance between consecutive occurrences in
// the sub-run).  Between two consecutive long intervals lie only short ones,
// so index gap m is a frame distance m*lo + 1 between the spikes closing
// them; between two short ones lie only long ones: m*(lo+1) - 1.  A slot with
// gap pair [g, g+h] thus allows the frame distances
//     long:  D1 = g*lo + 1,      D2 = D1 + h*lo
//     short: D1 = g*(lo+1) - 1,  D2 = D1 + h*(lo+1)
// and FsrWord's argument carries over per class (class spikes restricted to
// the current sub-run): a class spike without a class spike exactly D1 / D2
// earlier is flagged; the only violation that can escape is a short at index
// gap 1 (distance lo) -- flagged separately when 1 is not allowed (g >= 2).
// The first class spike of the word is checked against the slot's last
// occurrence frame directly.  Slots not yet holding a gap pair (first
// occurrence / first gap after a sub-run start) and every FSR event go
// through the exact step.  Cs / Cl receive the class masks for ssr_accept.
template <class SC>
SPK_HD uint32_t ssr_flags(const SC& sc, uint32_t So, uint32_t S, int base, int prevlast,
                          uint32_t& Cs, uint32_t& Cl) {
    const uint32_t Vf = fsr_flags(sc, So, S, base);
    const int lo = sc.lo;
    const uint32_t hw = sc.hw;
    // no class spikes before the first interval (lo >= kLim); branch-free:
    // the shifts below clamp to 0 and the masks clear C
    const uint32_t live = lo < kLim ? 0xffffffffu : 0u;
    const int hi = bit_flo(So);
    const uint32_t fb = bit_shl_clamp(1u, (uint32_t)hi);
    const int d0 = base + 31 - hi - prevlast;
    // spikes closing an interval of the current sub-run: frames >= sf
    const uint32_t sub = bit_shr_clamp(0xffffffffu, 0u, (uint32_t)max(sc.sf - base, 0)) & live;
    const uint32_t at_lo = bit_shr_clamp(So, 0u, (uint32_t)lo);
    const uint32_t at_lo1 = bit_shr_clamp(So, 0u, (uint32_t)lo + 1u);
    Cs = ((So & at_lo) | (d0 == lo ? fb : 0u)) & sub;
    Cl = ((So & at_lo1 & ~at_lo) | (d0 == lo + 1 ? fb : 0u)) & (hw != 0u ? sub : 0u);
    uint32_t V = Vf;
#pragma unroll
    for (int cls = 0; cls < 2; ++cls) {  // 0 = short (value lo), 1 = long (lo + 1)
        const uint32_t C = cls ? Cl : Cs;
        const bool x = ((lo + cls) & 1) != 0;  // parity slot of the value
        const int l = x ? sc.l1 : sc.l0;
        const int g = x ? sc.g1 : sc.g0;
        const int h = (int)(x ? sc.h1 : sc.h0);
        const int fl = x ? sc.fl1 : sc.fl0;
        const uint32_t CS = C & S;
        const bool est = (l >= sc.sub0) & (g < kLim);
        const uint32_t fcs = bit_shl_clamp(1u, (uint32_t)bit_flo(CS));  // CS's first spike
        const int stp = cls ? lo : lo + 1;
        const int D1 = g * stp + (cls ? 1 : -1);
        const int D2 = D1 + h * stp;  // (h = 0: D1 again, OR-idempotent)
        const uint32_t Q = bit_shr_clamp(C, 0u, (uint32_t)D1) | bit_shr_clamp(C, 0u, (uint32_t)D2);
        const int hic = bit_flo(C);
        const uint32_t fcw = bit_shl_clamp(1u, (uint32_t)hic);  // C's first spike (0 if none)
        const int dfirst = base + 31 - hic - fl;
        const bool badf = ((fcw & S) != 0u) & (dfirst != D1) & (dfirst != D2);
        const uint32_t gap1 = (cls == 0) & (g >= 2) ? CS & bit_shr_clamp(C, 0u, (uint32_t)lo) : 0u;
        const uint32_t Vc = (CS & ~(Q | fcw)) | (badf ? fcw : 0u) | gap1;
        V |= est ? Vc : fcs;
    }
    return V;
}

// bookkeeping of an accepted prefix A (no event inside) for SSR (branch-free:
// the lanes of a warp accept different prefixes)
template <class SC>
SPK_HD void ssr_accept(SC& sc, uint32_t A, uint32_t Cs, uint32_t Cl, int base) {
    const int n = bit_popc(A);
#pragma unroll
    for (int cls = 0; cls < 2; ++cls) {
        const uint32_t Ac = A & (cls ? Cl : Cs);
        const int b = bit_ffs(Ac);  // latest class spike: bit b-1 (b = 0: none)
        const int idx = sc.ii + bit_popc(bit_shr_clamp(A, 0u, (uint32_t)(b - 1))) - 1;
        const int fr = base + 32 - b;
        const bool have = Ac != 0u;
        const bool odd = ((sc.lo + cls) & 1) != 0;
        sc.l1 = bit_selp(have & odd, idx, sc.l1);
        sc.fl1 = bit_selp(have & odd, fr, sc.fl1);
        sc.l0 = bit_selp(have & !odd, idx, sc.l0);
        sc.fl0 = bit_selp(have & !odd, fr, sc.fl0);
    }
    sc.cnt += n;
    sc.ii += n;
    sc.last = bit_selp(A != 0u, base + 32 - bit_ffs(A), sc.last);
}

// SSR over one word: bulk acceptance up to each event, the event exact
template <class SC, class EMIT>
SPK_HD void ssr_word(SC& sc, uint32_t So, int base, EMIT&& emit) {
    uint32_t S = So;
    const int prevlast = sc.last;
    while (S) {
        uint32_t Cs, Cl;
        const uint32_t V = ssr_flags(sc, So, S, base, prevlast, Cs, Cl);
        const uint32_t A = S & ~bit_shr_clamp(0xffffffffu, 0u, V ? (uint32_t)bit_clz(V) : 32u);
        ssr_accept(sc, A, Cs, Cl, base);
        S &= ~A;
        if (!S) break;
        const int c = bit_clz(S);
        S ^= 0x80000000u >> c;
        int rs, cnt;
        const bool e = sc.step(base + c, rs, cnt);
        emit(e, rs, cnt);
    }
}

// `emit(pred, rs, cnt)` stores a closed run when pred is true.
template <class SC, class EMIT>
SPK_HD void fsr_word(SC& sc, uint32_t S, int base, EMIT&& emit) {
    if (!S) return;
    FsrWord w;
    w.load(S, base);
    while (w.S) w.iterate(sc, emit);
}

}  // namespace spk
