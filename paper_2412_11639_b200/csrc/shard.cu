// shard.cu -- exact time sharding of one long stream (the
// "Time" partition of BASELINE configs[4]).
//
// A run's extent and value depend on the whole history before it (the pair
// rule's accepted set only grows, reconstruct.cpp:17-36), so a halo alone is
// not exact.  The stitching instead uses the automaton itself:
//   * every shard is scanned on its own from a fresh state (k_segment with no
//     entry state): the speculative runs;
//   * in shard order, k_resolve re-runs the start of shard r from the TRUE
//     entry state beside the speculative automaton; once both have the same
//     future (Scan::same_future: same pair / last spike, and for SSR the same
//     parity-slot states relative to the interval index) every later decision
//     coincides, so the speculative runs from there on are the true runs --
//     except that the run open at the sync point started earlier (rs_true)
//     and holds `delta` more intervals;
//   * k_junction turns that into the true exit state (the next shard's entry)
//     and tells whether the run open at the shard entry closes inside it;
//   * k_close_chain carries the close of boundary-crossing runs (one run may
//     span many shards: a static pixel is one run) from right to left;
//   * k_stitch writes the true run list of each shard: prefix runs, then the
//     speculative runs from the synced one on, the last one closed with the
//     carried close.
// The sync usually happens within a few runs after the shard start; a pixel
// that never syncs is covered by the prefix list (its re-run went through the
// whole shard) or, if that overflows, by a full re-scan from the entry state.
#include "spk_common.cuh"
#include "spk_fsm.cuh"
#include "spk_kernels.cuh"

namespace spk {

namespace {

// first speculative run's start, shard frames (in-grid split: the rows hold
// stream frames, shard r's region at r*rstride + kSplitGap)
__device__ __forceinline__ int spec_first_start(const ShardArgs& a, int64_t p) {
    if (a.grid_sf > 0) {
        const int r = (int)blockIdx.y + 1;
        return (int)a.spec[p * a.nshards * a.rstride + r * a.rstride + kSplitGap].start - r * a.grid_sf;
    }
    return (int)a.spec[p * a.scap].start;
}

// shift a state's frame fields by -len (to the next shard's frames)
template <int METHOD>
__device__ __forceinline__ void shift_state(Scan<METHOD>& X, int len) {
    if (X.last != kNoSpike) X.last -= len;
    if (X.lo < kLim) X.rs -= len;
    if (X.fl0 != kNoSpike) X.fl0 -= len;
    if (X.fl1 != kNoSpike) X.fl1 -= len;
    if (X.sf != kNoSpike) X.sf -= len;
}

// FSR shortcut: when the speculative scan had no break in the whole shard, the
// shard's intervals all lie in its final pair, so the true automaton never
// breaks either iff E's pair, the boundary-crossing interval and that pair fit
// one pair {x, x+1} -- then its end state follows without a scan.  (Pixels
// whose speculative pair never completes in a long shard would otherwise keep
// their warp scanning to the shard end.)
// E: the true entry; S, scount: the speculative end state and run count of
// the shard; f1: the speculative first run's start (its second spike's frame
// is not needed: S.cnt counts the intervals after it)
__device__ bool fsr_no_break_core(const Scan<kFSR>& E, const Scan<kFSR>& S, uint32_t scount, int f1s,
                                  Scan<kFSR>& X) {
    if (scount > 1u) return false;  // the speculative scan broke in the shard
    if (S.last == kNoSpike) {  // no spike in the shard
        X = E;
        return true;
    }
    if (E.last == kNoSpike) {  // nothing before: the true scan is the speculative one
        X = S;
        return true;
    }
    const bool hasS = S.lo < kLim;  // >= 2 spikes in the shard
    const int f1 = hasS ? f1s : S.last;
    const int t0 = f1 - E.last;
    int lo = t0, hi = t0;
    if (E.lo < kLim) {
        lo = min(lo, E.lo);
        hi = max(hi, E.lo + (int)E.hw);
    }
    if (hasS) {
        lo = min(lo, S.lo);
        hi = max(hi, S.lo + (int)S.hw);
    }
    if (hi - lo > 1) return false;
    X = E;
    X.lo = lo;
    X.hw = (uint32_t)(hi - lo);
    if (E.lo >= kLim) {  // E held a lone spike: the run starts there
        X.rs = E.last;
        X.cnt = 1 + (hasS ? S.cnt : 0);
    } else {
        X.cnt = E.cnt + 1 + (hasS ? S.cnt : 0);
    }
    X.last = S.last;
    return true;
}

__device__ bool fsr_no_break(const ShardArgs& a, int64_t p, const Scan<kFSR>& E, Scan<kFSR>& X) {
    if (a.scount[p] > 1u) return false;
    Scan<kFSR> S;
    S.restore(a.sstate, a.npix, p);
    return fsr_no_break_core(E, S, a.scount[p], S.lo < kLim ? spec_first_start(a, p) : 0, X);
}

}  // namespace

// Thread per pixel in warp lockstep over 32-frame words: lanes load the
// transposed words as K2 does and walk their spikes with both automata until
// every lane of the warp has synced (or the shard ends).
template <int METHOD>
__global__ void __launch_bounds__(64) k_resolve(ShardArgs a) {
    int entry_shift = 0;
    if (a.grid_sf > 0) {  // in-grid split: shard r = blockIdx.y + 1, entry = spec end of r-1
        const int r = (int)blockIdx.y + 1;
        const int64_t n = a.npix;
        a.planes = reinterpret_cast<const char*>(a.planes) + (size_t)r * a.grid_sf * a.pitch;
        a.frames = min(a.grid_sf, a.total_frames - r * a.grid_sf);
        a.entry = a.sstate + (int64_t)(r - 1) * Scan<METHOD>::kFields * n;
        entry_shift = a.grid_sf;
        a.scount += (int64_t)r * n;
        a.sstate += (int64_t)r * Scan<METHOD>::kFields * n;
        a.prefix += (int64_t)r * n * a.pcap;
        a.sync += (int64_t)r * n;
        a.tstate += (int64_t)r * Scan<METHOD>::kFields * n;
        a.syncj += (int64_t)r * n;
    }
    const int lane = threadIdx.x & 31;
    const int64_t word = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (word * 32 >= a.npix) return;  // warp-uniform
    const int64_t p = word * 32 + lane;
    const bool valid = p < a.npix;
    const char* col = reinterpret_cast<const char*>(a.planes) + word * 4;
    const int rev = 31 - lane;
    const int ngroups = (a.frames + 31) >> 5;

    Scan<METHOD> T, S;
    T.init();
    S.init();
    if (valid) {
        T.restore(a.entry, a.npix, p);
        T.nrun = 0;
        if (entry_shift) shift_state(T, entry_shift);
    }
    spk_run_t* pre = a.prefix + (valid ? p * a.pcap : 0);
    int m = 0;
    int sj = 0, jsync = -1;  // speculative runs closed (before the sync)
    bool done = !valid;
    spk_sync_t out{0, 0, 0, -1};
    if constexpr (METHOD == kFSR) {
        Scan<kFSR> X;
        if (valid && a.scount != nullptr && fsr_no_break(a, p, T, X)) {
            T = X;  // reported below as "never synced, no closed run"
            done = true;
        }
    }
    for (int g = 0; g < ngroups; ++g) {
        if (__all_sync(kFull, done)) break;
        const int f = g * 32 + rev;
        uint32_t w = f < a.frames ? __ldg(reinterpret_cast<const uint32_t*>(col + (size_t)f * a.pitch)) : 0u;
        w = transpose32(w, lane);
        if (done) continue;
        const int base = g * 32;
        const uint32_t wo = w;
        const int prevT = T.last, prevS = S.last;
        while (w) {
            // both automata accept in bulk up to the next event of either
            if constexpr (METHOD == kFSR) {
                const uint32_t V = fsr_flags(T, wo, w, base) | fsr_flags(S, wo, w, base);
                const uint32_t A = w & ~bit_shr_clamp(0xffffffffu, 0u, V ? (uint32_t)__clz(V) : 32u);
                fsr_accept(T, A, base);
                fsr_accept(S, A, base);
                w &= ~A;
            } else {
                uint32_t CsT, ClT, CsS, ClS;
                const uint32_t V = ssr_flags(T, wo, w, base, prevT, CsT, ClT) |
                                   ssr_flags(S, wo, w, base, prevS, CsS, ClS);
                const uint32_t A = w & ~bit_shr_clamp(0xffffffffu, 0u, V ? (uint32_t)__clz(V) : 32u);
                ssr_accept(T, A, CsT, ClT, base);
                ssr_accept(S, A, CsS, ClS, base);
                w &= ~A;
            }
            if (!w) break;
            const int c = __clz(w);
            w ^= 0x80000000u >> c;
            const int n = base + c;
            int rs, cnt;
            if (T.step(n, rs, cnt)) {
                if (m < a.pcap) pre[m] = spk_run_t{(uint32_t)rs, (uint32_t)cnt};
                ++m;
            }
            sj += (int)S.step(n, rs, cnt);
            if (T.same_future(S)) {
                out = spk_sync_t{T.rs, S.rs, T.cnt - S.cnt, m};
                jsync = sj;
                done = true;
                break;
            }
        }
    }
    if (!valid) return;
    if (out.npre < 0) {
        // never synced: the true runs of the whole shard are the prefix list
        // (plus the run open at the end, kept in the true end state)
        out.npre = m <= a.pcap ? -2 : -1;
        T.nrun = m;  // closed true runs, all in the prefix list
        T.save(a.tstate, a.npix, p);
    } else if (m > a.pcap) {
        out.npre = -1;
    }
    a.sync[p] = out;
    if (a.syncj != nullptr) a.syncj[p] = jsync;  // index of the synced speculative run
}

namespace {

// the true automaton state at the end of the shard
template <int METHOD>
__device__ void true_end(const ShardArgs& a, int64_t p, const spk_sync_t& sy, Scan<METHOD>& X) {
    if (sy.npre >= 0) {
        X.restore(a.sstate, a.npix, p);
        if ((X.lo < kLim) & (X.rs == sy.rs_spec)) {  // the synced run is still open
            X.rs = sy.rs_true;
            X.cnt += sy.delta;
        }
    } else if (sy.npre == -2) {
        X.restore(a.tstate, a.npix, p);
    } else if (a.fbstate != nullptr) {
        X.restore(a.fbstate, a.npix, p);
    } else {
        // prefix overflow in a fast pass without the re-scan: flagged on the
        // host side (the pass is redone robustly); any in-bounds state will do
        X.restore(a.sstate, a.npix, p);
    }
}

// index of the speculative run that started at `start` (runs sorted by start)
__device__ int find_run(const spk_run_t* r, int n, int start) {
    int lo = 0, hi = n;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if ((int)r[mid].start < start)
            lo = mid + 1;
        else
            hi = mid;
    }
    return lo;
}

// The shard's true runs in order, read from where they live: the prefix
// runs then the speculative runs from the synced one (re-based); the prefix
// plus the open run of the true end state; or the full re-scan.  When the
// true end state has an interval, the last entry is the run open at the end.
template <int METHOD>
struct TrueList {
    const spk_run_t* pre = nullptr;
    const spk_run_t* tail = nullptr;
    int npre = 0, j = 0, ntail = 0;
    spk_run_t extra{0u, 0u};  // -2: the open run of the true end state
    bool has_extra = false;
    spk_sync_t sy;

    __device__ void init(const ShardArgs& a, int64_t p) {
        sy = a.sync[p];
        pre = a.prefix + p * a.pcap;
        if (sy.npre >= 0) {
            npre = sy.npre;
            tail = a.spec + p * a.scap;
            ntail = (int)min(a.scount[p], (uint32_t)a.scap);
            j = find_run(tail, ntail, sy.rs_spec);
        } else if (sy.npre == -2) {
            Scan<METHOD> T;
            T.restore(a.tstate, a.npix, p);
            npre = T.nrun;
            has_extra = T.lo < kLim;
            extra = spk_run_t{(uint32_t)T.rs, (uint32_t)T.cnt};
        } else if (a.fb != nullptr) {
            tail = a.fb + p * a.scap;
            ntail = (int)min(a.fbcount[p], (uint32_t)a.scap);
        } else {  // fast pass without the re-scan (redone robustly): in-bounds stand-in
            tail = a.spec + p * a.scap;
            ntail = (int)min(a.scount[p], (uint32_t)a.scap);
        }
    }
    __device__ int count() const { return npre + (sy.npre == -2 ? (int)has_extra : ntail - j); }
    __device__ spk_run_t at(int k) const {
        if (k < npre) return pre[k];
        if (sy.npre == -2) return extra;
        const int i = j + (k - npre);
        spk_run_t r = tail[i];
        if (sy.npre >= 0 && i == j) {
            r.start = (uint32_t)sy.rs_true;
            r.intervals += (uint32_t)sy.delta;
        }
        return r;
    }
};

}  // namespace

// True exit state (frames shifted to the next shard), the close of the run
// open at the shard entry as far as it is decided in this shard (see
// spk_close), and the stream-end close of the run open at the end (used when
// this is the last shard).
template <int METHOD>
__global__ void __launch_bounds__(128) k_junction(ShardArgs a) {
    const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= a.npix) return;
    const spk_sync_t sy = a.sync[p];
    Scan<METHOD> E, X;
    E.restore(a.entry, a.npix, p);
    true_end<METHOD>(a, p, sy, X);
    TrueList<METHOD> L;
    L.init(a, p);
    const int n = L.count();
    const bool open_end = X.lo < kLim;  // last entry = run open at the end

    // A = the true run covering the shard start (entry 0 when it starts before
    // the shard: the run open at the entry, or the one starting at the last
    // spike before the shard)
    spk_close_t ec{0, 0, 0, 0, 0, 0, 0, 0};
    if (n >= 1 && (int)L.at(0).start < 0) {
        if (n >= 2 || !open_end) {
            const spk_run_t r0 = L.at(0);
            const spk_run_t r1 = L.at(1);
            ec.a_state = 1;
            ec.a_intervals = (int32_t)r0.intervals;
            ec.a_end = (int32_t)r1.start;
            if ((int32_t)r1.start < 0) {  // A closed before the shard: B starts there
                if (n >= 3 || !open_end) {
                    ec.b_kind = 1;
                    ec.b_intervals = (int32_t)r1.intervals;
                    ec.b_end = n >= 3 ? (int32_t)L.at(2).start : X.last;
                } else {
                    ec.b_kind = 2;  // B is this shard's end run
                }
            }
        } else {
            ec.a_state = 2;  // A is this shard's end run
        }
    } else if (E.last != kNoSpike) {
        // one spike before the shard and no run formed here yet: the run that
        // will start at that spike covers this shard too
        ec.a_state = 2;
    }
    a.entry_close[p] = ec;
    // the run open at the end, closed by the end of the stream
    a.tail_close[p] = spk_close_t{open_end ? 1 : 0, X.cnt, X.last, 0, 0, 0, 0, 0};
    // exit state in the next shard's frames
    if (X.last != kNoSpike) X.last -= a.frames;
    if (X.lo < kLim) X.rs -= a.frames;
    if (X.fl0 != kNoSpike) X.fl0 -= a.frames;
    if (X.fl1 != kNoSpike) X.fl1 -= a.frames;
    if (X.sf != kNoSpike) X.sf -= a.frames;
    X.nrun = 0;
    X.save(a.exit_state, a.npix, p);
}

// close record of shard r from shard r+1's entry close and close record;
// frames -> shard r (shard_len = length of shard r).
__global__ void __launch_bounds__(256) k_close_chain(const spk_close_t* entry_next,
                                                     const spk_close_t* close_next, int shard_len,
                                                     int64_t npix, spk_close_t* close) {
    const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= npix) return;
    const spk_close_t ec = entry_next[p];
    const spk_close_t nc = close_next[p];
    spk_close_t c{0, 0, 0, 0, 0, 0, 0, 0};
    if (ec.a_state == 1) {
        c.a_state = 1;
        c.a_intervals = ec.a_intervals;
        c.a_end = ec.a_end;
        if (ec.b_kind == 1) {
            c.b_kind = 1;
            c.b_intervals = ec.b_intervals;
            c.b_end = ec.b_end;
        } else if (ec.b_kind == 2) {  // B is the next shard's end run
            c.b_kind = nc.a_state == 1 ? 1 : 0;
            c.b_intervals = nc.a_intervals;
            c.b_end = nc.a_end;
        }
    } else if (ec.a_state == 2) {  // A runs through the next shard: the next record
        c = nc;
    }
    c.a_end += shard_len;
    c.b_end += shard_len;
    close[p] = c;
}

// True run list of the shard, the run open at the end closed with `close`
// (plus run B when A closes before the shard end).
template <int METHOD>
__global__ void __launch_bounds__(128) k_stitch(ShardArgs a) {
    const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= a.npix) return;
    const spk_sync_t sy = a.sync[p];
    Scan<METHOD> X;
    true_end<METHOD>(a, p, sy, X);
    TrueList<METHOD> L;
    L.init(a, p);
    const int n = L.count();
    // The run covering the shard end gets its total from `close`: the open run
    // (last true entry), or -- one spike so far -- the run that starts at that
    // spike once a later one arrives; then run B when A closes inside the shard.
    const spk_close_t c = a.close[p];
    const bool open_end = (X.lo < kLim) & (n >= 1);
    const bool add_a = !open_end & (X.last != kNoSpike) & (c.a_state == 1);
    const bool has_a = open_end | add_a;
    const bool with_b = has_a & (c.b_kind == 1) & (c.a_end < a.frames);
    const int na = n + (int)add_a;
    const int nall = na + (int)with_b;
    auto entry = [&](int i) -> spk_run_t {
        if (i == na) return spk_run_t{(uint32_t)c.a_end, (uint32_t)c.b_intervals};
        if (add_a & (i == n)) return spk_run_t{(uint32_t)X.last, (uint32_t)c.a_intervals};
        spk_run_t r = L.at(i);
        if (open_end & (i == n - 1)) r.intervals = (uint32_t)c.a_intervals;
        return r;
    };
    // skip runs that ended before the shard (started before frame 0 and closed
    // at a spike before it); the first kept one may still start earlier
    int k0 = 0;
    while (k0 + 1 < nall && (int)entry(k0 + 1).start <= 0) ++k0;
    spk_run_t* out = a.region + p * a.rcap;
    int k = 0;
    for (int i = k0; i < nall; ++i) {
        if (k < a.rcap) out[k] = entry(i);
        ++k;
    }
    int32_t last = X.last == kNoSpike ? -1 : X.last;
    if (has_a) last = with_b ? c.b_end : c.a_end;
    a.rcount[p] = (uint32_t)k;
    a.rlast[p] = last;
}

// ------------------------------------------------------ in-grid time split --
// One stream cut in S shards on ONE GPU (capi.cu reconstruct_impl): all
// speculative scans in one K2 launch, all resolves in one k_resolve launch
// (shard r resolved from the speculative end state of shard r-1 instead of
// the true one), then this pass walks each pixel's shards in order.  The
// resolve of shard r is the true one iff its entry decides like the true
// entry (Scan::same_future, or both without an interval and the same last
// spike): the states can then differ only in the open run's bookkeeping, so
// the true runs are the resolved ones with the entry run's start / count
// corrected.  A pixel failing that (or overflowing a capacity) is flagged
// for a whole-stream re-scan (k_segment with flags).
namespace {

template <int METHOD>
__device__ bool decision_equal(const Scan<METHOD>& A, const Scan<METHOD>& B) {
    const bool ia = A.lo < kLim, ib = B.lo < kLim;
    if (ia != ib) return false;
    if (!ia) return A.last == B.last;
    return A.same_future(B);
}

}  // namespace

// a state's fields through the read-only path (FSR: the 6 it uses)
template <int METHOD>
__device__ __forceinline__ void load_state(Scan<METHOD>& X, const int32_t* __restrict__ st, int64_t n,
                                           int64_t p) {
    if constexpr (METHOD == kFSR) {
        X.init();
        X.last = __ldg(st + p);
        X.lo = __ldg(st + n + p);
        X.rs = __ldg(st + 2 * n + p);
        X.cnt = __ldg(st + 3 * n + p);
        X.nrun = __ldg(st + 4 * n + p);
        X.hw = (uint32_t)__ldg(st + 5 * n + p);
    } else {
        X.restore(st, n, p);
    }
}

template <int METHOD>
__global__ void __launch_bounds__(128) k_split_combine(SplitArgs a) {
    const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= a.npix) return;
    constexpr int F = Scan<METHOD>::kFields;
    const int S = a.nshards;
    const int64_t n = a.npix;
    spk_run_t* row = a.runs + p * S * a.rstride;
    uint32_t* sg = a.seg + p * S * 2;
    bool bad = false;
    uint32_t total = 0;
    int32_t last_abs = -1;
    Scan<METHOD> E;   // true entry of shard r (shard r frames)
    Scan<METHOD> Xp;  // speculative end state of shard r-1 (its own frames)
    E.init();
    Xp.init();
    for (int r = 0; r < S; ++r) {
        const int f0 = r * a.sf;
        const int len = min(a.sf, a.frames - f0);
        const int64_t base = (int64_t)r * a.rstride + kSplitGap;
        const uint32_t cr = __ldg(a.scount + r * n + p);
        Scan<METHOD> Xs;  // speculative end state of shard r
        load_state(Xs, a.sstate + (int64_t)r * F * n, n, p);
        const spk_sync_t sy = r > 0 ? a.sync[r * n + p] : spk_sync_t{0, 0, 0, 0};
        const int jr = r > 0 ? __ldg(a.syncj + r * n + p) : 0;
        if (cr > (uint32_t)a.scap) {  // speculative list overflowed
            bad = true;
            break;
        }
        Scan<METHOD> X = Xs;  // true end state of shard r (shard r frames)
        int64_t b = base, e = base + cr;
        if (r > 0) {
            Scan<METHOD> Ep = Xp;  // the entry the resolve used
            shift_state(Ep, a.sf);
            if (!decision_equal(E, Ep)) {
                // FSR: a shard whose speculative scan never broke is decided
                // by the pairs alone (fsr_no_break): no run closes in it
                bool ok = false;
                if constexpr (METHOD == kFSR) {
                    const int f1s = cr >= 1u ? (int)row[base].start - f0 : 0;
                    ok = fsr_no_break_core(E, Xs, cr, f1s, X);
                }
                if (!ok) {
                    bad = true;
                    break;
                }
                b = e = base;
                if ((r == S - 1) & (X.lo < kLim)) {
                    row[e] = spk_run_t{(uint32_t)(X.rs + f0), (uint32_t)X.cnt};
                    ++e;
                }
            } else {
                // the entry run (open at the shard start, with an interval) is
                // the only run whose bookkeeping differs: start E.rs, count + dcnt
                const bool adj = Ep.lo < kLim;
                const int eprs = Ep.rs, ers = E.rs, dcnt = E.cnt - Ep.cnt;
                auto fixed = [&](spk_run_t q) {
                    if (adj & ((int)q.start == eprs)) {
                        q.start = (uint32_t)ers;
                        q.intervals += (uint32_t)dcnt;
                    }
                    q.start += (uint32_t)f0;  // stream frames
                    return q;
                };
                const spk_run_t* pre = a.prefix + (r * n + p) * a.pcap;
                if (sy.npre == -1) {  // prefix list overflowed
                    bad = true;
                    break;
                }
                if (sy.npre >= 0) {
                    // the synced speculative run (its index: the speculative
                    // automaton's closures before the sync, counted by k_resolve)
                    const int64_t j = base + jr;
                    if (jr < 0 || (uint32_t)jr >= cr || sy.npre > kSplitGap) {
                        bad = true;
                        break;
                    }
                    const spk_run_t rj = row[j];
                    if (rj.start != (uint32_t)(sy.rs_spec + f0)) {
                        bad = true;
                        break;
                    }
                    for (int k = 0; k < sy.npre; ++k) row[j - sy.npre + k] = fixed(pre[k]);
                    const spk_run_t tj = fixed(spk_run_t{(uint32_t)sy.rs_true, rj.intervals + (uint32_t)sy.delta});
                    row[j] = tj;
                    b = j - sy.npre;
                    if ((X.lo < kLim) & (X.rs == sy.rs_spec)) {  // the synced run is still open
                        X.rs = (int)tj.start - f0;
                        X.cnt += (int)tj.intervals - (int)rj.intervals;
                    }
                } else {  // never synced: the prefix list + the open run of the true end state
                    load_state(X, a.tstate + (int64_t)r * F * n, n, p);
                    const int m = X.nrun;
                    if (m > a.pcap || m + 1 > a.scap) {
                        bad = true;
                        break;
                    }
                    for (int k = 0; k < m; ++k) row[base + k] = fixed(pre[k]);
                    e = base + m;
                    if (X.lo < kLim) {
                        if (adj & (X.rs == eprs)) {
                            X.rs = ers;
                            X.cnt += dcnt;
                        }
                        row[e] = spk_run_t{(uint32_t)(X.rs + f0), (uint32_t)X.cnt};
                        ++e;
                    }
                }
            }
        }
        // the run open at the shard end continues in the next shard (it comes
        // back there as the entry run); the last shard keeps it
        if ((r < S - 1) & (X.lo < kLim) & (e > b)) --e;
        SPK_CHECK((b >= (int64_t)r * a.rstride) & (b <= e) & (e <= (int64_t)(r + 1) * a.rstride));
        sg[2 * r] = (uint32_t)b;
        sg[2 * r + 1] = (uint32_t)e;
        total += (uint32_t)(e - b);
        if (X.last != kNoSpike) last_abs = X.last + f0;
        E = X;
        shift_state(E, len);
        Xp = Xs;
    }
    a.flags[p] = bad ? 1 : 0;
    if (bad) {
        atomicAdd(a.nflag, 1u);
        return;  // the re-scan writes seg / counts / last
    }
    a.counts[p] = total;
    a.last[p] = last_abs;
}

template __global__ void k_split_combine<kFSR>(SplitArgs);
template __global__ void k_split_combine<kSSR>(SplitArgs);

// the state at the start of a stream (Scan::init), for the first shard's entry
__global__ void __launch_bounds__(256) k_state_fresh(int32_t* st, int64_t npix) {
    const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= npix) return;
    Scan<kSSR> s;  // FSR and SSR share the layout
    s.init();
    s.save(st, npix, p);
}

template __global__ void k_resolve<kFSR>(ShardArgs);
template __global__ void k_resolve<kSSR>(ShardArgs);
template __global__ void k_junction<kFSR>(ShardArgs);
template __global__ void k_junction<kSSR>(ShardArgs);
template __global__ void k_stitch<kFSR>(ShardArgs);
template __global__ void k_stitch<kSSR>(ShardArgs);

}  // namespace spk
