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

// FSR shortcut: when the speculative scan had no break in the whole shard, the
// shard's intervals all lie in its final pair, so the true automaton never
// breaks either iff E's pair, the boundary-crossing interval and that pair fit
// one pair {x, x+1} -- then its end state follows without a scan.  (Pixels
// whose speculative pair never completes in a long shard would otherwise keep
// their warp scanning to the shard end.)
__device__ bool fsr_no_break(const ShardArgs& a, int64_t p, const Scan<kFSR>& E, Scan<kFSR>& X) {
    if (a.scount[p] > 1u) return false;  // the speculative scan broke in the shard
    Scan<kFSR> S;
    S.restore(a.sstate, a.npix, p);
    if (S.last == kNoSpike) {  // no spike in the shard
        X = E;
        return true;
    }
    if (E.last == kNoSpike) {  // nothing before: the true scan is the speculative one
        X = S;
        return true;
    }
    const bool hasS = S.lo < kLim;  // >= 2 spikes in the shard
    const int f1 = hasS ? (int)a.spec[p * a.scap].start : S.last;
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

}  // namespace

// Thread per pixel in warp lockstep over 32-frame words: lanes load the
// transposed words as K2 does and walk their spikes with both automata until
// every lane of the warp has synced (or the shard ends).
template <int METHOD>
__global__ void __launch_bounds__(64) k_resolve(ShardArgs a) {
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
    }
    spk_run_t* pre = a.prefix + (valid ? p * a.pcap : 0);
    int m = 0;
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
            S.step(n, rs, cnt);
            if (T.same_future(S)) {
                out = spk_sync_t{T.rs, S.rs, T.cnt - S.cnt, m};
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
