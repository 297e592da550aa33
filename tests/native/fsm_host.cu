// Host build of the product's streaming FSR/SSR state machine
// (paper_2412_11639_b200/csrc/spk_fsm.cuh) for CPU unit tests: the exact
// header the sm_100a kernels use, driven frame by frame on the CPU and
// compared with the oracle in tests/test_fsm_host.py.  Test code only.
#include <cstdint>
#include <vector>

#include "../../paper_2412_11639_b200/csrc/spk_fsm.cuh"
#include "../../paper_2412_11639_b200/csrc/spk_common.cuh"

namespace {
struct Collect {
    long* start;
    long* end;
    long* cnt;
    long cap;
    long n = 0;
    void run(int rs, int c, int e, int) {
        if (n < cap) {
            start[n] = rs;
            end[n] = e;
            cnt[n] = c;
        }
        ++n;
    }
    void done(int, int, int, int) {}
};
}  // namespace

extern "C" long fsm_runs(const uint8_t* bits, long frames, int method, long* start, long* end,
                         long* cnt, long cap) {
    Collect em{start, end, cnt, cap};
    if (method == 0) {
        spk::Fsm<spk::kFSR> f;
        f.init();
        for (long n = 0; n < frames; ++n)
            if (bits[n]) f.spike((int)n, em);
        f.finish((int)frames, em);
    } else {
        spk::Fsm<spk::kSSR> f;
        f.init();
        for (long n = 0; n < frames; ++n)
            if (bits[n]) f.spike((int)n, em);
        f.finish((int)frames, em);
    }
    return em.n;
}

// The branch-free Scan<METHOD> automaton of the segment kernel: runs as
// (start, intervals); a run ends where the next starts, the last at the final
// spike.
extern "C" long scan_runs(const uint8_t* bits, long frames, int method, long* start, long* end,
                          long* cnt, long cap) {
    long n = 0, last = -1;
    auto go = [&](auto& sc) {
        sc.init();
        for (long f = 0; f < frames; ++f) {
            if (!bits[f]) continue;
            int rs, c;
            if (sc.step((int)f, rs, c)) {
                if (n < cap) {
                    start[n] = rs;
                    cnt[n] = c;
                }
                ++n;
            }
            last = f;
        }
        int rs, c;
        if (sc.tail(rs, c)) {
            if (n < cap) {
                start[n] = rs;
                cnt[n] = c;
            }
            ++n;
        }
    };
    if (method == 0) {
        spk::Scan<spk::kFSR> sc;
        go(sc);
    } else {
        spk::Scan<spk::kSSR> sc;
        go(sc);
    }
    for (long k = 0; k < n && k < cap; ++k) end[k] = (k + 1 < n) ? start[k + 1] : last;
    return n;
}

// The segment kernel's word-level driver: 32-frame words with the first frame
// in bit 31; FSR through fsr_word (bulk acceptance), SSR spike by spike.
static long word_runs_impl(const uint8_t* bits, long frames, int method, long* start, long* end,
                           long* cnt, long cap, bool ssr_bulk) {
    long n = 0, last = -1;
    auto put = [&](bool e, int rs, int c) {
        if (e) {
            if (n < cap) {
                start[n] = rs;
                cnt[n] = c;
            }
            ++n;
        }
    };
    auto go = [&](auto& sc, bool bulk) {
        sc.init();
        for (long base = 0; base < frames; base += 32) {
            uint32_t w = 0;
            for (int b = 0; b < 32 && base + b < frames; ++b)
                if (bits[base + b]) {
                    w |= 0x80000000u >> b;
                    last = base + b;
                }
            if (bulk) {
                spk::fsr_word(sc, w, (int)base, put);
            } else if (ssr_bulk) {
                spk::ssr_word(sc, w, (int)base, put);
            } else {
                while (w) {
                    const int c = spk::bit_clz(w);
                    w ^= 0x80000000u >> c;
                    int rs, cc;
                    const bool e = sc.step((int)base + c, rs, cc);
                    put(e, rs, cc);
                }
            }
        }
        int rs, c;
        const bool e = sc.tail(rs, c);
        put(e, rs, c);
    };
    if (method == 0) {
        spk::Scan<spk::kFSR> sc;
        go(sc, true);
    } else {
        spk::Scan<spk::kSSR> sc;
        go(sc, false);
    }
    for (long k = 0; k < n && k < cap; ++k) end[k] = (k + 1 < n) ? start[k + 1] : last;
    return n;
}

extern "C" long word_runs(const uint8_t* bits, long frames, int method, long* start, long* end,
                          long* cnt, long cap) {
    return word_runs_impl(bits, frames, method, start, end, cnt, cap, false);
}

// SSR with the bit-parallel second-level test (ssr_word); FSR as word_runs
extern "C" long ssrword_runs(const uint8_t* bits, long frames, int method, long* start, long* end,
                             long* cnt, long cap) {
    return word_runs_impl(bits, frames, method, start, end, cnt, cap, true);
}

// The FSR window driver of the segment kernel (fsr_batch<SPK_WIN>).
extern "C" long batch_runs(const uint8_t* bits, long frames, int method, long* start, long* end,
                           long* cnt, long cap) {
    if (method != 0) return word_runs(bits, frames, method, start, end, cnt, cap);
    long n = 0, last = -1;
    auto put = [&](bool e, int rs, int c) {
        if (e) {
            if (n < cap) {
                start[n] = rs;
                cnt[n] = c;
            }
            ++n;
        }
    };
    const long ngroups = (frames + 31) / 32;
    std::vector<uint32_t> words(ngroups + 4, 0u);
    for (long f = 0; f < frames; ++f)
        if (bits[f]) {
            words[f / 32] |= 0x80000000u >> (f % 32);
            last = f;
        }
    spk::Scan<spk::kFSR> sc;
    sc.init();
    long wi = 0;
    int cpos = 0;
    while (wi < ngroups)
        wi += spk::fsr_batch<SPK_WIN>(sc, [&](int j) { return words[wi + j]; }, (int)(wi * 32), cpos, put);
    int rs, c;
    const bool e = sc.tail(rs, c);
    put(e, rs, c);
    for (long k = 0; k < n && k < cap; ++k) end[k] = (k + 1 < n) ? start[k + 1] : last;
    return n;
}

// The FSR driver of the segment kernel with quiet windows: after an
// iteration without an event, kQuiet words are tried at once (fsr_quiet),
// and the event window (fsr_batch) runs when they hold an event.
extern "C" long quiet_runs(const uint8_t* bits, long frames, int method, long* start, long* end,
                           long* cnt, long cap) {
    if (method != 0) return word_runs(bits, frames, method, start, end, cnt, cap);
    long n = 0, last = -1;
    auto put = [&](bool e, int rs, int c) {
        if (e) {
            if (n < cap) {
                start[n] = rs;
                cnt[n] = c;
            }
            ++n;
        }
    };
    const long ngroups = (frames + 31) / 32;
    std::vector<uint32_t> words(ngroups + spk::kQuiet, 0u);
    for (long f = 0; f < frames; ++f)
        if (bits[f]) {
            words[f / 32] |= 0x80000000u >> (f % 32);
            last = f;
        }
    spk::Scan<spk::kFSR> sc;
    sc.init();
    long wi = 0;
    int cpos = 0;
    bool quiet = false;
    while (wi < ngroups) {
        if (quiet && spk::fsr_quiet<spk::kQuiet>(sc, [&](int k) { return words[wi + k]; }, (int)(wi * 32),
                                                 cpos)) {
            wi += spk::kQuiet;
            continue;
        }
        const int k = spk::fsr_batch<SPK_WIN>(sc, [&](int j) { return words[wi + j]; }, (int)(wi * 32), cpos, put);
        quiet = k == SPK_WIN;
        wi += k;
    }
    int rs, c;
    const bool e = sc.tail(rs, c);
    put(e, rs, c);
    for (long k = 0; k < n && k < cap; ++k) end[k] = (k + 1 < n) ? start[k + 1] : last;
    return n;
}

// Scan<kSSR>::step_mem (parity slots in memory, as in K2's SSR spike loop);
// the first `warm` spikes go through step() so the slots move from registers
// to memory with some state in them.  FSR: the plain step.
extern "C" long scanmem_runs(const uint8_t* bits, long frames, int method, long* start, long* end,
                             long* cnt, long cap) {
    if (method == 0) return scan_runs(bits, frames, method, start, end, cnt, cap);
    long n = 0, last = -1, seen = 0;
    const long warm = frames % 7;
    spk::Scan<spk::kSSR> sc;
    sc.init();
    int4 slots[2];
    auto slot = [&](int k) -> int4& { return slots[k]; };
    auto put = [&](bool e, int rs, int c) {
        if (!e) return;
        if (n < cap) {
            start[n] = rs;
            cnt[n] = c;
        }
        ++n;
    };
    for (long f = 0; f < frames; ++f) {
        if (!bits[f]) continue;
        int rs, c;
        bool e;
        if (seen < warm) {
            e = sc.step((int)f, rs, c);
        } else {
            if (seen == warm) sc.store_slots(slot);
            e = sc.step_mem((int)f, slot, rs, c);
        }
        put(e, rs, c);
        ++seen;
        last = f;
    }
    int rs, c;
    const bool e = sc.tail(rs, c);
    put(e, rs, c);
    for (long k = 0; k < n && k < cap; ++k) end[k] = (k + 1 < n) ? start[k + 1] : last;
    return n;
}

// the u8 run-value rule as compiled for the kernels
extern "C" void host_run_u8(const uint32_t* n, const uint32_t* span, uint32_t* out, long m) {
    for (long i = 0; i < m; ++i) out[i] = spk::run_u8(n[i], span[i]);
}

// profiling aid: fsr_batch iterations and events (exact steps) for one pixel
extern "C" void batch_iters(const uint8_t* bits, long frames, long* iters, long* events) {
    const long ngroups = (frames + 31) / 32;
    std::vector<uint32_t> words(ngroups + 4, 0u);
    for (long f = 0; f < frames; ++f)
        if (bits[f]) words[f / 32] |= 0x80000000u >> (f % 32);
    spk::Scan<spk::kFSR> sc;
    sc.init();
    long wi = 0, it = 0, ev = 0;
    int cpos = 0;
    auto put = [&](bool, int, int) {};
    while (wi < ngroups) {
        const int k = spk::fsr_batch<SPK_WIN>(sc, [&](int j) { return words[wi + j]; }, (int)(wi * 32), cpos, put);
        ev += cpos != 0;
        wi += k;
        ++it;
    }
    *iters = it;
    *events = ev;
}

// SSR bulk words (ssr_word) leave exactly the automaton state of the
// per-spike steps after every word: returns the first word whose state
// differs, or -1.
extern "C" long ssr_state_check(const uint8_t* bits, long frames) {
    const long ng = (frames + 31) / 32;
    std::vector<uint32_t> w(ng + 1, 0u);
    for (long f = 0; f < frames; ++f)
        if (bits[f]) w[f / 32] |= 0x80000000u >> (f % 32);
    spk::Scan<spk::kSSR> a, b;
    a.init();
    b.init();
    auto put = [&](bool, int, int) {};
    for (long i = 0; i < ng; ++i) {
        const int base = (int)(i * 32);
        spk::ssr_word(a, w[i], base, put);
        for (uint32_t s = w[i]; s;) {
            const int c = spk::bit_clz(s);
            s ^= 0x80000000u >> c;
            int rs, cnt;
            b.step(base + c, rs, cnt);
        }
        const int32_t va[] = {a.last, a.lo, a.rs, a.cnt, (int32_t)a.hw, a.ii, a.sub0, a.l0, a.l1,
                              a.g0, a.g1, (int32_t)a.h0, (int32_t)a.h1, a.fl0, a.fl1, a.sf};
        const int32_t vb[] = {b.last, b.lo, b.rs, b.cnt, (int32_t)b.hw, b.ii, b.sub0, b.l0, b.l1,
                              b.g0, b.g1, (int32_t)b.h0, (int32_t)b.h1, b.fl0, b.fl1, b.sf};
        for (int k = 0; k < 16; ++k)
            if (va[k] != vb[k]) return i * 100 + k;
    }
    return -1;
}
