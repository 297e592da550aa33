"""The product's streaming FSR/SSR state machine (csrc/spk_fsm.cuh), compiled
for the host by nvcc, reproduces the oracle's batch segmentation exactly.

This is the header the sm_100a segment kernel runs; testing it on the CPU
pins the state-machine logic independently of the GPU plumbing.
"""
import ctypes as C
import zlib
import subprocess
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
SRC = ROOT / "tests" / "native" / "fsm_host.cu"
LIB = ROOT / "tests" / "native" / "libfsm_host.so"
HDR = ROOT / "paper_2412_11639_b200" / "csrc" / "spk_fsm.cuh"


@pytest.fixture(scope="module")
def fsm():
    if not LIB.exists() or LIB.stat().st_mtime < max(SRC.stat().st_mtime, HDR.stat().st_mtime,
                                                      (HDR.parent / "spk_common.cuh").stat().st_mtime):
        subprocess.run(["nvcc", "-O2", "-std=c++17", "-arch=sm_100a", "-Xcompiler", "-fPIC",
                        "-shared", "-diag-suppress", "20011", f"-I{ROOT / 'include'}", "-o",
                        str(LIB), str(SRC)], check=True)
    h = C.CDLL(str(LIB))
    h.fsm_runs.restype = C.c_long
    h.fsm_runs.argtypes = [C.c_void_p, C.c_long, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p,
                           C.c_long]

    h.scan_runs.restype = C.c_long
    h.scan_runs.argtypes = h.fsm_runs.argtypes
    h.word_runs.restype = C.c_long
    h.word_runs.argtypes = h.fsm_runs.argtypes
    h.batch_runs.restype = C.c_long
    h.batch_runs.argtypes = h.fsm_runs.argtypes
    h.quiet_runs.restype = C.c_long
    h.quiet_runs.argtypes = h.fsm_runs.argtypes
    h.ssr_state_check.restype = C.c_long
    h.ssr_state_check.argtypes = [C.c_void_p, C.c_long]
    h.ssrword_runs.restype = C.c_long
    h.ssrword_runs.argtypes = h.fsm_runs.argtypes
    h.scanmem_runs.restype = C.c_long
    h.scanmem_runs.argtypes = h.fsm_runs.argtypes

    def make(fn):
        def run(bits, m):
            cap = bits.size + 1
            s, e, c = (np.zeros(cap, np.int64) for _ in range(3))
            n = fn(bits.ctypes.data, bits.size, m, s.ctypes.data, e.ctypes.data,
                   c.ctypes.data, cap)
            return s[:n], e[:n], c[:n]
        return run
    return {"fsm": make(h.fsm_runs), "scan": make(h.scan_runs), "word": make(h.word_runs),
            "batch": make(h.batch_runs), "quiet": make(h.quiet_runs),
            "ssrword": make(h.ssrword_runs), "scanmem": make(h.scanmem_runs), "_h": h}


def if_stream(rng, t, segs, flips):
    b = np.zeros(t, np.uint8)
    r = rng.random()
    for k in range(segs):
        q = rng.uniform(0.005, 1.0)
        for n in range(k * t // segs, (k + 1) * t // segs):
            r += q
            if r >= 1 - 1e-9:
                b[n] = 1
                r -= 1
    return b ^ (rng.random(t) < flips).astype(np.uint8)


@pytest.mark.parametrize("kind", ["fsm", "scan", "word", "batch", "quiet", "ssrword", "scanmem"])
@pytest.mark.parametrize("family", ["noise", "if", "if_noisy", "if_rare_flips"])
def test_fsm_matches_oracle(fsm, oracle, family, kind):
    run = fsm[kind]
    rng = np.random.default_rng(zlib.crc32(family.encode()))
    for _ in range(2500):
        t = int(rng.integers(0, 700))
        if family == "noise":
            b = (rng.random(t) < rng.uniform(0.01, 0.95)).astype(np.uint8)
        else:
            flips = {"if": 0.0, "if_noisy": 0.03, "if_rare_flips": 0.002}[family]
            b = if_stream(rng, t, int(rng.integers(1, 5)), flips)
        for m in (0, 1):
            got, want = run(b, m), oracle.runs(b, m)
            assert all(np.array_equal(x, y) for x, y in zip(got, want)), (family, m, t)


@pytest.mark.parametrize("kind", ["fsm", "scan", "word", "batch", "quiet", "ssrword", "scanmem"])
def test_fsm_golden_rows(fsm, golden_dir, kind):
    z = np.load(golden_dir / "rows.npz")
    for name in sorted({k.split("/")[0] for k in z.files}):
        bits = z[f"{name}/bits"]
        for m, tag in ((0, "fsr"), (1, "ssr")):
            s, e, n = z[f"{name}/{tag}_seg"]
            keep = n > 0
            got = fsm[kind](bits, m)
            assert np.array_equal(got[0], s[keep]) and np.array_equal(got[1], e[keep]) \
                and np.array_equal(got[2], n[keep]), (name, tag)


def test_run_u8_exact_vs_integer_rule(fsm):
    """The kernels' u8 run value == round-half-away(255 N / span) computed with
    exact integers (SURVEY finding 6), over random and boundary (N, span)."""
    h = C.CDLL(str(LIB))
    h.host_run_u8.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_long]
    rng = np.random.default_rng(9)
    span = np.concatenate([rng.integers(1, 1 << 29, 200000), rng.integers(1, 2000, 200000),
                           np.arange(1, 3000)]).astype(np.uint32)
    n = (rng.random(span.size) * (span.astype(np.float64) + 1)).astype(np.uint64)
    n = np.minimum(n, span).astype(np.uint32)
    n[:1000] = span[:1000]          # N == span -> 255
    n[1000:2000] = 1                # smallest
    # exact half ties: 255 N / span = k + 1/2  <=>  510 N = (2k+1) span
    k = rng.integers(0, 255, 1000).astype(np.uint64)
    ts = (rng.integers(1, 1 << 20, 1000) * 510).astype(np.uint64)
    span[2000:3000] = ts.astype(np.uint32)
    n[2000:3000] = ((2 * k + 1) * ts // 510).astype(np.uint32)
    out = np.zeros(span.size, np.uint32)
    h.host_run_u8(n.ctypes.data, span.ctypes.data, out.ctypes.data, span.size)
    want = (510 * n.astype(np.uint64) + span) // (2 * span.astype(np.uint64))
    assert np.array_equal(out, want.astype(np.uint32))
    # and equals quantize() of the reference double
    v = 255.0 * n.astype(np.float64) / span.astype(np.float64)
    assert np.array_equal(out, np.floor(np.clip(v, 0, 255) + 0.5).astype(np.uint32))
    # every (N, span) with span <= 1536, and spans around the fast path's 2^22 limit
    sp = np.repeat(np.arange(1, 1537, dtype=np.uint32), 1537)
    nn = np.tile(np.arange(0, 1537, dtype=np.uint32), 1536)
    keep = nn <= sp
    sp, nn = sp[keep], nn[keep]
    edge = rng.integers((1 << 22) - 4000, (1 << 22) + 4000, 100000).astype(np.uint32)
    sp = np.concatenate([sp, edge])
    nn = np.concatenate([nn, (rng.random(edge.size) * (edge + 1.0)).astype(np.uint32)])
    nn = np.minimum(nn, sp)
    out = np.zeros(sp.size, np.uint32)
    h.host_run_u8(nn.ctypes.data, sp.ctypes.data, out.ctypes.data, sp.size)
    want = (510 * nn.astype(np.uint64) + sp) // (2 * sp.astype(np.uint64))
    assert np.array_equal(out, want.astype(np.uint32))


@pytest.mark.parametrize("kind", ["batch", "quiet", "ssrword"])
def test_bulk_drivers_long_streams(fsm, oracle, kind):
    """long stable runs (rates near integer reciprocals, slow drifts, rare
    flips): the bit-parallel tests accept many words in a row"""
    run = fsm[kind]
    rng = np.random.default_rng(20250)
    for _ in range(300):
        t = int(rng.integers(1000, 6000))
        r, b = rng.random(), np.zeros(t, np.uint8)
        base = 1.0 / (int(rng.integers(1, 40)) + rng.choice([0.0, 1e-4, 0.37, 0.5, 0.999]))
        drift = rng.uniform(-1e-6, 1e-6)
        for n in range(t):
            r += min(1.0, max(0.001, base + drift * n))
            if r >= 1 - 1e-9:
                b[n] = 1
                r -= 1
        b ^= (rng.random(t) < rng.choice([0.0, 0.0005, 0.01])).astype(np.uint8)
        for m in (0, 1):
            got, want = run(b, m), oracle.runs(b, m)
            assert all(np.array_equal(x, y) for x, y in zip(got, want)), (m, t)


@pytest.mark.parametrize("seed", range(6))
def test_ssr_bulk_state_equals_exact_steps(fsm, seed):
    """After every word, the SSR bulk driver (ssr_flags / ssr_accept) holds
    exactly the automaton state of the per-spike steps (all 16 fields)."""
    rng = np.random.default_rng(seed)
    for _ in range(300):
        t = int(rng.integers(1, 3000))
        kind = rng.integers(0, 3)
        if kind == 0:  # piecewise-constant rates (runs of regular spikes)
            bits = np.zeros(t, np.uint8)
            acc, q = rng.uniform(0, 1), rng.uniform(0.02, 1.0)
            for f in range(t):
                if rng.random() < 0.003:
                    q = rng.uniform(0.02, 1.0)
                acc += q
                if acc >= 1.0:
                    acc -= 1.0
                    bits[f] = 1
            bits ^= (rng.random(t) < rng.choice([0.0, 0.002, 0.01])).astype(np.uint8)
        elif kind == 1:
            bits = (rng.random(t) < rng.uniform(0.05, 0.9)).astype(np.uint8)
        else:  # slowly varying rate
            q = 0.05 + 0.4 * (1 + np.sin(np.arange(t) / rng.uniform(50, 900)))
            c = np.cumsum(q) + rng.uniform(0, 1)
            bits = (np.floor(c) != np.floor(c - q)).astype(np.uint8)
        r = fsm["_h"].ssr_state_check(bits.ctypes.data, t)
        assert r == -1, (seed, t, int(kind), divmod(r, 100))
