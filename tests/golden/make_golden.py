"""Generate tests/golden/*.npz from the UNMODIFIED reference library.

Run in the build container (needs oracle/_ref/libspikecam_ref.so, i.e.
/root/reference): `python tests/golden/make_golden.py`.  The fixtures are the
reference's own outputs on (a) the known-answer streams of proj/tests/
test_reconstruct.cpp and acceptance.cpp, re-created here from their published
parameters, and (b) small seeded volumes, so the GPU box can check parity
without the reference checkout.  Expected values are never written by hand.
"""
from __future__ import annotations

import hashlib
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
from oracle.oracle import Reference  # noqa: E402

OUT = Path(__file__).resolve().parent
REF = Reference()


def from_intervals(first, gaps, total):
    """helpers.hpp stream_from_intervals (proj/tests/helpers.hpp:12-20)."""
    pos = [first]
    for g in gaps:
        pos.append(pos[-1] + g)
    frames = max(total, pos[-1] + 1)
    b = np.zeros(frames, np.uint8)
    b[pos] = 1
    return b


def constant(q, frames):
    return REF.simulate_pixel(np.full(frames, q))


def mixed(rng, lo=64, hi=512, flips=0.0):
    """random_mixed_stream-like generator (proj/tests/helpers.hpp:24-48) on numpy's RNG."""
    frames = int(rng.integers(lo, hi + 1))
    runs = int(rng.integers(1, 5))
    bits, r = [], 0.0
    for _ in range(runs):
        q = rng.uniform(0.02, 1.0)
        for _ in range(frames // runs):
            r += q
            if r >= 1.0 - 1e-9:
                bits.append(1)
                r -= 1.0
            else:
                bits.append(0)
    b = np.array(bits, np.uint8)
    if flips:
        b ^= (rng.random(b.size) < flips).astype(np.uint8)
    return b


def rows():
    cases = {
        "worked_example": from_intervals(0, [3, 3, 4, 3, 7, 6, 7], 40),
        "worked_example_tight": from_intervals(0, [3, 3, 4, 3, 7, 6, 7], 0),
        "ssr_no_break": from_intervals(0, [3, 3, 4, 3], 20),
        "const_q03_1000": constant(0.3, 1000),
        "const_q03_2000": constant(0.3, 2000),
        "const_q03_1024": constant(0.3, 1024),
        "const_q05_256": constant(0.5, 256),
        "two_phase": REF.simulate_pixel(np.r_[np.full(500, 0.3), np.full(500, 0.125)]),
        "ssr_split": REF.simulate_pixel(np.r_[np.full(600, 1 / 3.1), np.full(600, 1 / 3.9)]),
        "tfp_example": from_intervals(3, [4] * 20, 84),
        "tfi_example": from_intervals(1, [2, 2, 2], 10),
        "periodic_2": from_intervals(1, [2] * 40, 0),
        "periodic_3": from_intervals(2, [3] * 40, 0),
        "periodic_5": from_intervals(4, [5] * 40, 0),
        "all_zero_50": np.zeros(50, np.uint8),
        "empty": np.zeros(0, np.uint8),
        "single_spike": from_intervals(7, [], 20),
        "two_spikes": from_intervals(3, [5], 12),
        "spike_at_0_and_end": from_intervals(0, [19], 20),
        "saturated": np.ones(100, np.uint8),
    }
    rng = np.random.default_rng(41)
    for i in range(40):
        cases[f"mixed_{i:02d}"] = mixed(rng)
    rng = np.random.default_rng(1019)
    for i in range(40):
        cases[f"noisy_{i:02d}"] = mixed(rng, flips=1 / 64)
    return cases


def save_rows():
    cases = rows()
    data = {}
    for name, b in cases.items():
        data[f"{name}/bits"] = b
        for m, tag in ((0, "fsr"), (1, "ssr")):
            s, e, n, v = REF.segments(b, m)
            data[f"{name}/{tag}_seg"] = np.stack([s, e, n]).astype(np.int64)
            data[f"{name}/{tag}_segval"] = v
        for m, tag, win in ((0, "fsr", 32), (1, "ssr", 32), (2, "tfi", 32), (3, "tfp32", 32),
                            (3, "tfp7", 7), (3, "tfp1", 1)):
            data[f"{name}/{tag}_pix"] = REF.reconstruct_pixel(b, m, win)
        d, v = REF.fsr_events(b)
        data[f"{name}/events"] = np.stack([d.astype(np.float64), v])
        for blk in (1 << 30, 32, 7):
            d2, v2 = REF.stream_events(b, blk)
            assert np.array_equal(d, d2) and np.array_equal(v, v2), (name, blk)
    np.savez_compressed(OUT / "rows.npz", **data)
    print("rows.npz:", len(cases), "streams")


def pack(bits, w, h):
    t = bits.shape[0]
    npix = w * h
    fb = (npix + 7) // 8
    planes = np.zeros((t, fb), np.uint8)
    for p in range(npix):
        planes[:, p >> 3] |= (bits[:, p].astype(np.uint8) & 1) << (p & 7)
    return planes


def scene_volume(w, h, t, rate):
    bits = np.zeros((t, w * h), np.uint8)
    for y in range(h):
        for x in range(w):
            r = np.array([rate(x, y, n) for n in range(t)], dtype=np.float64)
            bits[:, y * w + x] = REF.simulate_pixel(r)
    return bits


def save_volume(name, bits, w, h, methods):
    t = bits.shape[0]
    planes = pack(bits, w, h)
    fb = planes.shape[1]
    data = {"planes": planes, "geom": np.array([w, h, t], np.int64)}
    for m, tag, win in methods:
        f, u = REF.reconstruct(planes, fb, w, h, t, m, win, workers=3)
        s = REF.reconstruct_serial(planes, fb, w, h, t, m, win)
        assert np.array_equal(f.view(np.uint64), s.view(np.uint64)), (name, tag)
        data[f"{tag}/u8"] = u
        data[f"{tag}/f64_sha256"] = np.frombuffer(hashlib.sha256(f.tobytes()).digest(), np.uint8)
        if f.size <= 40000:
            data[f"{tag}/f64"] = f
    np.savez_compressed(OUT / f"vol_{name}.npz", **data)
    print(f"vol_{name}.npz", w, h, t)


def save_crit9():
    """proj/tests/acceptance.cpp:231-236 (criterion 9, the benchmark floor):
    400x250x320, static rates 0.05 + 0.9*((31x + 17y) mod 20)/19, default
    simulate options (threshold 1, residual 0) -- 20 distinct pixel streams.
    Stored: the planes and SHA-256 of the reference's FSR/SSR outputs (f64
    doubles and quantised uint8 frames; the frames themselves are 32 MB)."""
    w, h, t = 400, 250, 320
    streams = [REF.simulate_pixel(np.full(t, 0.05 + 0.9 * c / 19.0)) for c in range(20)]
    bits = np.zeros((t, w * h), np.uint8)
    for y in range(h):
        for x in range(w):
            bits[:, y * w + x] = streams[(x * 31 + y * 17) % 20]
    planes = pack(bits, w, h)
    fb = planes.shape[1]
    data = {"planes": planes, "geom": np.array([w, h, t], np.int64)}
    for m, tag in ((0, "fsr"), (1, "ssr")):
        f, u = REF.reconstruct(planes, fb, w, h, t, m, 32, workers=4)
        data[f"{tag}/f64_sha256"] = np.frombuffer(hashlib.sha256(f.tobytes()).digest(), np.uint8)
        data[f"{tag}/u8_sha256"] = np.frombuffer(hashlib.sha256(u.tobytes()).digest(), np.uint8)
    np.savez_compressed(OUT / "vol_crit9.npz", **data)
    print("vol_crit9.npz", w, h, t)


def save_records():
    """SPKR images of the golden volumes from the reference's --emit-records
    loop (proj/tools/spikecam_main.cpp:146-172 -> write_spkr), plus a
    long-duration case (> 255-frame segments split into several words)."""
    import tempfile
    data = {}
    vols = {}
    for name in ("par12x9", "bar64x48", "noise40x25", "odd9x1", "odd13x7"):
        g = np.load(OUT / f"vol_{name}.npz")
        vols[name] = (g["planes"], *(int(x) for x in g["geom"]))
    # sparse pixels: silent, single spike, ISI > 255, runs longer than 255 frames
    rng = np.random.default_rng(83)
    w, h, t = 7, 3, 2600
    bits = np.zeros((t, w * h), np.uint8)
    for p in range(w * h):
        kind = p % 5
        if kind == 1:
            bits[int(rng.integers(0, t)), p] = 1
        elif kind == 2:
            bits[int(rng.integers(0, 300))::int(rng.integers(256, 700)), p] = 1
        elif kind == 3:
            bits[int(rng.integers(0, 5))::int(rng.integers(2, 9)), p] = 1
        elif kind == 4:
            bits[:, p] = (rng.random(t) < 0.02).astype(np.uint8)
    vols["sparse7x3"] = (pack(bits, w, h), w, h, t)
    data["sparse7x3/planes"] = vols["sparse7x3"][0]
    data["sparse7x3/geom"] = np.array([w, h, t], np.int64)
    with tempfile.TemporaryDirectory() as d:
        for name, (planes, w, h, t) in vols.items():
            for m, tag in ((0, "fsr"), (1, "ssr")):
                f = Path(d) / f"{name}_{tag}.spkr"
                REF.emit_records(planes, planes.shape[1], w, h, t, m, 20000, f)
                data[f"{name}/{tag}"] = np.fromfile(f, np.uint8)
    np.savez_compressed(OUT / "records.npz", **data)
    print("records.npz:", len(vols), "volumes")


ALL = [(0, "fsr", 32), (1, "ssr", 32), (2, "tfi", 32), (3, "tfp32", 32), (3, "tfp16", 16),
       (3, "tfp3", 3)]


def main():
    save_rows()
    # proj/tests/test_reconstruct.cpp:250-267 scene (serial == parallel test)
    save_volume("par12x9", scene_volume(12, 9, 200, lambda x, y, n: 0.1 + 0.8 * (
        (x * 31 + y * 17 + n // 64) % 10) / 10.0), 12, 9, ALL)
    # proj/tests/acceptance.cpp:165-173 moving-bar scene
    def bar(x, y, n):
        bg = 0.12 + 0.55 * ((x * 7 + y * 13) % 32) / 31.0
        d = (x - (n // 8) % 64 + 64) % 64
        return 0.92 if d < 6 else bg
    save_volume("bar64x48", scene_volume(64, 48, 288, bar), 64, 48, ALL)
    rng = np.random.default_rng(61)
    save_volume("noise40x25", (rng.random((300, 40 * 25)) < 0.3).astype(np.uint8), 40, 25, ALL)
    rng = np.random.default_rng(67)
    save_volume("odd9x1", (rng.random((1100, 9)) < 0.4).astype(np.uint8), 9, 1, ALL)
    rng = np.random.default_rng(71)
    save_volume("odd13x7", (rng.random((45, 91)) < 0.2).astype(np.uint8), 13, 7, ALL)
    # SPK1 golden bytes (proj/tests/test_io.cpp:49-62)
    import tempfile
    with tempfile.TemporaryDirectory() as d:
        f = Path(d) / "g.spk"
        REF.write_spk(np.array([[1]], np.uint8), 1, 2, 1, 1, 20000, f)
        gold = np.fromfile(f, np.uint8)
        f2 = Path(d) / "pad.spk"
        REF.write_spk(np.array([[0xFF, 0x01]], np.uint8), 2, 9, 1, 1, 20000, f2)
        pad = np.fromfile(f2, np.uint8)
        vals = np.array([[0.0, 127.5, 127.49999, 254.5, 255.0, 0.5, 1.5, 2.5]], np.float64)
        f3 = Path(d) / "q.pgm"
        REF.write_pgm(vals, 8, 1, f3)
        pgm = np.fromfile(f3, np.uint8)[-8:]
    np.savez_compressed(OUT / "formats.npz", spk_golden=gold, spk_pad=pad, quant_in=vals,
                        quant_out=pgm)
    print("formats.npz")
    save_records()
    save_metrics()
    save_crit9()


def stab_rows(bits_list, depth):
    res = [REF.stability(b, depth) for b in bits_list]
    arr = np.array([[r["depth"], r["index"], r["verified_order"], int(r["absolute"])]
                    for r in res], np.int64)
    return arr, np.array([r["path"] for r in res])


def save_metrics():
    """Quality metrics (two_dimensional_entropy / mse / psnr, metrics.cpp:12-61)
    and stability_order (stability.cpp:112-128) from the reference library."""
    data = {}
    rng = np.random.default_rng(97)
    imgs = {"rand9x13": rng.uniform(-5.0, 260.0, (9, 13)), "const3x3": np.full((3, 3), 77.25),
            "ramp5x4": np.arange(20, dtype=np.float64).reshape(4, 5) * 12.75}
    for k, v in imgs.items():
        data[f"img/{k}"] = v
        data[f"img/{k}/te"] = np.float64(REF.te(v))
    # frames of the moving-bar volume: FSR values vs TFI frames as the reference images
    g = np.load(OUT / "vol_bar64x48.npz")
    planes = g["planes"]
    w, h, t = (int(x) for x in g["geom"])
    f, _ = REF.reconstruct(planes, planes.shape[1], w, h, t, 0, 32)
    _, tfi = REF.reconstruct(planes, planes.shape[1], w, h, t, 2, 32)
    f = f.reshape(t, h, w)
    tfi = tfi.reshape(t, h, w).astype(np.float64)
    data["bar/te_fsr"] = np.array([REF.te(f[n]) for n in range(t)])
    data["bar/mse_fsr_tfi"] = np.array([REF.mse(f[n], tfi[n]) for n in range(t)])
    data["bar/psnr_fsr_tfi"] = np.array([REF.psnr(f[n], tfi[n]) for n in range(t)])
    # stability_order on the known-answer rows and a constant-rate sweep
    # (cmd_verify_stability, spikecam_main.cpp:209-225: log-spaced q, length 2048)
    cases = rows()
    names = sorted(cases)
    data["rows/names"] = np.array(names)
    for depth in (1, 3, 8):
        a, pth = stab_rows([cases[n] for n in names], depth)
        data[f"rows/d{depth}"] = a
        data[f"rows/d{depth}/path"] = pth
    qs = 0.01 * (1.0 / 0.01) ** (np.arange(40) / 39.0)
    sweep = [REF.simulate_pixel(np.full(2048, q)) for q in qs]
    data["sweep/bits"] = np.stack(sweep)
    a, pth = stab_rows(sweep, 8)
    data["sweep/d8"] = a
    data["sweep/d8/path"] = pth
    # per-pixel reports of whole golden volumes (verify-stability --in)
    for name, depth in (("bar64x48", 8), ("noise40x25", 8), ("par12x9", 4), ("odd9x1", 8)):
        gv = np.load(OUT / f"vol_{name}.npz")
        pl = gv["planes"]
        w, h, t = (int(x) for x in gv["geom"])
        bits = np.stack([(pl[:, p >> 3] >> (p & 7)) & 1 for p in range(w * h)]).astype(np.uint8)
        a, pth = stab_rows(list(bits), depth)
        data[f"vol/{name}/d{depth}"] = a
        data[f"vol/{name}/d{depth}/path"] = pth
    np.savez_compressed(OUT / "metrics.npz", **data)
    print("metrics.npz")


if __name__ == "__main__":
    if sys.argv[1:] == ["records"]:
        save_records()
    elif sys.argv[1:] == ["metrics"]:
        save_metrics()
    else:
        main()
