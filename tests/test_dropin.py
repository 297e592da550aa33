"""The C++ drop-in (include/spikecam/b200.hpp) against the reference's outputs.

A C++ program (tests/native/dropin_test.cpp) uses the drop-in exactly as the
reference's callers use the reference library; its dumps are compared with
the golden fixtures generated from the unmodified reference
(tests/golden/make_golden.py).  Bar: bit-exact (segments, doubles, uint8).
"""
from __future__ import annotations

import hashlib
import subprocess
from pathlib import Path

import numpy as np
import pytest

from paper_2412_11639_b200 import build as pkg_build

HERE = Path(__file__).resolve().parent
SRC = HERE / "native" / "dropin_test.cpp"
EXE = HERE / "native" / "dropin_test"


@pytest.fixture(scope="module")
def exe():
    return pkg_build.build_cpp_program(SRC, EXE)


def run(exe, *args, timeout=600):
    r = subprocess.run([str(exe), *map(str, args)], capture_output=True, text=True, timeout=timeout)
    assert r.returncode == 0, r.stderr[-4000:]
    return r


def test_cpp_dropin_exports(exe):
    """The drop-in library resolves every symbol of the header (link check)."""
    out = subprocess.run(["nm", "-D", "--defined-only", str(pkg_build.CPP_LIB)], capture_output=True,
                         text=True, check=True).stdout
    demangled = subprocess.run(["c++filt"], input=out, capture_output=True, text=True).stdout
    for name in ["spikecam::reconstruct(", "spikecam::reconstruct_serial(", "spikecam::segment_fsr(",
                 "spikecam::segment_ssr(", "spikecam::fsr_events(", "spikecam::reconstruct_pixel(",
                 "spikecam::read_spk(", "spikecam::write_spk(", "spikecam::read_raw(",
                 "spikecam::write_image(", "spikecam::read_image(", "spikecam::reconstruct_u8(",
                 "spikecam::SpikeVolume::SpikeVolume(", "spikecam::ReconMethod::parse(",
                 "spikecam::two_dimensional_entropy(", "spikecam::mse(", "spikecam::psnr(",
                 "spikecam::stability_order("]:
        assert name in demangled, name


def test_cpp_dropin_host_selftest(exe, tmp_path):
    """Container / file-format / error rules of the drop-in; no GPU call."""
    run(exe, "selftest", tmp_path)


@pytest.mark.gpu
def test_cpp_dropin_gpucheck(exe):
    run(exe, "gpucheck")


def _segs(buf, off):
    k = int(np.frombuffer(buf, np.uint32, 1, off)[0])
    off += 4
    rec = np.frombuffer(buf, np.dtype([("s", "<i8"), ("e", "<i8"), ("n", "<i8"), ("v", "<f8")]), k, off)
    return rec, off + 32 * k


@pytest.mark.gpu
def test_cpp_dropin_rows_match_reference(exe, golden_dir, tmp_path):
    """segment_fsr / segment_ssr / reconstruct_pixel / fsr_events on the
    reference's known-answer and random streams (test_reconstruct.cpp cases)."""
    g = np.load(golden_dir / "rows.npz")
    names = sorted({k.split("/")[0] for k in g.files})
    with open(tmp_path / "in.bin", "wb") as f:
        f.write(np.uint32(len(names)).tobytes())
        for n in names:
            b = g[f"{n}/bits"].astype(np.uint8)
            f.write(np.uint32(b.size).tobytes())
            f.write(b.tobytes())
    run(exe, "rows", tmp_path / "in.bin", tmp_path / "out.bin")
    buf = (tmp_path / "out.bin").read_bytes()
    off = 0
    for n in names:
        t = g[f"{n}/bits"].size
        for tag in ("fsr", "ssr"):
            rec, off = _segs(buf, off)
            seg = g[f"{n}/{tag}_seg"]
            assert np.array_equal(rec["s"], seg[0]) and np.array_equal(rec["e"], seg[1]), (n, tag)
            assert np.array_equal(rec["n"], seg[2]), (n, tag)
            assert np.array_equal(rec["v"].view(np.uint64), g[f"{n}/{tag}_segval"].view(np.uint64)), (n, tag)
        for tag in ("fsr", "ssr", "tfi", "tfp32", "tfp7", "tfp1"):
            pix = np.frombuffer(buf, np.float64, t, off)
            off += 8 * t
            assert np.array_equal(pix.view(np.uint64), g[f"{n}/{tag}_pix"].view(np.uint64)), (n, tag)
        k = int(np.frombuffer(buf, np.uint32, 1, off)[0])
        off += 4
        ev = np.frombuffer(buf, np.dtype([("d", "<i8"), ("v", "<f8")]), k, off)
        off += 16 * k
        want = g[f"{n}/events"]
        assert np.array_equal(ev["d"], want[0].astype(np.int64)), n
        assert np.array_equal(ev["v"].view(np.uint64), want[1].view(np.uint64)), n
    assert off == len(buf)


VOLS = ["par12x9", "bar64x48", "noise40x25", "odd9x1", "odd13x7"]
TAGS = ["fsr", "ssr", "tfi", "tfp32", "tfp16", "tfp3"]


@pytest.mark.gpu
@pytest.mark.parametrize("name", VOLS)
def test_cpp_dropin_volume_matches_reference(exe, golden_dir, tmp_path, name):
    """read_spk -> reconstruct (IntensityImage doubles) and read_spk_packed ->
    reconstruct_u8 against the reference's volume outputs."""
    g = np.load(golden_dir / f"vol_{name}.npz")
    w, h, t = (int(x) for x in g["geom"])
    head = np.zeros(16, np.uint8)
    head[:4] = np.frombuffer(b"SPK1", np.uint8)
    head[4:8] = np.frombuffer(np.array([w, h], "<u2").tobytes(), np.uint8)
    head[8:16] = np.frombuffer(np.array([20000, t], "<u4").tobytes(), np.uint8)
    spk = tmp_path / "v.spk"
    spk.write_bytes(head.tobytes() + g["planes"].tobytes())
    run(exe, "vol", spk, tmp_path)
    for tag in TAGS:
        f64 = np.fromfile(tmp_path / f"{tag}.f64", np.float64)
        assert hashlib.sha256(f64.tobytes()).digest() == g[f"{tag}/f64_sha256"].tobytes(), tag
        u8 = np.fromfile(tmp_path / f"{tag}.u8", np.uint8).reshape(t, w * h)
        assert np.array_equal(u8, g[f"{tag}/u8"]), tag
        if t > 1:
            pgm = (tmp_path / f"{tag}_mid.pgm").read_bytes()
            assert np.array_equal(np.frombuffer(pgm[-w * h:], np.uint8), g[f"{tag}/u8"][t // 2]), tag


def _reports(buf):
    out, off = [], 0
    while off < len(buf):
        d, = np.frombuffer(buf, np.int32, 1, off)
        i, = np.frombuffer(buf, np.int64, 1, off + 4)
        vo, ab = np.frombuffer(buf, np.int32, 2, off + 12)
        n, = np.frombuffer(buf, np.uint32, 1, off + 20)
        path = buf[off + 24: off + 24 + int(n)].decode()
        out.append(([int(d), int(i), int(vo), int(ab)], path))
        off += 24 + int(n)
    return out


@pytest.mark.gpu
@pytest.mark.parametrize("depth", [1, 3, 8])
def test_cpp_dropin_stability_rows(exe, golden_dir, tmp_path, depth):
    """stability_order(SpikeLikeStream, depth) against the reference's reports."""
    rows = np.load(golden_dir / "rows.npz")
    gm = np.load(golden_dir / "metrics.npz")
    names = list(gm["rows/names"])
    with open(tmp_path / "in.bin", "wb") as f:
        f.write(np.uint32(len(names)).tobytes())
        for n in names:
            b = rows[f"{n}/bits"].astype(np.uint8)
            f.write(np.uint32(b.size).tobytes())
            f.write(b.tobytes())
    run(exe, "stab", tmp_path / "in.bin", tmp_path / "out.bin", depth)
    got = _reports((tmp_path / "out.bin").read_bytes())
    for i, n in enumerate(names):
        assert got[i][0] == [int(x) for x in gm[f"rows/d{depth}"][i]], n
        assert got[i][1] == str(gm[f"rows/d{depth}/path"][i]), n


@pytest.mark.gpu
def test_cpp_dropin_metrics_and_volume_stability(exe, golden_dir, tmp_path):
    """two_dimensional_entropy / mse / psnr and stability_order(SpikeVolume)
    through the C++ drop-in on the moving-bar volume."""
    g = np.load(golden_dir / "vol_bar64x48.npz")
    gm = np.load(golden_dir / "metrics.npz")
    w, h, t = (int(x) for x in g["geom"])
    head = np.zeros(16, np.uint8)
    head[:4] = np.frombuffer(b"SPK1", np.uint8)
    head[4:8] = np.frombuffer(np.array([w, h], "<u2").tobytes(), np.uint8)
    head[8:16] = np.frombuffer(np.array([20000, t], "<u4").tobytes(), np.uint8)
    spk = tmp_path / "v.spk"
    spk.write_bytes(head.tobytes() + g["planes"].tobytes())
    run(exe, "metrics", spk, tmp_path)
    te = np.fromfile(tmp_path / "te.f64", np.float64)
    want = gm["bar/te_fsr"]
    assert np.allclose(te, want, rtol=1e-12, atol=0)
    single = np.fromfile(tmp_path / "single.f64", np.float64).reshape(-1, 3)
    for k, n in enumerate(range(0, t, 37)):
        assert np.isclose(single[k, 0], want[n], rtol=1e-12, atol=0)
        assert np.isclose(single[k, 1], gm["bar/mse_fsr_tfi"][n], rtol=1e-12, atol=0)
        p = gm["bar/psnr_fsr_tfi"][n]
        assert (np.isinf(p) and np.isinf(single[k, 2])) or np.isclose(single[k, 2], p, rtol=1e-12)
    rep = _reports((tmp_path / "stab_d8.bin").read_bytes())
    wd = gm["vol/bar64x48/d8"]
    wp = gm["vol/bar64x48/d8/path"]
    assert len(rep) == w * h
    for p in range(w * h):
        assert rep[p][0] == [int(x) for x in wd[p]] and rep[p][1] == str(wp[p]), p


def _spk_file(path, planes, w, h, t):
    head = np.zeros(16, np.uint8)
    head[:4] = np.frombuffer(b"SPK1", np.uint8)
    head[4:8] = np.frombuffer(np.array([w, h], "<u2").tobytes(), np.uint8)
    head[8:16] = np.frombuffer(np.array([20000, t], "<u4").tobytes(), np.uint8)
    path.write_bytes(head.tobytes() + planes.tobytes())


@pytest.mark.gpu
@pytest.mark.parametrize("name", VOLS + ["sparse7x3"])
def test_cpp_dropin_emit_records_match_reference(exe, golden_dir, tmp_path, name):
    """The CLI's --emit-records loop (spikecam_main.cpp:146-172) compiled
    against the drop-in headers, and the whole-sensor emit_records (GPU),
    write the reference's SPKR bytes (tests/golden/records.npz); decode() of
    every pixel equals its uint8 frames; bench() runs."""
    rec = np.load(golden_dir / "records.npz")
    if name == "sparse7x3":
        planes, geom = rec["sparse7x3/planes"], rec["sparse7x3/geom"]
    else:
        g = np.load(golden_dir / f"vol_{name}.npz")
        planes, geom = g["planes"], g["geom"]
    w, h, t = (int(x) for x in geom)
    spk = tmp_path / "v.spk"
    _spk_file(spk, planes, w, h, t)
    run(exe, "records", spk, tmp_path)
    for tag in ("fsr", "ssr"):
        want = rec[f"{name}/{tag}"].tobytes()
        assert (tmp_path / f"{tag}_loop.spkr").read_bytes() == want, tag
        assert (tmp_path / f"{tag}_gpu.spkr").read_bytes() == want, tag
