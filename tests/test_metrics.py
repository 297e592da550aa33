"""Quality metrics and the stability check.

CPU: the oracle restatement (oracle/spk_oracle.c) against the reference's own
outputs in tests/golden/metrics.npz (make_golden.py save_metrics) and, where
oracle/_ref is built, against the reference on random inputs.
GPU: spk_frame_metrics / spk_stability through the C-ABI against the same
fixtures and the oracle.  Entropy and mse are float reductions: the bar is
1e-12 relative (the device sums in a fixed tree order, the reference
sequentially); stability reports are integers and must match exactly.
"""
from pathlib import Path

import numpy as np
import pytest
import torch

from oracle.oracle import Reference, ref_available

GOLD = np.load(Path(__file__).parent / "golden" / "metrics.npz")
RTOL = 1e-12
STAB_KEYS = ("depth", "index", "verified_order", "absolute")


def close(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    same_inf = np.isinf(a) & np.isinf(b) & (np.sign(a) == np.sign(b))
    with np.errstate(invalid="ignore"):
        return bool(np.all(same_inf | (np.abs(a - b) <= RTOL * np.maximum(np.abs(b), 1e-300))))


def golden_volume(name):
    g = np.load(Path(__file__).parent / "golden" / f"vol_{name}.npz")
    w, h, t = (int(x) for x in g["geom"])
    return g["planes"], w, h, t


def column_bits(planes, w, h):
    return np.stack([(planes[:, p >> 3] >> (p & 7)) & 1 for p in range(w * h)]).astype(np.uint8)


def rows_padded():
    """the golden rows as one volume: pixel i = row i, padded with silent frames
    (trailing zeros leave S1, hence stability_order, unchanged)"""
    rows = np.load(Path(__file__).parent / "golden" / "rows.npz")
    names = list(GOLD["rows/names"])
    bits = [rows[f"{n}/bits"] for n in names]
    t = max(b.size for b in bits)
    cols = np.zeros((t, len(bits)), np.uint8)
    for i, b in enumerate(bits):
        cols[: b.size, i] = b
    return names, cols


# ---------------------------------------------------------------- CPU ----
def test_oracle_te_images(oracle):
    for k in ("rand9x13", "const3x3", "ramp5x4"):
        assert close(oracle.te(GOLD[f"img/{k}"]), GOLD[f"img/{k}/te"]), k


def test_oracle_te_small_image_rejected(oracle):
    assert np.isnan(oracle.te(np.zeros((2, 9))))


@pytest.mark.parametrize("depth", [1, 3, 8])
def test_oracle_stability_rows(oracle, depth):
    names, cols = rows_padded()
    want = GOLD[f"rows/d{depth}"]
    paths = GOLD[f"rows/d{depth}/path"]
    for i, n in enumerate(names):
        r = oracle.stability(cols[:, i], depth)
        assert [r[k] for k in STAB_KEYS] == [int(x) for x in want[i]], (n, depth)
        assert r["path"] == str(paths[i]), n


def test_oracle_stability_sweep(oracle):
    """cmd_verify_stability's constant-rate sweep (spikecam_main.cpp:209-225)"""
    for i, b in enumerate(GOLD["sweep/bits"]):
        r = oracle.stability(b, 8)
        assert [r[k] for k in STAB_KEYS] == [int(x) for x in GOLD["sweep/d8"][i]]


@pytest.mark.parametrize("name,depth", [("bar64x48", 8), ("noise40x25", 8), ("par12x9", 4)])
def test_oracle_stability_volumes(oracle, name, depth):
    planes, w, h, t = golden_volume(name)
    bits = column_bits(planes, w, h)
    want = GOLD[f"vol/{name}/d{depth}"]
    paths = GOLD[f"vol/{name}/d{depth}/path"]
    for p in range(w * h):
        r = oracle.stability(bits[p], depth)
        assert [r[k] for k in STAB_KEYS] == [int(x) for x in want[p]], (name, p)
        assert r["path"] == str(paths[p])


@pytest.mark.skipif(not ref_available(), reason="oracle/_ref not built")
def test_oracle_pinned_to_reference_random(oracle):
    ref = Reference()
    rng = np.random.default_rng(2024)
    for i in range(60):
        hh, ww = int(rng.integers(3, 20)), int(rng.integers(3, 20))
        img = rng.uniform(-3, 258, (hh, ww))
        if i % 3 == 0:
            img = np.round(img)
        other = rng.integers(0, 256, (hh, ww)).astype(np.float64)
        assert close(oracle.te(img), ref.te(img))
        assert close(oracle.mse(img, other), ref.mse(img, other))
        t = int(rng.integers(0, 3000))
        q = rng.uniform(0.01, 1.0)
        b = ref.simulate_pixel(np.full(t, q), 1.0, rng.uniform(0, 1)) if t else np.zeros(0, np.uint8)
        if i % 2:
            b ^= (rng.random(t) < 0.002).astype(np.uint8)
        for depth in (1, 2, 5, 8, 12):
            assert oracle.stability(b, depth) == ref.stability(b, depth), (i, depth)


# ---------------------------------------------------------------- GPU ----
gpu = pytest.mark.gpu


def _spk():
    import paper_2412_11639_b200 as spk
    return spk


def _vol(planes, w, h, t):
    spk = _spk()
    return spk.PackedVolume.from_payload(np.ascontiguousarray(planes).reshape(-1), w, h, t)


@gpu
def test_gpu_te_images():
    spk = _spk()
    for k in ("rand9x13", "const3x3", "ramp5x4"):
        img = torch.tensor(GOLD[f"img/{k}"], device="cuda")
        assert close(spk.two_dimensional_entropy(img), GOLD[f"img/{k}/te"]), k
        q = torch.floor(img.clamp(0, 255) + 0.5).to(torch.uint8)
        assert close(spk.two_dimensional_entropy(q), GOLD[f"img/{k}/te"]), k


@gpu
def test_gpu_frame_metrics_bar():
    """entropy of every FSR frame of the moving-bar volume, and mse / psnr
    against the TFI frames as the reference images (the CLI's compare)"""
    spk = _spk()
    vol = _vol(*golden_volume("bar64x48"))
    f64 = spk.reconstruct(vol, "fsr", dtype=torch.float64)
    u8 = spk.reconstruct(vol, "fsr")
    tfi = spk.reconstruct(vol, "tfi")
    te, ms = spk.frame_metrics(f64, tfi)
    assert close(te.cpu().numpy(), GOLD["bar/te_fsr"])
    assert close(ms.cpu().numpy(), GOLD["bar/mse_fsr_tfi"])
    te8, _ = spk.frame_metrics(u8)
    assert close(te8.cpu().numpy(), GOLD["bar/te_fsr"])
    te32, _ = spk.frame_metrics(spk.reconstruct(vol, "fsr", dtype=torch.float32))
    assert te32.shape == te.shape
    for n in (0, 1, 100, 287):
        p = spk.psnr(f64[n], tfi[n])
        assert close(p, GOLD["bar/psnr_fsr_tfi"][n]), n
    rows = spk.compare(vol, ["fsr"], tfi, warmup=10)
    assert close(rows[0]["te"], np.mean(GOLD["bar/te_fsr"][10:]))
    assert close(rows[0]["mse"], np.mean(GOLD["bar/mse_fsr_tfi"][10:]))


@gpu
def test_gpu_frame_metrics_errors():
    spk = _spk()
    with pytest.raises(ValueError):
        spk.frame_metrics(torch.zeros((4, 2, 9), dtype=torch.uint8, device="cuda"))
    te, ms = spk.frame_metrics(torch.zeros((0, 5, 5), dtype=torch.uint8, device="cuda"))
    assert te.numel() == 0 and ms is None
    # mse alone is defined for any size
    a = torch.full((3, 1, 2), 7.0, dtype=torch.float64, device="cuda")
    r = torch.full((3, 1, 2), 5, dtype=torch.uint8, device="cuda")
    _, ms = spk.frame_metrics(a, r, te=False)
    assert torch.equal(ms.cpu(), torch.full((3,), 4.0, dtype=torch.float64))


def _check_stab(rep, want, paths, tag):
    spk = _spk()
    got = np.stack([rep[k].astype(np.int64) for k in STAB_KEYS], 1)
    bad = np.nonzero((got != want).any(1))[0]
    assert bad.size == 0, (tag, bad[:5], got[bad[:5]], want[bad[:5]])
    for p in range(len(rep)):
        assert spk.metrics.path_string(rep["path"][p], rep["path_len"][p]) == str(paths[p]), (tag, p)


@gpu
@pytest.mark.parametrize("name,depth", [("bar64x48", 8), ("noise40x25", 8), ("par12x9", 4),
                                        ("odd9x1", 8)])
def test_gpu_stability_golden_volumes(name, depth):
    spk = _spk()
    vol = _vol(*golden_volume(name))
    _check_stab(spk.stability(vol, depth), GOLD[f"vol/{name}/d{depth}"],
                GOLD[f"vol/{name}/d{depth}/path"], name)


@gpu
@pytest.mark.parametrize("depth", [1, 3, 8])
def test_gpu_stability_golden_rows(oracle, depth):
    spk = _spk()
    names, cols = rows_padded()
    t, n = cols.shape
    vol = _vol(oracle.pack(cols, n, 1), n, 1, t)
    _check_stab(spk.stability(vol, depth), GOLD[f"rows/d{depth}"], GOLD[f"rows/d{depth}/path"],
                f"rows d{depth}")


@gpu
def test_gpu_stability_sweep_and_verify(oracle):
    spk = _spk()
    sweep = GOLD["sweep/bits"]
    n, t = sweep.shape
    vol = _vol(oracle.pack(sweep.T.copy(), n, 1), n, 1, t)
    rep = spk.stability(vol, 8)
    got = np.stack([rep[k].astype(np.int64) for k in STAB_KEYS], 1)
    assert np.array_equal(got, GOLD["sweep/d8"])
    ok, fails = spk.verify_stability(vol, 8)
    assert ok and fails == []
    vol2 = _vol(*golden_volume("bar64x48"))
    ok, fails = spk.verify_stability(vol2, 8)
    want = GOLD["vol/bar64x48/d8"]
    first_row = int(np.nonzero(want[:, 0] > 0)[0][0]) // 64
    assert not ok and {f[1] for f in fails} == {first_row}
    assert len(fails) == int((want[first_row * 64:(first_row + 1) * 64, 0] > 0).sum())


@gpu
@pytest.mark.parametrize("scene,w,h,t,depth", [("moving", 40, 24, 3000, 8), ("static", 32, 16, 6000, 8),
                                               ("noise", 33, 7, 500, 5), ("sensor", 48, 20, 4000, 12)])
def test_gpu_stability_vs_oracle(oracle, scene, w, h, t, depth):
    spk = _spk()
    vol = spk.synth(scene, 3, w, h, t)
    rep = spk.stability(vol, depth)
    bits = column_bits(vol.planes.cpu().numpy(), w, h)
    for p in range(w * h):
        r = oracle.stability(bits[p], depth)
        assert [int(rep[k][p]) for k in STAB_KEYS] == [r[k] for k in STAB_KEYS], (scene, p)
        assert spk.metrics.path_string(rep["path"][p], rep["path_len"][p]) == r["path"]


@gpu
def test_gpu_stability_edges():
    spk = _spk()
    vol = spk.PackedVolume.empty(5, 3, 0)
    rep = spk.stability(vol, 8)
    assert (rep["depth"] == 0).all() and (rep["verified_order"] == 1).all() and (rep["absolute"] == 1).all()
    vol = spk.synth("noise", 0, 8, 2, 100)
    for bad in (0, 64):
        with pytest.raises(ValueError):
            spk.stability(vol, bad)
