"""Pin the C oracle (oracle/spk_oracle.c) against the reference's own outputs.

The fixtures in tests/golden/ were produced by the unmodified reference
library (tests/golden/make_golden.py); the known-answer assertions below are
the ones proj/tests/test_reconstruct.cpp, test_io.cpp and acceptance.cpp make
(cited per test).  CPU only.
"""
import numpy as np
import pytest

FSR, SSR, TFI, TFP = 0, 1, 2, 3


@pytest.fixture(scope="module")
def rows(golden_dir):
    z = np.load(golden_dir / "rows.npz")
    names = sorted({k.split("/")[0] for k in z.files})
    return z, names


def non_degenerate(seg):
    s, e, n = seg
    keep = n > 0
    return s[keep], e[keep], n[keep]


def test_rows_runs_match_reference(oracle, rows):
    z, names = rows
    for name in names:
        bits = z[f"{name}/bits"]
        for m, tag in ((FSR, "fsr"), (SSR, "ssr")):
            s, e, n = non_degenerate(z[f"{name}/{tag}_seg"])
            os_, oe, on = oracle.runs(bits, m)
            assert np.array_equal(os_, s) and np.array_equal(oe, e) and np.array_equal(on, n), \
                (name, tag)


def test_rows_pixel_values_bit_exact(oracle, rows):
    z, names = rows
    for name in names:
        bits = z[f"{name}/bits"]
        for m, tag, win in ((FSR, "fsr", 32), (SSR, "ssr", 32), (TFI, "tfi", 32),
                            (TFP, "tfp32", 32), (TFP, "tfp7", 7), (TFP, "tfp1", 1)):
            want = z[f"{name}/{tag}_pix"]
            got = oracle.row_f64(bits, m, win)
            assert np.array_equal(got.view(np.uint64), want.view(np.uint64)), (name, tag)


def test_rows_fsr_events(oracle, rows):
    z, names = rows
    for name in names:
        d, v = oracle.fsr_events(z[f"{name}/bits"])
        want = z[f"{name}/events"]
        assert np.array_equal(d, want[0].astype(np.int64)), name
        assert np.array_equal(v, want[1]), name


@pytest.mark.parametrize("vol", ["par12x9", "bar64x48", "noise40x25", "odd9x1", "odd13x7"])
def test_volumes_match_reference(oracle, golden_dir, vol):
    z = np.load(golden_dir / f"vol_{vol}.npz")
    w, h, t = (int(v) for v in z["geom"])
    planes = z["planes"]
    pitch = planes.shape[1]
    for tag in sorted({k.split("/")[0] for k in z.files if "/" in k}):
        m = {"fsr": FSR, "ssr": SSR, "tfi": TFI}.get(tag, TFP)
        win = int(tag[3:]) if tag.startswith("tfp") else 32
        u = oracle.reconstruct(planes, w, h, t, pitch, m, win, dtype=np.uint8)
        assert np.array_equal(u, z[f"{tag}/u8"]), (vol, tag)
        f = oracle.reconstruct(planes, w, h, t, pitch, m, win, dtype=np.float64)
        import hashlib
        assert hashlib.sha256(f.tobytes()).digest() == z[f"{tag}/f64_sha256"].tobytes(), (vol, tag)


# ---- known answers from the reference's unit tests --------------------------

def test_worked_example(oracle, rows):
    """test_reconstruct.cpp:59-71: S1 {3,3,4,3,7,6,7} -> [0,13) and [13,33)."""
    z, _ = rows
    s, e, n = oracle.runs(z["worked_example/bits"], FSR)
    assert list(s) == [0, 13] and list(e) == [13, 33] and list(n) == [4, 3]


def test_streaming_worked_example(oracle, rows):
    """test_reconstruct.cpp:160-178: event (13, 255/3.25), flush (20, 255*3/20), (1, carry)."""
    z, _ = rows
    d, v = oracle.fsr_events(z["worked_example_tight/bits"])
    assert list(d) == [13, 20, 1]
    assert v[0] == pytest.approx(255 / 3.25) and v[1] == pytest.approx(255 * 3 / 20)
    assert v[2] == v[1]


def test_constant_and_two_phase(oracle, rows):
    """test_reconstruct.cpp:73-87, 98-102, 240-248."""
    z, _ = rows
    assert len(oracle.runs(z["const_q03_1000/bits"], FSR)[0]) == 1
    s, e, n = oracle.runs(z["const_q03_2000/bits"], FSR)
    assert len(s) == 1 and 255 * n[0] / (e[0] - s[0]) == pytest.approx(76.5, rel=0.01)
    s, e, n = oracle.runs(z["const_q03_1024/bits"], FSR)
    err = abs(255 * n[0] / (e[0] - s[0]) - 76.5) / 76.5
    assert len(s) == 1 and err <= 2.0 / (n[0] * 3.0)
    s, e, _ = oracle.runs(z["two_phase/bits"], FSR)
    assert len(s) == 2 and abs(e[0] - 500) <= 16


def test_ssr_refines_and_splits(oracle, rows):
    """test_reconstruct.cpp:104-158, acceptance.cpp:197-229."""
    z, names = rows
    for name in ("ssr_no_break", "const_q03_1000"):
        a, b = oracle.runs(z[f"{name}/bits"], FSR), oracle.runs(z[f"{name}/bits"], SSR)
        assert all(np.array_equal(x, y) for x, y in zip(a, b))
    assert len(oracle.runs(z["ssr_split/bits"], FSR)[0]) == 1
    assert len(oracle.runs(z["ssr_split/bits"], SSR)[0]) >= 2
    for name in names:  # every SSR run inside one FSR run
        bits = z[f"{name}/bits"]
        fs, fe, _ = oracle.runs(bits, FSR)
        ss, se, _ = oracle.runs(bits, SSR)
        for a, b in zip(ss, se):
            k = np.searchsorted(fe, a, side="right")
            assert k < len(fs) and fs[k] <= a and b <= fe[k], name


def test_tfi_tfp_known_answers(oracle, rows):
    """test_reconstruct.cpp:200-238."""
    z, _ = rows
    assert oracle.row_f64(z["tfp_example/bits"], TFP, 32)[63] == pytest.approx(255 * 8 / 32)
    v = oracle.row_f64(z["tfi_example/bits"], TFI)
    assert v[0] == 0.0 and v[3] == pytest.approx(127.5) and v[9] == pytest.approx(127.5)
    for m, win in ((FSR, 32), (SSR, 32), (TFI, 32), (TFP, 32)):
        vals = oracle.row_f64(z["const_q05_256/bits"], m, win)
        assert np.allclose(vals[64:250], 127.5, rtol=0.01)
    for p in (2, 3, 5):
        bits = z[f"periodic_{p}/bits"]
        tfi = oracle.row_f64(bits, TFI)
        for k in (1, 2, 3):
            tfp = oracle.row_f64(bits, TFP, k * p)
            half = bits.size // 2
            assert np.allclose(tfi[half:], 255 / p) and np.allclose(tfp[half:], 255 / p)


def test_quantize_matches_reference_pgm(oracle, golden_dir):
    """quantize (io.cpp:78-81) through the reference's own write_image(pgm)."""
    z = np.load(golden_dir / "formats.npz")
    got = [oracle.quantize(v) for v in z["quant_in"][0]]
    assert got == list(z["quant_out"])
    assert oracle.quantize(127.5) == 128 and oracle.quantize(-3) == 0 and oracle.quantize(300) == 255


def test_spk1_packing_golden_bytes(oracle, golden_dir):
    """test_io.cpp:49-74: golden header+payload and zero pad bits."""
    z = np.load(golden_dir / "formats.npz")
    assert list(z["spk_golden"]) == [0x53, 0x50, 0x4B, 0x31, 2, 0, 1, 0, 0x20, 0x4E, 0, 0, 1, 0, 0,
                                     0, 1]
    assert list(oracle.pack(np.array([[1, 0]], np.uint8), 2, 1)[0]) == [1]
    planes = oracle.pack(np.ones((1, 9), np.uint8), 9, 1)
    assert list(planes[0]) == [0xFF, 0x01] == list(z["spk_pad"][16:])
    # msb-first toggle (test_io.cpp:130-140)
    assert oracle.unpack(np.array([[1]], np.uint8), 8, 1, 1, 1)[0, 0] == 1
    assert oracle.unpack(np.array([[1]], np.uint8), 8, 1, 1, 1, msb_first=True)[0, 7] == 1


def test_codec_encode(oracle):
    """codec.cpp:8-19: lround ties away, durations split at 255."""
    assert list(oracle.encode(300, 127.5)) == [255 << 8 | 128, 45 << 8 | 128]
    with pytest.raises(ValueError):
        oracle.encode(0, 1.0)
