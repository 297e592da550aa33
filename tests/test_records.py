"""SPKR segment records: GPU file image vs the reference.

Golden images come from the reference's own --emit-records loop
(tests/golden/make_golden.py:save_records -> oracle/ref_shim.cpp
ref_emit_records).  Bar: byte-identical SPKR images.  At full size the check
is a size-independent property: decoding a pixel's records (codec.cpp:33-43)
reproduces that pixel's uint8 frames exactly (lead 0, run values, carried
tail -- the same quantize rule).
"""
from __future__ import annotations

import numpy as np
import pytest

from paper_2412_11639_b200.records import decode, parse_spkr
from paper_2412_11639_b200.recon import IoError

VOLS = ["par12x9", "bar64x48", "noise40x25", "odd9x1", "odd13x7", "sparse7x3"]


def _vol(golden_dir, name):
    if name == "sparse7x3":
        g = np.load(golden_dir / "records.npz")
        planes, geom = g["sparse7x3/planes"], g["sparse7x3/geom"]
    else:
        g = np.load(golden_dir / f"vol_{name}.npz")
        planes, geom = g["planes"], g["geom"]
    w, h, t = (int(x) for x in geom)
    return planes, w, h, t


@pytest.mark.parametrize("name", VOLS)
def test_oracle_records_match_reference(oracle, golden_dir, name):
    """Pins the oracle's record restatement against the reference's bytes."""
    planes, w, h, t = _vol(golden_dir, name)
    gold = np.load(golden_dir / "records.npz")
    for m, tag in ((0, "fsr"), (1, "ssr")):
        assert oracle.records(planes, w, h, t, planes.shape[1], m) == gold[f"{name}/{tag}"].tobytes()


@pytest.mark.parametrize("name", VOLS)
def test_decoded_records_are_u8_frames(oracle, golden_dir, name):
    planes, w, h, t = _vol(golden_dir, name)
    gold = np.load(golden_dir / "records.npz")
    for m, tag in ((0, "fsr"), (1, "ssr")):
        rv = parse_spkr(gold[f"{name}/{tag}"])
        assert (rv.width, rv.height, rv.frame_count, rv.fps) == (w, h, t, 20000)
        frames = oracle.reconstruct(planes, w, h, t, planes.shape[1], m)
        for p in range(w * h):
            assert np.array_equal(decode(rv.words[p]), frames[:, p]), (tag, p)


def test_parse_spkr_errors(golden_dir):
    img = np.load(golden_dir / "records.npz")["odd13x7/fsr"].tobytes()
    with pytest.raises(IoError, match="magic"):
        parse_spkr(b"SPKX" + img[4:])
    with pytest.raises(IoError, match="truncated"):
        parse_spkr(img[:-1])
    with pytest.raises(IoError, match="trailing"):
        parse_spkr(img + b"\0")
    with pytest.raises(RuntimeError, match="zero-duration"):
        decode(np.array([0x0105, 0x0007], np.uint16))


@pytest.mark.gpu
@pytest.mark.parametrize("name", VOLS)
def test_gpu_records_match_reference(golden_dir, name):
    import torch

    import paper_2412_11639_b200 as spk
    planes, w, h, t = _vol(golden_dir, name)
    gold = np.load(golden_dir / "records.npz")
    vol = spk.PackedVolume.from_payload(planes.reshape(-1), w, h, t, device="cuda")
    for tag in ("fsr", "ssr"):
        img = spk.records(vol, tag)
        assert img.is_cuda and img.dtype == torch.uint8
        assert img.cpu().numpy().tobytes() == gold[f"{name}/{tag}"].tobytes(), tag
        host = spk.records_host(planes.reshape(-1), w, h, t, tag)
        assert host == gold[f"{name}/{tag}"].tobytes(), tag


@pytest.mark.gpu
def test_gpu_records_overflowed_run_lists(oracle, golden_dir):
    """Pixels with more runs than the run-list capacity take the rescan path."""
    import paper_2412_11639_b200 as spk
    from paper_2412_11639_b200 import _capi as capi
    planes, w, h, t = _vol(golden_dir, "noise40x25")
    vol = spk.PackedVolume.from_payload(planes.reshape(-1), w, h, t, device="cuda")
    gold = np.load(golden_dir / "records.npz")
    try:
        for cap in (1, 3, 17):
            capi.check(capi.lib().spk_set_run_capacity(cap))
            for tag in ("fsr", "ssr"):
                assert spk.records(vol, tag).cpu().numpy().tobytes() == gold[f"noise40x25/{tag}"].tobytes()
    finally:
        capi.lib().spk_set_run_capacity(0)


@pytest.mark.gpu
def test_gpu_records_edges():
    import paper_2412_11639_b200 as spk
    for w, h, t in ((5, 2, 0), (1, 1, 1), (3, 1, 256), (33, 1, 511)):
        vol = spk.synth("noise", 3, w, h, t, param=0.2, device="cuda") if t else \
            spk.PackedVolume.empty(w, h, 0, device="cuda")
        for tag in ("fsr", "ssr"):
            rv = parse_spkr(spk.records(vol, tag, fps=1234).cpu().numpy())
            assert (rv.width, rv.height, rv.fps, rv.frame_count) == (w, h, 1234, t)
            u8 = spk.reconstruct(vol, tag).reshape(t, -1).cpu().numpy() if t else \
                np.zeros((0, w * h), np.uint8)
            for p in range(w * h):
                got = decode(rv.words[p]) if rv.words[p].size else np.zeros(0, np.uint8)
                assert np.array_equal(got, u8[:, p]), (w, h, t, tag, p)
    with pytest.raises(ValueError):
        spk.records(spk.synth("noise", 1, 4, 4, 10, param=0.3, device="cuda"), "tfi")


@pytest.mark.gpu
@pytest.mark.parametrize("tag", ["fsr", "ssr"])
def test_gpu_records_full_length_property(tag):
    """C2's full stream length (40,000 frames) on a 400 x 20 band: decoded
    records == uint8 frames for every pixel."""
    import paper_2412_11639_b200 as spk
    w, h, t = 400, 20, 40000
    vol = spk.synth("moving", 0, w, h, t, device="cuda")
    rv = parse_spkr(spk.records(vol, tag).cpu().numpy())
    u8 = spk.reconstruct(vol, tag).reshape(t, -1).cpu().numpy()
    nwords = 0
    for p in range(w * h):
        nwords += rv.words[p].size
        assert np.array_equal(decode(rv.words[p]), u8[:, p]), p
    assert nwords < w * h * t / 20  # records are far smaller than frames
