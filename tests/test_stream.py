"""Streaming FSR (PixelReconState for every pixel, csrc/stream.cu): events
pushed block by block equal the reference's streaming events for any
blocking (golden rows, made with PixelReconState at block sizes 2^30, 32, 7)
and the oracle's fsr_events on whole volumes."""
from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _per_pixel(chunks, npix):
    """concatenate the (offsets, durations, intensities) of successive calls per pixel"""
    out = [([], []) for _ in range(npix)]
    for offs, d, v in chunks:
        offs, d, v = offs.cpu().numpy(), d.cpu().numpy(), v.cpu().numpy()
        for p in range(npix):
            out[p][0].extend(d[offs[p]:offs[p + 1]].tolist())
            out[p][1].extend(v[offs[p]:offs[p + 1]].tolist())
    return out


def _run(vol, blocks):
    import paper_2412_11639_b200 as spk
    es = spk.EventStream(vol.width, vol.height)
    chunks, f = [], 0
    for b in blocks:
        chunks.append(es.push(vol.planes[f:f + b]))
        f += b
    assert f == vol.frames and es.frames == f
    chunks.append(es.flush())
    es.close()
    return _per_pixel(chunks, vol.npix)


def test_golden_rows_any_blocking(golden_dir):
    import paper_2412_11639_b200 as spk
    g = np.load(golden_dir / "rows.npz")
    names = sorted({k.split("/")[0] for k in g.files})
    for name in names:
        bits = g[f"{name}/bits"].astype(np.uint8)
        t = bits.size
        want = g[f"{name}/events"]
        # 1x1 volume: one payload byte per frame, the spike in bit 0
        vol = spk.PackedVolume.from_payload(bits.copy(), 1, 1, t, device="cuda") \
            if t else spk.PackedVolume.empty(1, 1, 0, device="cuda")
        for blk in (1 << 30, 32, 7, 1):
            blocks = [min(blk, t - i) for i in range(0, t, blk)] if t else []
            d, v = _run(vol, blocks)[0]
            assert np.array_equal(np.array(d, np.int64), want[0].astype(np.int64)), (name, blk)
            assert np.array_equal(np.array(v, np.float64).view(np.int64), want[1].view(np.int64)), (name, blk)


@pytest.mark.parametrize("scene", ["moving", "noise", "static", "range"])
def test_volumes_vs_oracle(oracle, scene):
    import paper_2412_11639_b200 as spk
    w, h, t = 37, 5, 3000
    vol = spk.synth(scene, 3, w, h, t, param=0.25, device="cuda")
    rng = np.random.default_rng(7)
    blocks, f = [], 0
    while f < t:
        b = int(min(t - f, rng.choice([1, 5, 31, 32, 100, 1024, 2500])))
        blocks.append(b)
        f += b
    got = _run(vol, blocks)
    bits = vol.to_bytes().reshape(t, -1).cpu().numpy()
    for p in range(w * h):
        d, v = oracle.fsr_events(bits[:, p])
        assert np.array_equal(np.array(got[p][0], np.int64), d), (scene, p)
        assert np.array_equal(np.array(got[p][1], np.float64).view(np.int64), v.view(np.int64)), (scene, p)


def test_empty_pushes_and_zero_frames():
    import paper_2412_11639_b200 as spk
    es = spk.EventStream(3, 2)
    offs, d, v = es.flush()
    assert offs.tolist() == [0] * 7 and d.numel() == 0
    es = spk.EventStream(3, 2)
    vol = spk.PackedVolume.empty(3, 2, 10, device="cuda")
    vol.planes.zero_()
    es.push(vol.planes[:0])
    es.push(vol)
    offs, d, v = es.flush()
    assert d.tolist() == [10] * 6 and v.tolist() == [0.0] * 6
