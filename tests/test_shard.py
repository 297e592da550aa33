"""Pixel-band sharding (paper_2412_11639_b200/shard.py).

CPU: the band plan, the zero-copy band view (checked with the oracle) and the
all-gather layout over a real 2-rank gloo group.  GPU: bands reconstructed
one after another (independent launches, no inter-rank waiting) assemble to
exactly the single-GPU frames.
"""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2412_11639_b200.recon import PackedVolume
from paper_2412_11639_b200.shard import BAND_ALIGN, band_view, gather_bands, pixel_bands


@pytest.mark.parametrize("npix", [1, 9, 127, 128, 129, 1000, 100_000, 1_000_000])
@pytest.mark.parametrize("world", [1, 2, 3, 4, 7, 8])
def test_pixel_bands_partition(npix, world):
    bands = pixel_bands(npix, world)
    assert len(bands) == world
    assert bands[0][0] == 0 and bands[-1][1] == npix
    for (a0, a1), (b0, b1) in zip(bands, bands[1:]):
        assert a1 == b0
    for p0, p1 in bands:
        assert p0 <= p1 and (p0 == npix or p0 % BAND_ALIGN == 0)
    sizes = [p1 - p0 for p0, p1 in bands]
    if npix >= world * BAND_ALIGN:
        assert max(sizes) - min(sizes) <= BAND_ALIGN + npix % BAND_ALIGN


def _volume_cpu(oracle, w, h, t, seed, p=0.3):
    rng = np.random.default_rng(seed)
    bits = (rng.random((t, w * h)) < p).astype(np.uint8)
    pitch = ((w * h + 127) // 128) * 16
    planes = oracle.pack(bits, w, h, pitch)
    return PackedVolume(w, h, t, torch.from_numpy(planes)), planes, pitch


@pytest.mark.parametrize("world", [2, 3, 5])
def test_band_view_bits(oracle, world):
    """A band view reconstructs (oracle) to the full volume's band columns."""
    w, h, t = 37, 11, 120
    vol, planes, pitch = _volume_cpu(oracle, w, h, t, 3)
    for method in (0, 1, 3):
        full = oracle.reconstruct(planes, w, h, t, pitch, method)
        for p0, p1 in pixel_bands(w * h, world):
            if p1 == p0:
                continue
            v = band_view(vol, p0, p1)
            assert (v.width, v.height, v.frames) == (p1 - p0, 1, t)
            assert v.planes.stride(0) == pitch
            vp = np.ascontiguousarray(v.planes.numpy())
            band = oracle.reconstruct(vp, p1 - p0, 1, t, vp.shape[1], method)
            assert np.array_equal(band, full[:, p0:p1]), (method, p0, p1)


def test_band_view_rejects_unaligned(oracle):
    vol, _, _ = _volume_cpu(oracle, 64, 2, 4, 1)
    with pytest.raises(ValueError):
        band_view(vol, 16, 64)
    with pytest.raises(ValueError):
        band_view(vol, 0, 129)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _gather_worker(rank, world, port, w, h, t, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle.oracle import Oracle
        orc = Oracle()
        rng = np.random.default_rng(11)
        bits = (rng.random((t, w * h)) < 0.25).astype(np.uint8)
        planes = orc.pack(bits, w, h)
        pitch = planes.shape[1]
        full = orc.reconstruct(planes, w, h, t, pitch, 1)  # SSR uint8
        bands = pixel_bands(w * h, world)
        p0, p1 = bands[rank]
        bmax = max(b - a for a, b in bands)
        local = torch.zeros((t, bmax), dtype=torch.uint8)
        # this rank's band, computed from its own band of the input only
        local[:, : p1 - p0] = torch.from_numpy(
            orc.reconstruct(planes, w, h, t, pitch, 1, pix_begin=p0, pix_end=p1))
        got = gather_bands(local, w * h)
        q.put((rank, bool(np.array_equal(got.numpy(), full))))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("geom", [(300, 2, 50), (13, 7, 33)])
def test_gather_bands_gloo_world2(geom):
    w, h, t = geom
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gather_worker, args=(r, 2, port, w, h, t, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=180)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    res = dict(q.get(timeout=5) for _ in range(2))
    assert res == {0: True, 1: True}


@pytest.mark.gpu
@pytest.mark.parametrize("geom", [(400, 250, 1500), (37, 11, 700), (1000, 3, 2100)])
@pytest.mark.parametrize("method", ["fsr", "ssr", "tfi", "tfp"])
def test_bands_assemble_to_single_gpu(oracle, geom, method):
    import paper_2412_11639_b200 as spk
    from paper_2412_11639_b200.shard import reconstruct_band, reconstruct_sharded
    w, h, t = geom
    vol = spk.synth("moving", 5, w, h, t, device="cuda")
    for dtype in (torch.uint8, torch.float64):
        ref = spk.reconstruct(vol, method, dtype=dtype).reshape(t, -1)
        for world in (2, 3, 8):
            full = torch.full_like(ref, 7)
            for r in range(world):
                p0, p1, out = reconstruct_band(vol, method, r, world, dtype)
                full[:, p0:p1] = out[:, : p1 - p0]
            assert torch.equal(full, ref), (world, dtype)
        one = reconstruct_sharded(vol, method, dtype=dtype)  # no process group: world 1
        assert torch.equal(one.reshape(t, -1), ref)


# ---- time shards across ranks: the exchange schedule (gloo, CPU) ----------
class _FakeTimeShard:
    """Stands in for TimeShard's device work so the rank-to-rank protocol can
    run on CPU: every tensor a rank produces encodes who made it."""

    def __init__(self, vol, f0, f1, method, pcap, stream):
        self.npix = vol.npix
        self.rank = dist.get_rank()
        self.tail_close = torch.full((self.npix, 8), 1000 + self.rank, dtype=torch.int32)
        self.entry_close = torch.full((self.npix, 8), 2000 + self.rank, dtype=torch.int32)

    def speculate(self):
        pass

    def fresh_entry(self):
        return torch.zeros((17, self.npix), dtype=torch.int32)

    def resolve(self, entry):
        self.entry = entry.clone()
        return entry + (self.rank + 1)  # exit state = entry state "advanced" by this shard

    def close_from_next(self, ec_next, close_next):
        return ec_next * 10000 + close_next

    def stitch(self, close):
        self.close = close.clone()

    def expand(self, out):
        out[0, :] = self.entry[0, 0]
        out[1, :] = self.close[0, 0] % 1000003


def _timeshard_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2412_11639_b200.shard import reconstruct_time_sharded_dist
        vol = PackedVolume(4, 2, 5, torch.zeros((5, 16), dtype=torch.uint8))
        out = torch.zeros((5, 8), dtype=torch.int64)
        reconstruct_time_sharded_dist(vol, "fsr", out=out, shard_type=_FakeTimeShard)
        q.put((rank, int(out[0, 0]), int(out[1, 0])))
    finally:
        dist.destroy_process_group()


def test_time_shard_exchange_gloo_world3():
    """forward: rank r's entry = exit of rank r-1 (state advanced by every
    earlier shard); backward: rank r's close combines rank r+1's entry close and
    close record, recursively from the last rank's tail close."""
    world = 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_timeshard_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=180)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    got = {r: (e, c) for r, e, c in (q.get(timeout=5) for _ in range(world))}
    closes = {world - 1: 1000 + world - 1}
    for r in range(world - 2, -1, -1):
        closes[r] = (2000 + r + 1) * 10000 + closes[r + 1]
    for r in range(world):
        assert got[r][0] == sum(i + 1 for i in range(r)), (r, got[r])
        assert got[r][1] == closes[r] % 1000003, (r, got[r])
