"""Exact time sharding of one stream (SURVEY.md 8(e) "Time", BASELINE configs[4]).

Each shard is scanned on its own from a fresh state; the boundaries are
resolved with the true entry state (csrc/shard.cu).  The bar is bit-identity
with the single-pass reconstruction (itself pinned to the reference by
test_gpu_parity.py), over the validation cases SURVEY lists: breaks at a
boundary, runs spanning >= 3 shards (static scenes: one run per pixel),
pixels with 0 or 1 spikes in a shard, SSR gap sets completing after the
boundary, saturated (I = 1) and dark (ISI ~ 1000) pixels.
"""
from __future__ import annotations

import pytest
import torch

pytestmark = pytest.mark.gpu


def _check(vol, method, dtype=torch.uint8, **kw):
    import paper_2412_11639_b200 as spk
    from paper_2412_11639_b200.shard import reconstruct_time_sharded
    ref = spk.reconstruct(vol, method, dtype=dtype)
    got = reconstruct_time_sharded(vol, method, dtype=dtype, **kw)
    torch.cuda.synchronize()
    if dtype == torch.float64:
        assert torch.equal(got.view(torch.int64), ref.view(torch.int64)), (method, kw)
    else:
        mism = (got != ref).sum().item()
        assert mism == 0, (method, kw, mism)


@pytest.mark.parametrize("method", ["fsr", "ssr"])
@pytest.mark.parametrize("nshards", [2, 3, 7])
def test_moving_scene(method, nshards):
    import paper_2412_11639_b200 as spk
    vol = spk.synth("moving", 3, 400, 25, 6000, device="cuda")
    _check(vol, method, nshards=nshards)


@pytest.mark.parametrize("method", ["fsr", "ssr"])
def test_static_scene_runs_span_all_shards(method):
    import paper_2412_11639_b200 as spk
    vol = spk.synth("static", 5, 200, 10, 8000, device="cuda")
    _check(vol, method, nshards=8)
    _check(vol, method, dtype=torch.float64, nshards=5)


@pytest.mark.parametrize("method", ["fsr", "ssr"])
def test_extreme_range_scene(method):
    """configs[4] generator: dark (ISI up to 1000), saturated and mid pixels;
    shards shorter than the darkest ISIs, so some pixels see 0 or 1 spikes."""
    import paper_2412_11639_b200 as spk
    vol = spk.synth("range", 7, 160, 10, 9000, device="cuda")
    _check(vol, method, nshards=9)
    _check(vol, method, bounds=[0, 32, 96, 1000, 1001, 2500, 2531, 9000])


@pytest.mark.parametrize("method", ["fsr", "ssr"])
def test_noise_and_uneven_bounds(method):
    import paper_2412_11639_b200 as spk
    vol = spk.synth("noise", 9, 64, 7, 3000, param=0.3, device="cuda")
    _check(vol, method, bounds=[0, 1, 33, 700, 701, 2048, 2999, 3000])
    _check(vol, method, dtype=torch.float32, nshards=4)


@pytest.mark.parametrize("method", ["fsr", "ssr"])
@pytest.mark.parametrize("pcap", [1, 2, 5])
def test_prefix_overflow_paths(method, pcap):
    """a tiny prefix list forces the 'never synced' and full re-scan paths"""
    import paper_2412_11639_b200 as spk
    vol = spk.synth("moving", 11, 96, 8, 4000, device="cuda")
    _check(vol, method, nshards=5, prefix_cap=pcap)
    vol = spk.synth("noise", 12, 40, 3, 2000, param=0.45, device="cuda")
    _check(vol, method, nshards=6, prefix_cap=pcap)


def test_one_shard_and_single_pixel():
    import paper_2412_11639_b200 as spk
    vol = spk.synth("moving", 1, 33, 1, 2500, device="cuda")
    _check(vol, "fsr", nshards=1)
    vol = spk.synth("noise", 2, 1, 1, 3000, param=0.2, device="cuda")
    for m in ("fsr", "ssr"):
        _check(vol, m, nshards=11)


def test_randomized_bounds():
    """random scenes, methods and cut points (including 1-frame shards)"""
    import random

    import paper_2412_11639_b200 as spk
    rnd = random.Random(2412)
    for it in range(16):
        scene = rnd.choice(["moving", "static", "range", "noise", "sensor"])
        w, h, t = rnd.choice([(40, 3), (128, 2), (9, 5)]) + (rnd.randint(500, 5000),)
        vol = spk.synth(scene, it, w, h, t, param=rnd.uniform(0.05, 0.6), device="cuda")
        k = rnd.randint(2, 12)
        cuts = sorted(set(rnd.randint(1, t - 1) for _ in range(k - 1)))
        for method in ("fsr", "ssr"):
            _check(vol, method, bounds=[0] + cuts + [t], prefix_cap=rnd.choice([3, 16, 64]))


def test_dist_driver_single_rank():
    """the per-rank driver with no process group: one shard = the whole stream"""
    import paper_2412_11639_b200 as spk
    from paper_2412_11639_b200.shard import reconstruct_time_sharded_dist
    vol = spk.synth("moving", 4, 64, 9, 2000, device="cuda")
    for m in ("fsr", "ssr"):
        got = reconstruct_time_sharded_dist(vol, m)
        assert torch.equal(got, spk.reconstruct(vol, m).reshape(2000, -1))
