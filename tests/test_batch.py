"""Device batch (spk_reconstruct_batch, BASELINE configs[3]): the CUDA graph
of many reconstructions must give exactly the frames of per-volume calls --
on first capture, on replay, and after the inputs behind the same buffers
change (the graph reads the buffers, it does not bake their contents)."""
import pytest
import torch

import paper_2412_11639_b200 as spk

pytestmark = pytest.mark.gpu


def _vols(seed0, n, w, h, t):
    return [spk.synth(("static", "moving", "noise", "range")[i % 4], seed0 + i, w, h, t,
                      param=0.05) for i in range(n)]


@pytest.mark.parametrize("method", ["fsr", "ssr", "tfi", "tfp"])
@pytest.mark.parametrize("dtype", [torch.uint8, torch.float64])
def test_batch_equals_calls(method, dtype):
    w, h, t = 67, 23, 1700
    vols = _vols(3, 7, w, h, t)
    want = [spk.reconstruct(v, method, dtype=dtype).clone() for v in vols]
    outs = [torch.empty((t, w * h), dtype=dtype, device="cuda") for _ in vols]
    for rep in range(3):  # capture, then replays of the cached graph
        for o in outs:
            o.fill_(7)
        got = spk.reconstruct_batch(vols, method, outs=outs)
        torch.cuda.synchronize()
        for g, ref in zip(got, want):
            assert torch.equal(g, ref), (method, rep)


def test_batch_replay_reads_new_inputs():
    w, h, t = 50, 20, 2300
    vols = _vols(11, 5, w, h, t)
    outs = [torch.empty((t, w * h), dtype=torch.uint8, device="cuda") for _ in vols]
    spk.reconstruct_batch(vols, "fsr", outs=outs)
    for i, v in enumerate(vols):  # new contents behind the same plane buffers
        v.planes.copy_(spk.synth("moving", 100 + i, w, h, t).planes)
    got = spk.reconstruct_batch(vols, "fsr", outs=outs)
    torch.cuda.synchronize()
    for g, v in zip(got, vols):
        assert torch.equal(g, spk.reconstruct(v, "fsr"))


def test_batch_rejects_mixed_geometry():
    a = spk.synth("moving", 1, 40, 10, 500)
    b = spk.synth("moving", 2, 40, 10, 600)
    with pytest.raises(ValueError):
        spk.reconstruct_batch([a, b], "fsr")
