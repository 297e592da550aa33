"""The multi-GPU drivers with the real kernels: several processes (one rank
each, gloo, host-staged exchange) sharing cuda:0 -- the only GPU of the test
box.  Every rank launches libspikecam_b200.so; nothing waits on another
rank's kernels inside a launch (ranks exchange O(W*H) state between
launches), so sharing one device is sound.

* time shards (configs[4] style, reconstruct_time_sharded_dist): rank r
  generates and reconstructs frames [a_r, a_r+1) of one long stream; its
  frames must equal the same frames of a single pass;
* pixel bands (reconstruct_sharded): every rank reconstructs its band and the
  all-gather assembles the single-pass frames.
"""
import hashlib
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _digest(t: torch.Tensor) -> str:
    return hashlib.sha256(t.contiguous().cpu().numpy().tobytes()).hexdigest()


def _time_worker(rank, world, port, scene, w, h, t, method, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2412_11639_b200 as spk
        from paper_2412_11639_b200 import _capi as capi
        from paper_2412_11639_b200.shard import reconstruct_time_sharded_dist, time_bounds
        b = time_bounds(t, world)
        f0, f1 = b[rank], b[rank + 1]
        shard = spk.synth(scene, 7, w, h, f1 - f0, frame0=f0, param=0.3)
        capi.lib().spk_launch_count(1)
        out = reconstruct_time_sharded_dist(shard, method)
        torch.cuda.synchronize()
        q.put((rank, f0, f1, _digest(out), int(capi.lib().spk_launch_count(1))))
    finally:
        dist.destroy_process_group()


def _spawn(target, world, args):
    # the ranks share cuda:0 with this process: hand back what earlier tests
    # left cached (torch's allocator and the library's stream-ordered pool)
    from paper_2412_11639_b200 import _capi as capi
    torch.cuda.empty_cache()
    capi.check(capi.lib().spk_release_memory())
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=target, args=(r, world, port, *args, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=600)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    return [q.get(timeout=10) for _ in range(world)]


@pytest.mark.parametrize("scene,w,h,t,world", [("range", 400, 250, 24000, 3),
                                               ("moving", 400, 250, 12000, 4),
                                               ("noise", 64, 8, 3000, 2)])
@pytest.mark.parametrize("method", ["fsr", "ssr"])
def test_time_shards_across_processes(scene, w, h, t, world, method):
    import paper_2412_11639_b200 as spk
    torch.cuda.set_device(0)
    res = _spawn(_time_worker, world, (scene, w, h, t, method))
    full = spk.synth(scene, 7, w, h, t, param=0.3)
    ref = spk.reconstruct(full, method).reshape(t, w * h)
    for rank, f0, f1, dig, launches in res:
        assert launches > 0, rank  # the rank ran the sm_100a kernels
        assert dig == _digest(ref[f0:f1]), (rank, f0, f1)


def _band_worker(rank, world, port, w, h, t, method, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2412_11639_b200 as spk
        from paper_2412_11639_b200.shard import reconstruct_sharded
        vol = spk.synth("moving", 3, w, h, t)  # replicated input, every rank its band
        full = reconstruct_sharded(vol, method)
        torch.cuda.synchronize()
        q.put((rank, _digest(full.reshape(t, w * h))))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("method", ["fsr", "ssr", "tfp"])
def test_pixel_bands_across_processes(world, method):
    import paper_2412_11639_b200 as spk
    torch.cuda.set_device(0)
    w, h, t = 400, 250, 3000
    res = _spawn(_band_worker, world, (w, h, t, method))
    ref = spk.reconstruct(spk.synth("moving", 3, w, h, t), method).reshape(t, w * h)
    want = _digest(ref)
    assert all(d == want for _, d in res), res
