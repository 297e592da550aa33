"""Per-phase device time of the single-process time-sharded driver (CUDA events)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2412_11639_b200 as spk  # noqa: E402
from paper_2412_11639_b200.shard import TimeShard, fresh_state, time_bounds  # noqa: E402

scene, W, H, T, method, K = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]), sys.argv[5], int(sys.argv[6])
vol = spk.synth(scene, 0, W, H, T, device="cuda")
out = torch.empty((T, W * H), dtype=torch.uint8, device="cuda")
for rep in range(2):
    ev = {}

    def mark(k):
        ev[k] = torch.cuda.Event(enable_timing=True)
        ev[k].record()
    b = time_bounds(T, K)
    shards = [TimeShard(vol, b0, b1, method) for b0, b1 in zip(b, b[1:])]
    mark("start")
    for sh in shards:
        sh.speculate()
    mark("speculate")
    entry = fresh_state(vol.npix, vol.planes.device)
    for sh in shards:
        entry = sh.resolve(entry)
    mark("resolve")
    closes = [None] * K
    closes[-1] = shards[-1].tail_close
    for r in range(K - 2, -1, -1):
        closes[r] = shards[r].close_from_next(shards[r + 1].entry_close, closes[r + 1])
    for sh, c in zip(shards, closes):
        sh.stitch(c)
    mark("stitch")
    for sh in shards:
        sh.expand(out[sh.f0:sh.f1])
    mark("expand")
    torch.cuda.synchronize()
    keys = list(ev)
    print(rep, " ".join(f"{k1}={ev[k0].elapsed_time(ev[k1]):.2f}ms" for k0, k1 in zip(keys, keys[1:])),
          "fb:", sum(sh.fb is not None for sh in shards), "scap:", [sh.scap for sh in shards][:3], flush=True)
