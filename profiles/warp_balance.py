"""Lockstep vs free-running cost of the per-spike SSR loop: per warp (32
consecutive pixels), sum over 32-frame words of the max popcount over lanes
vs the max over lanes of the total spike count."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2412_11639_b200 as spk  # noqa: E402

for scene, W, H, T in (("moving", 400, 250, 40000), ("sensor", 1000, 1000, 4000)):
    v = spk.synth(scene, 0, W, H, T)
    lock = free = tot = 0.0
    npix = W * H
    for f0 in range(0, T, 4000):
        b = v.to_bytes()[f0:f0 + 4000].reshape(-1, npix) if False else None
        break
    bits = spk.PackedVolume(W, H, T, v.planes).to_bytes().reshape(T, npix)
    nw = T // 32
    pop = bits[: nw * 32].reshape(nw, 32, npix).sum(1, dtype=torch.int32)  # [word, pixel]
    nwarp = npix // 32
    pop = pop[:, : nwarp * 32].reshape(nw, nwarp, 32)
    lock = pop.max(2).values.sum(0).float()          # per warp
    free = pop.sum(0).max(1).values.float()          # per warp
    mean = pop.sum(0).float().mean(1)
    print(f"{scene}: lockstep {lock.mean():.0f}  free-running {free.mean():.0f}  mean lane {mean.mean():.0f} "
          f"(lockstep/free {float((lock / free).mean()):.3f})", flush=True)
