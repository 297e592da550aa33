"""Small reconstructions of every kernel family for compute-sanitizer
(memcheck / racecheck / synccheck): FSR and SSR (incl. the in-grid time
split and an overflowing noise pixel set -> k_fixup), TFI/TFP, the
multi-launch time-shard protocol, streaming, records and metrics.
compute-sanitizer --tool racecheck python profiles/sanitize_run.py"""
import os
import sys

import torch

sys.path.insert(0, ".")
import paper_2412_11639_b200 as spk  # noqa: E402
from paper_2412_11639_b200.shard import reconstruct_time_sharded  # noqa: E402

w, h = 72, 20
for scene, t, param in (("moving", 3000, 0.0), ("noise", 900, 0.3), ("range", 5000, 0.0)):
    vol = spk.synth(scene, 3, w, h, t, param=param)
    for m in ("fsr", "ssr", "tfi", "tfp"):
        spk.reconstruct(vol, m)
        spk.reconstruct(vol, m, dtype=torch.float64)
    for S in ("3", "1"):
        os.environ["SPK_SPLIT"] = S
        spk.reconstruct(vol, "fsr")
        spk.reconstruct(vol, "ssr")
    del os.environ["SPK_SPLIT"]
    reconstruct_time_sharded(vol, "fsr", nshards=3)
    reconstruct_time_sharded(vol, "ssr", nshards=3)
    spk.records(vol, "fsr")
    fr = spk.reconstruct(vol, "fsr")
    spk.frame_metrics(fr, ref=fr)
    spk.stability(vol, 4)
torch.cuda.synchronize()
print("sanitize_run done")
