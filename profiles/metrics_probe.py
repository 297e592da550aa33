"""Device time of the 8(f)#4 paths at the config sizes: per-frame entropy +
mse of a C2 reconstruction, and stability_order of every pixel of C1."""
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2412_11639_b200 as spk  # noqa: E402


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps * 1e3


vol = spk.synth("moving", 0, 400, 250, 40000)
u8 = spk.reconstruct(vol, "fsr")
ref = spk.reconstruct(vol, "tfi")
ms = timed(lambda: spk.frame_metrics(u8, ref))
print(f"C2 frame_metrics u8 (te+mse, 40000 frames): {ms:.2f} ms ({40000 / ms:.1f} k frames/s)", flush=True)
del u8, ref
for scene, w, h, t in (("static", 400, 250, 20000), ("moving", 400, 250, 40000)):
    v = spk.synth(scene, 0, w, h, t)
    ms = timed(lambda: spk.stability(v, 8), reps=1)
    ok, fails = spk.verify_stability(v, 8)
    print(f"{scene} {w}x{h}x{t} stability depth 8: {ms:.1f} ms, ok={ok}, first fails={fails[:2]}", flush=True)
