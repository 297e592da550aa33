"""Does K2 (ALU-bound) of one volume overlap K2b..K3 (HBM-bound) of another?
N volumes reconstructed back to back on 1, 2 or 4 streams (CUDA events)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2412_11639_b200 as spk  # noqa: E402

W, H = 400, 250
for scene, T, n in (("moving", 4000, 16), ("moving", 40000, 4), ("static", 4000, 16)):
    vols = [spk.synth(scene, i, W, H, T, device="cuda") for i in range(n)]
    outs = [torch.empty((T, W * H), dtype=torch.uint8, device="cuda") for _ in range(n)]
    for m in ("fsr", "ssr"):
        for ns in (1, 2, 4):
            ss = [torch.cuda.Stream() for _ in range(ns)]
            def go():
                for i in range(n):
                    spk.reconstruct(vols[i], m, out=outs[i], stream=ss[i % ns])
            go()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            best = 1e9
            for _ in range(3):
                torch.cuda.synchronize()
                e0.record()
                for s in ss:
                    s.wait_event(e0)
                go()
                for s in ss:
                    torch.cuda.current_stream().wait_stream(s)
                e1.record()
                torch.cuda.synchronize()
                best = min(best, e0.elapsed_time(e1))
            print(f"{scene} T={T} x{n} {m} streams={ns}: {best / n:.3f} ms/volume "
                  f"({n * T / best * 1e3 / 1e6:.2f} M fps)", flush=True)
    del vols, outs
