"""Direct-mode diagnostics on configs-sized scenes: step time by phase
(spk_set_timing) for u8 FSR/SSR.  python profiles/direct_probe.py"""
import ctypes as C
import sys

import torch

sys.path.insert(0, ".")
import paper_2412_11639_b200 as spk  # noqa: E402
from paper_2412_11639_b200 import _capi as capi  # noqa: E402

lib = capi.lib()
for scene, w, h, t in (("moving", 400, 250, 40000), ("static", 400, 250, 20000),
                       ("sensor", 1000, 1000, 20000)):
    vol = spk.synth(scene, 1, w, h, t, device="cuda")
    out = torch.empty((t, w * h), dtype=torch.uint8, device="cuda")
    for m in ("fsr", "ssr"):
        spk.reconstruct(vol, m, out=out)
        torch.cuda.synchronize()
        lib.spk_set_timing(1)
        spk.reconstruct(vol, m, out=out)
        torch.cuda.synchronize()
        ph = [C.c_float() for _ in range(4)]
        lib.spk_last_timing(*[C.byref(x) for x in ph])
        lib.spk_set_timing(0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            spk.reconstruct(vol, m, out=out)
        e1.record()
        torch.cuda.synchronize()
        print(f"{scene} {w}x{h}x{t} {m}: {e0.elapsed_time(e1) / 5:.3f} ms/step  phases "
              + " ".join(f"{x.value:.3f}" for x in ph), flush=True)
    del vol, out
