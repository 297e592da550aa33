"""configs[2] 1000x1000x20000: FSR/SSR device time per step (CUDA events)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2412_11639_b200 as spk  # noqa: E402

W, H, T = 1000, 1000, 20000
vol = spk.synth("sensor", 0, W, H, T, device="cuda")
out = torch.empty((T, W * H), dtype=torch.uint8, device="cuda")
for m in ("fsr", "ssr"):
    for _ in range(3):
        spk.reconstruct(vol, m, out=out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        spk.reconstruct(vol, m, out=out)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    pxf = W * H * T
    print(f"{m}: {ms:.2f} ms/step  {T / ms * 1e3 / 1e6:.3f} M fps  "
          f"{pxf * 1.125 / ms / 1e6 / 6553.3:.3f} of HBM roofline", flush=True)

# per-phase device times (timing mode runs the volume as one pixel part)
import ctypes as C  # noqa: E402

from paper_2412_11639_b200 import _capi as capi  # noqa: E402

lib = capi.lib()
for m in ("fsr", "ssr"):
    v = [C.c_float() for _ in range(4)]
    lib.spk_set_timing(1)
    acc = []
    for _ in range(4):
        spk.reconstruct(vol, m, out=out)
        torch.cuda.synchronize()
        capi.check(lib.spk_last_timing(*(C.byref(x) for x in v)))
        acc.append([x.value for x in v])
    lib.spk_set_timing(0)
    ph = [sum(a[i] for a in acc[1:]) / 3 for i in range(4)]
    print(f"{m} phases (seg, fin, exp, fix) ms: " + ", ".join(f"{p:.2f}" for p in ph), flush=True)
