"""Per-step time and per-phase device times of one scene:
python profiles/phases.py SCENE W H T [methods]"""
import ctypes as C
import sys

import torch

sys.path.insert(0, ".")
import os  # noqa: E402
from pathlib import Path  # noqa: E402

from paper_2412_11639_b200 import _capi as capi  # noqa: E402
if os.environ.get("SPK_PROBE_LIB"):  # A/B probes: another build of the library
    capi.LIB_PATH = Path(os.environ["SPK_PROBE_LIB"]).resolve()
    _h = C.CDLL(str(capi.LIB_PATH))
    for _name in list(capi.SIGNATURES):  # an older build lacks newer entry points
        if not hasattr(_h, _name):
            del capi.SIGNATURES[_name]
import paper_2412_11639_b200 as spk  # noqa: E402

scene, W, H, T = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
methods = sys.argv[5].split(",") if len(sys.argv) > 5 else ["fsr", "ssr"]
vol = spk.synth(scene, 0, W, H, T, device="cuda")
out = torch.empty((T, W * H), dtype=torch.uint8, device="cuda")
lib = capi.lib()
for m in methods:
    for _ in range(3):
        spk.reconstruct(vol, m, out=out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        spk.reconstruct(vol, m, out=out)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    v = [C.c_float() for _ in range(4)]
    lib.spk_set_timing(1)
    acc = []
    for _ in range(6):
        spk.reconstruct(vol, m, out=out)
        torch.cuda.synchronize()
        capi.check(lib.spk_last_timing(*(C.byref(x) for x in v)))
        acc.append([x.value for x in v])
        sh, fl = C.c_int32(1), C.c_int64(0)
        if hasattr(lib, "spk_last_split") and "spk_last_split" in capi.SIGNATURES:
            capi.check(lib.spk_last_split(C.byref(sh), C.byref(fl)))
    lib.spk_set_timing(0)
    ph = [sum(a[i] for a in acc[1:]) / 5 for i in range(4)]
    frac = W * H * T * 1.125 / ms / 1e6 / 6553.3
    print(f"{scene} {W}x{H}x{T} {m}: {ms:.3f} ms/step ({T / ms / 1e3:.2f} M fps, frac {frac:.3f}) | "
          f"seg {ph[0]:.3f} fin {ph[1]:.3f} exp {ph[2]:.3f} fix {ph[3]:.3f} | split {sh.value} "
          f"rescanned {fl.value}", flush=True)
