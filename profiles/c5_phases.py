"""configs[4] (400x250 x 1,000,000 frames, range scene) phase times of one
reconstruct (spk_set_timing): python profiles/c5_phases.py [T] [method]"""
import ctypes as C
import sys

import torch

sys.path.insert(0, ".")
import paper_2412_11639_b200 as spk  # noqa: E402
from paper_2412_11639_b200 import _capi as capi  # noqa: E402

T = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
m = sys.argv[2] if len(sys.argv) > 2 else "fsr"
lib = capi.lib()
vol = spk.synth("range", 0, 400, 250, T, device="cuda")
out = torch.empty((T, vol.npix), dtype=torch.uint8, device="cuda")
spk.reconstruct(vol, m, out=out)
torch.cuda.synchronize()
for _ in range(2):
    lib.spk_set_timing(1)
    spk.reconstruct(vol, m, out=out)
    torch.cuda.synchronize()
    ph = [C.c_float() for _ in range(4)]
    lib.spk_last_timing(*[C.byref(x) for x in ph])
    lib.spk_set_timing(0)
    tot = sum(x.value for x in ph)
    print(f"range 400x250x{T} {m}: total {tot:.2f} ms  segment {ph[0].value:.2f}  finalize {ph[1].value:.2f}"
          f"  expand {ph[2].value:.2f} ({T * vol.npix / (ph[2].value * 1e-3) / 1e12:.2f} TB/s)  fixup {ph[3].value:.3f}",
          flush=True)
