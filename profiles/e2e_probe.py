"""End-to-end host batch (spk_reconstruct_host_batch) frames/s on C2, N steps."""
import ctypes as C
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2412_11639_b200 as spk  # noqa: E402
from paper_2412_11639_b200 import _capi as capi  # noqa: E402

W, H, T = 400, 250, 40000
vol = spk.synth("moving", 0, W, H, T, device="cuda")
payload = torch.from_numpy(vol.payload()).pin_memory()
houts = [torch.empty((T, W * H), dtype=torch.uint8).pin_memory() for _ in range(3)]
g = capi.geom(W, H, T, 0)
lib = capi.lib()
for n in (8, 8):
    pin = (C.c_void_p * n)(*([payload.data_ptr()] * n))
    pout = (C.c_void_p * n)(*[houts[i % 3].data_ptr() for i in range(n)])
    lib.spk_reconstruct_host_batch(g, 1, pin, 0, 32, capi.SPK_OUT_U8, pout, W * H)
    t0 = time.perf_counter()
    capi.check(lib.spk_reconstruct_host_batch(g, n, pin, 0, 32, capi.SPK_OUT_U8, pout, W * H))
    el = time.perf_counter() - t0
    print(f"{sys.argv[1] if len(sys.argv) > 1 else ''} e2e {n} steps: {n * T / el / 1e3:.1f} k frames/s "
          f"({el / n * 1e3:.1f} ms/step)", flush=True)
