"""H2D of the C2 payload: spk_upload_planes (pitched 2D copy) vs a flat copy."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2412_11639_b200 as spk  # noqa: E402
from paper_2412_11639_b200 import _capi as capi  # noqa: E402

W, H, T = 400, 250, 40000
vol = spk.synth("moving", 0, W, H, T, device="cuda")
pay = torch.from_numpy(vol.payload()).pin_memory()
flat = torch.empty(pay.numel(), dtype=torch.uint8, device="cuda")
lib = capi.lib()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s = torch.cuda.current_stream().cuda_stream
for name, fn in (("spk_upload_planes", lambda: capi.check(lib.spk_upload_planes(
        vol.geom(), pay.data_ptr(), (W * H + 7) // 8, 0, vol.planes.data_ptr(), s))),
                 ("flat copy", lambda: flat.copy_(pay, non_blocking=True))):
    fn()
    torch.cuda.synchronize()
    e0.record()
    for _ in range(3):
        fn()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 3
    print(f"{name}: {ms:.2f} ms  {pay.numel() / ms / 1e6:.1f} GB/s", flush=True)
