"""Profiling driver for the 8(f)#4 kernels: per-frame metrics of a C2
reconstruction (te + mse) and stability_order of every C1 pixel, each once."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2412_11639_b200 as spk  # noqa: E402

vol = spk.synth("moving", 0, 400, 250, 40000, device="cuda")
u8 = spk.reconstruct(vol, "fsr")
ref = spk.reconstruct(vol, "tfi")
spk.frame_metrics(u8, ref)
del u8, ref, vol
v = spk.synth("static", 0, 400, 250, 20000, device="cuda")
spk.stability(v, 8)
torch.cuda.synchronize()
print("ok")
