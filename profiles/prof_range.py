"""One reconstruct of the configs[4] range scene (400x250, T frames) for ncu:
python profiles/prof_range.py [T] [method]"""
import sys

import torch

sys.path.insert(0, ".")
import paper_2412_11639_b200 as spk  # noqa: E402

T = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000
m = sys.argv[2] if len(sys.argv) > 2 else "fsr"
vol = spk.synth("range", 0, 400, 250, T, device="cuda")
out = torch.empty((T, vol.npix), dtype=torch.uint8, device="cuda")
spk.reconstruct(vol, m, out=out)
torch.cuda.synchronize()
