"""Profiling driver: C2 (moving 400x250x40000) reconstructed twice with one
method, so ncu can skip the first (cold) launch of each kernel."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2412_11639_b200 as spk  # noqa: E402

method = sys.argv[1] if len(sys.argv) > 1 else "fsr"
frames = int(sys.argv[2]) if len(sys.argv) > 2 else 40000
vol = spk.synth("moving", 0, 400, 250, frames, device="cuda")
out = torch.empty((frames, 400 * 250), dtype=torch.uint8, device="cuda")
for _ in range(2):
    spk.reconstruct(vol, method, out=out)
torch.cuda.synchronize()
print("ok", method, frames)
