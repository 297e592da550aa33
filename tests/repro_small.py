"""Small reproduction driver (debugging aid): one noise volume, FSR/SSR u8."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2412_11639_b200 as spk

w, h, t = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
m = sys.argv[4] if len(sys.argv) > 4 else "fsr"
v = spk.synth("noise", 7, w, h, t, param=0.3)
out = spk.reconstruct(v, m)
torch.cuda.synchronize()
print("ok", out.shape, int(out.sum()))
