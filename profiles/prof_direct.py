"""One direct-mode (uint8) reconstruction of a configs-sized scene for ncu:
python profiles/prof_direct.py SCENE W H T METHOD"""
import sys

import torch

sys.path.insert(0, ".")
import paper_2412_11639_b200 as spk  # noqa: E402

scene, w, h, t, m = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]), sys.argv[5]
vol = spk.synth(scene, 1, w, h, t, device="cuda")
out = torch.empty((t, w * h), dtype=torch.uint8, device="cuda")
spk.reconstruct(vol, m, out=out)
torch.cuda.synchronize()
