"""One reconstruct() call of a scene (for ncu launch lists):
python profiles/one_call.py SCENE W H T METHOD [SPK_SPLIT]"""
import os
import sys

import torch

sys.path.insert(0, ".")
if len(sys.argv) > 6:
    os.environ["SPK_SPLIT"] = sys.argv[6]
import paper_2412_11639_b200 as spk  # noqa: E402

scene, W, H, T, m = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]), sys.argv[5]
vol = spk.synth(scene, 0, W, H, T, device="cuda")
out = torch.empty((T, W * H), dtype=torch.uint8, device="cuda")
for _ in range(2):
    spk.reconstruct(vol, m, out=out)
torch.cuda.synchronize()
