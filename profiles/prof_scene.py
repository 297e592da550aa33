"""Profiling driver: one scene reconstructed twice (ncu can skip the cold
launch): python profiles/prof_scene.py SCENE W H T METHOD"""
import sys

import torch

sys.path.insert(0, ".")
import paper_2412_11639_b200 as spk  # noqa: E402

scene, W, H, T, method = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]), sys.argv[5]
vol = spk.synth(scene, 0, W, H, T, device="cuda")
out = torch.empty((T, W * H), dtype=torch.uint8, device="cuda")
for _ in range(2):
    spk.reconstruct(vol, method, out=out)
torch.cuda.synchronize()
print("ok", scene, W, H, T, method)
