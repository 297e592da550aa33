"""One reconstruction (for ncu captures): python profiles/one_recon.py scene w h t method [reps]"""
import sys
import torch
sys.path.insert(0, ".")
import paper_2412_11639_b200 as spk  # noqa: E402

scene, w, h, t, m = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]), sys.argv[5]
reps = int(sys.argv[6]) if len(sys.argv) > 6 else 2
vol = spk.synth(scene, 0, w, h, t, device="cuda")
out = torch.empty((t, w * h), dtype=torch.uint8, device="cuda")
for _ in range(reps):
    spk.reconstruct(vol, m, out=out)
torch.cuda.synchronize()
print("ok")
