"""Save the spike bits of 256 sampled pixels of a scene (one uint8 per frame)
for host-side modelling: python profiles/dump_pixels.py SCENE W H T OUT.npy"""
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_2412_11639_b200 as spk  # noqa: E402

scene, W, H, T, out = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]), sys.argv[5]
v = spk.synth(scene, 0, W, H, T, device="cuda")
pix = np.random.default_rng(0).choice(W * H, 256, replace=False)
cols = v.planes[:, :].cpu().numpy()
bits = np.stack([((cols[:, p >> 3] >> (p & 7)) & 1).astype(np.uint8) for p in pix])
np.save(out, bits)
print(out, bits.shape, bits.mean())
