"""Phase timing of one reconstruction per config (CUDA events through
spk_set_timing), plus a checksum of the frames so variants run in separate
processes (env knobs are read once) can be compared.

    python profiles/walk_probe.py [configs...]   # c1 c2 c3 c5s (C5 first 200k frames)
"""
import ctypes as C
import hashlib
import json
import sys

import torch

sys.path.insert(0, ".")
import paper_2412_11639_b200 as spk  # noqa: E402
from paper_2412_11639_b200 import _capi as capi  # noqa: E402

CFG = {
    "c1": ("static", 400, 250, 20000),
    "c2": ("moving", 400, 250, 40000),
    "c3": ("sensor", 1000, 1000, 20000),
    "c5s": ("range", 400, 250, 200000),
}
lib = capi.lib()
names = sys.argv[1:] or ["c2", "c1", "c3"]
for name in names:
    scene, w, h, t = CFG[name]
    vol = spk.synth(scene, 0, w, h, t, device="cuda")
    out = torch.empty((t, w * h), dtype=torch.uint8, device="cuda")
    for m in ("fsr", "ssr"):
        for _ in range(3):
            spk.reconstruct(vol, m, out=out)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 10
        e0.record()
        for _ in range(reps):
            spk.reconstruct(vol, m, out=out)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        v = [C.c_float() for _ in range(4)]
        lib.spk_set_timing(1)
        acc = [0.0] * 4
        for _ in range(5):
            spk.reconstruct(vol, m, out=out)
            capi.check(lib.spk_last_timing(*(C.byref(x) for x in v)))
            acc = [a + x.value / 5 for a, x in zip(acc, v)]
        lib.spk_set_timing(0)
        # checksum: per-frame sums + a strided sample hashed
        sums = torch.cat([out[i:i + 4096].to(torch.int64).sum(dim=1) for i in range(0, t, 4096)])
        hs = hashlib.sha256(sums.cpu().numpy().tobytes() + out[::97, ::13].cpu().numpy().tobytes()).hexdigest()[:16]
        pxf = w * h * t
        print(json.dumps({"cfg": name, "method": m, "ms": round(ms, 4),
                          "phases": [round(x, 4) for x in acc], "frac": pxf * 1.125 / (ms * 1e-3) / 1e9 / 6547.8,
                          "sha": hs}), flush=True)
    del vol, out
    torch.cuda.empty_cache()
