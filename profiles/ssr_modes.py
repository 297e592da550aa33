"""SSR segment time per scene for alternative builds of the library
(python profiles/ssr_modes.py lib1.so lib2.so ...)."""
import shutil
import subprocess
import sys

code = r'''
import sys, torch
sys.path.insert(0, ".")
import paper_2412_11639_b200 as spk
from paper_2412_11639_b200 import _capi as capi
import ctypes as C
lib = capi.lib()
res = []
for scene, t in (("moving", 40000), ("static", 20000), ("range", 100000)):
    vol = spk.synth(scene, 0, 400, 250, t, device="cuda")
    out = torch.empty((t, 100000), dtype=torch.uint8, device="cuda")
    for _ in range(2):
        spk.reconstruct(vol, "ssr", out=out)
    lib.spk_set_timing(1)
    v = [C.c_float() for _ in range(4)]
    seg = []
    for _ in range(5):
        spk.reconstruct(vol, "ssr", out=out)
        capi.check(lib.spk_last_timing(*(C.byref(x) for x in v)))
        seg.append(v[0].value)
    lib.spk_set_timing(0)
    res.append(f"{scene}:{sorted(seg)[2]:.2f}ms")
print(" ".join(res))
'''
for lib in sys.argv[1:]:
    shutil.copy(lib, "paper_2412_11639_b200/libspikecam_b200.so")
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True)
    print(lib, out.stdout.strip(), out.stderr.strip()[-300:])
