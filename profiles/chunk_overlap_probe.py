"""Feasibility probe for time-chunk pipelining of one volume (configs[1]).

K2 (integer-ALU bound) of time chunk c+1 beside the expansion (K2b..K3, HBM
bound) of chunk c.  Timing only: every chunk is segmented from a carried
state (spk_segment_state) into its own run list and expanded on its own.
Compares: whole volume in one call; chunks serialised on one stream; chunks
pipelined over two streams (expansion stream at high priority).
python profiles/chunk_overlap_probe.py [F]
"""
import ctypes as C
import sys

import torch

sys.path.insert(0, ".")
import paper_2412_11639_b200 as spk  # noqa: E402
from paper_2412_11639_b200 import _capi as capi  # noqa: E402

W, H, T = 400, 250, 40000
lib = capi.lib()
npix = W * H


def run(scene, method, F, mode):
    vol = spk.synth(scene, 1, W, H, T, device="cuda")
    pitch = vol.pitch
    out = torch.empty((T, npix), dtype=torch.uint8, device="cuda")
    nch = (T + F - 1) // F
    cap = max(64, F // 32)
    runs = [torch.empty((npix, cap, 2), dtype=torch.int32, device="cuda") for _ in range(nch)]
    counts = [torch.empty(npix, dtype=torch.int32, device="cuda") for _ in range(nch)]
    last = [torch.empty(npix, dtype=torch.int32, device="cuda") for _ in range(nch)]
    st = [torch.empty((17, npix), dtype=torch.int32, device="cuda") for _ in range(nch + 1)]
    sA = torch.cuda.Stream()
    sB = torch.cuda.Stream(priority=-1)
    mk = 0 if method == "fsr" else 1
    evs = [torch.cuda.Event() for _ in range(nch)]

    def geom(c):
        n = min(F, T - c * F)
        return capi.spk_geom(W, H, n, pitch), n

    def go():
        lib.spk_state_fresh(npix, st[0].data_ptr(), sA.cuda_stream)
        for c in range(nch):
            g, n = geom(c)
            planes = vol.planes.data_ptr() + c * F * pitch
            lib.spk_segment_state(C.byref(g), planes, mk, runs[c].data_ptr(), cap,
                                  counts[c].data_ptr(), last[c].data_ptr(), st[c].data_ptr(),
                                  st[c + 1].data_ptr(), sA.cuda_stream)
            evs[c].record(sA)
            s = sB if mode == "pipe" else sA
            s.wait_event(evs[c])
            lib.spk_expand_runs_u8(C.byref(g), runs[c].data_ptr(), cap, counts[c].data_ptr(),
                                   last[c].data_ptr(), out.data_ptr() + c * F * npix, npix,
                                   s.cuda_stream)
        sA.wait_stream(sB)

    if mode == "whole":
        def go():  # noqa: F811
            spk.reconstruct(vol, method, out=out, stream=sA)
    for _ in range(3):
        go()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(10):
        torch.cuda.synchronize()
        e0.record(sA)
        sB.wait_event(e0)
        go()
        e1.record(sA)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    return ts[len(ts) // 2]


for scene in ("moving", "static"):
    for method in ("fsr", "ssr"):
        whole = run(scene, method, T, "whole")
        line = f"{scene} {method}: whole {whole:.3f} ms"
        for F in [int(a) for a in sys.argv[1:]] or (20480, 10240, 5120):
            ser = run(scene, method, F, "serial")
            pipe = run(scene, method, F, "pipe")
            line += f" | F={F}: serial {ser:.3f} pipe {pipe:.3f}"
        print(line, flush=True)
