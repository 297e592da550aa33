"""configs[3]-style batch: host issue time vs device time of 64 calls
(two streams, like bench.py), and per-call device time alone."""
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2412_11639_b200 as spk  # noqa: E402

W, H, T, N = 400, 250, 4000, 64
vols = [spk.synth("static" if i % 2 == 0 else "moving", i, W, H, T, device="cuda") for i in range(N)]
outs = [torch.empty((T, W * H), dtype=torch.uint8, device="cuda") for _ in range(N)]
lanes = [torch.cuda.Stream() for _ in range(2)]
for m in ("fsr", "ssr"):
    def batch():
        for k, (v, o) in enumerate(zip(vols, outs)):
            spk.reconstruct(v, m, out=o, stream=lanes[k % 2])
    for _ in range(2):
        batch()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    for ln in lanes:
        ln.wait_stream(torch.cuda.current_stream())
    batch()
    t1 = time.perf_counter()
    for ln in lanes:
        torch.cuda.current_stream().wait_stream(ln)
    e1.record()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    # one stream, one volume at a time
    s = torch.cuda.current_stream()
    e2, e3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e2.record()
    for v, o in zip(vols, outs):
        spk.reconstruct(v, m, out=o)
    e3.record()
    torch.cuda.synchronize()
    print(f"{m}: 2 lanes {e0.elapsed_time(e1):.2f} ms device, host issue {1e3*(t1-t0):.2f} ms, "
          f"wall {1e3*(t2-t0):.2f} ms; 1 lane {e2.elapsed_time(e3):.2f} ms", flush=True)

# the same batch captured once in a CUDA graph and replayed
for m, nb in (("fsr", 2), ("fsr", 4), ("fsr", 8), ("ssr", 4)):
    s0 = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s0):
        for _ in range(2):  # warm (pools, attributes)
            for v, o in zip(vols, outs):
                spk.reconstruct(v, m, out=o, stream=s0)
    torch.cuda.synchronize()
    with torch.cuda.graph(g, stream=s0):
        fork = [torch.cuda.Stream() for _ in range(nb)]
        cur = torch.cuda.current_stream()
        for ln in fork:
            ln.wait_stream(cur)
        for k, (v, o) in enumerate(zip(vols, outs)):
            spk.reconstruct(v, m, out=o, stream=fork[k % nb])
        for ln in fork:
            cur.wait_stream(ln)
    ref = [o.clone() for o in outs]
    for _ in range(2):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    same = all(torch.equal(a, b) for a, b in zip(outs, ref))
    print(f"{m}: graph of 64 calls on {nb} branches {e0.elapsed_time(e1) / 5:.2f} ms, frames equal {same}",
          flush=True)
