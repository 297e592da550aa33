import sys, torch
sys.path.insert(0, ".")
import paper_2412_11639_b200 as spk
vol = spk.synth("moving", 0, 400, 250, 40000, device="cuda")
out = torch.empty((40000, 100000), dtype=torch.uint8, device="cuda")
for m in ("fsr", "ssr"):
    for _ in range(3):
        spk.reconstruct(vol, m, out=out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        spk.reconstruct(vol, m, out=out)
    e1.record(); torch.cuda.synchronize()
    print(m, "ms/step", e0.elapsed_time(e1) / 10)
