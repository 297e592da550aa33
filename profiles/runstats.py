import sys, torch
sys.path.insert(0, ".")
import paper_2412_11639_b200 as spk
for scene in ("moving", "static"):
    vol = spk.synth(scene, 0, 400, 250, 40000, device="cuda")
    for m in ("fsr", "ssr"):
        runs, counts, last = spk.segments(vol, m, run_cap=8192)
        c = counts.float()
        w = c.view(-1, 32)
        print(scene, m, "runs/px mean %.1f max %.0f | per-warp max mean %.1f | warp max/mean %.2f" % (
            c.mean(), c.max(), w.max(1).values.mean(), (w.max(1).values / w.mean(1).clamp(min=1)).mean()))
        hist = torch.histc(c, bins=10, min=0, max=float(c.max()))
        print("  hist", [int(x) for x in hist.tolist()])
