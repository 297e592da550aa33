"""Debug driver for time shards: python tests/ts_debug2.py scene W H T method b0,b1,... [param] [pcap]"""
import sys, torch
sys.path.insert(0, ".")
import paper_2412_11639_b200 as spk
from paper_2412_11639_b200.shard import TimeShard, fresh_state
scene, W, H, T, method = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]), sys.argv[5]
bounds = [int(x) for x in sys.argv[6].split(",")]
param = float(sys.argv[7]) if len(sys.argv) > 7 else 0.0
pcap = int(sys.argv[8]) if len(sys.argv) > 8 else 64
vol = spk.synth(scene, 7 if scene == "range" else 9, W, H, T, param=param, device="cuda")
shards = [TimeShard(vol, b0, b1, method, pcap) for b0, b1 in zip(bounds, bounds[1:])]
for sh in shards:
    sh.speculate()
torch.cuda.synchronize(); print("spec ok", flush=True)
entry = fresh_state(vol.npix, vol.planes.device)
for sh in shards:
    entry = sh.resolve(entry); torch.cuda.synchronize()
    print("resolve", sh.f0, torch.bincount((sh.sync[:, 3] + 2).long()).tolist(), "fb" if sh.fb is not None else "", flush=True)
closes = [None] * len(shards)
closes[-1] = shards[-1].tail_close
for r in range(len(shards) - 2, -1, -1):
    closes[r] = shards[r].close_from_next(shards[r + 1].entry_close, closes[r + 1])
torch.cuda.synchronize(); print("close ok", flush=True)
out = torch.empty((T, vol.npix), dtype=torch.uint8, device="cuda")
for sh, c in zip(shards, closes):
    sh.stitch(c); torch.cuda.synchronize()
    rr = sh.region[:, :, 0].cpu(); cnt = sh.region_counts.cpu(); lst = sh.region_last.cpu()
    bad = 0
    for p in range(sh.npix):
        n = int(cnt[p])
        if n > sh.rcap:
            bad += 1; continue
        st = rr[p, :n].tolist()
        ok = all(a < b for a, b in zip(st, st[1:])) and (n == 0 or (st[-1] < sh.frames and int(lst[p]) > st[-1])) and (n < 2 or st[1] > 0)
        if not ok and bad < 3:
            print("  bad", sh.f0, p, n, st[:4], st[-2:], int(lst[p]), sh.sync[p].tolist(), c[p].tolist(), flush=True)
        bad += not ok
    print("stitch", sh.f0, "bad", bad, flush=True)
    sh.expand(out[sh.f0:sh.f1]); torch.cuda.synchronize()
ref = spk.reconstruct(vol, method).reshape(T, -1)
badp = (ref != out).any(0).nonzero().flatten().tolist()
print("mismatch", int((ref != out).sum()), "pixels", len(badp))
runs, counts, last = spk.segments(vol, method, run_cap=4096)
for p in badp[:3]:
    n = int(counts[p]); rl = runs[p, :n].tolist()
    fr = (ref[:, p] != out[:, p]).nonzero().flatten().tolist()
    print("pixel", p, "frames", fr[:2], fr[-2:], "true runs near", [r for r in rl if fr[0] - 3000 < r[0] < fr[-1] + 50][:12], "last", int(last[p]))
    for sh, c in zip(shards, closes):
        if sh.f0 - 2000 <= fr[0] <= sh.f1 + 2000:
            n2 = int(sh.region_counts[p]); reg = sh.region[p, :n2].tolist()
            print("  shard", sh.f0, sh.f1, "sync", sh.sync[p].tolist(), "region", [(a + sh.f0, b) for a, b in reg][:5], "...", [(a + sh.f0, b) for a, b in reg][-3:], "last", int(sh.region_last[p]) + sh.f0, "close", c[p].tolist(), "ec", sh.entry_close[p].tolist())
