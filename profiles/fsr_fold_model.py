"""Iteration-count model of the FSR K2 loop (host, no GPU): per pixel the exact-step
events with and without folding pair completions into the bit-parallel test, and the
iterations of a K-word window loop; the warp pays its busiest lane.  Uses the host
generator of the configs[1] scene (bench.py moving_scene_cpu), 3 rows x 40,000 frames.
python profiles/fsr_fold_model.py"""
import sys, numpy as np
sys.path.insert(0, ".")
from bench import moving_scene_cpu
W, H, T = 400, 3, 40000
pl = moving_scene_cpu(W, H, T, 5)
bits = np.unpackbits(pl, axis=1, bitorder="little")[:, :W*H]  # [T, npix]
def events(sp, fold):
    ev = []
    lo = None; hw = 0; last = None
    for s in sp:
        if last is None:
            ev.append(s); last = s; continue
        t = s - last
        if lo is None:
            lo, hw = t, 0; ev.append(s)
        elif lo <= t <= lo + hw:
            pass
        elif hw == 0 and abs(t - lo) == 1:
            if not fold: ev.append(s)
            lo, hw = min(lo, t), 1
        else:
            ev.append(s); lo, hw = t, 0
        last = s
    return ev
def iters(ev, K):
    ev = np.array(ev + [10**9]); i = 0; cur = 0; it = 0
    while cur < T:
        w0 = cur // 32; end = (w0 + K) * 32
        while ev[i] < cur: i += 1
        if ev[i] < end: cur = ev[i] + 1
        else: cur = end
        it += 1
    return it
res = {}
for p in range(0, W*H, 7):
    sp = np.nonzero(bits[:, p])[0].tolist()
    for fold in (0, 1):
        ev = events(sp, fold)
        for K in (1, 2, 3, 4, 6, 8):
            res.setdefault((fold, K), []).append(iters(ev, K))
        res.setdefault((fold, 'ev'), []).append(len(ev))
for k, v in sorted(res.items(), key=str):
    v = np.array(v)
    # warp max over 32 consecutive sampled lanes
    m = v[: len(v)//32*32].reshape(-1, 32).max(1).mean()
    print(k, "mean", v.mean(), "warpmax~", m)
