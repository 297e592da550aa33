"""Fraction of runs whose uint8 value equals the previous run's (a change
that changes nothing): python profiles/same_value_runs.py SCENE W H T"""
import sys

import torch

sys.path.insert(0, ".")
import paper_2412_11639_b200 as spk  # noqa: E402

scene, W, H, T = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
vol = spk.synth(scene, 0, W, H, T, device="cuda")
for m in ("fsr", "ssr"):
    runs, counts, last = spk.segments(vol, m)
    cap = runs.shape[1]
    n = counts.clamp(max=cap).long()
    st = runs[..., 0].long()
    iv = runs[..., 1].double()
    nxt = torch.cat([st[:, 1:], torch.full_like(st[:, :1], 0)], dim=1)
    idx = torch.arange(cap, device="cuda")[None, :]
    nxt = torch.where(idx == (n - 1)[:, None], last.long()[:, None], nxt)
    span = (nxt - st).double().clamp(min=1)
    u8 = torch.floor((510.0 * iv + span) / (2.0 * span))
    valid = idx < n[:, None]
    same = (u8[:, 1:] == u8[:, :-1]) & valid[:, 1:]
    tot = int(valid.sum())
    print(f"{scene} {m}: runs {tot}, same value as previous run {int(same.sum())} "
          f"({100.0 * int(same.sum()) / max(tot, 1):.1f}%)")
