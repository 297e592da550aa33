"""K2 alone: one whole-stream launch vs all time shards' speculative scans in
one launch (spk_segment_shards), CUDA events.  Also checks that the
one-launch shards equal per-shard spk_segment_state calls.
python profiles/shard_k2_probe.py SCENE W H T [S,S,...]"""
import ctypes as C
import sys

import torch

sys.path.insert(0, ".")
import paper_2412_11639_b200 as spk  # noqa: E402
from paper_2412_11639_b200 import _capi as capi  # noqa: E402

scene, W, H, T = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
Ss = [int(x) for x in (sys.argv[5] if len(sys.argv) > 5 else "1,2,4,8,16").split(",")]
lib = capi.lib()
npix = W * H
vol = spk.synth(scene, 0, W, H, T, device="cuda")
i32 = dict(dtype=torch.int32, device="cuda")
for method in ("fsr",):
    mk = 0 if method == "fsr" else 1
    for S in Ss:
        words = (T + 31) // 32
        sf = ((words + S - 1) // S) * 32
        ns = (T + sf - 1) // sf
        cap = max(64, sf // 32) if S > 1 else max(64, T // 32)
        runs = torch.empty((ns, npix, cap, 2), **i32)
        counts = torch.empty((ns, npix), **i32)
        last = torch.empty((ns, npix), **i32)
        st = torch.empty((ns, 17, npix), **i32)
        g = capi.geom(W, H, T, vol.pitch)

        def go():
            if S == 1:
                capi.check(lib.spk_segment(g, vol.planes.data_ptr(), mk, runs.data_ptr(), cap,
                                           counts.data_ptr(), last.data_ptr(), None))
            else:
                capi.check(lib.spk_segment_shards(g, vol.planes.data_ptr(), mk, sf, runs.data_ptr(), cap,
                                                  counts.data_ptr(), last.data_ptr(), st.data_ptr(), None))
        for _ in range(2):
            go()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 5 if T > 100000 else 20
        e0.record()
        for _ in range(reps):
            go()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        ok = ""
        if S > 1 and npix * cap * 8 < 4e9:
            # shard 1 against its own per-shard call
            r = 1
            f0, f1 = r * sf, min(T, (r + 1) * sf)
            g1 = capi.geom(W, H, f1 - f0, vol.pitch)
            runs1 = torch.empty((npix, cap, 2), **i32)
            c1 = torch.empty((npix,), **i32)
            l1 = torch.empty((npix,), **i32)
            s1 = torch.empty((17, npix), **i32)
            capi.check(lib.spk_segment_state(g1, vol.planes[f0:f1].data_ptr(), mk, runs1.data_ptr(), cap,
                                             c1.data_ptr(), l1.data_ptr(), None, s1.data_ptr(), None))
            torch.cuda.synchronize()
            n = c1.clamp(max=cap)
            mask = torch.arange(cap, device="cuda")[None, :] < n[:, None]
            same = (torch.equal(c1, counts[r]) and torch.equal(l1, last[r]) and torch.equal(s1, st[r])
                    and torch.equal(runs1[mask], runs[r][mask]))
            ok = f" shard1==own call: {same}"
        print(f"{scene} {W}x{H}x{T} {method} S={S} ({ns} shards of {sf}): K2 {ms:.3f} ms, "
              f"max count {int(counts.max())} cap {cap}{ok}", flush=True)
        del runs, counts, last, st
        torch.cuda.empty_cache()
