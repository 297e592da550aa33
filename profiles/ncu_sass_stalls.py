import csv, subprocess, sys
rep, kernel, thr = sys.argv[1], sys.argv[2], int(sys.argv[3])
out = subprocess.run(["ncu", "-i", rep, "-k", f"regex:{kernel}", "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hi = [i for i, r in enumerate(rows) if r and r[0] == "Address"]
h = rows[hi[0]]
end = hi[1] - 1 if len(hi) > 1 else len(rows)
cols = ['stall_branch_resolving','stall_lg','stall_long_sb','stall_math','stall_mio','stall_not_selected','stall_selected','stall_short_sb','stall_wait','stall_drain','stall_dispatch']
idx = {c: h.index(c) for c in cols}
isrc = h.index("Source"); iall = h.index("Warp Stall Sampling (All Samples)")
for i, r in enumerate(rows[hi[0]+1:end]):
    try:
        tot = int(r[iall] or 0)
    except Exception:
        continue
    if tot >= thr:
        parts = " ".join(f"{c[6:]}={r[idx[c]]}" for c in cols if r[idx[c]] not in ("", "0"))
        print(f"{i:5d} {tot:6d} {r[isrc][:50]:50s} {parts}")
