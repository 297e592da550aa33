"""SASS of one kernel from an ncu report with per-instruction execution
counts, grouped into runs of equal count (~basic blocks): shows where the
warp instructions go.  python profiles/ncu_sass_blocks.py REP KERNEL_REGEX [min_share]"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
min_share = float(sys.argv[3]) if len(sys.argv) > 3 else 0.005
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                      "-k", f"regex:{kern}"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
h = rows[1]
ei, si = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
ins = []
for r in rows[2:]:
    try:
        ins.append((r[0][-5:], r[1].strip(), int(r[ei]), int(r[si])))
    except (ValueError, IndexError):
        pass
tot = sum(e for _, _, e, _ in ins)
print(f"total warp instructions {tot:,}")
blocks, cur = [], []
for x in ins:
    if cur and x[2] != cur[-1][2]:
        blocks.append(cur)
        cur = []
    cur.append(x)
blocks.append(cur)
for b in blocks:
    n = sum(x[2] for x in b)
    if n / tot < min_share:
        continue
    print(f"--- {len(b)} instrs x {b[0][2]:,} = {100*n/tot:.1f}%  stalls={sum(x[3] for x in b)}")
    for a, src, e, st in b:
        print(f"   {a} {st:6d} {src[:90]}")
