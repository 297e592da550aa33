"""Instructions of one kernel in an ncu report grouped by execution count
(a proxy for code regions: loop bodies share a count): python profiles/ncu_buckets.py REP KERNEL"""
import csv
import subprocess
import sys
from collections import Counter, defaultdict

rep, kern = sys.argv[1], sys.argv[2]
out = subprocess.run(["ncu", "-i", rep, "-k", f"regex:{kern}", "--page", "source", "--csv",
                      "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdrs = [i for i, r in enumerate(rows) if r and r[0] == "Address"]
h = rows[hdrs[0]]
isrc, ie = h.index("Source"), h.index("Instructions Executed")
iss = h.index("Warp Stall Sampling (All Samples)")
tot, stalls, n_of = Counter(), Counter(), Counter()
ops = defaultdict(Counter)
for r in rows[hdrs[0] + 1:(hdrs[1] - 1 if len(hdrs) > 1 else len(rows))]:
    try:
        n, st = int(r[ie] or 0), int(r[iss] or 0)
    except (ValueError, IndexError):
        continue
    if n == 0:
        continue
    tot[n] += n
    stalls[n] += st
    n_of[n] += 1
    op = r[isrc].split()[0] if not r[isrc].startswith("@") else r[isrc].split()[1]
    ops[n][op.split(".")[0]] += 1
T, S = sum(tot.values()), sum(stalls.values())
for n, v in sorted(tot.items(), key=lambda x: -x[1])[:14]:
    top = ", ".join(f"{o}:{c}" for o, c in ops[n].most_common(6))
    print(f"exec {n:>9d}  instrs {n_of[n]:>4d}  {v / T * 100:5.1f}% inst  {stalls[n] / max(S, 1) * 100:5.1f}% stall  [{top}]")
print("total warp-instructions", T)
