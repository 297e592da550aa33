"""Top SASS lines by warp-stall samples from an ncu report:
python profiles/ncu_hot_sass.py report.ncu-rep [n]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(txt)))
h = r[1]
si = h.index("Warp Stall Sampling (All Samples)")
ei = h.index("Instructions Executed")
rows = []
for x in r[2:]:
    try:
        rows.append((int(x[si]), int(x[ei]), x[0][-5:], x[1].strip()))
    except (ValueError, IndexError):
        pass
tot = sum(t[0] for t in rows)
print("total samples", tot, " instructions executed", sum(t[1] for t in rows))
for s, e, a, src in sorted(rows, key=lambda t: -t[0])[:n]:
    print(f"{s:7d} {100*s/tot:5.1f}% exec={e:9d} {a} {src[:80]}")
