"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list
(stdin): the second half of the launches (the timed call of one_call.py),
library kernels only."""
import csv
import sys

rows = [r for r in csv.reader(line for line in sys.stdin if not line.startswith("=="))]
h = rows[0]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
rs = rows[1:]
rs = rs[len(rs) // 2:]
tot = 0.0
for r in rs:
    if r[ki].startswith("k_synth") or "elementwise" in r[ki] or "fill" in r[ki]:
        continue
    v = float(r[vi].replace(",", "")) / 1e3
    tot += v
    print(f"{r[ki][:44]:44s} {v:10.1f} us")
print(f"total {tot:.1f} us")
