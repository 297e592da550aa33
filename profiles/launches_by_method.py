"""Split an ncu launch list by the segment kernel that precedes each launch."""
import csv
import sys
from collections import defaultdict


def main(path):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    cur, d = None, defaultdict(list)
    for r in rows[hdr + 1:]:
        if r[mi] != "gpu__time_duration.sum":
            continue
        name = r[ki].split("(")[0].replace("void ", "")
        if name.startswith("k_segment"):
            cur = name
        d[(cur, name)].append(float(r[vi].replace(",", "")))
    tot = defaultdict(float)
    for (cur, name), v in sorted(d.items(), key=lambda x: str(x)):
        m = sum(v) / len(v) / 1e3
        tot[cur] += m
        print(f"{str(cur):14s} {name:32s} n={len(v):3d} {m:9.1f} us")
    for cur, t in tot.items():
        print(f"{str(cur):14s} {'TOTAL per step':32s}       {t:9.1f} us")


if __name__ == "__main__":
    main(sys.argv[1])
