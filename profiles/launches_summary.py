"""Per-kernel summary of an ncu --csv launch list (metrics per launch)."""
import csv
import sys
from collections import defaultdict


def main(path, skip_prefix=("k_synth",)):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, mi, vi, ui = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value",
                                            "Metric Unit"))
    idi = h.index("ID")
    per = defaultdict(lambda: defaultdict(list))
    units = {}
    for r in rows[hdr + 1:]:
        name = r[ki].split("(")[0].replace("void ", "")
        per[name][r[mi]].append(float(r[vi].replace(",", "")))
        units[r[mi]] = r[ui]
    for name, mets in per.items():
        parts = [f"{name:28s} n={len(next(iter(mets.values())))}"]
        for m, v in sorted(mets.items()):
            parts.append(f"{m.split('__')[1][:24]}={sum(v)/len(v):.4g}{units[m]}")
        print("  ".join(parts))


if __name__ == "__main__":
    main(sys.argv[1])
