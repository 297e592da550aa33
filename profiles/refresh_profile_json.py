"""Refresh profiles/traffic_*.json and alu_*.json (read by bench.py) from an
ncu --set full capture of profiles/prof_c2.py:
python profiles/refresh_profile_json.py REP METHOD"""
import csv
import json
import subprocess
import sys
from pathlib import Path

rep, method = sys.argv[1], sys.argv[2]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[0]


def col(name):
    return h.index(name)


def num(v):
    return float(v.replace(",", ""))


seen = {}
for r in rows[2:]:
    k = r[col("Kernel Name")].split("(")[0].replace("void ", "")
    k = k.split("<")[0]
    seen[k] = r  # the last (warm) launch of each kernel
here = Path(__file__).resolve().parent
for kern in ("k_segment", "k_expand"):
    if kern not in seen:  # capture restricted to other kernels: keep the file
        continue
    r = seen[kern]
    rd, wr = num(r[col("dram__bytes_read.sum")]), num(r[col("dram__bytes_write.sum")])
    unit_r, unit_w = rows[1][col("dram__bytes_read.sum")], rows[1][col("dram__bytes_write.sum")]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    rd *= scale[unit_r]
    wr *= scale[unit_w]
    (here / f"traffic_{kern}_{method}.json").write_text(json.dumps({
        "bytes_per_launch": rd + wr, "dram_bytes_read": rd, "dram_bytes_write": wr,
        "source": f"{rep} (ncu --set full, C2 {method.upper()}, profiles/prof_c2.py)"}, indent=1) + "\n")
    if kern == "k_segment":
        stalls = []
        for i, n in enumerate(h):
            if n.startswith("smsp__average_warps_issue_stalled_") and n.endswith("_per_issue_active.ratio"):
                stalls.append((num(r[i]), n[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
        stalls.sort(reverse=True)
        (here / f"alu_{kern}_{method}.json").write_text(json.dumps({
            "alu_pipe_frac": round(num(r[col("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active")]) / 100, 3),
            "issue_active_frac": round(num(r[col("sm__inst_issued.avg.pct_of_peak_sustained_active")]) / 100, 3),
            "fma_pipe_frac": round(num(r[col("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active")]) / 100, 3),
            "top_stalls": ", ".join(f"{n} {v:.2f}" for v, n in stalls[:3] if n != "selected") + " warps/issue",
            "source": f"{rep} (sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active)"}, indent=1) + "\n")
    print(kern, method, rd + wr)
