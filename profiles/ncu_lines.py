"""Instructions executed and stall samples per CUDA source line of a kernel
in an ncu report (needs -lineinfo): python profiles/ncu_lines.py REP [n]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = []
fname = None
hdr = None
for rec in csv.reader(io.StringIO(txt)):
    if not rec:
        continue
    if rec[0] in ("File Name", "File Path"):
        fname = rec[1].split("/")[-1]
        hdr = None
        continue
    if rec[0] == "Line No" or rec[0] == "#":
        hdr = rec
        continue
    if hdr is None:
        continue
    if len(rec) > 2 and rec[2].startswith("0x"):  # a SASS row under the line
        continue
    try:
        ei = hdr.index("Instructions Executed")
        si = hdr.index("Warp Stall Sampling (All Samples)")
        rows.append((int(rec[ei] or 0), int(rec[si] or 0), fname, rec[0], rec[1].strip()))
    except (ValueError, IndexError):
        pass
te = sum(r[0] for r in rows) or 1
ts = sum(r[1] for r in rows) or 1
print(f"instructions executed {te:.3e}, stall samples {ts}")
for e, s, f, ln, src in sorted(rows, key=lambda r: -r[0])[:n]:
    print(f"{100*e/te:5.1f}% inst {100*s/ts:5.1f}% stall  {f}:{ln:5s} {src[:90]}")
