"""Hot SASS lines of one kernel in an ncu report (exec count, stall samples)."""
import csv
import subprocess
import sys


def main(rep, kernel, frac=0.003):
    out = subprocess.run(["ncu", "-i", rep, "-k", f"regex:{kernel}", "--page", "source", "--csv",
                          "--print-source", "sass"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdrs = [i for i, r in enumerate(rows) if r and r[0] == "Address"]
    h = rows[hdrs[0]]
    ia, isrc = h.index("Address"), h.index("Source")
    ie, iss = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
    ith = h.index("Avg. Threads Executed")
    end = hdrs[1] - 1 if len(hdrs) > 1 else len(rows)
    data = []
    for r in rows[hdrs[0] + 1:end]:
        try:
            data.append((r[isrc], int(r[ie] or 0), int(r[iss] or 0), float(r[ith] or 0)))
        except (ValueError, IndexError):
            pass
    tot = sum(d[1] for d in data)
    ts = sum(d[2] for d in data)
    print(f"warp-instructions {tot}  stall samples {ts}  sass lines {len(data)}")
    for i, d in enumerate(data):
        if d[1] > tot * frac or d[2] > ts * 0.01:
            print(f"{i:5d} {d[0][:72]:72s} {d[1]:>11d} {d[2]:>7d} {d[3]:5.1f}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], float(sys.argv[3]) if len(sys.argv) > 3 else 0.003)
