import csv, subprocess, sys
rep, kernel = sys.argv[1], sys.argv[2]
out = subprocess.run(["ncu", "-i", rep, "-k", f"regex:{kernel}", "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdrs = [i for i, r in enumerate(rows) if r and r[0] == "Address"]
h = rows[hdrs[0]]
isrc, ie, iss, ith = h.index("Source"), h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)"), h.index("Avg. Threads Executed")
end = hdrs[1] - 1 if len(hdrs) > 1 else len(rows)
for i, r in enumerate(rows[hdrs[0] + 1:end]):
    try:
        print(f"{i:5d} {int(r[ie] or 0):>10d} {int(r[iss] or 0):>6d} {float(r[ith] or 0):5.1f}  {r[isrc][:90]}")
    except Exception:
        pass
