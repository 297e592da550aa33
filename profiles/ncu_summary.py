"""Summarise an ncu report: per kernel time, DRAM bytes, throughputs (profiles/)."""
import csv
import subprocess
import sys

WANT = [
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "dram_rd"),
    ("dram__bytes_write.sum", "dram_wr"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram%"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm%"),
    ("sm__inst_executed.avg.per_cycle_active", "ipc"),
    ("smsp__inst_executed.sum", "warp_inst"),
    ("smsp__thread_inst_executed_per_inst_executed.ratio", "lanes/inst"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occ%"),
    ("launch__registers_per_thread", "regs"),
    ("lts__t_bytes.sum", "l2_bytes"),
]


def main(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h = rows[0]
    units = rows[1]
    for r in rows[2:]:
        name = r[h.index("Kernel Name")]
        parts = [name[:40]]
        for key, tag in WANT:
            if key in h:
                i = h.index(key)
                parts.append(f"{tag}={r[i]}{units[i] if units[i] not in ('', '%') else ''}")
        print("  ".join(parts))


if __name__ == "__main__":
    main(sys.argv[1])
