"""Per-kernel ncu figures of one configs[1] step, tied to the library build.

    # on the GPU box (one process per method; the first step is skipped):
    ncu --set full --clock-control none --launch-skip 9 --launch-count 8 \\
        -o gpurun_out/step_fsr python profiles/ncu_step_profile.py run fsr
    ncu ... -o gpurun_out/step_ssr python profiles/ncu_step_profile.py run ssr
    # here (or there):
    python profiles/ncu_step_profile.py summarize gpurun_out/step_fsr.ncu-rep gpurun_out/step_ssr.ncu-rep

`summarize` writes profiles/ncu_step.json: the SHA-256 (16 hex) of the
libspikecam_b200.so that was profiled and, per method and kernel, its DRAM
bytes per launch (dram__bytes_read.sum + dram__bytes_write.sum), ncu's cold,
serialised duration, the DRAM-throughput / ALU / FMA / issue percentages and
warp instructions.  bench.py reports these figures only when the hash matches
the library it loads.
"""
import csv
import hashlib
import io
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
LIB = ROOT / "paper_2412_11639_b200" / "libspikecam_b200.so"
SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9,
         "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0,
         "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0}


def run(method: str) -> None:
    import torch
    sys.path.insert(0, str(ROOT))
    import paper_2412_11639_b200 as spk
    vol = spk.synth("moving", 0, 400, 250, 40000, device="cuda")
    out = torch.empty((40000, 400 * 250), dtype=torch.uint8, device="cuda")
    for _ in range(2):
        spk.reconstruct(vol, method, out=out)
    torch.cuda.synchronize()
    from paper_2412_11639_b200.build import source_sha16
    print("ok", method, source_sha16())


def kernel_rows(rep: str):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    head, units = rows[0], rows[1]

    def val(r, name):
        if name not in head:
            return 0.0
        i = head.index(name)
        return float(r[i].replace(",", "")) * SCALE.get(units[i], 1.0)

    def pct(r, name):
        if name not in head:
            return None
        return round(float(r[head.index(name)].replace(",", "")) / 100.0, 4)

    out = {}
    for r in rows[2:]:
        name = r[head.index("Kernel Name")].split("(")[0].replace("void ", "").split("<")[0]
        k = {"dram_bytes": val(r, "dram__bytes_read.sum") + val(r, "dram__bytes_write.sum"),
             "dram_read": val(r, "dram__bytes_read.sum"),
             "dram_write": val(r, "dram__bytes_write.sum"),
             "ncu_ms": val(r, "gpu__time_duration.sum") * 1e3,
             "dram_throughput": pct(r, "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
             "alu_pipe": pct(r, "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active"),
             "fma_pipe": pct(r, "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active"),
             "issue_active": pct(r, "sm__inst_issued.avg.pct_of_peak_sustained_active"),
             "warp_inst": val(r, "smsp__inst_executed.sum")}
        if name.startswith("k_scan") or name.startswith("k_fin"):  # the finalize phase
            agg = out.setdefault("finalize", {"dram_bytes": 0.0, "ncu_ms": 0.0, "warp_inst": 0.0})
            for key in ("dram_bytes", "ncu_ms", "warp_inst"):
                agg[key] += k[key]
        out[name] = k  # one launch per kernel per step (scan kernels: the last)
    return out


def summarize(reps, out=None):
    sys.path.insert(0, str(ROOT))
    from paper_2412_11639_b200.build import source_sha16
    d = {"build_sha16": source_sha16(),
         "source": "ncu --set full --clock-control none, one warm configs[1] step per method "
                   "(profiles/ncu_step_profile.py)"}
    for rep in reps:
        method = "ssr" if "ssr" in Path(rep).name else "fsr"
        d[method] = kernel_rows(rep)
    Path(out or ROOT / "profiles" / "ncu_step.json").write_text(json.dumps(d, indent=1) + "\n")
    print(json.dumps(d, indent=1))


if __name__ == "__main__":
    if sys.argv[1] == "run":
        run(sys.argv[2])
    else:  # summarize REP... [--out FILE]
        args = sys.argv[2:]
        out = None
        if "--out" in args:
            i = args.index("--out")
            out = args[i + 1]
            del args[i:i + 2]
        summarize(args, out)
