#!/usr/bin/env python
"""Benchmark: FSR/SSR spike-stream reconstruction on B200 (arXiv 2412.11639).

Metric (BASELINE.json): reconstructed frames/s at 400x250, with Gpixel-frames/s
and the fraction of the HBM roofline.  One "step" = one pass of the hot path
(bit-packed planes -> one uint8 frame per timestep, all pixels) over the
BASELINE.json configs[1] workload: the moving scene, 400x250 px, 40,000
timesteps (synthetic, seeded; the paper's datasets are not available).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--method fsr|ssr]
    python bench.py --impl reference ...   # the reference CPU implementation

N>1 (torchrun, one rank per GPU): every rank reconstructs its own independent
stream (stream sharding, BASELINE configs[3] style): weak scaling, no
data-path collective; time = max over ranks of device time.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "reconstructed frames/sec at 400x250 (and Gpixel-frames/s); % of HBM roofline"
W, H, T = 400, 250, 40000
FPGA_FPS = 20000.0  # FSR/SSR on the XCVU9P FPGA, 400x250
BYTES_PER_PXF = 1.125  # 1 packed input bit + 1 uint8 output byte
CPU_SAMPLE_FRAMES = 2000
LONG_T = 1_000_000  # BASELINE configs[4]: one long stream, extreme dynamic range


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


def build_sha16() -> str:
    """Hash (16 hex) of the sources and flags the loaded sm_100a library was
    built from (paper_2412_11639_b200.build.source_sha16: nvcc's output is not
    byte-reproducible, so a build is identified by its sources)."""
    from paper_2412_11639_b200.build import source_sha16
    return source_sha16()


def step_profile(lib_sha: str):
    """Per-kernel ncu figures of one C2 step (profiles/ncu_step.json, written
    by profiles/ncu_step_profile.py from an ncu --set full capture), only when
    they were captured from this very build."""
    f = ROOT / "profiles" / "ncu_step.json"
    if not f.exists():
        return None
    d = json.loads(f.read_text())
    return d if d.get("build_sha16") == lib_sha else None


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


# ------------------------------------------------------------------ clocks --
class ClockSampler:
    """NVML samples of SM clock and throttle reasons during the timed region."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
        0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
        0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
        0x100: "display_clock_setting",
    }

    def __init__(self, index: int):
        self.samples, self.reasons, self.max_mhz = [], 0, None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:  # noqa: BLE001 -- clocks are reported as unavailable
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                self.reasons |= self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            except Exception:  # noqa: BLE001
                pass
            time.sleep(0.01)

    def __enter__(self):
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nv:
            self.t.join()

    def report(self):
        if not self.nv or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unavailable"]}
        names = [n for b, n in self.REASONS.items() if self.reasons & b and n != "gpu_idle"]
        return {"sm_mhz": float(np.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": names, "samples": len(self.samples)}


# ------------------------------------------------------------ CPU baseline --
def cpu_model() -> str:
    try:
        for ln in Path("/proc/cpuinfo").read_text().splitlines():
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_reference_fps(planes_host: np.ndarray, pitch: int, w: int, h: int, t: int, method: int,
                      repeats: int = 3, workers: int | None = None):
    """The reference's own bench() (proj/src/metrics.cpp:63-82) on the host:
    median of `repeats` reconstruct() calls with `workers` OpenMP threads
    (default: every host thread).  Returns (fps, threads used, kind)."""
    from oracle.oracle import Reference, ref_available

    cores = workers or os.cpu_count() or 1
    if ref_available():
        fps = Reference().bench_fps(planes_host, pitch, w, h, t, method, 32, repeats, cores)
        return fps, cores, "reference"
    from oracle.oracle import Oracle  # C restatement as the port baseline
    o = Oracle()
    t0 = time.perf_counter()
    for _ in range(repeats):
        o.reconstruct(planes_host, w, h, t, pitch, method, 32, dtype=np.float64, threads=cores)
    return repeats * t / (time.perf_counter() - t0), cores, "port"


def cpu_baseline_block(planes_host: np.ndarray, pitch: int, method: int, source: str,
                       long_planes: np.ndarray | None = None):
    """cpu_baseline: the reference on the box's host cores, every thread and
    one thread, on frames [0, CPU_SAMPLE_FRAMES) of the configs[1] stream
    (plus a longer sample, when given, for the frames-vs-T scaling)."""
    tcpu = planes_host.shape[0]
    fps_all, cores, kind = cpu_reference_fps(planes_host, pitch, W, H, tcpu, method)
    fps_one, _, _ = cpu_reference_fps(planes_host, pitch, W, H, tcpu, method, workers=1)
    blk = {"value": fps_all, "unit": "frames/s", "cores": cores, "kind": kind,
           "workers_1": fps_one, "cpu_model": cpu_model(),
           "sample": f"frames [0,{tcpu}) of the configs[1] stream ({source}); the reference "
                     f"bench(): median of 3 reconstruct() calls, {cores} OpenMP workers "
                     f"(workers_1: one)"}
    if long_planes is not None:
        tl = long_planes.shape[0]
        fps_l, _, _ = cpu_reference_fps(long_planes, pitch, W, H, tl, method)
        blk["t_scaling"] = {f"T={tcpu}": fps_all, f"T={tl}": fps_l,
                            "note": "reference frames/s at two sample lengths (all threads)"}
    return blk


def reference_stream(frames: int):
    """Frames [0, frames) of the configs[1] stream as host SPK planes: the
    device generator (spk_synth, the GPU arm's exact input) when a GPU is
    present, else the host port of the same scene construction."""
    try:
        import torch
        if torch.cuda.is_available():
            import paper_2412_11639_b200 as spk
            v = spk.synth("moving", 0, W, H, frames, device=torch.device("cuda", 0))
            return v.planes.cpu().numpy(), v.pitch, "device generator, seed 0: the GPU arm's input"
    except Exception:  # noqa: BLE001 -- no usable GPU: host generator below
        pass
    pl = moving_scene_cpu(W, H, frames, 0)
    return pl, pl.shape[1], "host generator (no GPU visible)"


def moving_scene_cpu(w: int, h: int, t: int, seed: int) -> np.ndarray:
    """Host-only generator of the configs[1] moving scene (fallback for the
    reference arm on a host without a GPU; same construction as the device
    generator: 16 seeded sinusoids in [0.01, 0.6] translating at 0.05 px/step,
    an occluding bar at 0.2 px/step, integrate-and-fire with threshold 1 and
    uniform initial residual -- a different random draw).
    Returns dense SPK1 planes [t, ceil(w*h/8)]."""
    rng = np.random.default_rng(seed)
    amp = 0.3 + rng.random(16)
    fx = 0.004 + 0.06 * rng.random(16)
    fy = 0.004 + 0.06 * rng.random(16)
    ph = 2 * np.pi * rng.random(16)
    bar_x0, bar_w, bar_i = 400 * rng.random(), 12 + 20 * rng.random(), 0.01 + 0.1 * rng.random()
    # texture on the 0.05-px lattice: x - 0.05 n = 0.05 * (20 x - n)
    k = np.arange(-(t - 1), 20 * (w - 1) + 1)
    ys = np.arange(h)
    arg = 2 * np.pi * (fx[None, None, :] * (0.05 * k)[None, :, None] +
                       fy[None, None, :] * ys[:, None, None]) + ph
    tex = (0.5 + 0.5 * (amp * np.sin(arg)).sum(-1) / amp.sum())
    tex = np.clip(0.01 + 0.59 * tex, 0.01, 0.6).astype(np.float32)  # [h, len(k)]
    xs = np.arange(w)
    idx = (20 * xs)[None, :] + (t - 1)  # index of k = 20x - n at n = 0
    residual = rng.random((h, w))
    rate_sum = np.zeros((h, w))
    fired = np.zeros((h, w))
    fb = (w * h + 7) // 8
    planes = np.zeros((t, fb), np.uint8)
    for n in range(t):
        q = tex[:, idx[0] - n].astype(np.float64)
        bx = np.fmod(bar_x0 + 0.2 * n, w + bar_w) - bar_w
        inbar = (xs >= bx) & (xs < bx + bar_w)
        q[:, inbar] = np.float32(bar_i)
        rate_sum += q
        bit = residual + rate_sum - fired >= 1.0 - 1e-9
        fired += bit
        planes[n] = np.packbits(bit.reshape(-1), bitorder="little")[:fb]
    return planes


def bench_config(frames: int, method: str, world: int) -> dict:
    """`config` of both arms (the driver compares them)."""
    return {"workload": f"configs[1] moving 400x250x{frames}", "method": method,
            "width": W, "height": H, "frames": frames,
            "parallelism": f"streams x{world} (one independent stream per GPU)",
            "l2": "no flush: 0.5 GB in + 4 GB out per step > 126 MB L2",
            "vs_baseline_ref": "FPGA 20,000 FPS (BASELINE.md, PAPER.md:199)"}


def run_reference_arm(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    method = {"fsr": 0, "ssr": 1}[args.method]
    tcpu = CPU_SAMPLE_FRAMES
    planes, pitch, source = reference_stream(tcpu)
    cores = os.cpu_count() or 1
    for _ in range(args.warmup):
        cpu_reference_fps(planes, pitch, W, H, tcpu, method, repeats=3)
    rates = []
    kind = "reference"
    for _ in range(args.steps):
        fps_i, cores, kind = cpu_reference_fps(planes, pitch, W, H, tcpu, method, repeats=3)
        rates.append(fps_i)
    fps = float(np.median(rates))
    fps_one, _, _ = cpu_reference_fps(planes, pitch, W, H, tcpu, method, repeats=3, workers=1)
    total = args.steps * tcpu / fps
    sample = (f"configs[1] moving scene, frames [0,{tcpu}) of the 400x250x{args.frames} stream "
              f"({source}); per step the reference bench() (median of 3 reconstruct() calls, "
              f"{cores} OpenMP workers); workers_1 = one worker")
    line = {
        "impl": "reference", "metric": METRIC, "value": fps, "unit": "frames/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * total / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": fps / FPGA_FPS, "dtype": "f64", "data": "synthetic",
        "config": bench_config(args.frames, args.method, world),
        "cpu_baseline": {"value": fps, "unit": "frames/s", "cores": cores, "kind": kind,
                         "workers_1": fps_one, "cpu_model": cpu_model(), "sample": sample},
        "e2e": {"value": fps, "unit": "frames/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------- GPU arm --
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--method", default="fsr", choices=["fsr", "ssr"])
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU baseline sample")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=8)
    ap.add_argument("--frames", type=int, default=T)
    ap.add_argument("--no-long", action="store_true", help="skip the configs[4] long-stream leg")
    ap.add_argument("--no-configs", action="store_true",
                    help="skip the configs[0], [2] and [3] legs (static, large sensor, batch of 64)")
    ap.add_argument("--long-frames", type=int, default=LONG_T)
    args = ap.parse_args()
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    if args.impl == "reference":
        return run_reference_arm(args)

    import torch
    import torch.distributed as dist

    import paper_2412_11639_b200 as spk
    from paper_2412_11639_b200 import _capi as capi

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    frames = args.frames
    lib = capi.lib()

    # each rank: its own seeded stream (stream sharding; weak scaling)
    vol = spk.synth("moving", rank, W, H, frames, device=dev)
    out = torch.empty((frames, W * H), dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)

    def step(method):
        spk.reconstruct(vol, method, out=out)

    def timed(method, steps, warmup):
        for _ in range(warmup):
            step(method)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        lib.spk_launch_count(1)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(steps):
            step(method)
        e1.record(stream)
        torch.cuda.synchronize()
        launches = lib.spk_launch_count(1)
        ms = e0.elapsed_time(e1)
        if world > 1:
            t = torch.tensor([ms], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
            dist.barrier()
        return ms, launches

    def kernel_times(method, steps):
        """mean per-phase device time (CUDA events on the launch stream):
        K2 segment, K2b/scan/K2c finalize, K3 expand, fixup"""
        import ctypes as C
        v = [C.c_float() for _ in range(4)]
        acc = [[] for _ in range(4)]
        lib.spk_set_timing(1)
        for _ in range(steps):
            step(method)
            capi.check(lib.spk_last_timing(*(C.byref(x) for x in v)))
            for a, x in zip(acc, v):
                a.append(x.value)
        lib.spk_set_timing(0)
        return [float(np.mean(a)) for a in acc]

    sampler = ClockSampler(local)
    with sampler:
        ms, launches = timed(args.method, args.steps, args.warmup)
    clocks = sampler.report()
    phases = kernel_times(args.method, max(3, min(20, args.steps)))
    other = "ssr" if args.method == "fsr" else "fsr"
    k2 = max(5, args.steps // 5)
    ms2, _ = timed(other, k2, 3)
    phases2 = kernel_times(other, max(3, min(20, k2)))

    peak, peak_kind = peaks()
    pxf = W * H * frames
    ms_step = ms / args.steps
    fps = world * frames / (ms_step * 1e-3)
    gpxf = world * pxf / (ms_step * 1e-3) / 1e9

    lib_sha = build_sha16()
    prof = step_profile(lib_sha)

    def roofline(ph, ms_step, method):
        """The path's HBM roofline: algorithmic bytes of one step (1.125 B per
        px-frame: the packed input bit + the uint8 output byte)
        over the device-timed step.  `kernels`: each phase's share of the step
        (CUDA events on the launch stream), its own algorithmic bytes (K2
        reads 0.125 B/px-frame, the finalize none, K3 writes 1 B/px-frame) over
        its time, and what binds it -- from the ncu --set full capture of this
        very build (profiles/ncu_step.json, matched by the hash of the library's
        sources and flags; null when the capture is of another build)."""
        seg, fin, exp, fix = ph
        step_gbs = pxf * BYTES_PER_PXF / (ms_step * 1e-3) / 1e9
        kp = (prof or {}).get(method, {})

        def kern(name, ms, alg_bytes, note):
            k = {"name": name, "ms": ms, "share": ms / ms_step,
                 "hbm_frac_algorithmic": (alg_bytes / (ms * 1e-3) / 1e9 / peak) if ms > 0 and alg_bytes else None,
                 "bound": note}
            if name in kp:
                k["ncu"] = kp[name]
            return k
        kernels = [kern("k_segment", seg, pxf * 0.125, "integer ALU pipe (issue), not HBM"),
                   kern("finalize", fin, 0.0, "latency (scattered 4-B stores)"),
                   kern("k_expand", exp, pxf * 1.0, "HBM write"),
                   kern("k_fixup", fix, 0.0, "-")]
        # ("finalize" is the aggregate of K2b + scans + K2c, already counted by name)
        traffic = sum(v.get("dram_bytes", 0.0) for k, v in kp.items() if k != "finalize") if kp else None
        return {"bound": "hbm", "scope": "whole step (K2 + finalize + K3 + fixup)",
                "achieved": step_gbs, "peak": peak, "unit": "GB/s", "frac": step_gbs / peak,
                "traffic": traffic, "algorithmic_bytes": pxf * BYTES_PER_PXF,
                "peak_kind": peak_kind, "build_sha16": lib_sha,
                "traffic_source": (prof or {}).get("source"), "kernels": kernels,
                "phases_ms": {"segment": seg, "finalize": fin, "expand": exp, "fixup": fix}}

    line = {
        "metric": METRIC, "value": fps, "unit": "frames/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": fps / FPGA_FPS, "dtype": "u8", "data": "synthetic",
        "config": bench_config(frames, args.method, world),
        "gpx_frames_per_s": gpxf,
        "roofline": roofline(phases, ms_step, args.method),
        "gpu_launches": int(launches),
        "clocks": clocks,
        other: {"value": world * frames / (ms2 / k2 * 1e-3),
                "ms_per_step": ms2 / k2,
                "roofline": roofline(phases2, ms2 / k2, other)},
    }

    # end to end through the C-ABI host boundary (pinned host buffers): the
    # pipelined batch call (upload + kernels of step i+1 under the download of
    # step i), every step with its own H2D of the payload and D2H of the frames
    if not args.no_e2e:
        import ctypes as C
        payload = torch.from_numpy(vol.payload()).pin_memory()
        houts = [torch.empty((frames, W * H), dtype=torch.uint8).pin_memory() for _ in range(2)]
        g = capi.geom(W, H, frames, 0)
        n = args.e2e_steps
        pin = (C.c_void_p * n)(*([payload.data_ptr()] * n))
        pout = (C.c_void_p * n)(*[houts[i % 2].data_ptr() for i in range(n)])
        kind = 0 if args.method == "fsr" else 1

        def e2e_batch(count):
            capi.check(lib.spk_reconstruct_host_batch(g, count, pin, kind, 32, capi.SPK_OUT_U8,
                                                      pout, W * H))
        e2e_batch(2)  # warm: both lanes' device buffers come from the pool afterwards
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        e2e_batch(n)
        el = time.perf_counter() - t0
        if world > 1:
            t = torch.tensor([el], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            el = float(t.item())
        step(args.method)  # device-path result of the same method for the check
        assert torch.equal(houts[(n - 1) % 2][-64:], out[-64:].cpu()), "e2e result differs from device path"
        # the PCIe ceiling of this box: one plain device -> pinned-host copy of a step's frames
        d2h_ms = []
        for _ in range(2):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            houts[0].copy_(out, non_blocking=True)
            e1.record()
            e1.synchronize()
            d2h_ms.append(e0.elapsed_time(e1))
        d2h_gbs = houts[0].numel() / (min(d2h_ms) * 1e-3) / 1e9
        line["e2e"] = {"value": world * frames * n / el, "unit": "frames/s",
                       "h2d_bytes_per_step": int(payload.numel()),
                       "d2h_bytes_per_step": int(houts[0].numel()),
                       "steps": n,
                       "path": "spk_reconstruct_host_batch (C-ABI, pinned host in/out, "
                               "H2D + kernels of step i+1 overlap the D2H of step i)",
                       "pcie_d2h_gbs": d2h_gbs,
                       "pcie_frac": houts[0].numel() * n / el / 1e9 / d2h_gbs,
                       "pcie_note": "4 GB of uint8 frames per step over PCIe: e2e is bound by the "
                                    "device-to-host copy (pcie_d2h_gbs = one plain 4 GB copy on "
                                    "this box; profiles/pcie_probe.py)"}

    if rank == 0 and not args.no_cpu:
        tcpu = min(CPU_SAMPLE_FRAMES, frames)
        host = vol.planes[:tcpu].cpu().numpy()
        longp = vol.planes[:min(4 * tcpu, frames)].cpu().numpy() if frames > tcpu else None
        line["cpu_baseline"] = cpu_baseline_block(host, vol.pitch, 0 if args.method == "fsr" else 1,
                                                  "device generator, seed 0: this arm's input",
                                                  longp)
    if not args.no_long or not args.no_configs:
        del vol, out
        if not args.no_e2e:
            del payload, houts
        torch.cuda.empty_cache()
    if not args.no_configs:
        line["configs"] = other_configs(args, rank, world, dev)
        torch.cuda.empty_cache()
        if rank == 0:
            line["metrics"] = metrics_leg(dev, not args.no_cpu)
            torch.cuda.empty_cache()
    if not args.no_long:
        line["long_stream"] = long_stream(args, rank, world, dev)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def _device_ms(fn, dev, world, steps=5, warmup=3):
    """mean ms of fn() over `steps` (CUDA events on the current stream; fn
    joins any side streams it uses), max over ranks"""
    import torch
    import torch.distributed as dist
    stream = torch.cuda.current_stream(dev)
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        fn()
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    return ms


def metrics_leg(dev, with_cpu):
    """SURVEY 8(f) row 4 on the device: the CLI's `compare` metrics (per-frame
    two_dimensional_entropy + mse against uint8 reference frames) over a
    configs[1] reconstruction, and `verify-stability --in` (stability_order of
    every pixel, depth 8) over configs[0] and configs[1]; beside them the
    reference's own functions on the host (single thread, bounded samples)."""
    import torch

    import paper_2412_11639_b200 as spk
    res = {}
    vol = spk.synth("moving", 0, W, H, T, device=dev)
    f64 = spk.reconstruct(vol, "fsr", dtype=torch.float64)
    ref = spk.reconstruct(vol, "tfi")
    ms = _device_ms(lambda: spk.frame_metrics(f64, ref), dev, 1, steps=3, warmup=1)
    res["compare"] = {"workload": f"configs[1] FSR f64 frames vs TFI uint8 frames, {T} frames",
                      "value": T / (ms * 1e-3), "unit": "frames/s", "ms": ms}
    if with_cpu:
        from oracle.oracle import Reference, ref_available
        if ref_available():
            r = Reference()
            sample = f64[:20].cpu().numpy()
            rs = ref[:20].cpu().numpy().astype(np.float64)
            t0 = time.perf_counter()
            for n in range(20):
                r.te(sample[n].reshape(H, W))
                r.mse(sample[n].reshape(H, W), rs[n].reshape(H, W))
            el = time.perf_counter() - t0
            res["compare"]["cpu_baseline"] = {"value": 20 / el, "unit": "frames/s", "cores": 1,
                                              "kind": "reference", "sample": "frames [0,20)"}
    del f64, ref
    for key, scene, t in (("configs[0]", "static", 20000), ("configs[1]", "moving", T)):
        v = spk.synth(scene, 0, W, H, t, device=dev)
        ms = _device_ms(lambda: spk.stability(v, 8), dev, 1, steps=2, warmup=1)
        rr = {"workload": f"verify-stability --in, depth 8, {key} {scene} {W}x{H}x{t}",
              "value": W * H / (ms * 1e-3), "unit": "pixels/s", "ms": ms}
        if with_cpu:
            from oracle.oracle import Reference, ref_available
            if ref_available():
                r = Reference()
                pl = v.planes[:, :8].cpu().numpy()  # pixels 0..63
                t0 = time.perf_counter()
                for p in range(64):
                    r.stability(((pl[:, p >> 3] >> (p & 7)) & 1).astype(np.uint8), 8)
                el = time.perf_counter() - t0
                rr["cpu_baseline"] = {"value": 64 / el, "unit": "pixels/s", "cores": 1,
                                      "kind": "reference", "sample": "pixels [0,64)"}
        res[f"stability {key}"] = rr
        del v
    return res


def other_configs(args, rank, world, dev):
    """The other BASELINE configs, device-resident like `value`:
    configs[0] static 400x250x20,000 and configs[2] sensor 1000x1000x20,000
    (single-GPU configs: rank 0), and configs[3] -- 64 independent 400x250
    streams of 4,000 frames, seeds 0..63 alternating the static and moving
    generators -- sharded across the ranks (64/N streams each, no exchange;
    volumes issued as one cached CUDA graph, spk_reconstruct_batch; the same
    calls issued one by one are reported beside it)."""
    import torch

    import paper_2412_11639_b200 as spk
    res = {}
    methods = ("fsr", "ssr")
    for key, scene, w, h, t in (("configs[0]", "static", 400, 250, 20000),
                                ("configs[2]", "sensor", 1000, 1000, 20000)):
        if rank != 0:
            continue
        vol = spk.synth(scene, 0, w, h, t, device=dev)
        out = torch.empty((t, w * h), dtype=torch.uint8, device=dev)
        r = {"workload": f"{key} {scene} {w}x{h}x{t}", "unit": "frames/s"}
        for m in methods:
            ms = _device_ms(lambda: spk.reconstruct(vol, m, out=out), dev, 1)
            r[m] = {"value": t / (ms * 1e-3), "ms_per_step": ms,
                    "step_frac": w * h * t * BYTES_PER_PXF / (ms * 1e-3) / 1e9 / peaks()[0]}
        res[key] = r
        del vol, out
        torch.cuda.empty_cache()
    nvol, t4 = 64, 4000
    mine = list(range(rank * nvol // world, (rank + 1) * nvol // world))
    vols = [spk.synth("static" if i % 2 == 0 else "moving", i, W, H, t4, device=dev) for i in mine]
    outs = [torch.empty((t4, W * H), dtype=torch.uint8, device=dev) for _ in mine]
    lanes = [torch.cuda.Stream(dev) for _ in range(2)]
    cur = torch.cuda.current_stream(dev)
    r = {"workload": f"configs[3] {nvol} x {W}x{H}x{t4} (static/moving by seed parity)",
         "unit": "frames/s", "scaling": "strong", "streams_per_rank": len(mine),
         "parallelism": f"streams x{world}",
         "path": "reconstruct_batch (spk_reconstruct_batch: the rank's calls as one cached CUDA graph "
                 "over 4 branches); per_call_ms: the same calls issued one by one on two streams"}
    for m in methods:
        def per_call():
            for ln in lanes:
                ln.wait_stream(cur)
            for k, (v, o) in enumerate(zip(vols, outs)):
                spk.reconstruct(v, m, out=o, stream=lanes[k % 2])
            for ln in lanes:
                cur.wait_stream(ln)
        ms_calls = _device_ms(per_call, dev, world, steps=3, warmup=2)
        ms = _device_ms(lambda: spk.reconstruct_batch(vols, m, outs=outs), dev, world, steps=3, warmup=2)
        r[m] = {"value": nvol * t4 / (ms * 1e-3), "ms_per_step": ms, "per_call_ms": ms_calls,
                "step_frac": nvol * W * H * t4 * BYTES_PER_PXF / (ms * 1e-3) / 1e9 / peaks()[0]}
    res["configs[3]"] = r
    return res


def long_stream(args, rank, world, dev):
    """BASELINE configs[4]: one 400x250 stream of LONG_T frames, time-sharded
    across the ranks (rank r holds and outputs frames [a_r, a_r+1); exact
    boundary resolution, csrc/shard.cu) -- strong scaling.  On one GPU the
    single-pass time and the 8-shard time (protocol overhead) are reported,
    and the two outputs are compared through per-frame checksums."""
    import torch
    import torch.distributed as dist

    import paper_2412_11639_b200 as spk
    from paper_2412_11639_b200.shard import (reconstruct_time_sharded,
                                             reconstruct_time_sharded_dist, time_bounds)
    T5 = args.long_frames
    b = time_bounds(T5, world)
    f0, f1 = b[rank], b[rank + 1]
    vol = spk.synth("range", 0, W, H, f1 - f0, frame0=f0, device=dev)
    out = torch.empty((f1 - f0, W * H), dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)

    def timed(fn, steps=5, warmup=3):
        for _ in range(warmup):
            fn()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(steps):
            fn()
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / steps
        if world > 1:
            t = torch.tensor([ms], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        return ms

    def sums():
        return torch.cat([out[i:i + 4096].to(torch.int32).sum(dim=1)
                          for i in range(0, out.shape[0], 4096)])

    res = {"workload": f"configs[4] range 400x250x{T5}", "method": args.method,
           "unit": "frames/s", "scaling": "strong", "frames": T5}
    if world > 1:
        ms = timed(lambda: reconstruct_time_sharded_dist(vol, args.method, out=out))
        res.update(value=T5 / (ms * 1e-3), ms_per_step=ms,
                   parallelism=f"time shards x{world} (exact boundary resolution)")
    else:
        import ctypes as C

        from paper_2412_11639_b200 import _capi as capi
        ms = timed(lambda: spk.reconstruct(vol, args.method, out=out))
        ref = sums()
        # the in-grid time split reconstruct() chose (capi.cu reconstruct_split)
        lib = capi.lib()
        lib.spk_set_timing(1)
        spk.reconstruct(vol, args.method, out=out)
        sh, fl = C.c_int32(), C.c_int64()
        capi.check(lib.spk_last_split(C.byref(sh), C.byref(fl)))
        lib.spk_set_timing(0)
        ms8 = timed(lambda: reconstruct_time_sharded(vol, args.method, nshards=8, out=out), 3, 3)
        res.update(value=T5 / (ms * 1e-3), ms_per_step=ms,
                   parallelism=(f"one GPU, one call: in-grid time split x{sh.value} "
                                f"(one K2 launch for all shards, exact stitching)" if sh.value > 1
                                else "one GPU, single pass"),
                   in_grid_split={"shards": sh.value, "pixels_rescanned": fl.value},
                   time_sharded_8_on_1gpu_ms=ms8,
                   time_sharded_equal=bool(torch.equal(sums(), ref)))
    pxf = W * H * T5
    res["step_frac"] = pxf * BYTES_PER_PXF / (ms * 1e-3) / 1e9 / peaks()[0]
    return res


if __name__ == "__main__":
    sys.exit(main())
