"""PCIe copy bandwidth on the box: one 4 GB pinned D2H / H2D copy vs the same
bytes as 2 or 4 concurrent chunks on separate streams (CUDA events)."""
import torch

n = 4_000_000_000
dev = torch.empty(n, dtype=torch.uint8, device="cuda")
host = torch.empty(n, dtype=torch.uint8).pin_memory()


def run(k, d2h=True):
    streams = [torch.cuda.Stream() for _ in range(k)]
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    chunk = n // k
    for i, s in enumerate(streams):
        s.wait_event(e0)
        with torch.cuda.stream(s):
            if d2h:
                host[i * chunk:(i + 1) * chunk].copy_(dev[i * chunk:(i + 1) * chunk], non_blocking=True)
            else:
                dev[i * chunk:(i + 1) * chunk].copy_(host[i * chunk:(i + 1) * chunk], non_blocking=True)
    for s in streams:
        e1.wait_stream(s) if hasattr(e1, "wait_stream") else torch.cuda.current_stream().wait_stream(s)
    torch.cuda.current_stream().wait_stream(streams[-1])
    for s in streams:
        torch.cuda.current_stream().wait_stream(s)
    e1.record()
    torch.cuda.synchronize()
    return n / e0.elapsed_time(e1) / 1e6


for k in (1, 2, 4, 8):
    print(f"D2H {k} stream(s): {run(k):.1f} GB/s   H2D: {run(k, False):.1f} GB/s", flush=True)


def bidir(h2d_bytes=500_000_000):
    """a 4 GB D2H and a concurrent H2D on another stream (the e2e pattern):
    does the upload share the download's bandwidth?"""
    hin = torch.empty(h2d_bytes, dtype=torch.uint8).pin_memory()
    din = torch.empty(h2d_bytes, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    torch.cuda.synchronize()
    e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    e0.record()
    s1.wait_event(e0)
    s2.wait_event(e0)
    with torch.cuda.stream(s1):
        host.copy_(dev, non_blocking=True)
        e1.record(s1)
    with torch.cuda.stream(s2):
        for _ in range(8):  # 8 uploads under one download
            din.copy_(hin, non_blocking=True)
        e2.record(s2)
    torch.cuda.synchronize()
    d = e0.elapsed_time(e1)
    u = e0.elapsed_time(e2)
    print(f"bidirectional: D2H 4 GB in {d:.1f} ms ({n / d / 1e6:.1f} GB/s) with 8 x {h2d_bytes / 1e9:.1f} GB "
          f"H2D in {u:.1f} ms ({8 * h2d_bytes / u / 1e6:.1f} GB/s)", flush=True)


bidir()
