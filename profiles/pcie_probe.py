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
