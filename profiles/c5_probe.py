"""configs[4] (400x250 x 1,000,000 frames, extreme dynamic range) on one GPU:
single-pass reconstruct vs exact time sharding (8 shards), compared through
per-frame checksums (the two 100 GB outputs cannot coexist); CUDA-event times."""
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2412_11639_b200 as spk  # noqa: E402
from paper_2412_11639_b200.shard import reconstruct_time_sharded  # noqa: E402

T = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
method = sys.argv[2] if len(sys.argv) > 2 else "fsr"
K = int(sys.argv[3]) if len(sys.argv) > 3 else 8
vol = spk.synth("range", 0, 400, 250, T, device="cuda")
torch.cuda.synchronize()
free, total = torch.cuda.mem_get_info()
print(f"planes {vol.planes.numel() / 1e9:.1f} GB, free {free / 1e9:.1f} / {total / 1e9:.1f} GB", flush=True)
out = torch.empty((T, vol.npix), dtype=torch.uint8, device="cuda")


def timed(fn):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1)


def frame_sums():
    """per-frame sums, a block of frames at a time (int32 is exact: <= 255 * W*H)"""
    return torch.cat([out[i:i + 4096].to(torch.int32).sum(dim=1) for i in range(0, T, 4096)])


ms_s = timed(lambda: reconstruct_time_sharded(vol, method, nshards=K, out=out))
ms_s2 = timed(lambda: reconstruct_time_sharded(vol, method, nshards=K, out=out))
cs_shard = frame_sums()
print(f"time-sharded K={K}: {ms_s:.1f} / {ms_s2:.1f} ms  ({T / ms_s2 * 1e3 / 1e6:.2f} M fps)", flush=True)
out.zero_()
try:
    ms_1 = timed(lambda: spk.reconstruct(vol, method, out=out))
    ms_1b = timed(lambda: spk.reconstruct(vol, method, out=out))
    cs_single = frame_sums()
    print(f"single pass: {ms_1:.1f} / {ms_1b:.1f} ms  ({T / ms_1b * 1e3 / 1e6:.2f} M fps)", flush=True)
    print("per-frame checksums equal:", bool(torch.equal(cs_shard, cs_single)),
          "total", int(cs_single.sum()), flush=True)
except Exception as e:  # noqa: BLE001
    print("single pass failed:", type(e).__name__, str(e)[:200], flush=True)

# per-phase device times of the single pass (CUDA events around each phase)
import ctypes as C  # noqa: E402

from paper_2412_11639_b200 import _capi as capi  # noqa: E402
lib = capi.lib()
lib.spk_set_timing(1)
spk.reconstruct(vol, method, out=out)
v = [C.c_float() for _ in range(4)]
capi.check(lib.spk_last_timing(*(C.byref(x) for x in v)))
lib.spk_set_timing(0)
print("phases ms: segment %.2f finalize %.2f expand %.2f fixup %.2f" % tuple(x.value for x in v), flush=True)
