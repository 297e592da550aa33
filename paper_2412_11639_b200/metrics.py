"""Quality metrics and the stability check on the device.

    te, mse = frame_metrics(frames, ref)     # per frame, float64 tensors
    compare(vol, ["fsr", "ssr"], ref, warmup=10)  # the CLI's `compare`
    rep = stability(vol, depth=8)            # stability_order of every pixel
    ok, fails = verify_stability(vol, depth=8)    # `verify-stability --in`

two_dimensional_entropy / mse / psnr follow proj/src/metrics.cpp:12-61,
compare follows proj/tools/spikecam_main.cpp:263-299, stability_order
proj/src/stability.cpp:61-128 and verify-stability --in
spikecam_main.cpp:189-207.  Entropy and mse sums are reduced in a fixed
order on the device: deterministic, and equal to the reference's sequential
sums up to double rounding.
"""
from __future__ import annotations

import ctypes as C
import math

import numpy as np
import torch

from . import _capi as capi
from .recon import PackedVolume, _stream, reconstruct

_FTYPE = {torch.uint8: capi.SPK_OUT_U8, torch.float32: capi.SPK_OUT_F32,
          torch.float64: capi.SPK_OUT_F64}


def _frames2d(frames: torch.Tensor, width: int | None, height: int | None):
    if frames.dim() == 3:
        t, h, w = frames.shape
        if t and not frames[0].is_contiguous():
            raise ValueError("frames must be row-contiguous")
        return frames.reshape(t, h * w) if frames.is_contiguous() else frames, w, h
    if frames.dim() == 2 and width and height:
        return frames, width, height
    raise ValueError("frames: [T, H, W], or [T, >= W*H] with width/height")


def frame_metrics(frames: torch.Tensor, ref: torch.Tensor | None = None, te: bool = True,
                  width: int | None = None, height: int | None = None, stream=None):
    """Per-frame two_dimensional_entropy (quantized values) and, with `ref`
    (reference images, same shape: uint8 as read back from PGM, or values), mse.  Returns (te, mse); an output
    not asked for is None."""
    if frames.dtype not in _FTYPE:
        raise ValueError("frames must be uint8, float32 or float64")
    f2, w, h = _frames2d(frames, width, height)
    t = int(f2.shape[0])
    dev = f2.device
    r2 = None
    if ref is not None:
        if ref.dtype not in _FTYPE:
            raise ValueError("reference images must be uint8, float32 or float64")
        r2, rw, rh = _frames2d(ref, width or w, height or h)
        if (rw, rh) != (w, h) or r2.shape[0] != t:
            raise ValueError("reference geometry differs")
    te_out = torch.empty(t, dtype=torch.float64, device=dev) if te else None
    mse_out = torch.empty(t, dtype=torch.float64, device=dev) if ref is not None else None
    g = capi.geom(w, h, t, 0)
    with torch.cuda.device(dev):
        capi.check(capi.lib().spk_frame_metrics(
            g, f2.data_ptr() if t else None, _FTYPE[frames.dtype], int(f2.stride(0)) if t else w * h,
            r2.data_ptr() if r2 is not None and t else None,
            _FTYPE[ref.dtype] if ref is not None else capi.SPK_OUT_U8,
            int(r2.stride(0)) if r2 is not None and t else w * h,
            te_out.data_ptr() if te_out is not None and t else None,
            mse_out.data_ptr() if mse_out is not None and t else None, _stream(stream)))
    return te_out, mse_out


def two_dimensional_entropy(frame: torch.Tensor) -> float:
    """metrics.cpp:12-43 of one [H, W] image (uint8 = quantized, or values)."""
    te, _ = frame_metrics(frame.unsqueeze(0))
    return float(te[0])


def mse(image: torch.Tensor, reference: torch.Tensor) -> float:
    """metrics.cpp:45-55 of one [H, W] image against a reference image."""
    if image.shape != reference.shape:
        raise ValueError("mse: dimension mismatch")
    _, m = frame_metrics(image.unsqueeze(0), reference.unsqueeze(0), te=False)
    return float(m[0])


def psnr(image: torch.Tensor, reference: torch.Tensor) -> float:
    """metrics.cpp:57-61: 10*log10(255^2 / mse); +inf for identical images."""
    m = mse(image, reference)
    return math.inf if m == 0.0 else 10.0 * math.log10(255.0 * 255.0 / m)


def compare(volume: PackedVolume, methods=("fsr", "ssr", "tfi", "tfp"), ref=None,
            warmup: int = 0, dtype: torch.dtype = torch.float64) -> list[dict]:
    """The CLI's `compare` (spikecam_main.cpp:263-299): per method, the mean
    entropy over frames [first, T) and, with reference images ([T, H, W];
    frames without one are skipped the way a missing PGM is, via a
    boolean `ref_mask`), the mean mse and its psnr.  `ref` may be a tensor or
    a (tensor, mask) pair."""
    t = volume.frames
    first = min(warmup, max(0, t - 1))
    ref_t, mask = (ref if isinstance(ref, tuple) else (ref, None))
    out = []
    for m in methods:
        frames = reconstruct(volume, m, dtype=dtype)[first:]
        r = ref_t[first:] if ref_t is not None else None
        te, ms = frame_metrics(frames, r)
        row = {"method": m if isinstance(m, str) else str(m), "te": float(te.mean()) if te.numel() else 0.0}
        if ms is not None:
            sel = ms if mask is None else ms[torch.as_tensor(mask[first:], device=ms.device)]
            if sel.numel():
                avg = float(sel.mean())
                row["mse"] = avg
                row["psnr"] = math.inf if avg == 0.0 else 10.0 * math.log10(255.0 * 255.0 / avg)
        out.append(row)
    return out


STAB_DTYPE = np.dtype([("depth", np.int32), ("verified_order", np.int32), ("absolute", np.int32),
                       ("path_len", np.int32), ("index", np.int64), ("path", np.uint64)])


def path_string(bits: int, length: int) -> str:
    """'-'/'+' path of a violation (bit j = branch j+1 -> j+2, '+' = 1)."""
    return "".join("+" if (int(bits) >> j) & 1 else "-" for j in range(int(length)))


def stability(volume: PackedVolume, depth: int = 8, stream=None) -> np.ndarray:
    """stability_order of every pixel (row-major), as a structured array of
    STAB_DTYPE (depth 0 = no violation)."""
    out = torch.empty(volume.npix * STAB_DTYPE.itemsize, dtype=torch.uint8,
                      device=volume.planes.device)
    with torch.cuda.device(volume.planes.device):
        capi.check(capi.lib().spk_stability(
            volume.geom(), volume.planes.data_ptr() if volume.frames else None, int(depth),
            out.data_ptr(), _stream(stream)))
    return out.cpu().numpy().view(STAB_DTYPE)


def verify_stability(volume: PackedVolume, depth: int = 8):
    """verify-stability --in (spikecam_main.cpp:189-207): (ok, failures) with
    the failures the CLI prints -- every failing pixel of the first row that
    has one -- as (x, y, depth, path, index)."""
    rep = stability(volume, depth)
    bad = np.nonzero(rep["depth"] > 0)[0]
    if bad.size == 0:
        return True, []
    y = int(bad[0]) // volume.width
    row = bad[(bad // volume.width) == y]
    fails = [(int(p) % volume.width, y, int(rep["depth"][p]),
              path_string(rep["path"][p], rep["path_len"][p]), int(rep["index"][p])) for p in row]
    return False, fails
