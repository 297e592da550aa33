"""Segment records (SPKR): the paper's 16-bit FPGA output words.

Mirror of the reference's record path: `--emit-records`
(proj/tools/spikecam_main.cpp:146-172) = segment_fsr / segment_ssr per pixel
-> encode_events (proj/src/codec.cpp:8-31) -> write_spkr / read_spkr
(proj/src/io.cpp:240-292), and decode (codec.cpp:33-43).  The records of a
whole volume are produced on the GPU as one SPKR file image
(spk_records, paper_2412_11639_b200/csrc/records.cu).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np
import torch

from . import _capi as capi
from .recon import DEFAULT_FPS, IoError, Method, PackedVolume, _method, _stream


class _DevBuf:
    """A raw device allocation seen through __cuda_array_interface__."""

    def __init__(self, ptr: int, nbytes: int):
        self.__cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1",
                                         "data": (ptr, False), "version": 3}


def records(volume: PackedVolume, method="fsr", fps: int = DEFAULT_FPS, stream=None) -> torch.Tensor:
    """SPKR file image of every pixel's FSR / SSR segment records, as a uint8
    tensor on the volume's device (write it with `write_spkr`)."""
    m = _method(method)
    if m.kind not in (Method.fsr, Method.ssr):
        raise ValueError("--emit-records needs method fsr or ssr")
    ptr, nbytes = C.c_void_p(), C.c_uint64()
    dev = volume.planes.device
    with torch.cuda.device(dev):
        s = _stream(stream)
        capi.check(capi.lib().spk_records(volume.geom(),
                                          volume.planes.data_ptr() if volume.frames else None,
                                          int(m.kind), int(fps) & 0xFFFFFFFF, C.byref(ptr),
                                          C.byref(nbytes), s))
        try:
            so = torch.cuda.ExternalStream(s) if s else torch.cuda.default_stream(dev)
            with torch.cuda.stream(so):  # copy out on the stream that wrote the image
                view = torch.as_tensor(_DevBuf(ptr.value, nbytes.value), device=dev)
                img = view.clone()
        finally:
            capi.check(capi.lib().spk_free_device(ptr, s))
    return img


def records_host(payload: np.ndarray, width: int, height: int, frames: int, method="fsr",
                 fps: int = DEFAULT_FPS) -> bytes:
    """Host boundary: dense SPK1 payload in, SPKR file image (bytes) out."""
    m = _method(method)
    if m.kind not in (Method.fsr, Method.ssr):
        raise ValueError("--emit-records needs method fsr or ssr")
    buf = np.ascontiguousarray(np.asarray(payload, dtype=np.uint8).reshape(-1))
    ptr, nbytes = C.c_void_p(), C.c_uint64()
    g = capi.geom(width, height, frames, 0)
    capi.check(capi.lib().spk_records_host(g, buf.ctypes.data if buf.size else None, int(m.kind),
                                           int(fps) & 0xFFFFFFFF, C.byref(ptr), C.byref(nbytes)))
    try:
        return C.string_at(ptr.value, nbytes.value)
    finally:
        capi.lib().spk_free_host(ptr)


@dataclass
class RecordVolume:
    """io.hpp:44-60: geometry header + per-pixel word lists (row-major)."""

    width: int = 0
    height: int = 0
    fps: int = DEFAULT_FPS
    frame_count: int = 0
    words: list[np.ndarray] = field(default_factory=list)

    def pixel(self, x: int, y: int) -> np.ndarray:
        return self.words[y * self.width + x]


def write_spkr(image, path) -> None:
    """Write an SPKR image (tensor / bytes from `records`) to `path`."""
    data = image.cpu().numpy().tobytes() if isinstance(image, torch.Tensor) else bytes(image)
    try:
        Path(path).write_bytes(data)
    except OSError as e:
        raise IoError(f"cannot create {path}") from e


def parse_spkr(data, name: str = "<image>") -> RecordVolume:
    """read_spkr (io.cpp:257-292) on an in-memory image."""
    b = np.frombuffer(bytes(data) if not isinstance(data, np.ndarray) else data.tobytes(), np.uint8)
    if b.size < 16 or bytes(b[:4]) != b"SPKR":
        raise IoError(f"bad SPKR magic in {name}")
    w = int(b[4]) | int(b[5]) << 8
    h = int(b[6]) | int(b[7]) << 8
    fps = int(np.frombuffer(b[8:12].tobytes(), "<u4")[0])
    frames = int(np.frombuffer(b[12:16].tobytes(), "<u4")[0])
    if w < 1 or h < 1:
        raise IoError(f"empty geometry in {name}")
    pos, words = 16, []
    for _ in range(w * h):
        if pos + 4 > b.size:
            raise IoError(f"truncated SPKR record table: {name}")
        n = int(np.frombuffer(b[pos:pos + 4].tobytes(), "<u4")[0])
        pos += 4
        if pos + 2 * n > b.size:
            raise IoError(f"truncated SPKR records: {name}")
        words.append(np.frombuffer(b[pos:pos + 2 * n].tobytes(), "<u2").copy())
        pos += 2 * n
    if pos != b.size:
        raise IoError(f"trailing bytes after SPKR records in {name}")
    return RecordVolume(w, h, fps, frames, words)


def read_spkr(path) -> RecordVolume:
    try:
        data = Path(path).read_bytes()
    except OSError as e:
        raise IoError(f"cannot open {path}") from e
    return parse_spkr(data, str(path))


def decode(words: np.ndarray) -> np.ndarray:
    """codec.cpp:33-43: each word -> `duration` frames of its intensity."""
    w = np.asarray(words, dtype=np.uint16)
    d = (w >> 8).astype(np.int64)
    if (d == 0).any():
        raise RuntimeError("decode: zero-duration record")
    return np.repeat((w & 0xFF).astype(np.uint8), d)
