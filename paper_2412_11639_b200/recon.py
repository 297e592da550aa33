"""Python host mirror of the reference's reconstruction interface.

Names, argument meaning and error behaviour follow proj/include/spikecam/
(reference paths relative to /root/reference):

    ReconMethod.parse / .name      reconstruct.hpp:10-18, reconstruct.cpp:177-196
    reconstruct(volume, method, workers, out)
                                   reconstruct.hpp:73-79, reconstruct.cpp:441-471
    segment_fsr / segment_ssr      reconstruct.hpp:30-40 (run lists, no degenerate
                                   lead/tail entries; see segments())
    read_spk / read_raw / write_spk
                                   io.hpp:20-31, io.cpp:173-223

The compute is the C-ABI library (libspikecam_b200.so) on the current CUDA
device; torch provides device memory and the stream.  There is no CPU path:
every call either launches the sm_100a kernels or raises.
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass
from pathlib import Path

import numpy as np
import torch

from . import _capi as capi

DEFAULT_FPS = 20000  # kDefaultFps, io.hpp:16
DEFAULT_RAW_WIDTH = 400
DEFAULT_RAW_HEIGHT = 250


class Method(enum.IntEnum):
    fsr = capi.SPK_FSR
    ssr = capi.SPK_SSR
    tfi = capi.SPK_TFI
    tfp = capi.SPK_TFP


@dataclass(frozen=True)
class ReconMethod:
    kind: Method = Method.fsr
    tfp_window: int = 32  # only for Method.tfp, >= 1

    @staticmethod
    def parse(name: str, window: int = 32) -> "ReconMethod":
        """ReconMethod::parse: ValueError (std::invalid_argument) on bad input."""
        if name in ("fsr", "ssr", "tfi"):
            return ReconMethod(Method[name])
        if name == "tfp":
            if window < 1:
                raise ValueError("tfp window must be >= 1")
            return ReconMethod(Method.tfp, window)
        raise ValueError(f"unknown reconstruction method: {name}")

    def name(self) -> str:
        return f"tfp-{self.tfp_window}" if self.kind == Method.tfp else self.kind.name


def _method(m) -> ReconMethod:
    if isinstance(m, ReconMethod):
        return m
    if isinstance(m, Method):
        return ReconMethod(m)
    if isinstance(m, str):
        if m.startswith("tfp-"):
            return ReconMethod.parse("tfp", int(m[4:]))
        return ReconMethod.parse(m)
    raise ValueError(f"unknown reconstruction method: {m!r}")


class IoError(RuntimeError):
    """spikecam::io_error (io.hpp:12-14)."""


def plane_bytes(width: int, height: int) -> int:
    """frame_bytes, io.cpp:48-50: ceil(W*H/8)."""
    return (int(width) * int(height) + 7) // 8


def plane_pitch(width: int, height: int) -> int:
    """Device pitch of one bit-plane (16-B multiple, >= 4*ceil(W*H/32))."""
    return int(capi.lib().spk_plane_pitch(int(width), int(height)))


def _stream(stream) -> int:
    if stream is None:
        return torch.cuda.current_stream().cuda_stream
    return stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)


@dataclass
class PackedVolume:
    """A W x H x T spike volume held on the GPU as pitched SPK1 bit-planes.

    The B200-resident form of SpikeVolume (core.hpp:15-49): plane n is
    planes[n], pixel p = y*W + x is bit p & 7 of byte p >> 3 (LSB-first).
    """

    width: int
    height: int
    frames: int
    planes: torch.Tensor  # uint8 [frames, pitch] on a CUDA device

    @property
    def pitch(self) -> int:
        return int(self.planes.stride(0)) if self.frames > 0 else plane_pitch(self.width, self.height)

    @property
    def npix(self) -> int:
        return self.width * self.height

    def geom(self) -> capi.spk_geom:
        return capi.geom(self.width, self.height, self.frames, self.pitch)

    @staticmethod
    def empty(width: int, height: int, frames: int, device=None) -> "PackedVolume":
        _check_dims(width, height, frames)
        dev = torch.device(device) if device is not None else torch.device("cuda")
        planes = torch.empty((frames, plane_pitch(width, height)), dtype=torch.uint8, device=dev)
        return PackedVolume(width, height, frames, planes)

    @staticmethod
    def from_payload(payload, width: int, height: int, frames: int | None = None,
                     msb_first: bool = False, device=None, stream=None) -> "PackedVolume":
        """Dense SPK1 payload (T planes of ceil(W*H/8) bytes) -> device planes."""
        buf = np.ascontiguousarray(np.frombuffer(memoryview(payload), dtype=np.uint8)
                                   if not isinstance(payload, np.ndarray) else payload.reshape(-1))
        fb = plane_bytes(width, height)
        if frames is None:
            frames = buf.size // fb
        if buf.size < frames * fb:
            raise ValueError("payload shorter than frames * ceil(W*H/8)")
        vol = PackedVolume.empty(width, height, frames, device)
        if frames:
            with torch.cuda.device(vol.planes.device):
                s = _stream(stream)
                capi.check(capi.lib().spk_upload_planes(
                    vol.geom(), buf.ctypes.data, fb, int(bool(msb_first)),
                    vol.planes.data_ptr(), s))
                # `buf` is host memory owned by this frame: finish the copy first
                torch.cuda.ExternalStream(s).synchronize() if s else torch.cuda.synchronize()
        return vol

    @staticmethod
    def from_bytes(bits: torch.Tensor, width: int, height: int, stream=None) -> "PackedVolume":
        """One byte per bit (SpikeVolume::raw(), frame-major) -> planes (pack_frame)."""
        if not bits.is_cuda:
            raise ValueError("from_bytes expects a CUDA tensor")
        bits = bits.contiguous().view(-1)
        npix = width * height
        frames = bits.numel() // npix
        vol = PackedVolume.empty(width, height, frames, bits.device)
        with torch.cuda.device(bits.device):
            capi.check(capi.lib().spk_pack_bytes(vol.geom(), bits.data_ptr(),
                                                 vol.planes.data_ptr(), _stream(stream)))
        return vol

    def to_bytes(self, stream=None) -> torch.Tensor:
        """unpack_frame: planes -> uint8 [T, H, W] of 0/1."""
        out = torch.empty((self.frames, self.height, self.width), dtype=torch.uint8,
                          device=self.planes.device)
        with torch.cuda.device(self.planes.device):
            capi.check(capi.lib().spk_unpack_planes(self.geom(), self.planes.data_ptr(),
                                                    out.data_ptr(), _stream(stream)))
        return out

    def payload(self) -> np.ndarray:
        """Dense SPK1 payload on the host (T * ceil(W*H/8) bytes)."""
        fb = plane_bytes(self.width, self.height)
        return self.planes[:, :fb].cpu().numpy().reshape(-1)


def _check_dims(width: int, height: int, frames: int) -> None:
    if width < 1 or height < 1 or frames < 0:
        raise ValueError("SpikeVolume: width/height must be >= 1, frames >= 0")


_OUT = {
    torch.uint8: ("spk_reconstruct_u8", 1),
    torch.float32: ("spk_reconstruct_f32", 4),
    torch.float64: ("spk_reconstruct_f64", 8),
}


def reconstruct(volume: PackedVolume, method="fsr", workers: int = 0,
                out: torch.Tensor | None = None, dtype: torch.dtype = torch.uint8,
                stream=None) -> torch.Tensor:
    """Per-frame reconstruction of the whole volume (reconstruct.cpp:441-471).

    Returns a [T, H, W] tensor on the volume's device: uint8 frames (the
    reference's quantize(), io.cpp:78-81), or float32 / float64 values
    (float64 is bit-identical to the reference doubles).  `out` may be a
    caller-owned [T, >=H*W] buffer (reused, like the reference's `out`).
    `workers` -- the reference's CPU thread count -- selects up to that many
    of the visible GPUs, one pixel band each (shard.reconstruct_devices); with
    one GPU, or workers <= 1, it is one call.  The result is identical for
    any worker count (reconstruct.hpp:70-72).  Multi-process sharding lives in
    paper_2412_11639_b200.shard.
    """
    m = _method(method)
    workers = int(workers)
    nbands = min(max(workers, 1), torch.cuda.device_count()) if volume.frames else 1
    if nbands > 1 and stream is None:
        from .shard import reconstruct_devices
        return reconstruct_devices(volume, m, list(range(nbands)), out=out, dtype=dtype)
    if out is not None:
        dtype = out.dtype
    if dtype not in _OUT:
        raise ValueError(f"unsupported output dtype {dtype}")
    fn, _ = _OUT[dtype]
    npix = volume.npix
    if out is None:
        out = torch.empty((volume.frames, npix), dtype=dtype, device=volume.planes.device)
    if out.dim() != 2 or out.shape[0] != volume.frames or out.shape[1] < npix or out.stride(1) != 1:
        raise ValueError("out must be a [frames, >= W*H] row-major tensor")
    out_pitch = out.stride(0) if volume.frames > 0 else npix
    with torch.cuda.device(volume.planes.device):
        capi.check(getattr(capi.lib(), fn)(
            volume.geom(), volume.planes.data_ptr() if volume.frames else None,
            int(m.kind), int(m.tfp_window), out.data_ptr() if volume.frames else None,
            out_pitch, _stream(stream)))
    if out.shape[1] == npix:
        return out.view(volume.frames, volume.height, volume.width)
    return out


def reconstruct_batch(volumes, method="fsr", outs=None, dtype: torch.dtype = torch.uint8,
                      stream=None) -> list[torch.Tensor]:
    """reconstruct() of many volumes of one geometry on one device (BASELINE
    configs[3]) as one CUDA graph (spk_reconstruct_batch): the calls are
    captured once over four branches and the graph is replayed while the
    same buffers come back (`outs`: caller-owned [T, >= H*W] tensors, reused
    like the reference's `out`; allocated when None).  Returns the outputs as
    [T, H, W] views; identical to per-volume reconstruct() calls."""
    from . import _capi as C_
    volumes = list(volumes)
    if not volumes:
        return []
    m = _method(method)
    v0 = volumes[0]
    for v in volumes:
        if (v.width, v.height, v.frames, v.pitch) != (v0.width, v0.height, v0.frames, v0.pitch):
            raise ValueError("reconstruct_batch: volumes must share width, height, frames and pitch")
        if v.planes.device != v0.planes.device:
            raise ValueError("reconstruct_batch: volumes must be on one device")
    npix = v0.npix
    dev = v0.planes.device
    if outs is None:
        outs = [torch.empty((v0.frames, npix), dtype=dtype, device=dev) for _ in volumes]
    outs = list(outs)
    if len(outs) != len(volumes):
        raise ValueError("reconstruct_batch: one output per volume")
    dtype = outs[0].dtype
    if dtype not in _OUT:
        raise ValueError(f"unsupported output dtype {dtype}")
    for o in outs:
        if (o.dtype != dtype or o.dim() != 2 or o.shape[0] != v0.frames or o.shape[1] < npix or
                o.stride(1) != 1 or o.stride(0) != outs[0].stride(0) or o.device != dev):
            raise ValueError("outs must be [frames, >= W*H] row-major tensors of one dtype and pitch")
    out_type = {torch.uint8: C_.SPK_OUT_U8, torch.float32: C_.SPK_OUT_F32,
                torch.float64: C_.SPK_OUT_F64}[dtype]
    if v0.frames > 0:
        planes = (C.c_void_p * len(volumes))(*[v.planes.data_ptr() for v in volumes])
        ptrs = (C.c_void_p * len(outs))(*[o.data_ptr() for o in outs])
        with torch.cuda.device(dev):
            capi.check(capi.lib().spk_reconstruct_batch(
                v0.geom(), len(volumes), planes, int(m.kind), int(m.tfp_window), out_type, ptrs,
                outs[0].stride(0), _stream(stream)))
    return [o.view(v0.frames, v0.height, v0.width) if o.shape[1] == npix else o for o in outs]


def segments(volume: PackedVolume, method="fsr", run_cap: int | None = None, stream=None):
    """Stable runs of every pixel (segment_fsr / segment_ssr without the
    degenerate lead/tail segments): returns (runs [npix, cap, 2] int64 as
    (start frame, intervals), counts [npix], last_spike [npix]).  A pixel's
    runs tile [runs[0].start, last_spike); counts > cap means truncation."""
    m = _method(method)
    if m.kind not in (Method.fsr, Method.ssr):
        raise ValueError("segments: method must be fsr or ssr")
    npix = volume.npix
    cap = int(run_cap) if run_cap else max(64, volume.frames // 8)
    dev = volume.planes.device
    runs = torch.empty((npix, cap, 2), dtype=torch.int32, device=dev)
    counts = torch.empty((npix,), dtype=torch.int32, device=dev)
    last = torch.empty((npix,), dtype=torch.int32, device=dev)
    with torch.cuda.device(dev):
        capi.check(capi.lib().spk_segment(
            volume.geom(), volume.planes.data_ptr() if volume.frames else None, int(m.kind),
            runs.data_ptr(), cap, counts.data_ptr(), last.data_ptr(), _stream(stream)))
    return runs, counts, last


def reconstruct_host(payload: np.ndarray, width: int, height: int, frames: int, method="fsr",
                     dtype=np.uint8, out: np.ndarray | None = None) -> np.ndarray:
    """Host boundary of reconstruct(): dense SPK1 payload in host memory ->
    host frames [T, W*H], through spk_reconstruct_host (upload, kernels,
    download inside one C-ABI call).  Pinned buffers give the best copy rate."""
    m = _method(method)
    code = {np.dtype(np.uint8): capi.SPK_OUT_U8, np.dtype(np.float32): capi.SPK_OUT_F32,
            np.dtype(np.float64): capi.SPK_OUT_F64}[np.dtype(dtype)]
    npix = width * height
    if out is None:
        out = np.empty((frames, npix), dtype=dtype)
    buf = np.ascontiguousarray(payload.reshape(-1))
    g = capi.geom(width, height, frames, 0)
    capi.check(capi.lib().spk_reconstruct_host(g, buf.ctypes.data, int(m.kind),
                                               int(m.tfp_window), code, out.ctypes.data,
                                               out.shape[1]))
    return out


def reconstruct_host_multi(payload: np.ndarray, width: int, height: int, frames: int, method="fsr",
                           dtype=np.uint8, devices=(0,), out: np.ndarray | None = None) -> np.ndarray:
    """reconstruct_host() over several GPUs: the pixels are cut into
    len(devices) bands (128-pixel boundaries), band i on CUDA device
    devices[i] (spk_reconstruct_host_multi).  Identical output for any band
    count, as the reference's `workers` (reconstruct.hpp:70-72)."""
    m = _method(method)
    code = {np.dtype(np.uint8): capi.SPK_OUT_U8, np.dtype(np.float32): capi.SPK_OUT_F32,
            np.dtype(np.float64): capi.SPK_OUT_F64}[np.dtype(dtype)]
    npix = width * height
    if out is None:
        out = np.empty((frames, npix), dtype=dtype)
    buf = np.ascontiguousarray(payload.reshape(-1))
    devs = np.ascontiguousarray(np.asarray(devices, dtype=np.int32))
    g = capi.geom(width, height, frames, 0)
    capi.check(capi.lib().spk_reconstruct_host_multi(g, buf.ctypes.data, int(m.kind),
                                                     int(m.tfp_window), code, out.ctypes.data,
                                                     out.shape[1], devs.ctypes.data, int(devs.size)))
    return out


def reconstruct_host_batch(payloads, width: int, height: int, frames: int, method="fsr",
                           dtype=np.uint8, outs=None) -> list:
    """Many volumes of one geometry through spk_reconstruct_host_batch: the
    upload + reconstruction of volume i+1 overlap the download of volume i.
    `payloads`: dense SPK1 payloads (numpy / pinned torch host tensors);
    `outs`: host [T, W*H] buffers (allocated when omitted)."""
    m = _method(method)
    code = {np.dtype(np.uint8): capi.SPK_OUT_U8, np.dtype(np.float32): capi.SPK_OUT_F32,
            np.dtype(np.float64): capi.SPK_OUT_F64}[np.dtype(dtype)]
    npix = width * height
    if outs is None:
        outs = [np.empty((frames, npix), dtype=dtype) for _ in payloads]
    if len(outs) != len(payloads):
        raise ValueError("one output buffer per payload")

    def addr(x):
        if isinstance(x, torch.Tensor):
            return x.data_ptr()
        return np.ascontiguousarray(x).ctypes.data

    keep = [np.ascontiguousarray(p) if not isinstance(p, torch.Tensor) else p for p in payloads]
    pin = (C.c_void_p * len(keep))(*[addr(p) for p in keep])
    pout = (C.c_void_p * len(outs))(*[addr(o) for o in outs])
    g = capi.geom(width, height, frames, 0)
    capi.check(capi.lib().spk_reconstruct_host_batch(g, len(keep), pin, int(m.kind),
                                                     int(m.tfp_window), code, pout,
                                                     outs[0].shape[1] if len(outs) else npix))
    return outs


def reconstruct_host_ptr(h_payload: int, width: int, height: int, frames: int, method,
                         out_code: int, h_out: int, out_pitch: int) -> None:
    """Raw-pointer form (pinned torch tensors in bench.py's e2e leg)."""
    m = _method(method)
    g = capi.geom(width, height, frames, 0)
    capi.check(capi.lib().spk_reconstruct_host(g, h_payload, int(m.kind), int(m.tfp_window),
                                               out_code, h_out, out_pitch))


# ------------------------------------------------------------------- files --
def _u16(b, o):
    return int(b[o]) | int(b[o + 1]) << 8


def _u32(b, o):
    return int(b[o]) | int(b[o + 1]) << 8 | int(b[o + 2]) << 16 | int(b[o + 3]) << 24


def read_spk(path, device=None) -> tuple[PackedVolume, int]:
    """read_spk (io.cpp:185-206): SPK1 file -> (device volume, fps)."""
    path = Path(path)
    try:
        data = np.fromfile(path, dtype=np.uint8)
    except OSError as e:
        raise IoError(f"cannot open {path}") from e
    if data.size < 16 or bytes(data[:4]) != b"SPK1":
        raise IoError(f"bad SPK1 magic in {path}")
    w, h = _u16(data, 4), _u16(data, 6)
    fps, frames = _u32(data, 8), _u32(data, 12)
    if w < 1 or h < 1:
        raise IoError(f"empty geometry in {path}")
    expect = 16 + plane_bytes(w, h) * frames
    if data.size != expect:
        raise IoError(f"SPK1 length mismatch in {path}: expected {expect} bytes, got {data.size}")
    return PackedVolume.from_payload(data[16:], w, h, frames, device=device), fps


def read_raw(path, width: int = DEFAULT_RAW_WIDTH, height: int = DEFAULT_RAW_HEIGHT,
             msb_first: bool = False, device=None) -> PackedVolume:
    """read_raw (io.cpp:208-223): headerless dump, frames from the file size."""
    path = Path(path)
    try:
        data = np.fromfile(path, dtype=np.uint8)
    except OSError as e:
        raise IoError(f"cannot open {path}") from e
    fb = plane_bytes(width, height)
    if data.size % fb != 0:
        raise IoError(f"raw file {path} ({data.size} bytes) is not a multiple of the {fb}-byte "
                      f"frame size for {width}x{height}; check --width/--height")
    return PackedVolume.from_payload(data, width, height, data.size // fb, msb_first=msb_first,
                                     device=device)


def write_spk(volume: PackedVolume, fps: int, path) -> None:
    """write_spk (io.cpp:173-183)."""
    head = np.zeros(16, dtype=np.uint8)
    head[:4] = np.frombuffer(b"SPK1", dtype=np.uint8)
    for off, val, n in ((4, volume.width, 2), (6, volume.height, 2), (8, fps, 4),
                        (12, volume.frames, 4)):
        for i in range(n):
            head[off + i] = (int(val) >> (8 * i)) & 0xFF
    try:
        with open(path, "wb") as f:
            f.write(head.tobytes())
            f.write(volume.payload().tobytes())
    except OSError as e:
        raise IoError(f"cannot create {path}") from e


# --------------------------------------------------------------- synthesis --
SCENES = {"noise": 0, "static": 1, "moving": 2, "sensor": 3, "range": 5}


def synth(scene, seed: int, width: int, height: int, frames: int, frame0: int = 0,
          param: float = 0.0, device=None, stream=None) -> PackedVolume:
    """Seeded synthetic integrate-and-fire volume generated on the GPU (input
    synthesis for benchmarks/tests, not part of the reconstruction path)."""
    code = SCENES[scene] if isinstance(scene, str) else int(scene)
    vol = PackedVolume.empty(width, height, frames, device)
    with torch.cuda.device(vol.planes.device):
        capi.check(capi.lib().spk_synth(code, int(seed) & (2**64 - 1), vol.geom(), int(frame0),
                                        float(param),
                                        vol.planes.data_ptr() if frames else None,
                                        _stream(stream)))
    return vol
