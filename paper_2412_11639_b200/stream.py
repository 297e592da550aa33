"""Streaming FSR for every pixel at once: the batched form of the reference's
PixelReconState (proj/include/spikecam/reconstruct.hpp:46-67,
proj/src/reconstruct.cpp:230-290).

    es = EventStream(W, H)
    for block in blocks:                 # PackedVolume or [n, pitch] planes on the GPU
        offsets, durations, intensities = es.push(block)
    offsets, durations, intensities = es.flush()

Pixel p's events of a call are durations/intensities[offsets[p]:offsets[p+1]]
-- the SegmentEvents PixelReconState::push_frame / flush yield for that
pixel, in order (identical to fsr_events over the whole stream).
"""
from __future__ import annotations

import ctypes as C

import torch

from . import _capi as capi
from .recon import PackedVolume, _stream, plane_pitch


class _DevBuf:
    def __init__(self, ptr: int, nbytes: int):
        self.__cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1",
                                         "data": (ptr, False), "version": 3}


class EventStream:
    def __init__(self, width: int, height: int, device=None, stream=None):
        self.width, self.height = int(width), int(height)
        self.npix = self.width * self.height
        self.device = torch.device(device) if device is not None else torch.device("cuda")
        self._lib = capi.lib()
        self._h = C.c_void_p()
        self._stream = stream
        with torch.cuda.device(self.device):
            capi.check(self._lib.spk_stream_create(self.width, self.height,
                                                   _stream(stream), C.byref(self._h)))

    @property
    def frames(self) -> int:
        return int(self._lib.spk_stream_frames(self._h))

    def _take(self, ev: C.c_void_p, offs: C.c_void_p, total: int, s: int):
        """copy the library's pool buffers into torch tensors and free them"""
        so = torch.cuda.ExternalStream(s) if s else torch.cuda.default_stream(self.device)
        try:
            with torch.cuda.stream(so):
                o = torch.as_tensor(_DevBuf(offs.value, (self.npix + 1) * 8), device=self.device)
                offsets = o.view(torch.int64).clone()
                if total:
                    e = torch.as_tensor(_DevBuf(ev.value, total * 16), device=self.device)
                    pairs = e.view(torch.int64).view(total, 2).clone()
                    durations = pairs[:, 0].contiguous()
                    intensities = pairs[:, 1].contiguous().view(torch.float64)
                else:
                    durations = torch.empty(0, dtype=torch.int64, device=self.device)
                    intensities = torch.empty(0, dtype=torch.float64, device=self.device)
        finally:
            capi.check(self._lib.spk_free_device(ev, s))
            capi.check(self._lib.spk_free_device(offs, s))
        return offsets, durations, intensities

    def push(self, block):
        """Frames of the next block: a PackedVolume of this geometry, or a
        [frames, pitch] uint8 tensor of pitched planes on the device."""
        if isinstance(block, PackedVolume):
            if (block.width, block.height) != (self.width, self.height):
                raise ValueError("block geometry differs from the stream's")
            planes, frames, pitch = block.planes, block.frames, block.pitch
        else:
            planes, frames = block, int(block.shape[0])
            pitch = int(block.stride(0)) if frames else plane_pitch(self.width, self.height)
        ev, offs, tot = C.c_void_p(), C.c_void_p(), C.c_uint64()
        with torch.cuda.device(self.device):
            s = _stream(self._stream)
            capi.check(self._lib.spk_stream_push(self._h, planes.data_ptr() if frames else None,
                                                 pitch, frames, C.byref(ev), C.byref(offs),
                                                 C.byref(tot), s))
            return self._take(ev, offs, int(tot.value), s)

    def flush(self):
        """The still-open spans (PixelReconState::flush); ends the stream."""
        ev, offs, tot = C.c_void_p(), C.c_void_p(), C.c_uint64()
        with torch.cuda.device(self.device):
            s = _stream(self._stream)
            capi.check(self._lib.spk_stream_flush(self._h, C.byref(ev), C.byref(offs),
                                                  C.byref(tot), s))
            return self._take(ev, offs, int(tot.value), s)

    def close(self):
        if self._h:
            self._lib.spk_stream_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001 -- interpreter shutdown
            pass
