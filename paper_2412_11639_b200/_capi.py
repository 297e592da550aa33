"""ctypes binding of libspikecam_b200.so (include/spikecam_b200.h).

Loading fails loudly when the library has not been built: there is no CPU
fallback anywhere in the package.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

import os

# SPIKECAM_B200_LIB: another build of the library (the bounds-checked one,
# build.build_checked(), for tests/test_checked_build.py)
LIB_PATH = Path(os.environ.get("SPIKECAM_B200_LIB") or
                Path(__file__).resolve().parent / "libspikecam_b200.so").resolve()

SPK_OK, SPK_EINVAL, SPK_ECUDA, SPK_ENOMEM = 0, 1, 2, 3
SPK_FSR, SPK_SSR, SPK_TFI, SPK_TFP = 0, 1, 2, 3
SPK_OUT_U8, SPK_OUT_F32, SPK_OUT_F64 = 0, 1, 2


class spk_geom(C.Structure):
    _fields_ = [
        ("width", C.c_int32),
        ("height", C.c_int32),
        ("frames", C.c_int64),
        ("plane_pitch", C.c_size_t),
    ]


class spk_run(C.Structure):
    _fields_ = [("start", C.c_uint32), ("intervals", C.c_uint32)]


# every symbol include/spikecam_b200.h declares, with its ctypes signature
_P = C.c_void_p
_G = C.POINTER(spk_geom)
SIGNATURES = {
    "spk_reconstruct_u8": (C.c_int, [_G, _P, C.c_int, C.c_int, _P, C.c_size_t, _P]),
    "spk_reconstruct_f32": (C.c_int, [_G, _P, C.c_int, C.c_int, _P, C.c_size_t, _P]),
    "spk_reconstruct_f64": (C.c_int, [_G, _P, C.c_int, C.c_int, _P, C.c_size_t, _P]),
    "spk_segment_shards": (C.c_int, [_G, _P, C.c_int, C.c_int64, _P, C.c_int64, _P, _P, _P, _P]),
    "spk_segment": (C.c_int, [_G, _P, C.c_int, _P, C.c_int64, _P, _P, _P]),
    "spk_pack_bytes": (C.c_int, [_G, _P, _P, _P]),
    "spk_unpack_planes": (C.c_int, [_G, _P, _P, _P]),
    "spk_upload_planes": (C.c_int, [_G, _P, C.c_size_t, C.c_int, _P, _P]),
    "spk_reconstruct_host": (C.c_int, [_G, _P, C.c_int, C.c_int, C.c_int, _P, C.c_size_t]),
    "spk_device_count": (C.c_int, []),
    "spk_release_memory": (C.c_int, []),
    "spk_reconstruct_host_multi": (C.c_int, [_G, _P, C.c_int, C.c_int, C.c_int, _P, C.c_size_t, _P,
                                             C.c_int32]),
    "spk_segment_host": (C.c_int, [_G, _P, C.c_int, _P, C.c_int64, _P, _P]),
    "spk_reconstruct_batch": (C.c_int, [_G, C.c_int32, _P, C.c_int, C.c_int, C.c_int, _P, C.c_size_t, _P]),
    "spk_batch_release": (C.c_int, []),
    "spk_reconstruct_host_batch": (C.c_int, [_G, C.c_int32, _P, C.c_int, C.c_int, C.c_int, _P,
                                             C.c_size_t]),
    "spk_records": (C.c_int, [_G, _P, C.c_int, C.c_uint32, _P, _P, _P]),
    "spk_records_host": (C.c_int, [_G, _P, C.c_int, C.c_uint32, _P, _P]),
    "spk_free_device": (C.c_int, [_P, _P]),
    "spk_free_host": (None, [_P]),
    "spk_segment_state": (C.c_int, [_G, _P, C.c_int, _P, C.c_int64, _P, _P, _P, _P, _P]),
    "spk_state_fresh": (C.c_int, [C.c_int64, _P, _P]),
    "spk_shard_resolve": (C.c_int, [_G, _P, C.c_int, _P, _P, C.c_int64, _P, _P, _P, C.c_int32, _P,
                                    _P, _P]),
    "spk_shard_junction": (C.c_int, [_G, C.c_int, _P, _P, _P, C.c_int32, _P, _P, C.c_int64, _P, _P,
                                     _P, _P, _P, _P, _P, _P, _P]),
    "spk_shard_close_chain": (C.c_int, [C.c_int64, _P, _P, C.c_int32, _P, _P]),
    "spk_shard_stitch": (C.c_int, [_G, C.c_int, _P, _P, _P, C.c_int32, _P, _P, C.c_int64, _P, _P, _P,
                                   _P, _P, _P, _P, C.c_int64, _P, _P, _P]),
    "spk_stream_create": (C.c_int, [C.c_int32, C.c_int32, _P, _P]),
    "spk_stream_push": (C.c_int, [_P, _P, C.c_size_t, C.c_int64, _P, _P, _P, _P]),
    "spk_stream_flush": (C.c_int, [_P, _P, _P, _P, _P]),
    "spk_stream_push_host": (C.c_int, [_P, _P, C.c_int64, _P, _P, _P]),
    "spk_stream_flush_host": (C.c_int, [_P, _P, _P, _P]),
    "spk_stream_frames": (C.c_int64, [_P]),
    "spk_stream_destroy": (C.c_int, [_P]),
    "spk_expand_runs_u8": (C.c_int, [_G, _P, C.c_int64, _P, _P, _P, C.c_size_t, _P]),
    "spk_expand_runs_f32": (C.c_int, [_G, _P, C.c_int64, _P, _P, _P, C.c_size_t, _P]),
    "spk_expand_runs_f64": (C.c_int, [_G, _P, C.c_int64, _P, _P, _P, C.c_size_t, _P]),
    "spk_set_run_capacity": (C.c_int, [C.c_int64]),
    "spk_plane_pitch": (C.c_size_t, [C.c_int32, C.c_int32]),
    "spk_launch_count": (C.c_int64, [C.c_int]),
    "spk_set_timing": (C.c_int, [C.c_int]),
    "spk_last_split": (C.c_int, [_P, _P]),
    "spk_last_timing": (C.c_int, [_P, _P, _P, _P]),
    "spk_last_error": (C.c_char_p, []),
    "spk_version": (C.c_int, []),
    "spk_synth": (C.c_int, [C.c_int, C.c_uint64, _G, C.c_int64, C.c_double, _P, _P]),
    "spk_frame_metrics": (C.c_int, [_G, _P, C.c_int, C.c_size_t, _P, C.c_int, C.c_size_t, _P, _P,
                                    _P]),
    "spk_stability": (C.c_int, [_G, _P, C.c_int, _P, _P]),
    "spk_frame_metrics_host": (C.c_int, [_G, _P, C.c_int, C.c_size_t, _P, C.c_int, C.c_size_t,
                                         _P, _P]),
    "spk_stability_host": (C.c_int, [_G, _P, C.c_int, _P]),
}

_lib = None


def lib() -> C.CDLL:
    """The loaded library; raises if it was not built (no fallback path)."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise RuntimeError(
                f"{LIB_PATH} is missing: build it with __graft_entry__.build() "
                "(the reconstruction path has no CPU fallback)")
        h = C.CDLL(str(LIB_PATH))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(h, name)
            fn.restype = res
            fn.argtypes = args
        _lib = h
    return _lib


class SpikecamError(RuntimeError):
    """SPK_ECUDA: device failure (std::runtime_error in the C++ wrapper)."""


def check(rc: int) -> None:
    """Map a C-ABI return code onto the reference's exception classes."""
    if rc == SPK_OK:
        return
    msg = lib().spk_last_error().decode(errors="replace")
    if rc == SPK_EINVAL:
        raise ValueError(msg)  # std::invalid_argument
    if rc == SPK_ENOMEM:
        raise MemoryError(msg)
    raise SpikecamError(msg)


def geom(width: int, height: int, frames: int, plane_pitch: int) -> spk_geom:
    return spk_geom(int(width), int(height), int(frames), int(plane_pitch))
