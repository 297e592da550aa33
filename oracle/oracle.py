"""ctypes face of the oracle libraries.  TEST INFRASTRUCTURE ONLY.

    liboracle.so             C restatement of the reference path (spk_oracle.c)
    _ref/libspikecam_ref.so  the unmodified reference sources + ref_shim.cpp

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg import
this module, and only as the checker / the CPU arm -- never as the product.
Both libraries are built by oracle/Makefile (`make -C oracle all ref`).
"""
from __future__ import annotations

import ctypes as C
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ORACLE_SO = HERE / "liboracle.so"
REF_SO = HERE / "_ref" / "libspikecam_ref.so"
REF_SRC = Path("/root/reference/proj")

FSR, SSR, TFI, TFP = 0, 1, 2, 3
METHODS = {"fsr": FSR, "ssr": SSR, "tfi": TFI, "tfp": TFP}

_P = C.c_void_p
_L = C.c_long


def build(ref: bool = True) -> None:
    """Compile the C restatement and, where /root/reference exists, the reference."""
    subprocess.run(["make", "-s", "-C", str(HERE), "all"], check=True)
    if ref and REF_SRC.exists():
        subprocess.run(["make", "-s", "-C", str(HERE), "ref"], check=True)
        # the reference's acceptance gate over the B200 path (integration/);
        # needs libspikecam_b200.so, so __graft_entry__.build() builds it first
        subprocess.run(["make", "-s", "-C", str(HERE), "b200"], check=True)


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


class Oracle:
    """C restatement (spk_oracle.c)."""

    def __init__(self, path: Path = ORACLE_SO):
        if not path.exists():
            build(ref=False)
        h = C.CDLL(str(path))
        h.orc_plane_bytes.restype = C.c_size_t
        h.orc_plane_bytes.argtypes = [C.c_int, C.c_int]
        h.orc_pack.argtypes = [_P, C.c_int, C.c_int, _L, _P, C.c_size_t]
        h.orc_unpack.argtypes = [_P, C.c_int, C.c_int, _L, C.c_size_t, C.c_int, _P]
        h.orc_quantize.restype = C.c_uint8
        h.orc_quantize.argtypes = [C.c_double]
        h.orc_row_f64.argtypes = [_P, _L, C.c_int, C.c_int, _P]
        for f in (h.orc_reconstruct_f64, h.orc_reconstruct_u8):
            f.argtypes = [_P, C.c_int, C.c_int, _L, C.c_size_t, C.c_int, C.c_int, _L, _L, _P,
                          C.c_size_t, C.c_int]
        h.orc_runs.restype = _L
        h.orc_runs.argtypes = [_P, _L, C.c_int, _P, _P, _P, _L]
        h.orc_fsr_events.restype = _L
        h.orc_fsr_events.argtypes = [_P, _L, _P, _P, _L]
        h.orc_encode.restype = _L
        h.orc_encode.argtypes = [_L, C.c_double, _P, _L]
        h.orc_te_u8.restype = C.c_double
        h.orc_te_u8.argtypes = [_P, C.c_int, C.c_int]
        h.orc_te_f64.restype = C.c_double
        h.orc_te_f64.argtypes = [_P, C.c_int, C.c_int]
        h.orc_mse.restype = C.c_double
        h.orc_mse.argtypes = [_P, _P, _L]
        h.orc_stability.argtypes = [_P, _L, C.c_int, _P, C.c_char_p, _L]
        self.h = h

    # framing
    def plane_bytes(self, w, h):
        return int(self.h.orc_plane_bytes(w, h))

    def pack(self, bits: np.ndarray, w: int, h: int, pitch: int | None = None) -> np.ndarray:
        bits = np.ascontiguousarray(bits, dtype=np.uint8).reshape(-1, w * h)
        t = bits.shape[0]
        pitch = pitch or self.plane_bytes(w, h)
        out = np.zeros((t, pitch), dtype=np.uint8)
        self.h.orc_pack(_ptr(bits), w, h, t, _ptr(out), pitch)
        return out

    def unpack(self, planes: np.ndarray, w: int, h: int, t: int, pitch: int,
               msb_first: bool = False) -> np.ndarray:
        planes = np.ascontiguousarray(planes, dtype=np.uint8)
        out = np.zeros((t, w * h), dtype=np.uint8)
        self.h.orc_unpack(_ptr(planes), w, h, t, pitch, int(msb_first), _ptr(out))
        return out

    def quantize(self, v: float) -> int:
        return int(self.h.orc_quantize(v))

    # rows
    def row_f64(self, bits: np.ndarray, method: int, window: int = 32) -> np.ndarray:
        bits = np.ascontiguousarray(bits, dtype=np.uint8)
        out = np.zeros(bits.size, dtype=np.float64)
        if self.h.orc_row_f64(_ptr(bits), bits.size, method, window, _ptr(out)) != 0:
            raise ValueError("bad method/window")
        return out

    def runs(self, bits: np.ndarray, method: int):
        bits = np.ascontiguousarray(bits, dtype=np.uint8)
        cap = max(1, bits.size)
        s, e, c = (np.zeros(cap, dtype=np.int64) for _ in range(3))
        n = self.h.orc_runs(_ptr(bits), bits.size, method, _ptr(s), _ptr(e), _ptr(c), cap)
        return s[:n], e[:n], c[:n]

    def fsr_events(self, bits: np.ndarray):
        bits = np.ascontiguousarray(bits, dtype=np.uint8)
        cap = bits.size + 2
        d = np.zeros(cap, dtype=np.int64)
        v = np.zeros(cap, dtype=np.float64)
        n = self.h.orc_fsr_events(_ptr(bits), bits.size, _ptr(d), _ptr(v), cap)
        return d[:n], v[:n]

    def encode(self, duration: int, intensity: float) -> np.ndarray:
        cap = duration // 255 + 2
        w = np.zeros(cap, dtype=np.uint16)
        n = self.h.orc_encode(duration, intensity, _ptr(w), cap)
        if n < 0:
            raise ValueError("encode: bad duration/intensity")
        return w[:n]

    def pixel_records(self, bits: np.ndarray, method: int) -> np.ndarray:
        """encode_events of one pixel's segments (spikecam_main.cpp:146-172):
        lead [0, s0) at 0, each run at 255*N/span, tail [s_last, T) carrying
        the last run's value (build_segments, reconstruct.cpp:107-130)."""
        bits = np.ascontiguousarray(bits, dtype=np.uint8)
        t = bits.size
        if t == 0:
            return np.zeros(0, np.uint16)
        spikes = np.flatnonzero(bits)
        segs = []
        if spikes.size == 0:
            segs.append((t, 0.0))
        else:
            if spikes[0] > 0:
                segs.append((int(spikes[0]), 0.0))
            carry = 0.0
            for a, b, n in zip(*self.runs(bits, method)):
                carry = 255.0 * float(n) / float(b - a)
                segs.append((int(b - a), carry))
            segs.append((int(t - spikes[-1]), carry))
        return np.concatenate([self.encode(d, v) for d, v in segs])

    def records(self, planes: np.ndarray, w: int, h: int, t: int, pitch: int, method: int,
                fps: int = 20000) -> bytes:
        """SPKR file image (write_spkr, io.cpp:240-255) of a packed volume."""
        bits = self.unpack(planes, w, h, t, pitch)
        out = [b"SPKR", np.array([w, h], "<u2").tobytes(), np.array([fps, t], "<u4").tobytes()]
        for p in range(w * h):
            words = self.pixel_records(bits[:, p], method) if t else np.zeros(0, np.uint16)
            out.append(np.array([words.size], "<u4").tobytes())
            out.append(words.astype("<u2").tobytes())
        return b"".join(out)

    # volumes (planes: [T, pitch] uint8, LSB-first)
    # quality metrics and the stability check (metrics.cpp:12-61, stability.cpp:61-128)
    def te(self, frame: np.ndarray) -> float:
        """two_dimensional_entropy of one [H, W] frame (uint8 = quantized, or doubles)."""
        f = np.ascontiguousarray(frame)
        hh, ww = f.shape
        if f.dtype == np.uint8:
            return float(self.h.orc_te_u8(_ptr(f), ww, hh))
        f = f.astype(np.float64)
        return float(self.h.orc_te_f64(_ptr(f), ww, hh))

    def mse(self, a: np.ndarray, b: np.ndarray) -> float:
        a = np.ascontiguousarray(a, dtype=np.float64).reshape(-1)
        b = np.ascontiguousarray(b, dtype=np.float64).reshape(-1)
        return float(self.h.orc_mse(_ptr(a), _ptr(b), a.size))

    def stability(self, bits: np.ndarray, depth: int = 8) -> dict:
        bits = np.ascontiguousarray(bits, dtype=np.uint8)
        out = np.zeros(4, np.int64)
        path = C.create_string_buffer(64)
        if self.h.orc_stability(_ptr(bits), bits.size, depth, _ptr(out), path, 64):
            raise ValueError("stability_order: max_depth must be in [1, 60]")
        return _stab_result(out, path)

    def reconstruct(self, planes: np.ndarray, w: int, h: int, t: int, pitch: int, method: int,
                    window: int = 32, dtype=np.uint8, pix_begin: int = 0,
                    pix_end: int | None = None, threads: int = 0) -> np.ndarray:
        planes = np.ascontiguousarray(planes, dtype=np.uint8)
        pix_end = w * h if pix_end is None else pix_end
        n = pix_end - pix_begin
        out = np.zeros((t, n), dtype=dtype)
        fn = self.h.orc_reconstruct_u8 if dtype == np.uint8 else self.h.orc_reconstruct_f64
        rc = fn(_ptr(planes), w, h, t, pitch, method, window, pix_begin, pix_end, _ptr(out), n,
                threads)
        if rc != 0:
            raise ValueError("bad method/window")
        return out


def _stab_result(out, path):
    return {"depth": int(out[0]), "index": int(out[1]), "verified_order": int(out[2]),
            "absolute": bool(out[3]), "path": path.value.decode()}


class Reference:
    """The unmodified reference library (oracle/_ref/libspikecam_ref.so)."""

    def __init__(self, path: Path = REF_SO):
        if not path.exists():
            if REF_SRC.exists():
                build(ref=True)
            else:
                raise FileNotFoundError(f"{path} not built (needs /root/reference)")
        h = C.CDLL(str(path))
        h.ref_last_error.restype = C.c_char_p
        h.ref_reconstruct.restype = _L
        h.ref_reconstruct.argtypes = [_P, C.c_size_t, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                      C.c_int, _P, _P]
        h.ref_reconstruct_serial.restype = _L
        h.ref_reconstruct_serial.argtypes = [_P, C.c_size_t, C.c_int, C.c_int, C.c_int, C.c_int,
                                             C.c_int, _P]
        h.ref_bench_fps.restype = C.c_double
        h.ref_bench_fps.argtypes = [_P, C.c_size_t, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                    C.c_int, C.c_int]
        h.ref_segments.restype = _L
        h.ref_segments.argtypes = [_P, _L, C.c_int, _P, _P, _P, _P, _L]
        h.ref_reconstruct_pixel.restype = _L
        h.ref_reconstruct_pixel.argtypes = [_P, _L, C.c_int, C.c_int, _P]
        h.ref_stream_events.restype = _L
        h.ref_stream_events.argtypes = [_P, _L, _L, _P, _P, _L]
        h.ref_fsr_events.restype = _L
        h.ref_fsr_events.argtypes = [_P, _L, _P, _P, _L]
        h.ref_simulate_pixel.restype = _L
        h.ref_simulate_pixel.argtypes = [_P, _L, C.c_double, C.c_double, _P]
        h.ref_pixel_seed.restype = C.c_uint64
        h.ref_pixel_seed.argtypes = [C.c_uint64, C.c_int, C.c_int]
        h.ref_write_spk.restype = _L
        h.ref_write_spk.argtypes = [_P, C.c_size_t, C.c_int, C.c_int, C.c_int, C.c_uint32,
                                    C.c_char_p]
        h.ref_read.restype = _L
        h.ref_read.argtypes = [C.c_char_p, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_int),
                               C.POINTER(C.c_int), C.POINTER(C.c_uint32), _P, C.c_size_t]
        h.ref_write_pgm.restype = _L
        h.ref_write_pgm.argtypes = [_P, C.c_int, C.c_int, C.c_char_p]
        h.ref_encode_events.restype = _L
        h.ref_encode_events.argtypes = [_P, _P, _L, _P, _L]
        h.ref_emit_records.restype = _L
        h.ref_emit_records.argtypes = [_P, C.c_size_t, C.c_int, C.c_int, C.c_int, C.c_int,
                                       C.c_uint32, C.c_char_p]
        for f in (h.ref_te,):
            f.restype = C.c_double
            f.argtypes = [_P, C.c_int, C.c_int]
        for f in (h.ref_mse, h.ref_psnr):
            f.restype = C.c_double
            f.argtypes = [_P, _P, C.c_int, C.c_int]
        h.ref_stability.restype = _L
        h.ref_stability.argtypes = [_P, _L, C.c_int, _P, C.c_char_p, _L]
        self.h = h

    def _err(self):
        return self.h.ref_last_error().decode()

    def reconstruct(self, planes, pitch, w, h, t, method, window=32, workers=0):
        planes = np.ascontiguousarray(planes, dtype=np.uint8)
        f = np.zeros((t, w * h), dtype=np.float64)
        u = np.zeros((t, w * h), dtype=np.uint8)
        if self.h.ref_reconstruct(_ptr(planes), pitch, w, h, t, method, window, workers, _ptr(f),
                                  _ptr(u)) != 0:
            raise ValueError(self._err())
        return f, u

    def reconstruct_serial(self, planes, pitch, w, h, t, method, window=32):
        planes = np.ascontiguousarray(planes, dtype=np.uint8)
        f = np.zeros((t, w * h), dtype=np.float64)
        if self.h.ref_reconstruct_serial(_ptr(planes), pitch, w, h, t, method, window, _ptr(f)):
            raise ValueError(self._err())
        return f

    def bench_fps(self, planes, pitch, w, h, t, method, window=32, repeats=3, workers=1):
        planes = np.ascontiguousarray(planes, dtype=np.uint8)
        return float(self.h.ref_bench_fps(_ptr(planes), pitch, w, h, t, method, window, repeats,
                                          workers))

    def segments(self, bits, method):
        bits = np.ascontiguousarray(bits, dtype=np.uint8)
        cap = bits.size + 2
        s, e, n = (np.zeros(cap, dtype=np.int64) for _ in range(3))
        v = np.zeros(cap, dtype=np.float64)
        k = self.h.ref_segments(_ptr(bits), bits.size, method, _ptr(s), _ptr(e), _ptr(n), _ptr(v),
                                cap)
        if k < 0:
            raise ValueError(self._err())
        return s[:k], e[:k], n[:k], v[:k]

    def reconstruct_pixel(self, bits, method, window=32):
        bits = np.ascontiguousarray(bits, dtype=np.uint8)
        out = np.zeros(bits.size, dtype=np.float64)
        if self.h.ref_reconstruct_pixel(_ptr(bits), bits.size, method, window, _ptr(out)) < 0:
            raise ValueError(self._err())
        return out

    def stream_events(self, bits, block):
        bits = np.ascontiguousarray(bits, dtype=np.uint8)
        cap = bits.size + 2
        d = np.zeros(cap, dtype=np.int64)
        v = np.zeros(cap, dtype=np.float64)
        k = self.h.ref_stream_events(_ptr(bits), bits.size, block, _ptr(d), _ptr(v), cap)
        return d[:k], v[:k]

    def fsr_events(self, bits):
        bits = np.ascontiguousarray(bits, dtype=np.uint8)
        cap = bits.size + 2
        d = np.zeros(cap, dtype=np.int64)
        v = np.zeros(cap, dtype=np.float64)
        k = self.h.ref_fsr_events(_ptr(bits), bits.size, _ptr(d), _ptr(v), cap)
        return d[:k], v[:k]

    def simulate_pixel(self, rates, threshold=1.0, residual=0.0):
        rates = np.ascontiguousarray(rates, dtype=np.float64)
        bits = np.zeros(rates.size, dtype=np.uint8)
        if self.h.ref_simulate_pixel(_ptr(rates), rates.size, threshold, residual, _ptr(bits)):
            raise ValueError(self._err())
        return bits

    def pixel_seed(self, seed, x, y):
        return int(self.h.ref_pixel_seed(seed, x, y))

    def write_spk(self, planes, pitch, w, h, t, fps, path):
        planes = np.ascontiguousarray(planes, dtype=np.uint8)
        if self.h.ref_write_spk(_ptr(planes), pitch, w, h, t, fps, str(path).encode()):
            raise OSError(self._err())

    def read(self, path, kind=0, w=400, h=250, cap=1 << 28):
        wo, ho, fo = C.c_int(), C.c_int(), C.c_uint32()
        buf = np.zeros(cap, dtype=np.uint8)
        t = self.h.ref_read(str(path).encode(), kind, w, h, C.byref(wo), C.byref(ho), C.byref(fo),
                            _ptr(buf), cap)
        if t < 0:
            raise OSError(self._err())
        return buf[: t * wo.value * ho.value].reshape(t, wo.value * ho.value), wo.value, ho.value, \
            fo.value

    def write_pgm(self, values, w, h, path):
        values = np.ascontiguousarray(values, dtype=np.float64)
        if self.h.ref_write_pgm(_ptr(values), w, h, str(path).encode()):
            raise OSError(self._err())

    def encode_events(self, durations, intensities):
        d = np.ascontiguousarray(durations, dtype=np.int64)
        v = np.ascontiguousarray(intensities, dtype=np.float64)
        cap = int(d.sum() // 255 + d.size + 2) if d.size else 1
        words = np.zeros(cap, dtype=np.uint16)
        n = self.h.ref_encode_events(_ptr(d), _ptr(v), d.size, _ptr(words), cap)
        if n < 0:
            raise ValueError(self._err())
        return words[:n]

    def emit_records(self, planes, pitch, w, h, t, method, fps, path):
        """The CLI's --emit-records output (SPKR file) for a packed volume."""
        planes = np.ascontiguousarray(planes, dtype=np.uint8)
        if self.h.ref_emit_records(_ptr(planes), pitch, w, h, t, method, fps, str(path).encode()) < 0:
            raise ValueError(self._err())


    def te(self, values: np.ndarray) -> float:
        """two_dimensional_entropy of one [H, W] image of doubles."""
        v = np.ascontiguousarray(values, dtype=np.float64)
        r = self.h.ref_te(_ptr(v), v.shape[1], v.shape[0])
        if np.isnan(r):
            raise ValueError(self._err())
        return float(r)

    def mse(self, a: np.ndarray, b: np.ndarray) -> float:
        a = np.ascontiguousarray(a, dtype=np.float64)
        b = np.ascontiguousarray(b, dtype=np.float64)
        return float(self.h.ref_mse(_ptr(a), _ptr(b), a.shape[1], a.shape[0]))

    def psnr(self, a: np.ndarray, b: np.ndarray) -> float:
        a = np.ascontiguousarray(a, dtype=np.float64)
        b = np.ascontiguousarray(b, dtype=np.float64)
        return float(self.h.ref_psnr(_ptr(a), _ptr(b), a.shape[1], a.shape[0]))

    def stability(self, bits: np.ndarray, depth: int = 8) -> dict:
        bits = np.ascontiguousarray(bits, dtype=np.uint8)
        out = np.zeros(4, np.int64)
        path = C.create_string_buffer(256)
        if self.h.ref_stability(_ptr(bits), bits.size, depth, _ptr(out), path, 256) < 0:
            raise ValueError(self._err())
        return _stab_result(out, path)


def ref_available() -> bool:
    return REF_SO.exists()
