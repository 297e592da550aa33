"""C-ABI library: loads, exports every symbol include/spikecam_b200.h declares,
and rejects bad arguments the way the reference does -- all without a GPU
(validation happens before any CUDA call)."""
import ctypes as C
import re
from pathlib import Path

import numpy as np
import pytest

from paper_2412_11639_b200 import _capi as capi

ROOT = Path(__file__).resolve().parents[1]


def declared_symbols():
    text = (ROOT / "include" / "spikecam_b200.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(spk_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = capi.lib()
    names = declared_symbols()
    assert len(names) >= 14
    for n in names:
        assert hasattr(lib, n), n
        assert n in capi.SIGNATURES, f"{n} has no ctypes signature"
    assert set(capi.SIGNATURES) == set(names)


def test_library_is_sm100a_only():
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", str(capi.LIB_PATH)], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out
    assert not re.search(r"sm_(?!100a)\d+", out), out


def test_version_and_pitch():
    lib = capi.lib()
    assert lib.spk_version() >= 100
    assert lib.spk_plane_pitch(400, 250) == 12512  # 12500 B plane -> 16-B multiple
    assert lib.spk_plane_pitch(1000, 1000) == 125008
    assert lib.spk_plane_pitch(9, 1) == 16


def g(w=4, h=4, t=8, pitch=16):
    return capi.geom(w, h, t, pitch)


@pytest.mark.parametrize("fn", ["spk_reconstruct_u8", "spk_reconstruct_f32", "spk_reconstruct_f64"])
def test_invalid_arguments(fn):
    lib = capi.lib()
    f = getattr(lib, fn)
    dummy = C.c_void_p(16)  # never dereferenced: validation fails first
    assert f(g(), dummy, 7, 32, dummy, 16, None) == capi.SPK_EINVAL
    assert b"unknown reconstruction method" in lib.spk_last_error()
    assert f(g(), dummy, capi.SPK_TFP, 0, dummy, 16, None) == capi.SPK_EINVAL
    assert b"tfp window must be >= 1" in lib.spk_last_error()
    assert f(g(w=0), dummy, 0, 32, dummy, 16, None) == capi.SPK_EINVAL
    assert f(g(pitch=2), dummy, 0, 32, dummy, 16, None) == capi.SPK_EINVAL
    assert f(g(), dummy, 0, 32, dummy, 15, None) == capi.SPK_EINVAL  # out_pitch < W*H
    assert f(None, dummy, 0, 32, dummy, 16, None) == capi.SPK_EINVAL
    # T == 0 is a valid empty volume: nothing to launch
    assert f(g(t=0), None, 0, 32, None, 16, None) == capi.SPK_OK


def test_other_entry_points_validate():
    lib = capi.lib()
    d = C.c_void_p(16)
    assert lib.spk_segment(g(), d, capi.SPK_TFI, d, 8, d, d, None) == capi.SPK_EINVAL
    assert lib.spk_segment(g(), d, capi.SPK_FSR, d, 0, d, d, None) == capi.SPK_EINVAL
    assert lib.spk_set_run_capacity(-1) == capi.SPK_EINVAL
    assert lib.spk_set_run_capacity(0) == capi.SPK_OK
    assert lib.spk_synth(4, 1, g(), 0, 0.0, d, None) == capi.SPK_EINVAL
    assert lib.spk_upload_planes(g(), d, 1, 0, d, None) == capi.SPK_EINVAL  # src_pitch < 2
    assert lib.spk_reconstruct_host(g(), d, 0, 32, 9, d, 16) == capi.SPK_EINVAL
    assert lib.spk_launch_count(1) >= 0 and lib.spk_launch_count(0) == 0


def test_python_error_mapping():
    with pytest.raises(ValueError, match="unknown reconstruction method"):
        capi.check(capi.lib().spk_reconstruct_u8(g(), C.c_void_p(16), 9, 32, C.c_void_p(16), 16,
                                                 None))
