"""In-grid time split (capi.cu reconstruct_split, csrc/shard.cu
k_split_combine): one stream's scan cut in S time shards inside one
reconstruction must give exactly the frames of the one-pass scan -- every
scene family, odd pixel counts, shard counts that leave a short last shard,
pixels re-scanned whole (sparse spikes: lone spikes across shards), list
overflows (noise: k_fixup), FSR and SSR, uint8 and float64.  SPK_SPLIT=S
forces S shards (1 = one pass); the default chooses S from the sensor size
(BASELINE 400x250 streams split, 1000x1000 ones do not)."""
import ctypes as C
import os

import numpy as np
import pytest
import torch

import paper_2412_11639_b200 as spk
from paper_2412_11639_b200 import _capi as capi

pytestmark = pytest.mark.gpu


def _run(vol, method, S, dtype=torch.uint8):
    os.environ["SPK_SPLIT"] = str(S)
    lib = capi.lib()
    try:
        lib.spk_set_timing(1)
        out = spk.reconstruct(vol, method, dtype=dtype)
        torch.cuda.synchronize()
        sh, fl = C.c_int32(), C.c_int64()
        capi.check(lib.spk_last_split(C.byref(sh), C.byref(fl)))
    finally:
        lib.spk_set_timing(0)
        del os.environ["SPK_SPLIT"]
    return out, sh.value, fl.value


CASES = [  # scene, w, h, frames, param
    ("moving", 96, 40, 9000, 0.0),
    ("static", 67, 33, 12000, 0.0),
    ("range", 80, 41, 20000, 0.0),
    ("sensor", 50, 50, 10000, 0.0),
    ("noise", 40, 24, 3000, 0.3),     # dense: shard list overflows -> k_fixup
    ("noise", 64, 16, 8000, 0.002),   # sparse: lone spikes across shards
]


@pytest.mark.parametrize("scene,w,h,t,param", CASES)
@pytest.mark.parametrize("method", ["fsr", "ssr"])
def test_split_equals_one_pass(scene, w, h, t, param, method):
    vol = spk.synth(scene, 11, w, h, t, param=param)
    ref, s1, _ = _run(vol, method, 1)
    assert s1 == 1
    for S in (2, 3, 7, 16):
        got, sh, flagged = _run(vol, method, S)
        assert sh == min(S, (t + 31) // 32)
        assert torch.equal(got, ref), (scene, method, S, flagged)


@pytest.mark.parametrize("method", ["fsr", "ssr"])
def test_split_f64_and_oracle(method, oracle):
    w, h, t = 48, 21, 7000
    vol = spk.synth("moving", 5, w, h, t)
    got, sh, _ = _run(vol, method, 5, dtype=torch.float64)
    ref, _, _ = _run(vol, method, 1, dtype=torch.float64)
    assert sh == 5 and torch.equal(got, ref)
    host = vol.planes.cpu().numpy()
    m = 0 if method == "fsr" else 1
    want = oracle.reconstruct(host, w, h, t, vol.pitch, m, dtype=np.float64)
    assert np.array_equal(got.reshape(t, -1).cpu().numpy(), want)


def test_split_default_choice():
    """Long 400x250 FSR streams split (one K2 wave would leave SMs uneven);
    the 1000x1000 sensor (many waves) and shorter streams do not."""
    lib = capi.lib()
    for (w, h, t), split in (((400, 250, 80000), True), ((1000, 1000, 4096), False),
                             ((400, 250, 40000), False)):
        vol = spk.synth("static", 1, w, h, t)
        lib.spk_set_timing(1)
        try:
            spk.reconstruct(vol, "fsr")
            sh, fl = C.c_int32(), C.c_int64()
            capi.check(lib.spk_last_split(C.byref(sh), C.byref(fl)))
        finally:
            lib.spk_set_timing(0)
        assert (sh.value > 1) == split, (w, h, t, sh.value)
        assert fl.value == 0
