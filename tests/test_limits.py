"""Workspace limits of the expand stage: the change stream's
32-bit offsets (pixel parts when npix * cap would pass 2^32) and the K2c
grid.y bound (threads stride over a pixel's run blocks).  The limits are lowered
through test hooks (SPK_TEST_PART_ENTRIES / SPK_TEST_GRID_Y, read once per
process) so the split paths run on small volumes; each subprocess compares
its frames with the oracle."""
import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]

CHILD = r"""
import sys, numpy as np, torch
sys.path.insert(0, %r)
import paper_2412_11639_b200 as spk
from paper_2412_11639_b200 import _capi as capi
from oracle.oracle import Oracle
w, h, t = 300, 7, 3000
for method in (0, 1):
    v = spk.synth("moving", 5, w, h, t)
    capi.lib().spk_set_run_capacity(int(sys.argv[1]))
    got = spk.reconstruct(v, spk.ReconMethod(spk.Method(method))).reshape(t, w * h).cpu().numpy()
    want = Oracle().reconstruct(v.planes.cpu().numpy(), w, h, t, v.pitch, method)
    assert np.array_equal(got, want), method
    runs, counts, last = spk.segments(v, spk.ReconMethod(spk.Method(method)), run_cap=3000)
    e = torch.empty((t, w * h), dtype=torch.uint8, device="cuda")
    capi.check(capi.lib().spk_expand_runs_u8(v.geom(), runs.data_ptr(), 3000, counts.data_ptr(),
                                             last.data_ptr(), e.data_ptr(), w * h, None))
    assert np.array_equal(e.cpu().numpy(), want), method
print("ok")
"""


def _run(env_extra, cap):
    env = dict(os.environ, **env_extra)
    r = subprocess.run([sys.executable, "-c", CHILD % str(ROOT), str(cap)], env=env,
                       capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr[-3000:]


@pytest.mark.gpu
def test_expand_in_pixel_parts():
    # 2100 pixels x cap 1500 = 3.15M entries; parts of 2048 entries per... at most
    # 1,000,000 entries -> 512-pixel groups x 1 (parts of 512 pixels)
    _run({"SPK_TEST_PART_ENTRIES": "1000000"}, 1500)


@pytest.mark.gpu
def test_fin_scatter_segment_slabs():
    # cap 3000 -> 47 run blocks of 64; grid.y limited to 5 -> each thread strides over ~10
    _run({"SPK_TEST_GRID_Y": "5"}, 3000)


@pytest.mark.gpu
def test_exact_length_change_stream():
    # the change stream allocated after the scan at its exact length (the path
    # of >= 1 GiB worst cases: 1000x1000 sensors, 1M-frame streams), forced on a
    # small volume; also with pixel parts (each part reads back its own total)
    _run({"SPK_TEST_EXACT_STREAM": "1"}, 1500)
    _run({"SPK_TEST_EXACT_STREAM": "1", "SPK_TEST_PART_ENTRIES": "1000000"}, 700)
