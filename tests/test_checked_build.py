"""The kernels' index invariants, asserted: compute-sanitizer is closed on
the GPU pool, so the GPU parity tests also run against the bounds-checked
build (build.build_checked(): -DSPK_CHECKED, SPK_CHECK traps on a change
outside its sub-tile, a stream slot past the change stream, a run list
segment outside its shard region, ...).  A violated check fails the kernel
and the child's tests."""
import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]

def test_checked_build_has_the_checks():
    """the checked build carries the traps (BPT.TRAP in its SASS), the
    product build none"""
    import shutil
    from paper_2412_11639_b200.build import CHECKED_LIB, LIB, build_checked
    lib = CHECKED_LIB if CHECKED_LIB.exists() else build_checked()
    cuobjdump = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"

    def traps(path):
        out = subprocess.run([cuobjdump, "-sass", str(path)], capture_output=True, text=True).stdout
        return out.count("BPT.TRAP")
    assert traps(lib) > 100
    assert traps(LIB) == 0


@pytest.mark.gpu
def test_gpu_suite_on_checked_build():
    from paper_2412_11639_b200.build import CHECKED_LIB, build_checked
    lib = CHECKED_LIB if CHECKED_LIB.exists() else build_checked()
    env = dict(os.environ, SPIKECAM_B200_LIB=str(lib))
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider",
                        "tests/test_gpu_parity.py", "tests/test_split.py", "tests/test_time_shards.py",
                        "tests/test_batch.py", "tests/test_limits.py", "tests/test_stream.py",
                        "tests/test_records.py"],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=1800)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert "passed" in r.stdout
