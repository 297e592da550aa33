"""The reference's own caller over the B200 path.

oracle/_ref/acceptance_b200 is the reference's acceptance gate
(proj/tests/acceptance.cpp) linked against the UNMODIFIED reference sources
with spikecam::reconstruct bound to libspikecam_b200.so by
integration/reconstruct_b200.cpp (recipe: oracle/Makefile target `b200`).
Every reconstruct() of the gate -- the moving-bar scene of criterion 7 and
bench() of criterion 9 (1000 fps floor, FSR/SSR within 2x) -- runs on the GPU.
"""
import os
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
BIN = ROOT / "oracle" / "_ref" / "acceptance_b200"


@pytest.mark.gpu
def test_reference_acceptance_gate_on_b200():
    if not BIN.exists():
        pytest.skip("acceptance_b200 not built (needs /root/reference at build time)")
    env = dict(os.environ, SPK_B200_TRACE="1")
    r = subprocess.run([str(BIN)], capture_output=True, text=True, timeout=900, env=env,
                       cwd=ROOT / "oracle" / "_ref")
    out = r.stdout
    passes = [ln for ln in out.splitlines() if ln.startswith("[PASS]")]
    fails = [ln for ln in out.splitlines() if ln.startswith("[FAIL]")]
    assert r.returncode == 0 and not fails, out + r.stderr[-2000:]
    assert len(passes) == 10, out
    # the gate's reconstructions went through the C-ABI (criteria 7 and 9)
    assert "[b200] reconstruct fsr -> spk_reconstruct_host" in r.stderr
    assert "[b200] reconstruct ssr -> spk_reconstruct_host" in r.stderr
    print(out)


def test_acceptance_b200_links_the_c_abi():
    """CPU check: the binding binary resolves spikecam::reconstruct to the
    C-ABI library (no GPU needed to inspect the link)."""
    if not BIN.exists():
        pytest.skip("acceptance_b200 not built")
    ldd = subprocess.run(["ldd", str(BIN)], capture_output=True, text=True).stdout
    assert "libspikecam_b200.so" in ldd
    syms = subprocess.run(["nm", "-D", "--undefined-only", str(BIN)], capture_output=True,
                          text=True).stdout
    assert "spk_reconstruct_host" in syms
