"""Oracle restatement == the compiled reference (oracle/_ref) on seeded volumes.

Skipped where the reference library was not built (it needs /root/reference;
the driver's CPU run happens in the build container, where it exists).
"""
import numpy as np
import pytest

from oracle.oracle import Reference, ref_available

pytestmark = pytest.mark.skipif(not ref_available(), reason="oracle/_ref not built")


@pytest.mark.parametrize("seed", range(4))
def test_random_volumes_all_methods(oracle, seed):
    ref = Reference()
    rng = np.random.default_rng(100 + seed)
    w, h, t = int(rng.integers(1, 33)), int(rng.integers(1, 20)), int(rng.integers(0, 900))
    npix = w * h
    bits = np.zeros((t, npix), np.uint8)
    for p in range(npix):
        rates = np.full(t, rng.uniform(0.005, 1.0))
        if t and rng.random() < 0.5:
            rates[int(rng.integers(0, t)):] = rng.uniform(0.005, 1.0)
        bits[:, p] = ref.simulate_pixel(rates, 1.0, rng.uniform(0, 1))
    bits ^= (rng.random(bits.shape) < rng.choice([0.0, 0.01, 0.05])).astype(np.uint8)
    planes = oracle.pack(bits, w, h) if t else np.zeros((0, (npix + 7) // 8), np.uint8)
    pitch = (npix + 7) // 8
    for m, win in ((0, 32), (1, 32), (2, 32), (3, 1), (3, 32), (3, 77)):
        rf, ru = ref.reconstruct(planes, pitch, w, h, t, m, win)
        of = oracle.reconstruct(planes, w, h, t, pitch, m, win, dtype=np.float64)
        ou = oracle.reconstruct(planes, w, h, t, pitch, m, win, dtype=np.uint8)
        assert np.array_equal(rf.view(np.uint64), of.view(np.uint64)), (m, win)
        assert np.array_equal(ru, ou), (m, win)


def test_streaming_equals_batch_any_blocking(oracle):
    """acceptance.cpp:116-138 on 300 streams: oracle events == reference events."""
    ref = Reference()
    rng = np.random.default_rng(1009)
    for _ in range(300):
        t = int(rng.integers(64, 513))
        b = (rng.random(t) < rng.uniform(0.05, 0.8)).astype(np.uint8)
        d, v = oracle.fsr_events(b)
        for blk in (1 << 30, 32, 7):
            rd, rv = ref.stream_events(b, blk)
            assert np.array_equal(d, rd) and np.array_equal(v, rv)
