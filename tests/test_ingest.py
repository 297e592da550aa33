"""Ingest pipeline: host payloads -> pitched device
planes -> frames -> host, pipelined over volumes (spk_reconstruct_host_batch).
Bar: every volume's frames identical to its own single host call and to the
oracle."""
from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("geom", [(400, 25, 3000), (37, 11, 1500), (9, 1, 700)])
@pytest.mark.parametrize("method", ["fsr", "ssr", "tfi", "tfp"])
def test_batch_equals_single_calls(oracle, geom, method):
    import paper_2412_11639_b200 as spk
    w, h, t = geom
    pays = [spk.synth(sc, k, w, h, t, param=0.3, device="cuda").payload()
            for k, sc in enumerate(["moving", "static", "noise", "range", "sensor"])]
    outs = spk.reconstruct_host_batch(pays, w, h, t, method)
    for p, o in zip(pays, outs):
        ref = spk.reconstruct_host(p, w, h, t, method)
        assert np.array_equal(o, ref), method
    # and the oracle on the first volume
    fb = (w * h + 7) // 8
    planes = pays[0].reshape(t, fb)
    m = {"fsr": 0, "ssr": 1, "tfi": 2, "tfp": 3}[method]
    assert np.array_equal(outs[0], oracle.reconstruct(planes, w, h, t, fb, m))


def test_batch_f64_and_edges():
    import paper_2412_11639_b200 as spk
    w, h, t = 50, 3, 1200
    pays = [spk.synth("moving", k, w, h, t, device="cuda").payload() for k in range(3)]
    outs = spk.reconstruct_host_batch(pays, w, h, t, "fsr", dtype=np.float64)
    for p, o in zip(pays, outs):
        assert np.array_equal(o.view(np.int64), spk.reconstruct_host(p, w, h, t, "fsr", dtype=np.float64).view(np.int64))
    assert spk.reconstruct_host_batch([], w, h, t, "fsr") == []
    with pytest.raises(ValueError):
        spk.reconstruct_host_batch(pays, w, h, t, "fsr", outs=[np.empty((t, w * h), np.uint8)])
