"""Host-side mirror of the reference API: method parsing, formats, file errors."""
import numpy as np
import pytest

from paper_2412_11639_b200 import IoError, Method, ReconMethod, plane_bytes, plane_pitch, read_raw, read_spk


def test_recon_method_parse_and_name():
    """ReconMethod::parse / name (reconstruct.cpp:177-196, test_reconstruct.cpp:269-272)."""
    assert ReconMethod.parse("fsr").kind == Method.fsr
    assert ReconMethod.parse("ssr").name() == "ssr"
    assert ReconMethod.parse("tfp", 16).name() == "tfp-16"
    assert ReconMethod().tfp_window == 32
    with pytest.raises(ValueError):
        ReconMethod.parse("magic")
    with pytest.raises(ValueError):
        ReconMethod.parse("tfp", 0)


def test_plane_geometry():
    assert plane_bytes(400, 250) == 12500 and plane_bytes(9, 1) == 2
    assert plane_pitch(400, 250) % 16 == 0 and plane_pitch(400, 250) >= 12500


def test_read_spk_errors(tmp_path):
    """test_io.cpp:76-98: bad magic and truncation messages."""
    bad = tmp_path / "bad.spk"
    bad.write_bytes(b"NOPE" + bytes(12))
    with pytest.raises(IoError, match="magic"):
        read_spk(bad)
    trunc = tmp_path / "trunc.spk"
    head = b"SPK1" + (4).to_bytes(2, "little") + (4).to_bytes(2, "little") + \
        (20000).to_bytes(4, "little") + (2).to_bytes(4, "little")
    trunc.write_bytes(head + bytes(3))  # 4x4 -> 2 B/frame, 2 frames -> 20 B expected
    with pytest.raises(IoError, match=r"expected 20 bytes, got 19"):
        read_spk(trunc)
    with pytest.raises(IoError, match="cannot open"):
        read_spk(tmp_path / "missing.spk")


def test_read_raw_size_check(tmp_path):
    """test_io.cpp:100-110: frame count from the file size, else io_error."""
    f = tmp_path / "dump.raw"
    f.write_bytes(bytes(12501))
    with pytest.raises(IoError, match="not a multiple"):
        read_raw(f, 400, 250)
