"""spikecam-b200: B200-native FSR/SSR spike-camera reconstruction (arXiv 2412.11639).

The hot path -- bit-packed spike planes -> per-timestep frames -- runs in
hand-written sm_100a CUDA kernels behind a C-ABI (include/spikecam_b200.h,
libspikecam_b200.so).  This package is the Python host mirror of the
reference's C++ API (proj/include/spikecam/); torch supplies device memory,
streams and torch.distributed.  See DESIGN.md.
"""
from .recon import (  # noqa: F401
    DEFAULT_FPS,
    IoError,
    Method,
    PackedVolume,
    ReconMethod,
    plane_bytes,
    plane_pitch,
    read_raw,
    read_spk,
    reconstruct,
    reconstruct_batch,
    reconstruct_host,
    reconstruct_host_batch,
    reconstruct_host_multi,
    segments,
    synth,
    write_spk,
)
from .stream import EventStream  # noqa: F401
from .metrics import (  # noqa: F401
    compare, frame_metrics, mse, psnr, stability, two_dimensional_entropy, verify_stability)
from .records import RecordVolume, decode, read_spkr, records, records_host, write_spkr  # noqa: F401
from ._capi import LIB_PATH, SpikecamError  # noqa: F401

__version__ = "0.1.0"
