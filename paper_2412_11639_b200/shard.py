"""Multi-GPU reconstruction by pixel bands ("Pixels").

Every pixel's frames depend only on that pixel's own stream -- the
reference's parallel split is a pixel range per OpenMP thread
(proj/src/reconstruct.cpp:456-466, output "identical for any worker count",
reconstruct.hpp:70-72).  So the multi-GPU form gives each rank (one process
per GPU) a contiguous pixel band and needs no exchange on the data path; the
only collective is the optional gather of the finished frames.

Bands start on 128-pixel boundaries: the band's bit-planes are then a
zero-copy view of the full planes (byte offset p0/8, same pitch, 16-B
aligned) and its output columns stay 16-B aligned for the vector stores.
A band is handed to the C-ABI as a (p1-p0) x 1 volume.

Time sharding (needed only when one stream's planes exceed a GPU; C5's
12.5 GB fits in 180 GB) is not exact with a halo alone -- a run's set of
accepted intervals depends on its whole history (reconstruct.cpp:17-36) --
and is documented in DESIGN.md, not implemented.
"""
from __future__ import annotations

import torch
import torch.distributed as dist

from .recon import PackedVolume, reconstruct

BAND_ALIGN = 128


def pixel_bands(npix: int, world: int, align: int = BAND_ALIGN) -> list[tuple[int, int]]:
    """Contiguous [p0, p1) pixel bands, one per rank, starts aligned to `align`,
    sizes as equal as the alignment allows (ranks past the end get empty bands)."""
    if world < 1:
        raise ValueError("world must be >= 1")
    units = (npix + align - 1) // align
    bands = []
    for r in range(world):
        u0 = units * r // world
        u1 = units * (r + 1) // world
        bands.append((min(npix, u0 * align), min(npix, u1 * align)))
    return bands


def band_view(volume: PackedVolume, p0: int, p1: int) -> PackedVolume:
    """Pixels [p0, p1) of `volume` as a (p1-p0) x 1 volume sharing its planes."""
    if p0 % 32 or not 0 <= p0 < p1 <= volume.npix:
        raise ValueError(f"bad band [{p0}, {p1}) for {volume.npix} pixels")
    planes = volume.planes[:, p0 // 8: (p1 + 7) // 8]
    return PackedVolume(p1 - p0, 1, volume.frames, planes)


def _group_info(group) -> tuple[int, int]:
    if dist.is_available() and dist.is_initialized():
        return dist.get_rank(group), dist.get_world_size(group)
    return 0, 1


def reconstruct_band(volume: PackedVolume, method="fsr", rank: int = 0, world: int = 1,
                     dtype: torch.dtype = torch.uint8, out: torch.Tensor | None = None,
                     stream=None):
    """This rank's band: returns (p0, p1, frames [T, bmax]) where columns
    [0, p1-p0) hold pixels p0.. of every frame (bmax = the widest band, so
    the buffer is ready for an equal-size all-gather)."""
    bands = pixel_bands(volume.npix, world)
    p0, p1 = bands[rank]
    bmax = max(b1 - b0 for b0, b1 in bands)
    if out is None:
        out = torch.empty((volume.frames, bmax), dtype=dtype, device=volume.planes.device)
    if p1 > p0:
        reconstruct(band_view(volume, p0, p1), method, out=out, stream=stream)
    return p0, p1, out


def gather_bands(local: torch.Tensor, npix: int, group=None) -> torch.Tensor:
    """All-gather every rank's [T, bmax] band buffer and lay the bands out as
    full frames [T, npix] on every rank (one collective, then one copy per band)."""
    rank, world = _group_info(group)
    bands = pixel_bands(npix, world)
    if world == 1:
        return local[:, :npix].contiguous()
    t, bmax = local.shape
    flat = torch.empty((world * t, bmax), dtype=local.dtype, device=local.device)
    dist.all_gather_into_tensor(flat, local.contiguous(), group=group)
    stacked = flat.view(world, t, bmax)
    full = torch.empty((t, npix), dtype=local.dtype, device=local.device)
    for r, (p0, p1) in enumerate(bands):
        if p1 > p0:
            full[:, p0:p1] = stacked[r, :, : p1 - p0]
    return full


def reconstruct_sharded(volume: PackedVolume, method="fsr", group=None,
                        dtype: torch.dtype = torch.uint8, gather: bool = True, stream=None):
    """reconstruct() over every rank of `group`: each rank reconstructs its
    pixel band of `volume` (replicated or band-complete on every rank); with
    gather=True every rank returns the full [T, H, W] frames, identical to a
    single-GPU reconstruct(); otherwise (p0, p1, band frames)."""
    rank, world = _group_info(group)
    p0, p1, local = reconstruct_band(volume, method, rank, world, dtype, stream=stream)
    if not gather:
        return p0, p1, local[:, : p1 - p0]
    full = gather_bands(local, volume.npix, group)
    return full.view(volume.frames, volume.height, volume.width)
