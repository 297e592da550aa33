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

Time shards (configs[4]: one long stream cut in frame ranges, one per
rank) are below (`TimeShard`, `reconstruct_time_sharded`,
`reconstruct_time_sharded_dist`).  A halo alone is not exact -- a run's set
of accepted intervals depends on its whole history (reconstruct.cpp:17-36)
-- so every shard is scanned speculatively from a fresh state and the true
boundary state is resolved exactly (csrc/shard.cu).
"""
from __future__ import annotations

import torch
import torch.distributed as dist

from .recon import Method, PackedVolume, reconstruct

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
    if _staged(group) and local.is_cuda:  # gloo: through the host
        flat_h = torch.empty((world * t, bmax), dtype=local.dtype)
        dist.all_gather_into_tensor(flat_h, local.contiguous().cpu(), group=group)
        flat = flat_h.to(local.device)
    else:
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


def reconstruct_devices(volume: PackedVolume, method, devices: list[int],
                        out: torch.Tensor | None = None, dtype: torch.dtype = torch.uint8):
    """One process, several GPUs (the `workers` of reconstruct()): pixel band
    i is copied to devices[i], reconstructed there on its own stream and its
    columns copied back into `out` on the volume's device."""
    home = volume.planes.device
    npix, t = volume.npix, volume.frames
    if out is None:
        out = torch.empty((t, npix), dtype=dtype, device=home)
    bands = pixel_bands(npix, len(devices))
    pending = []
    for (p0, p1), d in zip(bands, devices):
        if p1 <= p0:
            continue
        dev = torch.device("cuda", d)
        s = torch.cuda.Stream(dev)
        with torch.cuda.device(dev), torch.cuda.stream(s):
            view = band_view(volume, p0, p1)
            bv = PackedVolume(view.width, 1, t, view.planes.to(dev, non_blocking=True))
            frames = reconstruct(bv, method, out=torch.empty((t, p1 - p0), dtype=out.dtype, device=dev),
                                 stream=s)
        pending.append((p0, p1, frames.reshape(t, p1 - p0), s))
    for p0, p1, frames, s in pending:
        s.synchronize()
        out[:, p0:p1].copy_(frames.to(home))
    return out.view(t, volume.height, volume.width) if out.shape[1] == npix else out


# ------------------------------------------------------------ time shards --
# One long stream cut in frame ranges (BASELINE configs[4]): exact, see
# csrc/shard.cu and DESIGN.md "Time sharding".  `TimeShard` holds one shard's
# device buffers; the driver below runs all shards of a volume in one process
# (one GPU); reconstruct_time_sharded_dist runs one shard per rank.

STATE_FIELDS = 17
SYNC_DT = 4   # spk_sync: 4 x int32
CLOSE_DT = 8  # spk_close: 8 x int32


def _ptr(t):
    return t.data_ptr() if t is not None else None


class TimeShard:
    """Frames [f0, f1) of a volume: speculative scan, then resolve / junction /
    stitch / expand through the C-ABI -- all asynchronous on `stream` (every
    torch allocation and reduction below runs on that stream too).

    Fast pass (robust=False): no host synchronisation.  The speculative run
    lists get a fixed capacity and the resolve no fallback re-scan; either
    overflowing (noise-like pixels) only sets the device flag `overflow`, and
    the driver re-runs the protocol robustly when any shard's flag is set --
    one host check after the whole pass.  Robust pass: capacities grown and
    fallback scans taken as needed (host checks between the launches)."""

    def __init__(self, volume: PackedVolume, f0: int, f1: int, method, prefix_cap: int = 64,
                 stream=None, robust: bool = False):
        from .recon import _method, _stream
        from . import _capi as capi
        self.capi, self.lib = capi, capi.lib()
        m = _method(method)
        if m.kind not in (Method.fsr, Method.ssr):
            raise ValueError("time sharding applies to fsr / ssr")
        self.kind = int(m.kind)
        self.vol = volume
        self.f0, self.f1 = f0, f1
        self.frames = f1 - f0
        self.npix = volume.npix
        self.dev = volume.planes.device
        self.planes = volume.planes[f0:f1]
        self.stream = _stream(stream)
        self.ts = (torch.cuda.ExternalStream(self.stream, device=self.dev) if self.stream
                   else torch.cuda.current_stream(self.dev))
        self.robust = robust
        self.pcap = int(prefix_cap)
        self.g = capi.geom(volume.width, volume.height, self.frames, volume.pitch)
        i32 = dict(dtype=torch.int32, device=self.dev)
        with torch.cuda.stream(self.ts):
            self.prefix = torch.empty((self.npix, self.pcap, 2), **i32)
            self.sync = torch.empty((self.npix, SYNC_DT), **i32)
            self.tstate = torch.empty((STATE_FIELDS, self.npix), **i32)
            self.exit_state = torch.empty((STATE_FIELDS, self.npix), **i32)
            self.entry_close = torch.empty((self.npix, CLOSE_DT), **i32)
            self.tail_close = torch.empty((self.npix, CLOSE_DT), **i32)
            self.overflow = torch.zeros((), dtype=torch.bool, device=self.dev)
        self.fb = self.fb_counts = self.fb_state = None

    def _segment(self, state_in):
        """runs of this shard from `state_in` (None = fresh); robust: the
        capacity grows until no pixel overflows, else overflow is flagged"""
        cap = max(64, self.frames // 64)
        i32 = dict(dtype=torch.int32, device=self.dev)
        while True:
            runs = torch.empty((self.npix, cap, 2), **i32)
            counts = torch.empty((self.npix,), **i32)
            last = torch.empty((self.npix,), **i32)
            state = torch.empty((STATE_FIELDS, self.npix), **i32)
            self.capi.check(self.lib.spk_segment_state(
                self.g, _ptr(self.planes) if self.frames else None, self.kind, _ptr(runs), cap,
                _ptr(counts), _ptr(last), _ptr(state_in), _ptr(state), self.stream))
            if not self.robust:
                if self.npix:
                    self.overflow |= counts.max() > cap
                return runs, counts, last, state, cap
            need = int(counts.max().item()) if self.npix else 0
            if need <= cap:
                return runs, counts, last, state, cap
            cap = need

    def speculate(self):
        with torch.cuda.stream(self.ts):
            self.spec, self.spec_counts, _, self.spec_state, self.scap = self._segment(None)

    def fresh_entry(self) -> torch.Tensor:
        """entry state of the first shard (start of the stream)"""
        return fresh_state(self.npix, self.dev, self.stream)

    def resolve(self, entry: torch.Tensor):
        """true entry state -> sync records, exit state, entry / tail closes"""
        with torch.cuda.stream(self.ts):
            return self._resolve(entry)

    def _resolve(self, entry):
        self.entry = entry
        self.capi.check(self.lib.spk_shard_resolve(
            self.g, _ptr(self.planes) if self.frames else None, self.kind, _ptr(entry),
            _ptr(self.spec), self.scap, _ptr(self.spec_counts), _ptr(self.spec_state),
            _ptr(self.prefix), self.pcap, _ptr(self.sync), _ptr(self.tstate), self.stream))
        if not self.robust:
            if self.npix:
                self.overflow |= (self.sync[:, 3] == -1).any()  # a prefix overflowed
        elif bool((self.sync[:, 3] == -1).any().item()):  # a prefix overflowed: full re-scan
            self.fb, self.fb_counts, _, self.fb_state, fbcap = self._segment(entry)
            if fbcap != self.scap:  # keep one capacity for both lists
                pad = torch.empty((self.npix, max(fbcap, self.scap), 2), dtype=torch.int32,
                                  device=self.dev)
                if fbcap < self.scap:
                    pad[:, :fbcap] = self.fb
                    self.fb = pad
                else:
                    pad[:, :self.scap] = self.spec
                    self.spec = pad
                    self.scap = fbcap
        self.capi.check(self.lib.spk_shard_junction(
            self.g, self.kind, _ptr(entry), _ptr(self.sync), _ptr(self.prefix), self.pcap,
            _ptr(self.tstate), _ptr(self.spec), self.scap, _ptr(self.spec_counts),
            _ptr(self.spec_state), _ptr(self.fb), _ptr(self.fb_counts), _ptr(self.fb_state),
            _ptr(self.exit_state), _ptr(self.entry_close), _ptr(self.tail_close), self.stream))
        return self.exit_state

    def close_from_next(self, entry_close_next, close_next):
        with torch.cuda.stream(self.ts):
            close = torch.empty((self.npix, CLOSE_DT), dtype=torch.int32, device=self.dev)
        self.capi.check(self.lib.spk_shard_close_chain(
            self.npix, _ptr(entry_close_next), _ptr(close_next), self.frames, _ptr(close),
            self.stream))
        return close

    def stitch(self, close: torch.Tensor):
        rcap = self.scap + self.pcap + 1
        i32 = dict(dtype=torch.int32, device=self.dev)
        with torch.cuda.stream(self.ts):
            self.region = torch.empty((self.npix, rcap, 2), **i32)
            self.region_counts = torch.empty((self.npix,), **i32)
            self.region_last = torch.empty((self.npix,), **i32)
        self.rcap = rcap
        self.capi.check(self.lib.spk_shard_stitch(
            self.g, self.kind, _ptr(self.entry), _ptr(self.sync), _ptr(self.prefix), self.pcap,
            _ptr(self.tstate), _ptr(self.spec), self.scap, _ptr(self.spec_counts),
            _ptr(self.spec_state), _ptr(self.fb), _ptr(self.fb_counts), _ptr(self.fb_state),
            _ptr(close), _ptr(self.region), rcap, _ptr(self.region_counts),
            _ptr(self.region_last), self.stream))

    def expand(self, out: torch.Tensor):
        """this shard's frames into `out` ([frames, >= W*H], row-major)"""
        fn = {torch.uint8: "spk_expand_runs_u8", torch.float32: "spk_expand_runs_f32",
              torch.float64: "spk_expand_runs_f64"}[out.dtype]
        g = self.capi.geom(self.vol.width, self.vol.height, self.frames, 0)
        self.capi.check(getattr(self.lib, fn)(
            g, _ptr(self.region), self.rcap, _ptr(self.region_counts), _ptr(self.region_last),
            _ptr(out), out.stride(0), self.stream))


def fresh_state(npix: int, device, stream=None) -> torch.Tensor:
    from .recon import _stream
    from . import _capi as capi
    st = torch.empty((STATE_FIELDS, npix), dtype=torch.int32, device=device)
    capi.check(capi.lib().spk_state_fresh(npix, st.data_ptr(), _stream(stream)))
    return st


def time_bounds(frames: int, nshards: int) -> list[int]:
    """[0 = a_0 < a_1 < ... < a_K = frames], shard lengths multiples of 32 frames"""
    words = (frames + 31) // 32
    b = [min(frames, (words * r // nshards) * 32) for r in range(nshards + 1)]
    b[-1] = frames
    return sorted(set(b))


def reconstruct_time_sharded(volume: PackedVolume, method="fsr", nshards: int = 2,
                             bounds: list[int] | None = None, dtype: torch.dtype = torch.uint8,
                             prefix_cap: int = 64, out: torch.Tensor | None = None, stream=None):
    """reconstruct() of one volume cut into time shards processed independently
    (one GPU, all shards in this process); bit-identical to reconstruct().
    The fast pass issues every launch without a host synchronisation; one
    check at the end decides whether the robust pass must redo it."""
    bounds = bounds or time_bounds(volume.frames, nshards)
    if bounds[0] != 0 or bounds[-1] != volume.frames or any(b1 <= b0 for b0, b1 in zip(bounds, bounds[1:])):
        raise ValueError("bounds must increase strictly from 0 to the frame count")
    if out is None:
        out = torch.empty((volume.frames, volume.npix), dtype=dtype, device=volume.planes.device)
    with torch.cuda.device(volume.planes.device):
        shards = _time_sharded_pass(volume, method, bounds, prefix_cap, out, stream, robust=False)
        if bool(torch.stack([sh.overflow for sh in shards]).any().item()):
            _time_sharded_pass(volume, method, bounds, prefix_cap, out, stream, robust=True)
    return out.view(volume.frames, volume.height, volume.width)


def _time_sharded_pass(volume, method, bounds, prefix_cap, out, stream, robust):
    shards = [TimeShard(volume, b0, b1, method, prefix_cap, stream, robust)
              for b0, b1 in zip(bounds, bounds[1:])]
    for sh in shards:                      # independent: the speculative scans
        sh.speculate()
    entry = fresh_state(volume.npix, volume.planes.device, stream)
    for sh in shards:                      # forward: true entry states
        entry = sh.resolve(entry)
    closes = [None] * len(shards)          # backward: closes of crossing runs
    closes[-1] = shards[-1].tail_close
    for r in range(len(shards) - 2, -1, -1):
        closes[r] = shards[r].close_from_next(shards[r + 1].entry_close, closes[r + 1])
    for sh, c in zip(shards, closes):      # independent: stitch + frames
        sh.stitch(c)
        sh.expand(out[sh.f0:sh.f1])
    return shards


def _staged(group):
    """gloo moves host tensors: device tensors are staged through the host"""
    return dist.get_backend(group) == "gloo"


def _send(t: torch.Tensor, dst: int, group):
    if _staged(group) and t.is_cuda:
        t = t.cpu()
    dist.send(t, dst=dst, group=group)


def _recv(t: torch.Tensor, src: int, group):
    if _staged(group) and t.is_cuda:
        h = torch.empty(t.shape, dtype=t.dtype)
        dist.recv(h, src=src, group=group)
        t.copy_(h)
    else:
        dist.recv(t, src=src, group=group)


def reconstruct_time_sharded_dist(shard: PackedVolume, method="fsr", group=None,
                                  dtype: torch.dtype = torch.uint8, prefix_cap: int = 64,
                                  out: torch.Tensor | None = None, stream=None,
                                  shard_type=TimeShard):
    """One time shard per rank (rank r holds frames [a_r, a_{r+1}) of the
    stream as `shard`, ranks in time order): returns this rank's frames,
    identical to the same frames of a single-pass reconstruct().

    Data path: none; the only exchange is O(W*H) per boundary -- the true
    automaton state forward (rank r -> r+1, 68 B/px) and the close records of
    boundary-crossing runs backward (rank r+1 -> r, 2 x 32 B/px).  NCCL moves
    device tensors; gloo (several ranks sharing one GPU, tests) stages them
    through the host.  The fast pass has no host synchronisation of its own;
    one all-reduce of the ranks' overflow flags at the end decides whether
    the robust pass must redo it."""
    rank, world = _group_info(group)
    if out is None:
        out = torch.empty((shard.frames, shard.npix), dtype=dtype, device=shard.planes.device)
    sh = _time_shard_dist_pass(shard, method, group, prefix_cap, out, stream, shard_type, False)
    flag = getattr(sh, "overflow", None)
    if flag is not None and world > 1:
        f = flag.to(torch.int32).reshape(1)
        if _staged(group):
            f = f.cpu()
        dist.all_reduce(f, op=dist.ReduceOp.MAX, group=group)
        flag = f
    if flag is not None and bool(flag.any().item()):
        _time_shard_dist_pass(shard, method, group, prefix_cap, out, stream, shard_type, True)
    return out


def _time_shard_dist_pass(shard, method, group, prefix_cap, out, stream, shard_type, robust):
    rank, world = _group_info(group)
    peer = (lambda r: dist.get_global_rank(group, r)) if group is not None else (lambda r: r)
    if shard_type is TimeShard:
        sh = TimeShard(shard, 0, shard.frames, method, prefix_cap, stream, robust)
    else:
        sh = shard_type(shard, 0, shard.frames, method, prefix_cap, stream)
    ts = getattr(sh, "ts", None)
    if ts is None:  # (test doubles without a device stream)
        return _time_shard_dist_steps(sh, shard, group, rank, world, peer, out)
    with torch.cuda.stream(ts):  # the collectives order against the shard's stream
        return _time_shard_dist_steps(sh, shard, group, rank, world, peer, out)


def _time_shard_dist_steps(sh, shard, group, rank, world, peer, out):
    dev = shard.planes.device
    sh.speculate()                              # independent on every rank
    if rank == 0:
        entry = sh.fresh_entry()
    else:                                       # forward: true entry state
        entry = torch.empty((STATE_FIELDS, shard.npix), dtype=torch.int32, device=dev)
        _recv(entry, peer(rank - 1), group)
    exit_state = sh.resolve(entry)
    if rank + 1 < world:
        _send(exit_state, peer(rank + 1), group)
    if rank + 1 == world:                       # backward: closes of crossing runs
        close = sh.tail_close
    else:
        ec_next = torch.empty((shard.npix, CLOSE_DT), dtype=torch.int32, device=dev)
        close_next = torch.empty_like(ec_next)
        _recv(ec_next, peer(rank + 1), group)
        _recv(close_next, peer(rank + 1), group)
        close = sh.close_from_next(ec_next, close_next)
    if rank > 0:
        _send(sh.entry_close, peer(rank - 1), group)
        _send(close, peer(rank - 1), group)
    sh.stitch(close)                            # independent: stitch + frames
    sh.expand(out)
    return sh
