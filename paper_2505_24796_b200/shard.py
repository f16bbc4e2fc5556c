"""Multi-GPU partitioning of the render path.

One process per GPU (torchrun), NCCL over NVLink for the only exchange step.
The reference renders one frame on one CPU thread (src/tilesplat/raster.py:
177-193); its tiles are independent, which is what both modes
below exploit:

* **views** -- a batch of cameras is split into contiguous blocks, one per
  rank.  Every rank holds a full replica of the scene and renders its own
  views; there is no collective on the data path (weak scaling).
* **tile bands** -- one huge frame (config 3, 3840x2160) is split into
  contiguous tile-row bands.  Every rank runs the replicated, band-agnostic
  K1 preprocess in geometry-only mode (no SH read), reads the per-tile-row
  splat counts (``tcgs_tile_row_counts``) and computes the SAME
  prefix-balanced partition locally (no communication), evaluates the SH
  colour of only the Gaussians that reach its band (``tcgs_colour``), then
  bins and blends its band.  The frame reaches rank 0 through NVLink peer
  memory (K7 writes into rank 0's frame) or one grouped NCCL send/recv
  (``gather_bands``); the fragment counters are summed with one tiny
  all-reduce.

The partition/gather helpers are plain torch.distributed code, so they are
covered on CPU with the gloo backend (tests/test_shard.py); the render itself
needs the B200.
"""

from __future__ import annotations

from dataclasses import dataclass

import ctypes

import numpy as np
import torch
import torch.distributed as dist

from . import _abi
from .raster import FragmentStats, Frame, GaussianCloud, Renderer, camera_struct

TILE = 16


def view_blocks(n_views: int, world: int) -> list[tuple[int, int]]:
    """Contiguous [begin, end) view ranges, one per rank; sizes differ by at most one."""
    if n_views < 0 or world < 1:
        raise ValueError("n_views must be >= 0 and world >= 1")
    base, extra = divmod(n_views, world)
    out, b = [], 0
    for r in range(world):
        e = b + base + (1 if r < extra else 0)
        out.append((b, e))
        b = e
    return out


def band_partition(row_counts, world: int, min_rows: int = 1) -> list[tuple[int, int]]:
    """Prefix-balanced contiguous tile-row bands [y0, y1) for ``world`` ranks.

    ``row_counts[y]`` is the splat count of tile row y (a proxy for K7 work).
    Every rank calls this on identical replicated counts, so every rank gets
    the identical partition with no communication.  Band r ends at the first
    row where the prefix reaches (r+1)/world of the total, keeping at least
    ``min_rows`` rows per band; bands cover every row exactly once.
    """
    c = np.asarray(row_counts, dtype=np.float64).reshape(-1)
    rows = int(c.shape[0])
    if world < 1:
        raise ValueError("world must be >= 1")
    if rows < world * min_rows:
        raise ValueError(f"{rows} tile rows cannot be split into {world} bands of >= {min_rows} rows")
    # +1 per row so empty rows still carry the per-tile fixed cost and the split is well defined
    w = c + 1.0
    pre = np.concatenate([[0.0], np.cumsum(w)])
    total = pre[-1]
    bounds = [0]
    for r in range(1, world):
        target = total * r / world
        y = int(np.searchsorted(pre, target, side="left"))
        # y is the first boundary whose prefix >= target; pick the closer of y-1 / y
        if y > 0 and abs(pre[y - 1] - target) <= abs(pre[min(y, rows)] - target):
            y -= 1
        lo = bounds[-1] + min_rows
        hi = rows - (world - r) * min_rows
        bounds.append(int(min(max(y, lo), hi)))
    bounds.append(rows)
    return [(bounds[r], bounds[r + 1]) for r in range(world)]


def band_pixel_rows(band: tuple[int, int], height: int) -> tuple[int, int]:
    """Image rows [r0, r1) covered by tile rows [y0, y1)."""
    return band[0] * TILE, min(band[1] * TILE, height)


def gather_bands(parts: list[torch.Tensor], full: list[torch.Tensor] | None, bands: list[tuple[int, int]],
                 height: int, group=None, dst: int = 0) -> None:
    """Assemble per-rank band slices into full frames on rank ``dst`` with ONE grouped send/recv.

    ``parts[i]`` is this rank's full-frame-shaped output i ([H, ...]); only its
    band rows are sent.  On ``dst``, ``full[i]`` receives every other rank's
    rows in place (its own rows are copied locally).  Bands are contiguous row
    ranges of row-major [H, W, ...] tensors, so each transfer is one
    contiguous message (NCCL: ncclGroupStart / ncclSend|ncclRecv x (G-1) /
    ncclGroupEnd through ``batch_isend_irecv``).
    """
    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    ops = []
    if rank == dst:
        if full is None or len(full) != len(parts):
            raise ValueError("rank dst needs one full-frame tensor per part")
        for i, p in enumerate(parts):
            r0, r1 = band_pixel_rows(bands[dst], height)
            if full[i].data_ptr() != p.data_ptr():
                full[i][r0:r1].copy_(p[r0:r1])
        for src in range(world):
            if src == dst:
                continue
            r0, r1 = band_pixel_rows(bands[src], height)
            if r1 <= r0:
                continue
            for i in range(len(parts)):
                ops.append(dist.P2POp(dist.irecv, full[i][r0:r1], dist.get_global_rank(group, src)
                                      if group is not None else src, group))
    else:
        r0, r1 = band_pixel_rows(bands[rank], height)
        if r1 > r0:
            for p in parts:
                ops.append(dist.P2POp(dist.isend, p[r0:r1].contiguous(), dist.get_global_rank(group, dst)
                                      if group is not None else dst, group))
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()


_SUMMED = ("f_blend", "f_cull", "f_skip", "n_splats", "pixels_terminated", "exp_calls")


def reduce_stats(st: FragmentStats, device, group=None) -> FragmentStats:
    """Whole-frame FragmentStats from per-band ones: band counters add; ``dropped`` and
    ``n_visible`` come from the replicated K1 and are identical on every rank."""
    t = torch.tensor([getattr(st, k) for k in _SUMMED], dtype=torch.int64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    vals = dict(zip(_SUMMED, (int(x) for x in t.tolist())))
    return FragmentStats(dropped=st.dropped, n_visible=st.n_visible, stage_ms=dict(st.stage_ms), **vals)


@dataclass
class BandFrame:
    band: tuple[int, int]
    bands: list[tuple[int, int]]
    local: Frame                 # this rank's full-size buffers (only band rows written)
    rgb: torch.Tensor | None     # assembled frame on rank 0, else None
    T: torch.Tensor | None
    n_contrib: torch.Tensor | None
    stats: FragmentStats | None  # whole-frame stats (all ranks)


class _CudaArray:
    """``__cuda_array_interface__`` view of raw device memory (wrapped by torch.as_tensor, not owned)."""

    def __init__(self, ptr: int, shape: tuple, typestr: str):
        self.__cuda_array_interface__ = {"shape": shape, "typestr": typestr, "data": (ptr, False), "version": 3,
                                         "strides": None}


class PeerFrame:
    """Rank 0's full-frame outputs (rgb [H,W,3] f32, T [H,W] f32, n_contrib [H,W] i32), double-buffered in one
    allocation, mapped into every rank of ``group`` with CUDA IPC (NVLink peer memory between GPUs of one box).

    Every rank passes a slot's tensors as K7's outputs: K7 stores the pixels of its tile-row band straight
    into rank 0's frame, tile by tile, so the band gather disappears.

    Ordering.  Frame k uses slot k % 2.  Rank 0 may read frame k (for example an async D2H on its current
    stream) until it enqueues frame k + 1's completion all-reduce; every other rank's K7 of frame k + 2 -- the
    next writer of that slot -- is stream-ordered after that all-reduce.  So a frame returned to rank 0 stays
    intact while rank 0 consumes it on its current stream (or synchronously) before rendering frame k + 2.
    """

    SLOTS = 2

    def __init__(self, lib, W: int, H: int, device, group=None):
        self.lib, self.group = lib, group
        self.rank = dist.get_rank(group)
        n = W * H
        self.slot_bytes = 20 * n  # 12 n (rgb) + 4 n (T) + 4 n (n_contrib)
        self.nbytes = self.SLOTS * self.slot_bytes
        handle = None
        with torch.cuda.device(device):
            if self.rank == 0:
                p = ctypes.c_void_p()
                _abi.check(lib.tcgs_frame_alloc(self.nbytes, ctypes.byref(p)), "tcgs_frame_alloc")
                self.ptr = p.value
                h = ctypes.create_string_buffer(_abi.IPC_HANDLE_BYTES)
                _abi.check(lib.tcgs_ipc_get_handle(ctypes.c_void_p(self.ptr), h), "tcgs_ipc_get_handle")
                handle = h.raw
            box = [handle]
            dist.broadcast_object_list(box, src=dist.get_global_rank(group, 0) if group is not None else 0,
                                       group=group)
            if self.rank != 0:
                p = ctypes.c_void_p()
                _abi.check(lib.tcgs_ipc_open(ctypes.create_string_buffer(box[0], _abi.IPC_HANDLE_BYTES),
                                             ctypes.byref(p)), "tcgs_ipc_open")
                self.ptr = p.value
            dev = torch.device(device)
            self.slots = []
            for k in range(self.SLOTS):
                base = self.ptr + k * self.slot_bytes
                self.slots.append((torch.as_tensor(_CudaArray(base, (H, W, 3), "<f4"), device=dev),
                                   torch.as_tensor(_CudaArray(base + 12 * n, (H, W), "<f4"), device=dev),
                                   torch.as_tensor(_CudaArray(base + 16 * n, (H, W), "<i4"), device=dev)))
            if self.rank == 0:
                for rgb, T, cnt in self.slots:
                    rgb.zero_()
                    T.fill_(1.0)
                    cnt.zero_()
                torch.cuda.synchronize(dev)
        dist.barrier(group)

    def slot(self, k: int):
        """(rgb, T, n_contrib) of frame k's slot."""
        return self.slots[k % self.SLOTS]

    def close(self):
        dist.barrier(self.group)
        if self.rank == 0:
            self.lib.tcgs_frame_free(ctypes.c_void_p(self.ptr))
        else:
            self.lib.tcgs_ipc_close(ctypes.c_void_p(self.ptr))


class BandRenderer:
    """Renders one frame split into tile-row bands across the ranks of ``group``.

    Per frame: K1 (replicated) -> tile-row counts (one 8*tiles_y-byte D2H) -> local partition ->
    K2-K6 + K7 on the band -> the frame on rank 0, either by one NCCL gather (``output="gather"``)
    or written there directly by every rank's K7 through CUDA IPC peer mappings (``output="peer"``,
    completion signalled by one tiny all-reduce / barrier).
    """

    def __init__(self, device, backend="tcgs", group=None, gather_extras: bool = True, output: str = "gather"):
        if output not in ("gather", "peer"):
            raise ValueError("output must be 'gather' or 'peer'")
        self.r = Renderer(device, backend)
        self.device = self.r.device
        self.group = group
        self.gather_extras = gather_extras
        self.output = output
        self._full = {}
        self._peer = {}
        self._rows = None
        self._flag = None
        self._frames = 0  # frames rendered: selects the peer frame's slot (the same on every rank)

    def peer_frame(self, W: int, H: int) -> PeerFrame:
        if (W, H) not in self._peer:
            self._peer[(W, H)] = PeerFrame(self.r.lib, W, H, self.device, self.group)
        return self._peer[(W, H)]

    def close(self):
        for pf in self._peer.values():
            pf.close()
        self._peer = {}

    def _complete(self):
        """Rank 0 may use the frame once every rank's K7 has finished writing into it."""
        if dist.get_backend(self.group) == "nccl":
            if self._flag is None:
                self._flag = torch.zeros(1, dtype=torch.int32, device=self.device)
            dist.all_reduce(self._flag, group=self.group)  # ordered after K7 on every rank's stream
        else:
            torch.cuda.synchronize(self.device)
            dist.barrier(self.group)

    def partition(self, cloud: GaussianCloud, cam) -> list[tuple[int, int]]:
        c = camera_struct(cam)
        tiles_y = (c.height + TILE - 1) // TILE
        if self._rows is None or self._rows.numel() < tiles_y:
            self._rows = torch.empty(tiles_y, dtype=torch.int64, device=self.device)
        st = torch.cuda.current_stream(self.device).cuda_stream
        _abi.check(self.r.lib.tcgs_tile_row_counts(self.r.ws.data_ptr(), cloud.P, c, self.r.max_splats,
                                                   self._rows.data_ptr(), st), "tcgs_tile_row_counts")
        counts = self._rows[:tiles_y].cpu().numpy()
        return band_partition(counts, dist.get_world_size(self.group))

    def full_buffers(self, W: int, H: int):
        key = (W, H)
        if key not in self._full:
            self._full[key] = (torch.zeros((H, W, 3), dtype=torch.float32, device=self.device),
                               torch.ones((H, W), dtype=torch.float32, device=self.device),
                               torch.zeros((H, W), dtype=torch.int32, device=self.device))
        return self._full[key]

    def render(self, cloud: GaussianCloud, cam, with_stats: bool = True, timers=None) -> BandFrame:
        """One frame: ``timers`` (5 CUDA events) bracket K1 | partition + K2-K6 | K7 | gather.  With peer output,
        rank 0's returned tensors are valid until it renders the frame after next (see ``PeerFrame``)."""
        rank = dist.get_rank(self.group)
        ev = timers
        with torch.cuda.device(self.device):
            if ev:
                ev[0].record()
            # several ranks: geometry for every Gaussian (no SH read), then SH only for the Gaussians that reach
            # this rank's band; one rank: K1's own staged colour (its band is the whole frame)
            defer = dist.get_world_size(self.group) > 1
            self.r.preprocess(cloud, cam, defer_colour=defer)
            if ev:
                ev[1].record()
            bands = self.partition(cloud, cam)
            band = bands[rank]
            if defer:
                self.r.colour(cloud, cam, band)
            c = camera_struct(cam)
            outs = None
            if self.output == "peer":
                pf = self.peer_frame(c.width, c.height)
                outs = pf.slot(self._frames)
            self._frames += 1
            if with_stats:
                frame = self.r.finish(cloud, cam, band, with_stats=True, outputs=outs)
            else:
                rgb, T, cnt = self.r.bin_blend(cloud, cam, band, outputs=outs, timers=ev)
                frame = Frame(rgb, T, cnt, None)
            H, W = frame.rgb.shape[0], frame.rgb.shape[1]
            parts = [frame.rgb, frame.T, frame.n_contrib] if self.gather_extras else [frame.rgb]
            if self.output == "peer":
                self._complete()
                full = parts if rank == 0 else None
            else:
                full = list(self.full_buffers(W, H))[:len(parts)] if rank == 0 else None
                gather_bands(parts, full, bands, H, self.group)
            if ev:
                ev[4].record()
            stats = reduce_stats(frame.stats, self.device, self.group) if with_stats else None
        if rank == 0:
            f = full + [None] * (3 - len(full))
            return BandFrame(band, bands, frame, f[0], f[1], f[2], stats)
        return BandFrame(band, bands, frame, None, None, None, stats)
