"""Patch scheduler: plan-shaped tiles over a large volume, 1..N GPUs
(reference: tiling.py:1-237).

Geometry is the reference's (tiling.py:83-162), restated: per axis the input
patch p, the network shrinkage m = p - o and an input overlap v >= m with
(v - m) even; tiles step by p - v, interior seams trim (v - m)/2 from each
side, the last tile is clamped to the volume end and keeps whatever earlier
tiles did not write.  Every output voxel is written exactly once.

Execution is B200-native: each GPU holds one ``PlanRunner`` (CUDA graph),
receives a contiguous block of tiles (x-major order, so a device's tiles
share input rows), uploads only the input slab those tiles read, runs the
tiles back to back with device-to-device patch extraction, writes the kept
regions into a device-resident output slab and copies that slab to the host
once.  There is no collective: tiles are independent (tiling.py:19-21).
"""

from __future__ import annotations

import math
import os
import threading
from dataclasses import dataclass

import numpy as np

from .errors import ExecutionError, TileError

WORKERS_ENV = "VOXPLAN_WORKERS"


@dataclass(frozen=True)
class Tile:
    index: tuple
    in_lo: tuple
    keep_lo: tuple
    keep_hi: tuple
    out_lo: tuple

    def input_window(self, patch_in):
        return tuple(slice(lo, lo + p) for lo, p in zip(self.in_lo, patch_in))

    @property
    def local_window(self):
        return tuple(slice(a, b) for a, b in zip(self.keep_lo, self.keep_hi))

    @property
    def out_window(self):
        return tuple(slice(o, o + b - a) for o, a, b in zip(self.out_lo, self.keep_lo, self.keep_hi))


@dataclass(frozen=True)
class TileGrid:
    counts: tuple
    tiles: tuple
    patch_in: tuple
    patch_out: tuple
    volume_in: tuple
    volume_out: tuple
    overlap: tuple


def axis_cuts(extent, patch, shrink, overlap):
    """[(in_lo, keep_lo, keep_hi)] along one axis, keep_* in output coords."""
    if patch > extent:
        raise TileError("volume extent %d is smaller than the plan's input patch %d"
                        % (extent, patch))
    if overlap < shrink:
        raise TileError("overlap %d is below the network's shrinkage %d" % (overlap, shrink))
    if (overlap - shrink) % 2:
        raise TileError("overlap minus shrinkage must be even, got %d - %d" % (overlap, shrink))
    step = patch - overlap
    if step < 1:
        raise TileError("overlap %d leaves no fresh output per tile of extent %d"
                        % (overlap, patch))
    out = patch - shrink
    if extent == patch:
        return [(0, 0, out)]
    trim = (overlap - shrink) // 2
    n = 1 + math.ceil((extent - patch) / step)
    starts = [min(i * step, extent - patch) for i in range(n)]
    keep_hi = [s + out - (trim if i < n - 1 else 0) for i, s in enumerate(starts)]
    keep_lo = [0] + keep_hi[:-1]
    return list(zip(starts, keep_lo, keep_hi))


def plan_tiles(volume_spatial, patch_in, patch_out, overlap=None) -> TileGrid:
    vol = tuple(int(v) for v in volume_spatial)
    pin = tuple(int(v) for v in patch_in)
    pout = tuple(int(v) for v in patch_out)
    shrink = tuple(a - b for a, b in zip(pin, pout))
    if min(shrink) < 0:
        raise TileError("output patch larger than input patch")
    if overlap is None:
        ov = shrink
    elif np.isscalar(overlap):
        ov = (int(overlap),) * 3
    else:
        ov = tuple(int(v) for v in overlap)
    axes = [axis_cuts(vol[d], pin[d], shrink[d], ov[d]) for d in range(3)]
    tiles = []
    for ix, cx in enumerate(axes[0]):
        for iy, cy in enumerate(axes[1]):
            for iz, cz in enumerate(axes[2]):
                cs = (cx, cy, cz)
                tiles.append(Tile(index=(ix, iy, iz),
                                  in_lo=tuple(c[0] for c in cs),
                                  keep_lo=tuple(c[1] - c[0] for c in cs),
                                  keep_hi=tuple(c[2] - c[0] for c in cs),
                                  out_lo=tuple(c[1] for c in cs)))
    return TileGrid(counts=tuple(len(a) for a in axes), tiles=tuple(tiles), patch_in=pin,
                    patch_out=pout, volume_in=vol,
                    volume_out=tuple(v - s for v, s in zip(vol, shrink)), overlap=ov)


def worker_count(requested=None) -> int:
    cap = os.environ.get(WORKERS_ENV)
    if requested is None:
        requested = int(cap) if cap else 1
    elif cap:
        requested = min(int(requested), int(cap))
    return max(1, int(requested))


def _plan_io(plan):
    if len(plan.inputs) != 1 or len(plan.outputs) != 1:
        raise TileError("tiled execution needs a single-input single-output plan")
    return plan.inputs[0][2], plan.outputs[0][0], plan.outputs[0][2]


def grid_for(plan, volume_spatial, overlap=None) -> TileGrid:
    in_dims, _, out_dims = _plan_io(plan)
    return plan_tiles(volume_spatial, in_dims[2:], out_dims[2:], overlap)


def partition(n_tiles: int, parts: int, rank: int) -> range:
    """Contiguous block of tile indices for one device / rank."""
    lo = (n_tiles * rank) // parts
    hi = (n_tiles * (rank + 1)) // parts
    return range(lo, hi)


class DeviceTiler:
    """Runs a block of tiles of one grid on one GPU, volume slab resident.

    ``streams`` PlanRunners (each with its own graph, buffers and CUDA
    stream) take the tiles round robin, so consecutive patches overlap: the
    deep U-net levels of one patch leave most SMs idle (few output tiles),
    and the next patch's large levels fill them.  Patches are independent,
    so this changes no result."""

    def __init__(self, plan, grid: TileGrid, device, backend=None, streams=None, batch=None):
        import torch
        from .plan import rebatch
        from .runner import PlanRunner
        self.torch = torch
        self.grid = grid
        self.device = torch.device(device)
        n = int(streams if streams is not None else os.environ.get("VOXPLAN_STREAMS", "2"))
        # patches per launch: the deep U-net levels of several patches share
        # one kernel (their few output tiles alone leave most SMs idle).
        # Config-5 volume, 2 streams: 1 -> 170.6 ms, 2 -> 149.9, 3 -> 138.4,
        # 4 -> 136.0 ms

        self.batch = max(1, int(batch if batch is not None else
                                os.environ.get("VOXPLAN_PATCH_BATCH", "4")))
        if plan.inputs[0][2][0] != 1:
            self.batch = 1                 # the volume's own batch already fills the plan
        bplan = rebatch(plan, self.batch) if self.batch > 1 else plan
        with torch.cuda.device(self.device):
            self.runners = [PlanRunner(bplan, backend=backend, device=self.device)
                            for _ in range(max(1, n))]
        self.runner = self.runners[0]
        self.in_name = plan.inputs[0][0]

    def slab_bounds(self, tiles):
        lo = [min(t.in_lo[d] for t in tiles) for d in range(3)]
        hi = [max(t.in_lo[d] + self.grid.patch_in[d] for t in tiles) for d in range(3)]
        olo = [min(t.out_lo[d] for t in tiles) for d in range(3)]
        ohi = [max(t.out_lo[d] + t.keep_hi[d] - t.keep_lo[d] for t in tiles) for d in range(3)]
        return lo, hi, olo, ohi

    def upload(self, volume, tiles):
        """Copy the input slab the tiles read to the device (one H2D)."""
        torch = self.torch
        lo, hi, olo, ohi = self.slab_bounds(tiles)
        win = (slice(None), slice(None)) + tuple(slice(a, b) for a, b in zip(lo, hi))
        host = torch.from_numpy(np.ascontiguousarray(volume[win], dtype=np.float32))
        with torch.cuda.device(self.device):
            self.slab = host.pin_memory().to(self.device, non_blocking=True)
            out_shape = (host.shape[0],) + tuple(
                self.runner._out_std[next(iter(self.runner._out_std))].shape[1:2])
            self.out_slab = torch.empty(out_shape + tuple(b - a for a, b in zip(olo, ohi)),
                                        dtype=torch.float32, device=self.device)
        self.lo, self.olo = lo, olo

    @property
    def launches_per_tile(self) -> float:
        return self.runner.launches / self.batch

    def launches_for(self, n_tiles: int) -> int:
        """Kernel launches to run n_tiles (batches of self.batch patches)."""
        return self.runner.launches * -(-n_tiles // self.batch)

    def run(self, tiles):
        """Run the tiles from the resident slab into the resident output slab
        (enqueued; the current stream is made to wait for all of them)."""
        torch = self.torch
        pin = self.grid.patch_in
        with torch.cuda.device(self.device):
            cur = torch.cuda.current_stream(self.device)
            for r in self.runners:
                r.stream.wait_stream(cur)       # slab / output slab are ready
            B = self.batch
            groups = [tiles[i:i + B] for i in range(0, len(tiles), B)]
            for gi, group in enumerate(groups):
                r = self.runners[gi % len(self.runners)]
                xin = r._in_std[self.in_name]
                with torch.cuda.stream(r.stream):
                    for b in range(B):
                        t = group[min(b, len(group) - 1)]   # a short last group repeats
                        src = tuple(slice(a - l, a - l + p)
                                    for a, l, p in zip(t.in_lo, self.lo, pin))
                        xin[b:b + 1].copy_(self.slab[(slice(None), slice(None)) + src])
                res = next(iter(r.run_on_stream({self.in_name: xin}).values()))
                with torch.cuda.stream(r.stream):
                    for b, t in enumerate(group):
                        dst = tuple(slice(o - l, o - l + (e - a)) for o, l, a, e in
                                    zip(t.out_lo, self.olo, t.keep_lo, t.keep_hi))
                        self.out_slab[(slice(None), slice(None)) + dst].copy_(
                            res[(slice(b, b + 1), slice(None)) + t.local_window])
            for r in self.runners:
                cur.wait_stream(r.stream)

    def download(self, out: np.ndarray, tiles):
        """Copy the output slab into the host volume (one D2H)."""
        _, _, olo, ohi = self.slab_bounds(tiles)
        host = self.out_slab.cpu().numpy()
        win = (slice(None), slice(None)) + tuple(slice(a, b) for a, b in zip(olo, ohi))
        # tiles of one block may not tile a full box: copy only what they wrote
        for t in tiles:
            dst = (slice(None), slice(None)) + t.out_window
            src = (slice(None), slice(None)) + tuple(
                slice(o - l, o - l + (b - a))
                for o, l, a, b in zip(t.out_lo, olo, t.keep_lo, t.keep_hi))
            out[dst] = host[src]
        del win


def run_tiled(plan, volume, *, overlap=None, backend=None, workers=None, grid=None,
              devices=None) -> np.ndarray:
    """Run ``plan`` patchwise over a (batch, fmap, x, y, z) volume (tiling.py:189-237).

    ``devices``: list of CUDA devices (default: ``workers`` devices, default 1,
    capped by ``VOXPLAN_WORKERS`` and the visible GPU count).  Each device gets
    a contiguous block of tiles and one host thread.
    """
    import torch
    volume = np.asarray(volume)
    if volume.ndim != 5:
        raise ExecutionError("tiled input must have rank 5, got rank %d" % volume.ndim)
    in_dims, _, out_dims = _plan_io(plan)
    if tuple(volume.shape[:2]) != tuple(in_dims[:2]):
        raise ExecutionError("volume batch/fmaps %s do not match the plan's %s"
                             % (volume.shape[:2], tuple(in_dims[:2])))
    if grid is None:
        grid = grid_for(plan, volume.shape[2:], overlap)
    elif tuple(grid.volume_in) != tuple(volume.shape[2:]):
        raise TileError("tile grid was planned for a different volume shape")
    if devices is None:
        ndev = min(worker_count(workers), max(1, torch.cuda.device_count()))
        devices = ["cuda:%d" % i for i in range(ndev)]
    devices = list(devices)[:len(grid.tiles)]
    out = np.empty(tuple(out_dims[:2]) + tuple(grid.volume_out), dtype=np.float32)
    blocks = [[grid.tiles[i] for i in partition(len(grid.tiles), len(devices), r)]
              for r in range(len(devices))]
    errors = []

    def work(r):
        try:
            if not blocks[r]:
                return
            dt = DeviceTiler(plan, grid, devices[r], backend)
            dt.upload(volume, blocks[r])
            dt.run(blocks[r])
            torch.cuda.synchronize(dt.device)
            dt.download(out, blocks[r])
        except Exception as exc:  # surfaced below
            errors.append(exc)

    if len(devices) == 1:
        work(0)
    else:
        threads = [threading.Thread(target=work, args=(r,)) for r in range(len(devices))]
        for t in threads:
            t.start()
        for t in threads:
            t.join()
    if errors:
        raise errors[0]
    return out
