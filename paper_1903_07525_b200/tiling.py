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


def slab_bounds(grid: TileGrid, tiles):
    """(in_lo, in_hi, out_lo, out_hi) of the input slab a block of tiles
    reads and of the output region it writes (bounding boxes)."""
    lo = [min(t.in_lo[d] for t in tiles) for d in range(3)]
    hi = [max(t.in_lo[d] + grid.patch_in[d] for t in tiles) for d in range(3)]
    olo = [min(t.out_lo[d] for t in tiles) for d in range(3)]
    ohi = [max(t.out_lo[d] + t.keep_hi[d] - t.keep_lo[d] for t in tiles) for d in range(3)]
    return lo, hi, olo, ohi


def rank_tiles(grid: TileGrid, world: int, rank: int):
    """The contiguous block of tiles rank ``rank`` of ``world`` runs."""
    return [grid.tiles[i] for i in partition(len(grid.tiles), world, rank)]


def gather_volume(out_slab, grid: TileGrid, rank: int, world: int, dist, full=None):
    """Assemble the output volume on rank 0 from every rank's output slab
    (the region ``slab_bounds(rank_tiles(...))`` of each rank) over
    torch.distributed point-to-point: NCCL between GPUs, or gloo (host
    tensors).  Each tile's kept window is copied out of its owner's slab, so
    any partition assembles every output voxel exactly once, also when a
    rank's block is not whole x-rows and its bounding box holds voxels it
    never wrote.  Returns the (batch, fmaps, X, Y, Z) volume on rank 0 (in
    ``full`` when given), None elsewhere.  This is the only exchange of a
    multi-GPU run (patches are independent)."""
    import torch
    host_only = dist.get_backend() == "gloo"
    if rank != 0:
        mine = out_slab.contiguous()
        dist.send(mine.cpu() if host_only else mine, dst=0)
        return None
    if full is None:
        full = torch.empty(tuple(out_slab.shape[:2]) + tuple(grid.volume_out),
                           dtype=out_slab.dtype, device=out_slab.device)
    for r in range(world):
        tiles = rank_tiles(grid, world, r)
        if not tiles:
            continue
        _, _, olo, ohi = slab_bounds(grid, tiles)
        if r == 0:
            src = out_slab
        else:
            shape = tuple(out_slab.shape[:2]) + tuple(b - a for a, b in zip(olo, ohi))
            buf = torch.empty(shape, dtype=out_slab.dtype,
                              device="cpu" if host_only else out_slab.device)
            dist.recv(buf, src=r)
            src = buf.to(full.device)
        for t in tiles:
            win = tuple(slice(o - l, o - l + (e - a)) for o, l, a, e in
                        zip(t.out_lo, olo, t.keep_lo, t.keep_hi))
            full[(slice(None), slice(None)) + t.out_window].copy_(
                src[(slice(None), slice(None)) + win])
    return full


class DeviceTiler:
    """Runs blocks of tiles of one grid on one GPU.

    ``streams`` PlanRunners (each with its own graph, buffers and CUDA
    stream) take the patch batches round robin, so consecutive batches
    overlap: the deep U-net levels of one batch leave most SMs idle (few
    output tiles), and the next batch's large levels fill them.  Patches are
    independent, so this changes no result.

    Two ways to feed it:
      * resident (``bind_slabs`` + ``run``): an input slab and an output slab
        already in HBM (the bench's device-timed value);
      * streamed (``run_host``): tiles are processed x-row by x-row (a row =
        the tiles sharing one x cut); each row's input slab is uploaded on a
        copy stream while the previous row computes, and each row's output is
        downloaded while the next one computes (two-deep device rings), so
        PCIe traffic overlaps the convolutions.  Page-locked host arrays
        (``staging.pinned_empty``) move by direct DMA; pageable ones go through
        pinned staging chunks copied by a thread pool."""

    def __init__(self, plan, grid: TileGrid, device, backend=None, streams=None, batch=None,
                 probe=None):
        import torch
        from .plan import rebatch
        from .runner import PlanRunner
        self.torch = torch
        self.grid = grid
        self.device = torch.device(device)
        n = int(streams if streams is not None else os.environ.get("VOXPLAN_STREAMS", "1"))
        # patches per launch: the deep U-net levels of several patches share
        # one kernel (their few output tiles alone leave most SMs idle).
        # Config-5 volume (round 1 kernels, 2 streams): 1 -> 170.6 ms,
        # 4 -> 131.5, 8 -> 124.1, 12 -> 123.5, 16 -> 123.1 ms; with the round-2
        # epilogues (1 stream): 12 -> 111.3, 18 -> 109.8, 24 -> 108.8,
        # 36 -> 108.4, 72 -> 106.9, 96 -> 106.5 ms (tools/ab_bench5.sh).  36
        # is one x-row of config 5's (8,6,6) tile grid, the largest batch the
        # streamed run_host (row by row) can form without padding.  Runner
        # streams: with the lean epilogue and no PDL inside the batches, one
        # stream measured 116.2 ms vs 116.9 ms for two (the persistent convs
        # fill every SM, so a second stream only interleaves), and a single
        # stream keeps the in-step kernel timing free of the other stream's
        # work.
        self.batch = max(1, int(batch if batch is not None else
                                os.environ.get("VOXPLAN_PATCH_BATCH", "36")))
        if batch is None:
            # never more than one x-row of this grid (no padded batches)
            self.batch = min(self.batch, max(len(r) for r in self.rows(list(grid.tiles))))
        self.vol_batch = int(plan.inputs[0][2][0])
        if self.vol_batch != 1:
            self.batch = 1                 # the volume's own batch already fills the plan
        bplan = rebatch(plan, self.batch) if self.batch > 1 else plan
        with torch.cuda.device(self.device):
            # no programmatic dependent launch inside the patch batches
            # (PlanRunner.pdl: 116.9 vs 118.7 ms for the config-5 volume)
            pdl = os.environ.get("VOXPLAN_PDL", "0") == "1"
            self.runners = [PlanRunner(bplan, backend=backend, device=self.device, pdl=pdl,
                                       probe=probe if i == 0 else None)
                            for i in range(max(1, n))]
            self.copy_in = torch.cuda.Stream(device=self.device)
            self.copy_out = torch.cuda.Stream(device=self.device)
        self.runner = self.runners[0]
        self.in_name = plan.inputs[0][0]
        self.out_fmaps = int(plan.outputs[0][2][1])
        self._rings = None
        self.slab = self.out_slab = None

    # ------------------------------------------------------------ geometry
    def slab_bounds(self, tiles):
        return slab_bounds(self.grid, tiles)

    @staticmethod
    def rows(tiles):
        """Tiles grouped by x cut (consecutive runs of equal in_lo[0])."""
        out = []
        for t in tiles:
            if out and out[-1][0].in_lo[0] == t.in_lo[0]:
                out[-1].append(t)
            else:
                out.append([t])
        return out

    @property
    def launches_per_tile(self) -> float:
        return self.runner.launches / self.batch

    def launches_for(self, n_tiles: int) -> int:
        """Kernel launches to run n_tiles (batches of self.batch patches): the
        network plus one gather and one scatter launch per batch."""
        return (self.runner.launches + 2) * -(-n_tiles // self.batch)

    # ------------------------------------------------------------ resident
    def bind_slabs(self, slab, lo, out_slab, olo):
        """Device input slab (n, c, X, Y, Z) whose voxel (0,0,0) is volume
        coordinate ``lo``, and output slab whose (0,0,0) is output ``olo``."""
        self.slab, self.lo, self.out_slab, self.olo = slab, tuple(lo), out_slab, tuple(olo)

    def upload(self, volume, tiles):
        """Copy the input slab the tiles read to the device and allocate the
        matching output slab (resident mode)."""
        torch = self.torch
        lo, hi, olo, ohi = self.slab_bounds(tiles)
        win = (slice(None), slice(None)) + tuple(slice(a, b) for a, b in zip(lo, hi))
        with torch.cuda.device(self.device):
            slab = torch.from_numpy(np.ascontiguousarray(volume[win], dtype=np.float32)).to(
                self.device)
            out_slab = torch.empty((volume.shape[0], self.out_fmaps) +
                                   tuple(b - a for a, b in zip(olo, ohi)),
                                   dtype=torch.float32, device=self.device)
        self.bind_slabs(slab, lo, out_slab, olo)

    def run(self, tiles):
        """Run the tiles from the bound input slab into the bound output slab
        (enqueued; the current stream is made to wait for all of them).  With
        one runner the whole tile list -- every batch's patch gather, network
        and kept-window scatter -- replays as one CUDA graph, captured on the
        first call for this (tile list, slab pair)."""
        torch = self.torch
        with torch.cuda.device(self.device):
            cur = torch.cuda.current_stream(self.device)
            for r in self.runners:
                r.stream.wait_stream(cur)       # slab / output slab are ready
            g = self._volume_graph(tiles, self.slab, self.lo, self.out_slab, self.olo)
            if g is not None:
                with torch.cuda.stream(self.runner.stream):
                    g.replay()
            else:
                self._enqueue(tiles, self.slab, self.lo, self.out_slab, self.olo)
            for r in self.runners:
                cur.wait_stream(r.stream)

    def _volume_graph(self, tiles, slab, lo, out_slab, olo):
        """One CUDA graph over every batch of ``tiles`` (single runner only;
        cached per tile list and slab pointers, VOXPLAN_VOLUME_GRAPH=0 off)."""
        torch = self.torch
        if len(self.runners) != 1 or os.environ.get("VOXPLAN_VOLUME_GRAPH", "1") != "1":
            return None
        # keyed by the tiles' geometry relative to the slabs, so the rows of
        # the streamed run_host (same layout, two ring slots) share graphs
        geo = tuple((tuple(a - l for a, l in zip(t.in_lo, lo)),
                     tuple(o - l for o, l in zip(t.out_lo, olo)),
                     tuple(t.keep_lo), tuple(t.keep_hi)) for t in tiles)
        key = (geo, slab.data_ptr(), out_slab.data_ptr(), tuple(slab.shape), tuple(slab.stride()),
               tuple(out_slab.shape), tuple(out_slab.stride()))
        cache = self.__dict__.setdefault("_vgraphs", {})
        g = cache.get(key)
        if g is None:
            r = self.runner
            r.ensure_graph()                     # kernels configured, pool bound
            torch.cuda.synchronize(self.device)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=r.stream, capture_error_mode="thread_local"):
                self._enqueue(tiles, slab, lo, out_slab, olo, raw=True)
            if len(cache) >= 8:
                cache.pop(next(iter(cache)))
            cache[key] = g
        return g

    def _windows(self, group, slab, lo, out_slab, olo, xin, res):
        """(gather, scatter) window pairs of one patch batch."""
        pin = self.grid.patch_in
        whole = self.vol_batch > 1
        gather, scatter = [], []
        for b in range(self.batch):
            t = group[min(b, len(group) - 1)]   # a short last group repeats
            src = tuple(slice(a - l, a - l + p) for a, l, p in zip(t.in_lo, lo, pin))
            dst_b = slice(None) if whole else slice(b, b + 1)
            gather.append((slab[(slice(None), slice(None)) + src], xin[dst_b]))
        for b, t in enumerate(group):
            dst = tuple(slice(o - l, o - l + (e - a)) for o, l, a, e in
                        zip(t.out_lo, olo, t.keep_lo, t.keep_hi))
            src_b = slice(None) if whole else slice(b, b + 1)
            scatter.append((res[(src_b, slice(None)) + t.local_window],
                            out_slab[(slice(None), slice(None)) + dst]))
        return gather, scatter

    def _enqueue(self, tiles, slab, lo, out_slab, olo, start=0, raw=False):
        """Enqueue the tiles' batches on the runner streams (round robin from
        runner `start`); returns the next runner index.  Each batch: one
        gather launch (the patches' input windows into the runner's input
        buffer), the network, one scatter launch (kept windows into the
        output slab).  ``raw``: launch the network's kernels directly (inside
        a capture of the whole volume) instead of replaying its graph."""
        from .device import copy_windows, current_stream_handle, pack_zwin_windows
        torch = self.torch
        B = self.batch
        # rebatched plans (volume batch 1) stack B patches along the batch
        # axis; a plan whose own batch is > 1 runs one patch of the whole
        # volume batch per launch (B == 1)
        groups = [tiles[i:i + B] for i in range(0, len(tiles), B)]
        k = start
        nocopy = os.environ.get("VOXPLAN_DEBUG_NOCOPY") == "1"   # timing experiments only
        for group in groups:
            r = self.runners[k % len(self.runners)]
            k += 1
            xin = r._in_std[self.in_name]
            res = next(iter(r._out_std.values()))
            gather, scatter = self._windows(group, slab, lo, out_slab, olo, xin, res)
            # inside the volume graph, a z-window network input is packed
            # straight from the slab windows (the gather fused into the pack)
            zw = r.zwin_input if (raw and r._n_in_calls == 1 and not nocopy and
                                  self.vol_batch == 1 and B <= 64) else None   # ZWIN_MAX
            if zw is not None and zw[0] != self.in_name:
                zw = None
            with torch.cuda.stream(r.stream):
                if zw is not None:
                    pack_zwin_windows([src for src, _ in gather], zw[1], zw[2], zw[3],
                                      current_stream_handle())
                    r.launch_raw(skip_inputs=True)
                elif not nocopy:
                    copy_windows(gather, current_stream_handle())
                if raw and zw is None:
                    r.launch_raw()
                elif not raw:
                    r.run_on_stream({self.in_name: xin})
                if not nocopy:
                    copy_windows(scatter, current_stream_handle())
        return k

    # ------------------------------------------------------------ streamed
    def _ring(self, nb, cin, in_ext, out_ext):
        """Two input and two output row slabs on the device (flat buffers for
        the largest row, viewed per row so every row slab is contiguous)."""
        torch = self.torch
        nin = nb * cin * int(np.prod(in_ext))
        nout = nb * self.out_fmaps * int(np.prod(out_ext))
        if self._rings is None or self._rings[0] < nin or self._rings[1] < nout:
            with torch.cuda.device(self.device):
                ins = [torch.empty(nin, dtype=torch.float32, device=self.device)
                       for _ in range(2)]
                outs = [torch.empty(nout, dtype=torch.float32, device=self.device)
                        for _ in range(2)]
            self._rings = (nin, nout, ins, outs)
        return self._rings[2], self._rings[3]

    def run_host(self, volume, out, tiles):
        """Stream the tiles' input rows from host ``volume`` and their kept
        outputs into host ``out`` (both (n, c, X, Y, Z) float32).  Returns
        when ``out`` holds the results."""
        from . import staging
        torch = self.torch
        rows = self.rows(list(tiles))
        if not rows:
            return
        bounds = [self.slab_bounds(r) for r in rows]
        in_ext = [max(b[1][d] - b[0][d] for b in bounds) for d in range(3)]
        out_ext = [max(b[3][d] - b[2][d] for b in bounds) for d in range(3)]
        nb, cin = int(volume.shape[0]), int(volume.shape[1])
        ins, outs = self._ring(nb, cin, in_ext, out_ext)
        vol_t = torch.from_numpy(volume) if staging.is_pinned(volume) else None
        out_t = torch.from_numpy(out) if staging.is_pinned(out) else None
        if getattr(self, "_stager", None) is None:
            self._stager = staging.RowStager()     # pinned slots, reused across calls
        stager = self._stager
        ev_in = [None, None]        # input slot free: its row's compute is done
        ev_out = [None, None]       # output slot free: its row's download is done
        k = 0

        def full_yz(lo, hi, shape):
            return lo[1] == 0 and lo[2] == 0 and hi[1] == shape[3] and hi[2] == shape[4]

        with torch.cuda.device(self.device):
            cur = torch.cuda.current_stream(self.device)
            self.copy_in.wait_stream(cur)
            self.copy_out.wait_stream(cur)
            for ri, (row, (lo, hi, olo, ohi)) in enumerate(zip(rows, bounds)):
                slot = ri % 2
                ishape = (nb, cin) + tuple(b - a for a, b in zip(lo, hi))
                oshape = (nb, self.out_fmaps) + tuple(b - a for a, b in zip(olo, ohi))
                xin = ins[slot][:int(np.prod(ishape))].view(ishape)
                yout = outs[slot][:int(np.prod(oshape))].view(oshape)
                win = (slice(None), slice(None)) + tuple(slice(a, b) for a, b in zip(lo, hi))
                owin = (slice(None), slice(None)) + tuple(slice(a, b) for a, b in zip(olo, ohi))
                # ---- upload row ri once row ri-2's compute released the slot
                if ev_in[slot] is not None:
                    self.copy_in.wait_event(ev_in[slot])
                if vol_t is not None and full_yz(lo, hi, volume.shape):
                    with torch.cuda.stream(self.copy_in):
                        for b in range(nb):
                            for c in range(cin):   # contiguous x-range of one fmap
                                xin[b, c].copy_(vol_t[b, c, lo[0]:hi[0]], non_blocking=True)
                else:
                    stager.upload(slot, volume[win], xin, self.copy_in)
                up = torch.cuda.Event()
                up.record(self.copy_in)
                # ---- compute (after the upload, and once row ri-2's output
                # left this slot)
                for r in self.runners:
                    r.stream.wait_event(up)
                    if ev_out[slot] is not None:
                        r.stream.wait_event(ev_out[slot])
                g = self._volume_graph(row, xin, lo, yout, olo)
                if g is not None:
                    with torch.cuda.stream(self.runner.stream):
                        g.replay()
                else:
                    k = self._enqueue(row, xin, lo, yout, olo, start=k)
                done = []
                for r in self.runners:
                    e = torch.cuda.Event()
                    e.record(r.stream)
                    done.append(e)
                # ---- download the row's kept output
                for e in done:
                    self.copy_out.wait_event(e)
                freed = torch.cuda.Event()
                freed.record(self.copy_out)
                ev_in[slot] = freed
                if out_t is not None and full_yz(olo, ohi, out.shape):
                    with torch.cuda.stream(self.copy_out):
                        for b in range(nb):
                            for c in range(self.out_fmaps):
                                out_t[b, c, olo[0]:ohi[0]].copy_(yout[b, c], non_blocking=True)
                else:
                    stager.download(slot, yout, out[owin], self.copy_out)
                fin = torch.cuda.Event()
                fin.record(self.copy_out)
                ev_out[slot] = fin
            for r in self.runners:
                cur.wait_stream(r.stream)
            cur.wait_stream(self.copy_out)
        self.copy_out.synchronize()
        stager.finish()


_TILER_CACHE: dict = {}
_TILER_LOCK = threading.Lock()


def device_tiler(plan, grid: TileGrid, device, backend=None, slot=0) -> DeviceTiler:
    """A cached DeviceTiler per (plan, grid, device, worker slot, backend,
    batching knobs): repeated run_tiled calls reuse bound runners and
    captured graphs; two workers on the same device get separate tilers."""
    key = (id(plan), grid.patch_in, grid.volume_in, grid.overlap, str(device), int(slot),
           repr(backend),
           os.environ.get("VOXPLAN_PATCH_BATCH", "36"), os.environ.get("VOXPLAN_STREAMS", "1"))
    with _TILER_LOCK:
        hit = _TILER_CACHE.get(key)
        if hit is not None and hit[0] is plan:
            return hit[1]
    dt = DeviceTiler(plan, grid, device, backend)
    with _TILER_LOCK:
        if len(_TILER_CACHE) >= 8:
            _TILER_CACHE.pop(next(iter(_TILER_CACHE)))
        _TILER_CACHE[key] = (plan, dt)
    return dt


def run_tiled(plan, volume, *, overlap=None, backend=None, workers=None, grid=None,
              devices=None, out=None) -> np.ndarray:
    """Run ``plan`` patchwise over a (batch, fmap, x, y, z) volume (tiling.py:189-237).

    ``devices``: list of CUDA devices (default: ``workers`` devices, default 1,
    capped by ``VOXPLAN_WORKERS`` and the visible GPU count).  Each device gets
    a contiguous block of tiles and one host thread, and streams its input
    rows in and its output rows out (DeviceTiler.run_host).  ``out``: an
    optional preallocated (e.g. page-locked) result array.
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
    shape = tuple(out_dims[:2]) + tuple(grid.volume_out)
    if out is None:
        out = np.empty(shape, dtype=np.float32)
    elif tuple(out.shape) != shape or out.dtype != np.float32:
        raise ExecutionError("out must be a float32 array of shape %s" % (shape,))
    if volume.dtype != np.float32:
        volume = volume.astype(np.float32)
    blocks = [[grid.tiles[i] for i in partition(len(grid.tiles), len(devices), r)]
              for r in range(len(devices))]
    errors = []

    def work(r):
        try:
            if not blocks[r]:
                return
            dt = device_tiler(plan, grid, devices[r], backend, slot=r)
            dt.run_host(volume, out, blocks[r])
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


def run_tiled_file(plan, in_path, out_path, *, overlap=None, backend=None, workers=None,
                   devices=None, grid=None):
    """File to file: stream a PZNV volume through ``run_tiled`` into a new PZNV
    file (formats.open_volume / create_volume memory maps: input rows are
    paged in and output rows written back while the GPU works on the
    neighbouring rows; neither volume is ever held in host memory as a
    whole).  The output file is byte-identical to
    ``write_volume(out_path, run_tiled(plan, read_volume(in_path)))``."""
    from .formats import create_volume, open_volume
    vol = open_volume(in_path)
    _, _, out_dims = _plan_io(plan)
    if grid is None:
        grid = grid_for(plan, vol.shape[2:], overlap)
    out = create_volume(out_path, tuple(out_dims[:2]) + tuple(grid.volume_out))
    try:
        run_tiled(plan, vol, overlap=overlap, backend=backend, workers=workers, grid=grid,
                  devices=devices, out=out)
        out.flush()
    finally:
        del out, vol
    return out_path
