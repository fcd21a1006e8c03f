"""CPU-only checks: the C-ABI library loads and exports every declared symbol,
host-side packing, backend registry rules, tiling geometry vs the reference,
and the multi-rank tile partition over a gloo process group."""

import json
import os
import re

import numpy as np
import pytest

from vxb_testutil import GOLDEN, ROOT

from paper_1903_07525_b200 import _lib, backend, tiling
from paper_1903_07525_b200.errors import ExecutionError, TileError


def _declared_symbols():
    hdr = open(os.path.join(ROOT, "include", "vxb.h")).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[a-z_0-9]+\s*\*?\s*(vxb_[a-z_0-9]+)\s*\(",
                                 hdr, re.M)))


def test_header_symbols_all_bound_and_exported():
    syms = _declared_symbols()
    assert len(syms) >= 20
    bound = {name for name, _, _ in _lib.SIGNATURES}
    assert set(syms) == bound, set(syms) ^ bound
    if not _lib.library_available():
        pytest.skip("libvxb.so not built")
    L = _lib.lib()
    for s in syms:
        assert hasattr(L, s)
    assert L.vxb_abi_version() == _lib.ABI_VERSION == 5


def test_host_packing_sizes_and_selection():
    if not _lib.library_available():
        pytest.skip("libvxb.so not built")
    L = _lib.lib()
    k3, s1 = _lib.i3((3, 3, 3)), _lib.i3((1, 1, 1))
    assert L.vxb_conv_select(16, 16, k3, s1) == _lib.PATH_TC
    assert L.vxb_conv_select(16, 16, k3, _lib.i3((2, 2, 2))) == _lib.PATH_DIRECT
    # C16 -> N tile 16, one channel-pair group of 27 steps, 32 B rows
    assert L.vxb_conv_weights_bytes(16, 16, k3, s1, 0) == 27 * 16 * 32
    # odd chunk (Cin=8): z-pair steps 3*3*2
    assert L.vxb_conv_weights_bytes(8, 16, k3, s1, 0) == 18 * 16 * 32
    # Cout 512 -> two N tiles of 256
    assert L.vxb_conv_weights_bytes(256, 512, k3, s1, 0) == 2 * 16 * 27 * 256 * 32
    w = np.random.default_rng(0).standard_normal((16, 16, 3, 3, 3)).astype(np.float32)
    n = L.vxb_conv_weights_bytes(16, 16, k3, s1, 0)
    dst = np.zeros(n, np.uint8)
    assert L.vxb_conv_pack_weights(w.ctypes.data, 16, 16, k3, s1, 0, dst.ctypes.data, n) == 0
    # C16 3x3x3 folds the x taps into N: device step (dy, dz) holds three
    # nt-row blocks [dx=2; dx=1; dx=0].  Inside a block: row n, k-half h,
    # lane l at (n/8)*256 + h*128 + (n%8)*16 + 2l
    bf = dst.view(np.uint16)
    from oracle.ref_numpy import bf16_round

    def at(buf, byte):
        return (np.array([buf[byte // 2]], np.uint16).astype(np.uint32) << 16).view(np.float32)[0]

    for (co, ci) in [(0, 0), (5, 3), (9, 12), (15, 15)]:
        h, l = ci // 8, ci % 8
        row = (co // 8) * 256 + h * 128 + (co % 8) * 16 + 2 * l
        for dx in range(3):
            for (dy, dz) in [(0, 0), (1, 2), (2, 1)]:
                step = dy * 3 + dz
                byte = step * 3 * 16 * 32 + (2 - dx) * 16 * 32 + row
                assert at(bf, byte) == bf16_round(w[co, ci, dx, dy, dz])
    # C128 (3*nt > 256) stays unfolded: step = (dx, dy, dz) tap order
    w2 = np.random.default_rng(1).standard_normal((128, 16, 3, 3, 3)).astype(np.float32)
    n2 = L.vxb_conv_weights_bytes(16, 128, k3, s1, 0)
    assert n2 == 27 * 128 * 32
    dst2 = np.zeros(n2, np.uint8)
    assert L.vxb_conv_pack_weights(w2.ctypes.data, 16, 128, k3, s1, 0, dst2.ctypes.data, n2) == 0
    bf2 = dst2.view(np.uint16)
    for (co, ci, dx, dy, dz) in [(0, 0, 0, 0, 0), (77, 9, 2, 1, 0), (127, 15, 1, 2, 2)]:
        h, l = ci // 8, ci % 8
        step = (dx * 3 + dy) * 3 + dz
        byte = step * 128 * 32 + (co // 8) * 256 + h * 128 + (co % 8) * 16 + 2 * l
        assert at(bf2, byte) == bf16_round(w2[co, ci, dx, dy, dz])
    # 1x3x3 folds along y with 16-row x tiles; x = 18 would pad 14 of 32 rows
    k133 = _lib.i3((1, 3, 3))
    assert L.vxb_conv_select_shape(28, 28, k133, s1, _lib.i3((18, 192, 192))) == _lib.PATH_TC_UNFOLDED
    assert L.vxb_conv_select_shape(28, 28, k133, s1, _lib.i3((32, 128, 128))) == _lib.PATH_TC
    assert L.vxb_conv_select_shape(28, 28, k3, s1, _lib.i3((18, 192, 192))) == _lib.PATH_TC
    assert L.vxb_conv_select_shape(28, 28, k3, _lib.i3((2, 2, 2)), _lib.i3((9, 9, 9))) == \
        _lib.PATH_DIRECT
    # deep levels with few output tiles split their fmaps into narrower N tiles
    assert L.vxb_conv_select_shape(768, 256, k3, s1, _lib.i3((16, 16, 16))) in \
        (_lib.PATH_TC_N128, _lib.PATH_TC_N64)
    assert L.vxb_conv_select_shape(80, 80, k3, s1, _lib.i3((18, 12, 12))) in \
        (_lib.PATH_TC_N64, _lib.PATH_TC_N32, _lib.PATH_TC_N16)
    # ... unless a launch covers enough batch entries (rebatched patches)
    assert L.vxb_conv_select_shape_b(80, 80, k3, s1, _lib.i3((18, 12, 12)), 1) == \
        L.vxb_conv_select_shape(80, 80, k3, s1, _lib.i3((18, 12, 12)))
    assert L.vxb_conv_select_shape_b(80, 80, k3, s1, _lib.i3((18, 12, 12)), 12) == _lib.PATH_TC
    assert L.vxb_conv_select_shape(128, 128, k3, s1, _lib.i3((32, 128, 128))) == _lib.PATH_TC
    assert L.vxb_conv_weights_bytes(768, 256, k3, s1, _lib.PATH_TC_N64) == \
        L.vxb_conv_weights_bytes(768, 256, k3, s1, _lib.PATH_TC)
    # unfolded C16 image: same size, plain tap order
    du = np.zeros(n, np.uint8)
    assert L.vxb_conv_pack_weights(w.ctypes.data, 16, 16, k3, s1, _lib.PATH_TC_UNFOLDED,
                                   du.ctypes.data, n) == 0
    bu = du.view(np.uint16)
    for (co, ci, dx, dy, dz) in [(0, 0, 0, 0, 0), (9, 12, 2, 1, 0), (15, 15, 1, 2, 2)]:
        h, l = ci // 8, ci % 8
        step = (dx * 3 + dy) * 3 + dz
        byte = step * 16 * 32 + (co // 8) * 256 + h * 128 + (co % 8) * 16 + 2 * l
        assert at(bu, byte) == bf16_round(w[co, ci, dx, dy, dz])
    assert L.vxb_conv_pack_weights(w.ctypes.data, 16, 16, k3, s1, 0, dst.ctypes.data, 10) != 0
    assert b"need" in L.vxb_last_error()


def test_backend_registry_rules(monkeypatch):
    with pytest.raises(ExecutionError):
        backend.get_backend("nope")
    monkeypatch.setattr(_lib, "LIB_PATH", "/nonexistent/libvxb.so")
    monkeypatch.setattr(_lib, "_LIB", None)
    with pytest.raises(ExecutionError):
        backend.get_backend("b200")
    with pytest.raises(ExecutionError):
        _lib.lib()
    assert backend.available_backends() == ()
    monkeypatch.setenv(backend.BACKEND_ENV, "bogus")
    with pytest.raises(ExecutionError):
        backend.get_backend()


def test_tiles_match_reference_geometry():
    for case in json.load(open(os.path.join(GOLDEN, "tiles.json"))):
        g = tiling.plan_tiles(case["volume"], case["patch_in"], case["patch_out"], case["overlap"])
        assert list(g.counts) == case["counts"]
        assert list(g.volume_out) == case["volume_out"]
        got = [[list(t.index), list(t.in_lo), list(t.keep_lo), list(t.keep_hi), list(t.out_lo)]
               for t in g.tiles]
        assert got == case["tiles"]


@pytest.mark.parametrize("vol,pin,pout,ov", [
    ((40, 40, 40), (16, 16, 16), (16, 16, 16), None),
    ((37, 50, 29), (12, 20, 9), (8, 16, 5), None),
    ((31, 33, 35), (10, 12, 14), (6, 8, 10), 8),
    ((18, 1024, 1024), (18, 192, 192), (18, 192, 192), 0),
])
def test_exactly_once_coverage(vol, pin, pout, ov):
    g = tiling.plan_tiles(vol, pin, pout, ov)
    cover = np.zeros(g.volume_out, np.int32)
    for t in g.tiles:
        cover[t.out_window] += 1
        assert all(0 <= a < b <= p for a, b, p in zip(t.keep_lo, t.keep_hi, pout))
    assert (cover == 1).all()


def test_tile_errors():
    with pytest.raises(TileError):
        tiling.plan_tiles((10, 10, 10), (12, 8, 8), (12, 8, 8))
    with pytest.raises(TileError):
        tiling.plan_tiles((20, 20, 20), (8, 8, 8), (6, 6, 6), 3)   # odd surplus
    with pytest.raises(TileError):
        tiling.plan_tiles((20, 20, 20), (8, 8, 8), (4, 4, 4), 2)   # below shrinkage


def test_partition_blocks():
    for n, parts in [(288, 1), (288, 2), (288, 8), (7, 3), (5, 8)]:
        seen = []
        for r in range(parts):
            seen += list(tiling.partition(n, parts, r))
        assert seen == list(range(n))


def _rank_main(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    g = tiling.plan_tiles((128, 1024, 1024), (18, 192, 192), (18, 192, 192), 0)
    mine = [g.tiles[i] for i in tiling.partition(len(g.tiles), world, rank)]
    vox = sum(int(np.prod(np.array(t.keep_hi) - np.array(t.keep_lo))) for t in mine)
    t = torch.tensor([float(vox), float(rank + 1)])
    tot = t.clone()
    dist.all_reduce(tot[:1], op=dist.ReduceOp.SUM)
    mx = t[1:].clone()
    dist.all_reduce(mx, op=dist.ReduceOp.MAX)    # bench.py: max-over-ranks timing
    if rank == 0:
        q.put((tot[0].item(), mx.item()))
    dist.destroy_process_group()


def test_two_rank_tile_partition_gloo():
    import multiprocessing as mp
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_rank_main, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    total, mx = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
    assert total == 128 * 1024 * 1024
    assert mx == 2.0


def _gather_main(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    g = tiling.plan_tiles((22, 30, 27), (8, 12, 11), (6, 10, 9), (4, 4, 4))
    mine = tiling.rank_tiles(g, world, rank)
    lo, hi, olo, ohi = tiling.slab_bounds(g, mine)
    slab = torch.full((1, 2) + tuple(b - a for a, b in zip(olo, ohi)), float("nan"),
                      dtype=torch.float64)
    for t in mine:        # what a tile's run would write: a code of the global voxel
        for d in range(3):
            assert lo[d] <= t.in_lo[d] and t.in_lo[d] + g.patch_in[d] <= hi[d]
        w = [np.arange(o, o + (e - a)) for o, a, e in zip(t.out_lo, t.keep_lo, t.keep_hi)]
        code = (w[0][:, None, None] * 10000 + w[1][None, :, None] * 100 + w[2][None, None, :])
        loc = tuple(slice(o - l, o - l + len(v)) for o, l, v in zip(t.out_lo, olo, w))
        for c in range(2):
            slab[(0, c) + loc] = torch.from_numpy(code + c * 1e6)
    full = tiling.gather_volume(slab, g, rank, world, dist)
    if rank == 0:
        q.put(full.numpy())
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gather_volume_gloo_assembles_exactly_once(world):
    """Ranks own contiguous tile blocks (split mid x-row for these grids);
    rank 0's gather must place every tile's kept window, never a neighbour's
    unwritten bounding-box voxels (tiling.gather_volume)."""
    import multiprocessing as mp
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_gather_main, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    full = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    g = tiling.plan_tiles((22, 30, 27), (8, 12, 11), (6, 10, 9), (4, 4, 4))
    assert len(g.tiles) % world != 0 or any(
        len({t.in_lo[0] for t in tiling.rank_tiles(g, world, r)}) > 1 for r in range(world))
    X, Y, Z = g.volume_out
    want = (np.arange(X)[:, None, None] * 10000 + np.arange(Y)[None, :, None] * 100
            + np.arange(Z)[None, None, :])
    assert full.shape == (1, 2, X, Y, Z)
    assert not np.isnan(full).any()
    np.testing.assert_array_equal(full[0, 0], want)
    np.testing.assert_array_equal(full[0, 1], want + 1e6)


def test_tiler_windows_and_row_batches():
    """DeviceTiler's batch geometry on the host (CPU tensors, no CUDA): the
    gather windows of a batch are exactly each tile's input window of the
    slab, the scatter windows each tile's kept output window, a short last
    group repeats its last tile for the gather only, and batches never span
    more than one x-row of the grid."""
    import torch
    grid = tiling.plan_tiles((9, 40, 30), (4, 16, 16), (4, 16, 16), overlap=0)
    rows = tiling.DeviceTiler.rows(list(grid.tiles))
    assert sum(len(r) for r in rows) == len(grid.tiles)
    assert all(len({t.in_lo[0] for t in r}) == 1 for r in rows)
    dt = object.__new__(tiling.DeviceTiler)      # geometry only: no runners
    dt.grid, dt.batch, dt.vol_batch = grid, 4, 1
    vol = torch.arange(9 * 40 * 30, dtype=torch.float32).reshape(1, 1, 9, 40, 30)
    lo, hi, olo, ohi = tiling.slab_bounds(grid, grid.tiles)
    slab = vol[(slice(None), slice(None)) + tuple(slice(a, b) for a, b in zip(lo, hi))]
    out_slab = torch.zeros((1, 2) + tuple(b - a for a, b in zip(olo, ohi)))
    xin = torch.zeros((4, 1) + tuple(grid.patch_in))
    res = torch.arange(4 * 2 * int(np.prod(grid.patch_in)), dtype=torch.float32).reshape(
        (4, 2) + tuple(grid.patch_in))
    group = list(grid.tiles[:3])                  # short group of 3 in a batch of 4
    gather, scatter = dt._windows(group, slab, lo, out_slab, olo, xin, res)
    assert len(gather) == 4 and len(scatter) == 3
    for b, (src, dst) in enumerate(gather):
        t = group[min(b, 2)]
        want = vol[(slice(None), slice(None)) + t.input_window(grid.patch_in)]
        assert torch.equal(src, want) and dst.shape == want.shape
    for b, (src, dst) in enumerate(scatter):
        t = group[b]
        assert torch.equal(src, res[(slice(b, b + 1), slice(None)) + t.local_window])
        dst.copy_(src)
        full = torch.zeros((1, 2, 9, 40, 30))
        full[(slice(None), slice(None)) + tuple(slice(a, b) for a, b in zip(olo, ohi))] = out_slab
        assert torch.equal(full[(slice(None), slice(None)) + t.out_window], src)
