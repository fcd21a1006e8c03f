"""Multi-rank tiled execution on the device, checked bit for bit against one
rank (the reference pins multi-worker tiling bit-identical to serial,
pkg/tests/test_tiling.py:164-170).

The GPU box has one B200, so the ranks share cuda:0.  They never wait on
each other's kernels: each runs its own DeviceTiler over its contiguous
block of tiles, and the only exchange is the final gather to rank 0
(tiling.gather_volume) over gloo (host tensors).  On a multi-GPU node the
same code runs one rank per GPU with NCCL (bench.py --gpus N).
"""

import multiprocessing as mp
import os
import socket

import numpy as np
import pytest

from vxb_testutil import cuda_ready

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not cuda_ready(), reason="needs CUDA + libvxb.so")]

VOL = (18, 96, 96)            # 3 x 2 x 2 = 12 tiles of 6 x 48 x 48


def _net():
    import paper_1903_07525_b200 as P
    from paper_1903_07525_b200 import configs as C
    spec, store = C.config5(patch=(6, 48, 48), feats=(8, 12, 16, 20))
    plan, _ = P.compile_network(spec, store, fixpoint=True, fuse_deconv_add=True)
    return plan


def _volume():
    return np.random.default_rng(21).uniform(0, 1, (1, 1) + VOL).astype(np.float32)


def _rank_main(rank, world, port, path):
    import torch
    import torch.distributed as dist
    from paper_1903_07525_b200 import tiling
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    plan = _net()
    grid = tiling.grid_for(plan, VOL, overlap=0)
    mine = tiling.rank_tiles(grid, world, rank)
    dt = tiling.DeviceTiler(plan, grid, "cuda:0")
    dt.upload(_volume(), mine)
    dt.run(mine)
    torch.cuda.synchronize()
    full = tiling.gather_volume(dt.out_slab, grid, rank, world, dist)
    if rank == 0:
        np.save(path, full.cpu().numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_ranks_gather_bit_identical_to_one_rank(world, tmp_path):
    import paper_1903_07525_b200 as P
    plan = _net()
    want = P.run_tiled(plan, _volume(), overlap=0)
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    path = str(tmp_path / "full.npy")
    ctx = mp.get_context("spawn")
    procs = [ctx.Process(target=_rank_main, args=(r, world, port, path)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    got = np.load(path)
    assert got.shape == want.shape
    assert np.array_equal(got, want)


def test_run_tiled_two_workers_one_device_bit_identical():
    """run_tiled(devices=[cuda:0, cuda:0]): two host threads, two tilers on
    the same device, each streaming its block; equals the one-device run."""
    import paper_1903_07525_b200 as P
    plan = _net()
    vol = _volume()
    want = P.run_tiled(plan, vol, overlap=0)
    got = P.run_tiled(plan, vol, overlap=0, devices=["cuda:0", "cuda:0"])
    assert np.array_equal(got, want)
