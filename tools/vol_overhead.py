"""Config-5 volume step vs its parts: 24 back-to-back batch graphs with no
gather/scatter, the gathers/scatters alone, and DeviceTiler.run."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1903_07525_b200 as P
from paper_1903_07525_b200 import configs as C, tiling

dev = torch.device("cuda", 0)
spec, store = C.config5()
plan, _ = P.compile_network(spec, store, fixpoint=True, fuse_deconv_add=True)
grid = P.grid_for(plan, C.VOLUME5, overlap=0)
dt = tiling.DeviceTiler(plan, grid, dev)
tiles = list(grid.tiles)
lo, hi, olo, ohi = dt.slab_bounds(tiles)
slab = torch.rand((1, 1) + tuple(b - a for a, b in zip(lo, hi)), device=dev)
out_slab = torch.empty((1, dt.out_fmaps) + tuple(b - a for a, b in zip(olo, ohi)), device=dev)
dt.bind_slabs(slab, lo, out_slab, olo)
flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
r = dt.runner
xin = r._in_std[dt.in_name]
nb = -(-len(tiles) // dt.batch)


def timed(fn, n=5):
    ts = []
    for _ in range(n):
        flush.fill_(1)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return float(np.median(ts))


for _ in range(2):
    dt.run(tiles)
torch.cuda.synchronize()
cs = torch.cuda.current_stream()


def graphs_only():
    r.stream.wait_stream(cs)
    for _ in range(nb):
        r.run_on_stream({dt.in_name: xin})
    cs.wait_stream(r.stream)


print("dt.run(all tiles)          %.2f ms" % timed(lambda: dt.run(tiles)))
print("%d graph replays only      %.2f ms" % (nb, timed(graphs_only)))
os.environ["VOXPLAN_DEBUG_NOCOPY"] = "1"
print("dt.run, no gather/scatter  %.2f ms" % timed(lambda: dt.run(tiles)))
os.environ.pop("VOXPLAN_DEBUG_NOCOPY")
