"""Flushed step time of configs 1/3/4 under runner options (FUSE_INPUT=1) and
the library's env knobs (set by the caller): one line per run."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1903_07525_b200 as P  # noqa: E402
from bench_util import build_nets  # noqa: E402

cfg = int(os.environ.get("CFG", "1"))
dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
name, spec, store, x = build_nets(cfg)[0]
plan, _ = P.compile_network(spec, store, fixpoint=True, fuse_deconv_add=True)
kw = {}
if os.environ.get("FUSE_INPUT") == "1":
    kw["fuse_input"] = True
r = P.PlanRunner(plan, backend="b200", device=dev, **kw)
xd = r.input_buffers()
xd[plan.inputs[0][0]].copy_(torch.from_numpy(x))
flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
cs = torch.cuda.current_stream(dev)
for _ in range(5):
    r.run_device(r.input_buffers())
torch.cuda.synchronize()
ts = []
for it in range(30):
    flush.fill_(1.0)
    torch.cuda.synchronize()
    torch.cuda._sleep(200_000)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(cs)
    r.run_device(r.input_buffers())
    e1.record(cs)
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1) * 1e3)
warm = []
for it in range(30):
    torch.cuda._sleep(200_000)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(cs)
    r.run_device(r.input_buffers())
    e1.record(cs)
    torch.cuda.synchronize()
    warm.append(e0.elapsed_time(e1) * 1e3)
print("cfg%d %s launches %d: flushed median %.1f us (min %.1f)  warm median %.1f us" % (
    cfg, os.environ.get("TAG", ""), r.launches, np.median(ts), min(ts), np.median(warm)), flush=True)
