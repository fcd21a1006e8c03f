"""One network of a BASELINE config through PlanRunner.run_device (graph),
for launch lists: prints the lowered op order.  Usage: CFG=4 python tools/cfg_launches.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1903_07525_b200 as P  # noqa: E402
from paper_1903_07525_b200 import configs as C  # noqa: E402

cfg = int(os.environ.get("CFG", "4"))
dev = torch.device("cuda", 0)
spec, store = {1: C.config1, 3: C.config3, 4: C.config4, 5: C.config5}[cfg]()
plan, _ = P.compile_network(spec, store, fixpoint=True, fuse_deconv_add=True)
r = P.PlanRunner(plan, device=dev, fuse_pool=os.environ.get("FUSEPOOL", "1") == "1")
lo, hi = C.input_range(cfg)
x = C.make_input(spec, 0, lo, hi)
bufs = r.input_buffers()
bufs[plan.inputs[0][0]].copy_(torch.from_numpy(x))
for _ in range(int(os.environ.get("ITERS", "3"))):
    r.run_device(bufs)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda._sleep(200000)
r.stream.wait_stream(torch.cuda.current_stream())
e0.record(r.stream)
for _ in range(10):
    r.run_device(bufs)
e1.record(r.stream)
torch.cuda.synchronize()
print("config %d: %.3f ms per forward, %d launches" % (cfg, e0.elapsed_time(e1) / 10, r.launches))
for i, (kind, st, info) in enumerate(r._ops):
    print(i, kind.name, getattr(st, "name", ""), tuple(info["out"].dims))
