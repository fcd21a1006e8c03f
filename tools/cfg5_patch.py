"""One config-5 patch (BATCH patches per launch) through PlanRunner.run_device
(graph), for launch lists."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1903_07525_b200 as P
from paper_1903_07525_b200 import configs as C

dev = torch.device("cuda", 0)
spec, store = C.config5()
plan, _ = P.compile_network(spec, store, fixpoint=True, fuse_deconv_add=True)
B = int(os.environ.get("BATCH", "1"))          # patches per launch (plan.rebatch)
if B > 1:
    from paper_1903_07525_b200.plan import rebatch
    plan = rebatch(plan, B)
r = P.PlanRunner(plan, device=dev)
x = np.concatenate([C.make_input(spec, i, 0.0, 1.0) for i in range(B)], axis=0)
bufs = r.input_buffers()
bufs[plan.inputs[0][0]].copy_(torch.from_numpy(x))
for _ in range(int(os.environ.get("ITERS", "3"))):
    r.run_device(bufs)
torch.cuda.synchronize()
s = r.stream
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda._sleep(200000)
s.wait_stream(torch.cuda.current_stream())
e0.record(s)
for _ in range(20):
    r.run_device(bufs)
e1.record(s)
torch.cuda.synchronize()
print("patch ms %.3f launches %d" % (e0.elapsed_time(e1) / 20, r.launches))
for i, (kind, st, info) in enumerate(r._ops):
    print(i, kind.name, getattr(st, "name", None) or getattr(st, "layer", ""))
