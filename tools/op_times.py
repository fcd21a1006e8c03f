"""Per-op device times of one config-5 patch batch, launched op by op with
events between ops (no graph), vs the same batch as one graph: how much of
the batch is kernel-boundary overhead."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1903_07525_b200 as P
from paper_1903_07525_b200 import configs as C
from paper_1903_07525_b200.plan import rebatch

dev = torch.device("cuda", 0)
B = int(os.environ.get("BATCH", "36"))
spec, store = C.config5()
plan, _ = P.compile_network(spec, store, fixpoint=True, fuse_deconv_add=True)
plan = rebatch(plan, B)
pdl = os.environ.get("PDL", "0") == "1"
r = P.PlanRunner(plan, device=dev, pdl=pdl)
x = np.concatenate([C.make_input(spec, i, 0.0, 1.0) for i in range(B)], axis=0)
bufs = r.input_buffers()
bufs[plan.inputs[0][0]].copy_(torch.from_numpy(x))
for _ in range(2):
    r.run_device(bufs)
torch.cuda.synchronize()
# graph timing
s = r.stream
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.wait_stream(torch.cuda.current_stream())
e0.record(s)
for _ in range(5):
    r.run_device(bufs)
e1.record(s)
torch.cuda.synchronize()
g_ms = e0.elapsed_time(e1) / 5
# op by op
L = P._lib if hasattr(P, "_lib") else None
from paper_1903_07525_b200 import _lib
lib = _lib.lib()
prev = lib.vxb_set_pdl(int(pdl))
evs = [torch.cuda.Event(enable_timing=True) for _ in range(len(r._calls) + 1)]
with torch.cuda.stream(s):
    for _ in range(2):
        evs[0].record(s)
        for i, c in enumerate(r._calls):
            c()
            evs[i + 1].record(s)
torch.cuda.synchronize()
lib.vxb_set_pdl(prev)
ops = [evs[i].elapsed_time(evs[i + 1]) for i in range(len(r._calls))]
names = ["input"] * r._n_in_calls + r.op_names + ["out"] * (len(r._calls) - r._n_in_calls - len(r.op_names))
print("graph %.3f ms; op by op total %.3f ms (sum of ops %.3f)" % (g_ms, evs[0].elapsed_time(evs[-1]), sum(ops)))
for n, t in zip(names, ops):
    print("  %-12s %8.1f us" % (n, t * 1e3))
