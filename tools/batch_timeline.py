"""Timeline of the config-2 PlanBatch schedule without a graph: input packs on
a side stream (background priority, independent launches), each network's
body on the main stream after its pack, events around every piece.  Prints
start/end (us from the step start) of each pack and each body, and each
body's duration next to its duration when run alone."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1903_07525_b200 as P  # noqa: E402
from paper_1903_07525_b200 import configs as C  # noqa: E402

dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
runners = []
for k in C.SWEEP_K:
    for c in C.SWEEP_C:
        spec, store = C.config2(c, k)
        plan, _ = P.compile_network(spec, store, fixpoint=True)
        r = P.PlanRunner(plan, device=dev)
        for t in r.input_buffers().values():
            t.copy_(torch.rand(t.shape) * 2 - 1)
        r._indep_flag[0] = True
        runners.append(("c%d_k%s" % (c, "".join(map(str, k))), r))
batch = P.PlanBatch([r for _, r in runners])
order = batch.order
main, side = torch.cuda.Stream(), torch.cuda.Stream()
flush = torch.empty(512 * 1024 * 1024, dtype=torch.uint8, device=dev)


def ev():
    return torch.cuda.Event(enable_timing=True)


def run(timeline):
    flush.fill_(1)
    torch.cuda.synchronize()
    t0 = ev()
    cur = torch.cuda.current_stream()
    torch.cuda._sleep(500_000)
    t0.record(cur)
    main.wait_stream(cur)
    side.wait_stream(cur)
    rec = []
    done = []
    with torch.cuda.stream(side):
        for i in order:
            name, r = runners[i]
            a, b = ev(), ev()
            a.record(side)
            for c in r._calls[:r._n_in_calls]:
                c()
            b.record(side)
            done.append(b)
            rec.append((name, "pack", a, b))
    with torch.cuda.stream(main):
        for i, d in zip(order, done):
            name, r = runners[i]
            main.wait_event(d)
            a, b = ev(), ev()
            a.record(main)
            for c in r._calls[r._n_in_calls:]:
                c()
            b.record(main)
            rec.append((name, "body", a, b))
    cur.wait_stream(main)
    cur.wait_stream(side)
    torch.cuda.synchronize()
    return [(n, kind, t0.elapsed_time(a) * 1e3, t0.elapsed_time(b) * 1e3) for n, kind, a, b in rec]


def alone(r):
    ts = []
    for _ in range(5):
        flush.fill_(1)
        torch.cuda.synchronize()
        a, b = ev(), ev()
        with torch.cuda.stream(main):
            for c in r._calls[:r._n_in_calls]:
                c()
            main.synchronize()
            a.record(main)
            for c in r._calls[r._n_in_calls:]:
                c()
            b.record(main)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    return float(np.median(ts))


for _ in range(3):
    run(None)
res = run(None)
solo = {n: alone(r) for n, r in runners}
end = max(e for _, _, _, e in res)
print("step (no graph) %.1f us" % end)
for n, kind, s, e in res:
    extra = "  alone %.1f" % solo[n] if kind == "body" else ""
    print("%-10s %-4s %8.1f -> %8.1f  (%.1f us)%s" % (n, kind, s, e, e - s, extra))
