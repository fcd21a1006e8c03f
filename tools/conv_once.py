"""A few launches of one conv shape (for ncu captures / quick timing).
Env: CIN, COUT, K (e.g. 133), SPATIAL (x,y,z), ACT, BASE=1 (residual operand),
F32OUT=1 (fp32 NCDHW output), X3=1 (split-bf16 precision), ITERS."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1903_07525_b200 import device as D, ops as K  # noqa: E402

dev = torch.device("cuda", 0)
cin = int(os.environ.get("CIN", "28"))
cout = int(os.environ.get("COUT", str(cin)))
k = tuple(int(v) for v in os.environ.get("K", "333"))
sp = tuple(int(v) for v in os.environ.get("SPATIAL", "72,192,192").split(","))
act = os.environ.get("ACT", "elu")
fa = None if act == "none" else (act, 1.0)
prec = "x3" if os.environ.get("X3") == "1" else "bf16"
dt = "split" if prec == "x3" else "bf16"
x = D.to_device_blocked(np.random.default_rng(0).uniform(-1, 1, (1, cin) + sp).astype(np.float32),
                        dtype=dt)
pad = tuple(v // 2 for v in k)
if os.environ.get("F32OUT") == "1":
    out = D.standard(torch.empty((1, cout) + sp, device=dev))
else:
    out = D.empty_blocked(1, cout, sp, dt)
base = None
if os.environ.get("BASE") == "1":
    base = D.to_device_blocked(np.random.default_rng(1).uniform(-1, 1, (1, cout) + sp)
                               .astype(np.float32), dtype=dt)
w = (np.random.default_rng(2).standard_normal((cout, cin) + k) * 0.05).astype(np.float32)
pk = K.pack_conv(w, np.zeros(cout, np.float32), base_scale=np.ones(cout, np.float32)
                 if base is not None else None, precision=prec, out_shape=sp)
n = int(os.environ.get("ITERS", "5"))
for _ in range(2):
    K.conv3d(x, pk, out, pad=pad, base=base, fused_act=fa)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(n):
    K.conv3d(x, pk, out, pad=pad, base=base, fused_act=fa)
e1.record()
torch.cuda.synchronize()
print("cin %d cout %d k %s sp %s base %s: %.1f us/launch" % (cin, cout, k, sp, base is not None,
                                                           e0.elapsed_time(e1) / n * 1e3))
