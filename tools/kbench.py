"""Kernel-only timing of the conv sweep layers (graph-captured launches)."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1903_07525_b200 import device as D, ops as K

dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
res = {}
only = os.environ.get("ONLY")
REPS = int(os.environ.get("REPS", "1"))
_act = os.environ.get("ACT", "elu")
FA = None if _act == "none" else (_act, 1.0)
F32OUT = os.environ.get("F32OUT") == "1"   # fp32 NCDHW output (the network-output epilogue)
spatial = tuple(int(v) for v in os.environ.get("SPATIAL", "32,128,128").split(","))
for k in ((3, 3, 3), (1, 3, 3)):
    for c in (8, 16, 32, 64, 128):
        name = "c%d_k%s" % (c, "".join(map(str, k)))
        if only and name not in only.split(","):
            continue
        rng = np.random.default_rng(c)
        x = D.empty_blocked(1, c, spatial)
        x.t.copy_(torch.randn(x.t.shape, device=dev).to(torch.bfloat16))
        x.t[..., (c % 8 or 8):] = 0 if c % 8 else x.t[..., 8:]
        out = (D.standard(torch.empty((1, c) + spatial, device=dev)) if F32OUT
               else D.empty_blocked(1, c, spatial))
        w = (rng.standard_normal((c, c) + k) * 0.05).astype(np.float32)
        pk = K.pack_conv(w, np.zeros(c, np.float32))
        pad = tuple(v // 2 for v in k)
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            K.conv3d(x, pk, out, pad=pad, fused_act=FA)
        s.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            K.conv3d(x, pk, out, pad=pad, fused_act=FA)
        flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)
        times = []
        for it in range(12):
            flush.fill_(it)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(s):
                torch.cuda._sleep(200_000)
                e0.record(s)
                for _ in range(REPS):
                    g.replay()
                e1.record(s)
            s.synchronize()
            times.append(e0.elapsed_time(e1) / REPS)
        ms = float(np.median(times[2:]))
        vox = int(np.prod(spatial))
        flops = 2.0 * c * c * int(np.prod(k)) * vox
        by = 2.0 * 2 * c * vox
        res[name] = {"us": ms * 1e3, "tflops": flops / ms / 1e9, "gbs": by / ms / 1e6}
        print(name, json.dumps(res[name]), flush=True)
tag = os.environ.get("TAG", "default")
os.makedirs("gpurun_out", exist_ok=True)
with open("gpurun_out/kbench_%s.json" % tag, "w") as fh:
    json.dump(res, fh)
