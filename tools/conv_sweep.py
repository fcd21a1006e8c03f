"""Time one conv shape under several tile choices (N path x slice cap).

Env: LAYERS = "cin:cout:kkk:x,y,z:batch[:base]" entries separated by ';'
     (default: the config-5 deep-level convs at 12 patches per launch),
     PATHS (comma list of auto,tc,unf,n128,n64,n32,n16), BXS (comma list),
     ITERS.  Prints us per launch (L2-warm back-to-back launches)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1903_07525_b200 import _lib, device as D, ops as K  # noqa: E402

DEFAULT = ";".join([
    "28:36:133:18,96,96:12", "36:36:333:18,96,96:12",
    "36:48:133:18,48,48:12", "48:48:333:18,48,48:12",
    "48:64:133:18,24,24:12", "64:64:333:18,24,24:12", "64:64:333:18,24,24:12:1",
    "64:80:133:18,12,12:12", "80:80:333:18,12,12:12", "80:80:333:18,12,12:12:1",
    "28:28:133:18,192,192:12",
])
PATHS = {"auto": 0, "tc": _lib.PATH_TC, "unf": _lib.PATH_TC_UNFOLDED, "n128": _lib.PATH_TC_N128,
         "n64": _lib.PATH_TC_N64, "n32": _lib.PATH_TC_N32, "n16": _lib.PATH_TC_N16}

dev = torch.device("cuda", 0)
iters = int(os.environ.get("ITERS", "20"))
paths = os.environ.get("PATHS", "auto,tc,n64,n32,unf").split(",")
bxs = os.environ.get("BXS", "8,6,4,3,2,1").split(",")
for spec in os.environ.get("LAYERS", DEFAULT).split(";"):
    f = spec.split(":")
    cin, cout, k = int(f[0]), int(f[1]), tuple(int(v) for v in f[2])
    sp = tuple(int(v) for v in f[3].split(","))
    nb = int(f[4])
    has_base = len(f) > 5 and f[5] == "1"
    rng = np.random.default_rng(0)
    x = D.to_device_blocked(rng.uniform(-1, 1, (nb, cin) + sp).astype(np.float32))
    out = D.empty_blocked(nb, cout, sp)
    base = D.to_device_blocked(rng.uniform(-1, 1, (nb, cout) + sp).astype(np.float32)) \
        if has_base else None
    w = (rng.standard_normal((cout, cin) + k) * 0.05).astype(np.float32)
    pad = tuple(v // 2 for v in k)
    res = []
    for pn in paths:
        try:
            pk = K.pack_conv(w, np.zeros(cout, np.float32),
                             base_scale=np.ones(cout, np.float32) if has_base else None,
                             path=PATHS[pn], out_shape=sp)
        except Exception as e:  # path not valid for this shape
            res.append("%s: %s" % (pn, str(e)[:40]))
            continue
        for bx in bxs:
            os.environ["VXB_TC_BX"] = bx
            try:
                for _ in range(2):
                    K.conv3d(x, pk, out, pad=pad, base=base, fused_act=("elu", 1.0))
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                for _ in range(iters):
                    K.conv3d(x, pk, out, pad=pad, base=base, fused_act=("elu", 1.0))
                e1.record()
                torch.cuda.synchronize()
                res.append("%s/bx%s %.1f" % (pn, bx, e0.elapsed_time(e1) / iters * 1e3))
            except Exception as e:
                res.append("%s/bx%s err" % (pn, bx))
    os.environ.pop("VXB_TC_BX", None)
    flops = 2.0 * cin * cout * np.prod(k) * nb * np.prod(sp)
    print("%s (%.1f GF):" % (spec, flops / 1e9))
    print("   " + "  ".join(res), flush=True)
