"""Streamed fold (VXB_TC_STREAM=2) against the tiled fold walk on a few shapes."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1903_07525_b200 import device as D, ops as K  # noqa: E402

os.environ["VXB_PRINT"] = os.environ.get("VXB_PRINT", "0")


def run(x, w, b, pad, base, mode, pool=False):
    os.environ["VXB_TC_STREAM"] = mode
    xd = D.to_device_blocked(x)
    osp = tuple(s + 2 * p - k + 1 for s, p, k in zip(x.shape[2:], pad, w.shape[2:]))
    out = D.empty_blocked(x.shape[0], w.shape[0], osp)
    bd = D.to_device_blocked(base) if base is not None else None
    pk = K.pack_conv(w, b, base_scale=np.ones(w.shape[0], np.float32) if base is not None else None)
    K.conv3d(xd, pk, out, pad=pad, base=bd, fused_act=("elu", 1.0))
    torch.cuda.synchronize()
    return D.to_host_standard(out)


cases = [(1, 28, (18, 32, 16), (1, 1, 1)), (2, 28, (18, 20, 12), (1, 1, 1)),
         (1, 32, (32, 16, 16), (1, 1, 1)), (1, 16, (7, 16, 8), (1, 1, 1)),
         (1, 28, (20, 18, 10), (0, 0, 0)), (3, 8, (5, 33, 9), (1, 1, 1)),
         (1, 48, (18, 16, 16), (1, 1, 1)), (1, 64, (9, 16, 8), (1, 1, 1))]
for n, c, sp, pad in cases:
    rng = np.random.default_rng(c + sp[0])
    x = rng.uniform(-1, 1, (n, c) + sp).astype(np.float32)
    w = (rng.standard_normal((c, c, 3, 3, 3)) * 0.1).astype(np.float32)
    b = rng.standard_normal(c).astype(np.float32)
    osp = tuple(s + 2 * p - 2 for s, p in zip(sp, pad))
    for use_base in (False, True):
        base = rng.uniform(-1, 1, (n, c) + osp).astype(np.float32) if use_base else None
        ref = run(x, w, b, pad, base, "0")
        got = run(x, w, b, pad, base, "2")
        d = np.abs(got - ref).max()
        print("n %d c %d sp %s pad %s base %d: max |stream - tiled| %.3e (max |ref| %.2f)" % (
            n, c, sp, pad, use_base, d, np.abs(ref).max()), flush=True)
