"""Per-CTA timeline of one conv3d_tc launch (VXB_TC_DEBUG globaltimer marks)."""
import os
import sys

import numpy as np
import torch

os.environ["VXB_TC_DEBUG"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1903_07525_b200 import _lib, device as D, ops as K

dev = torch.device("cuda", 0)
spatial = tuple(int(v) for v in os.environ.get("SPATIAL", "32,128,128").split(","))
_act = os.environ.get("ACT", "elu")
FA = None if _act == "none" else (_act, 1.0)
for case in os.environ.get("CASES", "8:333,16:333,32:333").split(","):
    parts = case.split(":")             # C:KKK or CIN:COUT:KKK
    c = int(parts[0])
    cout = int(parts[1]) if len(parts) == 3 else c
    ks = parts[-1]
    k = tuple(int(v) for v in ks)
    x = D.empty_blocked(1, c, spatial)
    x.t.copy_(torch.randn(x.t.shape, device=dev).to(torch.bfloat16))
    if os.environ.get("ZERO_INPUT"):
        x.t.zero_()
    if os.environ.get("F32IN"):
        x = D.standard(torch.randn((1, c) + spatial, device=dev))
    out = D.empty_blocked(1, cout, spatial)
    base = None
    if os.environ.get("BASE") == "1":        # residual operand (the c2 convs of config 5)
        base = D.empty_blocked(1, cout, spatial)
        base.t.copy_(torch.randn(base.t.shape, device=dev).to(torch.bfloat16))
    w = (np.random.default_rng(0).standard_normal((cout, c) + k) * 0.05).astype(np.float32)
    pk = K.pack_conv(w, np.zeros(cout, np.float32),
                     base_scale=np.ones(cout, np.float32) if base is not None else None)
    pad = tuple(v // 2 for v in k)
    for _ in range(3):
        K.conv3d(x, pk, out, pad=pad, fused_act=FA, base=base)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        K.conv3d(x, pk, out, pad=pad, fused_act=FA, base=base)
    e1.record()
    torch.cuda.synchronize()
    ev_us = e0.elapsed_time(e1) / 10 * 1e3
    buf = np.zeros(1024 * 64 * 8, np.uint64)
    _lib.lib().vxb_debug_read(buf.ctypes.data, buf.size)
    t = buf.reshape(1024, 64, 8).astype(np.int64)
    ctas = np.nonzero(t[:, 0, 5] > 0)[0]
    t = t[ctas]
    t0 = t[:, 0, 5].min()
    used = t[:, :, 0] > 0
    rel = np.where(t > 0, t - t0, -1)
    ntile = used.sum(1)
    print("== C%d k%s: event %.1f us, ctas %d, tiles/cta min %d max %d" % (
        c, ks, ev_us, len(ctas), ntile.min(), ntile.max()))
    print("  span start->end %.2f us; start spread %.2f us; end spread %.2f" % (
        rel[:, 0, 6].max() / 1e3, rel[:, 0, 5].max() / 1e3,
        (rel[:, 0, 6].max() - rel[:, 0, 6].min()) / 1e3))
    print("  setup (start->first TMA) mean %.2f us" % ((rel[:, 0, 0] - rel[:, 0, 5]).mean() / 1e3))
    for nm, a, b in (("tma issue->A landed", 0, 1), ("landed->MMA committed", 1, 2),
                     ("committed->epi start", 2, 3), ("epilogue", 3, 4), ("epi first tmem ld", 3, 7),
                     ("epi after first ld", 7, 4)):
        d = (rel[:, :, b] - rel[:, :, a])[used & (rel[:, :, b] >= 0)]
        print("  %-24s mean %7.2f us  p50 %7.2f  max %7.2f" % (nm, d.mean() / 1e3,
                                                              np.median(d) / 1e3, d.max() / 1e3))
    if int(os.environ.get("VXB_TC_DBGMODE", "0")) & 1024:
        g0 = (rel[:, :, 7] - rel[:, :, 1])[used & (rel[:, :, 7] >= 0)]
        g1 = (rel[:, :, 2] - rel[:, :, 7])[used & (rel[:, :, 7] >= 0)]
        print("  group0 %.2f us  group1 %.2f us" % (g0.mean() / 1e3, g1.mean() / 1e3))
    ck = (t[:, 1:, 6] - t[:, 1:, 5]).astype(np.float64)
    ns = (t[:, 1:, 2] - t[:, 1:, 1]).astype(np.float64)
    ok = used[:, 1:] & (t[:, 1:, 5] > 0) & (t[:, 1:, 6] > 0) & (ns > 0)
    if ok.any():
        print("  SM clock during MMA issue: %.0f MHz" % (ck[ok].sum() / ns[ok].sum() * 1e3))
    d = (rel[:, 1:, 1] - rel[:, :-1, 2])[used[:, 1:]]
    print("  MMA idle between tiles  mean %7.2f us" % (d.mean() / 1e3))
    last = np.array([rel[i, ntile[i] - 1, 4] for i in range(len(ctas))])
    print("  last epi end -> cta end mean %.2f us" % ((rel[:, 0, 6] - last).mean() / 1e3))
    i = int(np.argmax(ntile))
    print("  cta %d timeline (us):" % i,
          [tuple((rel[i, j, :5] / 1e3).round(1)) for j in range(min(ntile[i], 6))])
