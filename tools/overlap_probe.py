"""Can the fp32 -> bf16 input pack of one network run beside the conv of
another?  The persistent conv leaves one CTA's worth of registers per SM; a
pack launched after it on a second stream can fill that slot.  Prints conv
alone, pack alone, both serialised and both overlapped (us)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1903_07525_b200 import device as D, ops as K

dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
spatial = (32, 128, 128)
sa, sb = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=10):
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)
    ts = []
    for it in range(reps + 2):
        flush.fill_(it)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        cur = torch.cuda.current_stream()
        e0.record(cur)
        sa.wait_stream(cur)
        sb.wait_stream(cur)
        fn()
        cur.wait_stream(sa)
        cur.wait_stream(sb)
        e1.record(cur)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    return float(np.median(ts[2:]))


for c, k in ((128, (3, 3, 3)), (128, (1, 3, 3)), (64, (3, 3, 3)), (32, (3, 3, 3)), (16, (3, 3, 3))):
    xf = D.standard(torch.rand((1, c) + spatial, device=dev))
    xb = D.empty_blocked(1, c, spatial)
    xin = D.empty_blocked(1, c, spatial)
    xin.t.copy_(torch.randn(xin.t.shape, device=dev).to(torch.bfloat16))
    out = D.empty_blocked(1, c, spatial)
    w = (np.random.default_rng(0).standard_normal((c, c) + k) * 0.05).astype(np.float32)
    pk = K.pack_conv(w, np.zeros(c, np.float32))
    pad = tuple(v // 2 for v in k)

    def conv(s):
        with torch.cuda.stream(s):
            K.conv3d(xin, pk, out, pad=pad, fused_act=("elu", 1.0))

    def pack(s):
        with torch.cuda.stream(s):
            D.copy(xf, xb, stream=s.cuda_stream)

    t_conv = timed(lambda: conv(sa))
    t_pack = timed(lambda: pack(sa))
    t_ser = timed(lambda: (conv(sa), pack(sa)))
    t_ovl = timed(lambda: (conv(sa), pack(sb)))
    print("C%d k%s: conv %.1f  pack %.1f  serial %.1f  overlapped %.1f" %
          (c, "".join(map(str, k)), t_conv, t_pack, t_ser, t_ovl), flush=True)
