"""Driver for the reference's own compiled conv kernel — TEST INFRASTRUCTURE ONLY.

``oracle/_ref/_kernels*.so`` is the reference's ``_kernels.pyx`` + ``convcore.h``
(pkg/src/voxplan/_kernels.pyx:44-179, convcore.h:19-52) compiled from its own
sources by ``oracle/build_ref.sh``.  This module restates, on the host, the
marshalling the reference runtime does around that kernel for one conv step
(executor._bind_conv executor.py:134-164, kernels_cy.conv3d kernels_cy.py:30-57,
ops.pad_copy ops.py:105-110, blocked.to_blocked/from_blocked blocked.py:209-231)
so the CPU baseline times the reference's real inner loop.

Parallelism mirrors the reference's only mechanism, independent patches on a
thread pool (tiling.py:189-237): the output is cut into x-slabs, each slab is
one ``_kernels.conv3d`` call on its input window; the kernel releases the GIL
(_kernels.pyx:94) so slabs run on separate cores.
"""

from __future__ import annotations

import glob
import importlib.util
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np

REF_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_ref")
ACT_CODE = {None: 0, "relu": 1, "elu": 2, "sigmoid": 3}
_MOD = None


def available() -> bool:
    return bool(glob.glob(os.path.join(REF_DIR, "_kernels*.so")))


def kernels():
    global _MOD
    if _MOD is None:
        paths = glob.glob(os.path.join(REF_DIR, "_kernels*.so"))
        if not paths:
            raise RuntimeError("oracle/_ref not built (run oracle/build_ref.sh)")
        spec = importlib.util.spec_from_file_location("_kernels", paths[0])
        mod = importlib.util.module_from_spec(spec)
        spec.loader.exec_module(mod)
        _MOD = mod
    return _MOD


def to_blocked(std, simd=8):
    """standard (b, f, x, y, z) -> (b, ceil(f/S), x, y, z, S), tails zero."""
    b, f, x, y, z = std.shape
    nb = -(-f // simd)
    lifted = np.zeros((b, nb * simd, x, y, z), np.float32)
    lifted[:, :f] = std
    return np.ascontiguousarray(lifted.reshape(b, nb, simd, x, y, z).transpose(0, 1, 3, 4, 5, 2))


def from_blocked(view, fmaps):
    b, nb, x, y, z, s = view.shape
    return np.ascontiguousarray(view.transpose(0, 1, 5, 2, 3, 4).reshape(b, nb * s, x, y, z)[:, :fmaps])


def lane_kernel(w, simd=8):
    """(fo, fi, k...) -> (OB, IB, kx, ky, kz, in_lane, out_lane), C-contiguous
    (blocked.kernel_to_blocked + kernels_cy._lane_kernel)."""
    fo, fi, kx, ky, kz = w.shape
    ob, ib = -(-fo // simd), -(-fi // simd)
    lifted = np.zeros((ob * simd, ib * simd, kx, ky, kz), np.float32)
    lifted[:fo, :fi] = w
    seven = lifted.reshape(ob, simd, ib, simd, kx, ky, kz).transpose(0, 2, 4, 5, 6, 3, 1)
    return np.ascontiguousarray(seven)


class ConvStep:
    """One bound conv step of the reference engine, reusable across runs."""

    def __init__(self, w, bias, pad=(0, 0, 0), act=None, alpha=1.0, base_scale=None,
                 simd=8, patch=(4, 4, 8)):
        self.w = np.asarray(w, np.float32)
        self.fo, self.fi = self.w.shape[:2]
        self.k = self.w.shape[2:]
        self.pad = tuple(pad)
        self.simd = simd
        self.kt = lane_kernel(self.w, simd)
        ob = self.kt.shape[0]
        self.bias = np.zeros(ob * simd, np.float32)
        self.bias[:self.fo] = np.asarray(bias, np.float32)
        self.scale = None
        if base_scale is not None:
            self.scale = np.zeros(ob * simd, np.float32)
            self.scale[:self.fo] = np.asarray(base_scale, np.float32)
        self.code = ACT_CODE[act]
        self.alpha = float(alpha)
        self.patch = tuple(int(p) for p in patch)

    def prepare(self, x_std):
        """Pad step + to_blocked (done once per run in the reference)."""
        px, py, pz = self.pad
        xp = np.pad(np.asarray(x_std, np.float32), ((0, 0), (0, 0), (px, px), (py, py), (pz, pz)))
        return to_blocked(xp, self.simd)

    def run_blocked(self, xb, out_b, base_b=None, x_range=None):
        """Compute output x rows [x0, x1) into out_b (blocked, full extent)."""
        kx = self.k[0]
        ox = out_b.shape[2]
        x0, x1 = x_range or (0, ox)
        inp = np.ascontiguousarray(xb[:, :, x0:x1 + kx - 1])
        out = out_b[:, :, x0:x1]
        additive = base_b is not None
        base = np.ascontiguousarray(base_b[:, :, x0:x1]) if additive else inp
        scale = self.scale if (additive and self.scale is not None) else self.bias
        k = kernels()
        k.conv3d(inp, self.kt, self.bias, out, base, scale, additive,
                 additive and self.scale is not None, 1, 1, 1,
                 self.patch[0], self.patch[1], self.patch[2], self.code, self.alpha)

    def __call__(self, x_std, base_std=None, threads=1, x_range=None):
        xb = self.prepare(x_std)
        n, _, X, Y, Z, s = xb.shape
        ox, oy, oz = X - self.k[0] + 1, Y - self.k[1] + 1, Z - self.k[2] + 1
        out = np.zeros((n, -(-self.fo // s), ox, oy, oz, s), np.float32)
        base_b = to_blocked(np.asarray(base_std, np.float32), s) if base_std is not None else None
        lo, hi = x_range or (0, ox)
        if threads <= 1:
            self.run_blocked(xb, out, base_b, (lo, hi))
        else:
            cuts = np.linspace(lo, hi, threads + 1).astype(int)
            with ThreadPoolExecutor(max_workers=threads) as pool:
                list(pool.map(lambda i: self.run_blocked(xb, out, base_b, (cuts[i], cuts[i + 1])),
                              [i for i in range(threads) if cuts[i + 1] > cuts[i]]))
        tail = self.fo % s
        if tail:
            out[:, -1, ..., tail:] = 0  # ops.zero_tail (ops.py:18-23)
        return from_blocked(out[:, :, lo:hi], self.fo)
