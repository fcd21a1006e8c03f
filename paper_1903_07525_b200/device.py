"""Device-side blocked tensors and thin wrappers over the C ABI.

A ``DTensor`` is a view of one activation tensor in HBM.  The production
layout is the reference's channel-blocked layout (blocked.py:1-9) with
S = 8 lanes, stored as bf16: a torch tensor of shape
(batch, ceil(C/8), X, Y, Z, 8) whose last dim is contiguous.  Views may be
strided (crop windows, halo interiors, channel slices of a concat buffer);
the C ABI takes element strides.  Standard NCDHW fp32 tensors appear only
at the network boundary (``blocked=False``).

torch is used only as the HBM allocator and stream provider; every byte of
arithmetic runs in libvxb.so.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import ExecutionError, LayoutError

LANES = 8


def chunks(c: int) -> int:
    return -(-int(c) // LANES)


def _torch():
    import torch
    return torch


def current_stream_handle() -> int:
    torch = _torch()
    return torch.cuda.current_stream().cuda_stream


@dataclass
class DTensor:
    """A logical (n, c, x, y, z) tensor backed by a torch storage view."""

    t: object                 # torch.Tensor: 6-D blocked or 5-D standard view
    c: int                    # logical fmap count
    blocked: bool = True
    # split bf16 (VXB_BF16X2): t is (n, 2*ceil(C/8), x, y, z, 8) bf16 with
    # chunk 2j = hi plane and 2j+1 = lo plane of fmap chunk j
    split: bool = False

    @property
    def n(self) -> int:
        return int(self.t.shape[0])

    @property
    def spatial(self) -> tuple[int, int, int]:
        if self.blocked:
            return tuple(int(v) for v in self.t.shape[2:5])
        return tuple(int(v) for v in self.t.shape[2:5])

    @property
    def dims(self) -> tuple[int, int, int, int, int]:
        x, y, z = self.spatial
        return (self.n, self.c, x, y, z)

    @property
    def dtype_code(self) -> int:
        torch = _torch()
        if self.split:
            return _lib.VXB_BF16X2
        if self.t.dtype == torch.bfloat16:
            return _lib.VXB_BF16
        if self.t.dtype == torch.float32:
            return _lib.VXB_F32
        raise LayoutError("unsupported device dtype %s" % self.t.dtype)

    def vxb(self) -> _lib.VxbTensor:
        v = _lib.VxbTensor()
        v.data = self.t.data_ptr()
        v.dtype = self.dtype_code
        v.blocked = 1 if self.blocked else 0
        n, c, x, y, z = self.dims
        v.n, v.c, v.x, v.y, v.z = n, c, x, y, z
        st = self.t.stride()
        if self.blocked and st[5] != 1:
            raise LayoutError("blocked view must have a contiguous lane axis")
        for i in range(5):
            v.s[i] = int(st[i])
        if self.split:
            v.s[1] = 2 * int(st[1])      # one fmap chunk = a hi and a lo plane
        return v

    def window(self, lo, size) -> "DTensor":
        """Spatial sub-view [lo, lo+size) (crop), no copy."""
        sl = tuple(slice(int(a), int(a) + int(b)) for a, b in zip(lo, size))
        return DTensor(self.t[(slice(None), slice(None)) + sl], self.c, self.blocked, self.split)


def empty_blocked(n, c, spatial, dtype="bf16", device=None, zero=False) -> DTensor:
    """dtype: "bf16", "fp32" or "split" (hi + lo bf16 planes per chunk)."""
    torch = _torch()
    td = torch.float32 if dtype == "fp32" else torch.bfloat16
    x, y, z = (int(v) for v in spatial)
    planes = 2 if dtype == "split" else 1
    shape = (int(n), planes * chunks(c), x, y, z, LANES)
    dev = device or torch.device("cuda", torch.cuda.current_device())
    t = torch.zeros(shape, dtype=td, device=dev) if zero else torch.empty(shape, dtype=td, device=dev)
    return DTensor(t, int(c), True, dtype == "split")


def standard(t, c=None) -> DTensor:
    """Wrap a 5-D (n, c, x, y, z) torch tensor as a standard-layout view."""
    return DTensor(t, int(c if c is not None else t.shape[1]), False)


def null_tensor() -> _lib.VxbTensor:
    return _lib.VxbTensor()


def copy_windows(pairs, stream=None) -> None:
    """vxb_copy_windows: [(src, dst), ...] fp32 (n, c, x, y, z) torch views of
    equal shapes (z contiguous), moved in one launch per 16 pairs."""
    if not pairs:
        return
    L = _lib.lib()
    n = len(pairs)
    srcs, dsts = (_lib.VxbTensor * n)(), (_lib.VxbTensor * n)()
    for i, (a, b) in enumerate(pairs):
        srcs[i] = standard(a).vxb()
        dsts[i] = standard(b).vxb()
    _lib.check(L.vxb_copy_windows(srcs, dsts, n, stream or current_stream_handle()),
               "vxb_copy_windows")


def copy(src: DTensor, dst: DTensor, stream=None, independent=False) -> None:
    """vxb_copy; ``independent`` (vxb_copy_ex VXB_COPY_INDEPENDENT): the copy
    touches nothing the previous kernel in the stream does, so it may run
    beside that kernel (a network-input pack)."""
    L = _lib.lib()
    s, d = src.vxb(), dst.vxb()
    h = stream or current_stream_handle()
    if independent:
        _lib.check(L.vxb_copy_ex(ctypes.byref(s), ctypes.byref(d), _lib.COPY_INDEPENDENT, h),
                   "vxb_copy_ex")
    else:
        _lib.check(L.vxb_copy(ctypes.byref(s), ctypes.byref(d), h), "vxb_copy")


def pack_zwin_windows(windows, dst: DTensor, kz: int, pz: int, stream=None) -> None:
    """vxb_pack_zwin_windows: batch entry b of ``dst`` packed from the fp32
    (1, 1, x, y, z) torch view ``windows[b]`` (windows of one volume)."""
    L = _lib.lib()
    n = len(windows)
    srcs = (_lib.VxbTensor * n)()
    for i, w in enumerate(windows):
        srcs[i] = standard(w).vxb()
    d = dst.vxb()
    _lib.check(L.vxb_pack_zwin_windows(srcs, n, ctypes.byref(d), int(kz), int(pz),
                                       stream or current_stream_handle()),
               "vxb_pack_zwin_windows")


def pack_zwin(src: DTensor, dst: DTensor, kz: int, pz: int, stream=None,
              independent=False) -> None:
    """vxb_pack_zwin: z-window pack of a 1-channel fp32 input (lane l = z tap l)."""
    L = _lib.lib()
    s, d = src.vxb(), dst.vxb()
    flags = _lib.COPY_INDEPENDENT if independent else 0
    _lib.check(L.vxb_pack_zwin(ctypes.byref(s), ctypes.byref(d), int(kz), int(pz), flags,
                               stream or current_stream_handle()), "vxb_pack_zwin")


def zero(t: DTensor, stream=None) -> None:
    L = _lib.lib()
    v = t.vxb()
    _lib.check(L.vxb_zero(ctypes.byref(v), stream or current_stream_handle()), "vxb_zero")


def to_device_blocked(arr: np.ndarray, dtype="bf16", device=None) -> DTensor:
    """Standard (n, c, x, y, z) host array -> blocked device tensor (to_blocked)."""
    torch = _torch()
    arr = np.ascontiguousarray(np.asarray(arr, dtype=np.float32))
    if arr.ndim != 5:
        raise LayoutError("expected a rank-5 image, got rank %d" % arr.ndim)
    dev = device or torch.device("cuda", torch.cuda.current_device())
    src = standard(torch.from_numpy(arr).to(dev))
    out = empty_blocked(arr.shape[0], arr.shape[1], arr.shape[2:], dtype, dev)
    copy(src, out)
    return out


def to_host_standard(t: DTensor) -> np.ndarray:
    """Blocked device tensor -> standard fp32 host array (from_blocked)."""
    torch = _torch()
    n, c, x, y, z = t.dims
    out = torch.empty((n, c, x, y, z), dtype=torch.float32, device=t.t.device)
    copy(t, standard(out))
    return out.cpu().numpy()


def device_vector(vec, n=None, device=None):
    """fp32 per-fmap vector on the device (bias, base_scale, BN coefficients)."""
    torch = _torch()
    a = np.asarray(vec, dtype=np.float32).reshape(-1)
    if n is not None and a.shape[0] != n:
        raise ExecutionError("vector has %d entries, expected %d" % (a.shape[0], n))
    dev = device or torch.device("cuda", torch.cuda.current_device())
    return torch.from_numpy(np.ascontiguousarray(a)).to(dev)
