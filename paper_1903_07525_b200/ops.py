"""Functional layer over the C ABI: packed weights + one call per plan step.

Each function here is the device counterpart of one reference callable
(cited per function).  Arguments are ``DTensor`` views; launches go to the
current torch CUDA stream.  Nothing here falls back to the CPU.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib
from .device import DTensor, current_stream_handle, device_vector, null_tensor
from .errors import ExecutionError

_ACT = _lib.ACT_CODE


def _act(fused_act):
    if fused_act is None:
        return 0, 0.0
    kind, alpha = fused_act
    if kind not in _ACT:
        raise ExecutionError("unknown activation %r" % (kind,))
    return _ACT[kind], float(alpha)


@dataclass
class PackedConv:
    """A conv's weights packed once per bind for the chosen kernel path.

    Replaces blocked.kernel_to_blocked + kernels_cy._lane_kernel
    (blocked.py:260-278, kernels_cy.py:22-27): the reference transposes the
    kernel into lane order once per invocation; here the host packs it into
    the tensor-core slab layout (bf16) or the CUDA-core layout (fp32).
    """

    w: object            # torch uint8 device buffer
    bias: object         # torch fp32 device [cout]
    scale: object        # torch fp32 device [cout] or None
    cin0: int
    cin1: int
    cout: int
    k: tuple
    stride: tuple
    path: int
    prec: int = 0        # _lib.PREC_BF16 / PREC_X3 (split-bf16 inputs)

    @property
    def cin(self) -> int:
        return self.cin0 + self.cin1


PRECISIONS = {"bf16": _lib.PREC_BF16, "x3": _lib.PREC_X3}


def pack_conv(kernel, bias, *, stride=(1, 1, 1), base_scale=None, cin_split=None,
              path=0, out_shape=None, batch=1, device=None, precision="bf16") -> PackedConv:
    """Pack a standard (cout, cin, kx, ky, kz) fp32 kernel bank for vxb_conv3d.
    ``out_shape`` (x, y, z) of the output, when known, lets the library pick
    the tile layout (vxb_conv_select_shape_b, ``batch`` volumes per launch).
    ``precision="x3"`` packs for a
    split-bf16 input: bf16(W) against its hi and lo planes and
    bf16(W - bf16(W)) against hi (VXB_PREC_X3)."""
    import torch
    L = _lib.lib()
    w = np.ascontiguousarray(np.asarray(kernel, dtype=np.float32))
    if w.ndim != 5:
        raise ExecutionError("conv kernel must be rank 5 (cout, cin, kx, ky, kz)")
    cout, cin = int(w.shape[0]), int(w.shape[1])
    k = tuple(int(v) for v in w.shape[2:])
    cin0 = cin if cin_split is None else int(cin_split)
    cin1 = cin - cin0
    stride = tuple(int(s) for s in stride)
    if path == 0:
        if out_shape is not None:
            path = L.vxb_conv_select_shape_b(cin, cout, _lib.i3(k), _lib.i3(stride),
                                             _lib.i3(tuple(out_shape)), int(batch))
        else:
            path = L.vxb_conv_select(cin, cout, _lib.i3(k), _lib.i3(stride))
    if cin1 and path not in _lib.TC_PATHS:
        raise ExecutionError("a two-input (fused concat) conv needs the tensor-core path")
    prec = PRECISIONS[precision]
    nbytes = L.vxb_conv_weights_bytes3(cin0, cin1, cout, _lib.i3(k), _lib.i3(stride), path, prec)
    host = np.zeros(max(nbytes, 1), dtype=np.uint8)
    _lib.check(L.vxb_conv_pack_weights3(w.ctypes.data, cin0, cin1, cout, _lib.i3(k),
                                        _lib.i3(stride), path, prec, host.ctypes.data, nbytes),
               "vxb_conv_pack_weights3")
    dev = device or torch.device("cuda", torch.cuda.current_device())
    scale = None if base_scale is None else device_vector(base_scale, cout, dev)
    return PackedConv(torch.from_numpy(host).to(dev), device_vector(bias, cout, dev), scale,
                      cin0, cin1, cout, k, stride, path, prec)


@dataclass
class Head:
    """A 1x1x1 conv fused into the producing conv's epilogue (vxb_conv_desc
    head_*): w (cout_h, cin) and b on the device, its fused activation."""
    w: object
    b: object
    cout: int
    act: tuple = None


def make_head(kernel, bias, fused_act=None, device=None) -> Head:
    w = np.asarray(kernel, np.float32)
    cout = int(w.shape[0])
    return Head(device_vector(w.reshape(-1), device=device), device_vector(bias, cout, device),
                cout, fused_act)


def conv3d(x: DTensor, pk: PackedConv, out: DTensor, *, pad=(0, 0, 0), base: DTensor = None,
           fused_act=None, x2: DTensor = None, off=(0, 0, 0), off2=(0, 0, 0),
           pool_out: DTensor = None, head: Head = None, head_out: DTensor = None,
           stream=None) -> None:
    """Fused conv step (kernels_cy.conv3d -> _kernels.conv3d, _kernels.pyx:44-179).
    ``pool_out`` (n, cout, x, y/2, z/2): also write the 1x2x2 max pool of the
    stored output (the following MaxPool step, ops.py:63-86, fused).
    ``head`` / ``head_out``: the network's next 1x1x1 conv computed in this
    conv's epilogue into the fp32 NCDHW ``head_out`` (``out`` is not written)."""
    L = _lib.lib()
    d = _lib.VxbConvDesc()
    d.in0 = x.vxb()
    d.in1 = x2.vxb() if x2 is not None else null_tensor()
    d.off0 = _lib.i3(off)
    d.off1 = _lib.i3(off2)
    d.out = out.vxb()
    d.base = base.vxb() if base is not None else null_tensor()
    d.w_packed = pk.w.data_ptr()
    d.bias = pk.bias.data_ptr()
    d.base_scale = pk.scale.data_ptr() if (pk.scale is not None and base is not None) else None
    d.cin, d.cout = pk.cin, pk.cout
    d.k = _lib.i3(pk.k)
    d.stride = _lib.i3(pk.stride)
    d.pad = _lib.i3(pad)
    d.act, d.alpha = _act(fused_act)
    d.path = pk.path
    d.prec = pk.prec
    if pool_out is not None:
        d.pool_mode = 1
        d.pool_out = pool_out.vxb()
    if head is not None:
        d.head_w = head.w.data_ptr()
        d.head_b = head.b.data_ptr()
        d.head_cout = head.cout
        d.head_act, d.head_alpha = _act(head.act)
        d.head_out = head_out.vxb()
    _lib.check(L.vxb_conv3d(ctypes.byref(d), stream or current_stream_handle()), "vxb_conv3d")


def conv3d_subimage(x: DTensor, w_std_dev, bias_dev, out: DTensor, *, cin, cout, k, stride,
                    in_block, out_block, origin, extent, first, last, base: DTensor = None,
                    scale_dev=None, fused_act=None, stream=None) -> None:
    """Sub-image primitive (kernels_py.subimage / _kernels.subimage, _kernels.pyx:182-271)."""
    L = _lib.lib()
    d = _lib.VxbConvDesc()
    d.in0 = x.vxb()
    d.in1 = null_tensor()
    d.out = out.vxb()
    d.base = base.vxb() if base is not None else null_tensor()
    d.bias = bias_dev.data_ptr()
    d.base_scale = scale_dev.data_ptr() if scale_dev is not None else None
    d.cin, d.cout = int(cin), int(cout)
    d.k = _lib.i3(k)
    d.stride = _lib.i3(stride)
    d.act, d.alpha = _act(fused_act)
    _lib.check(L.vxb_conv3d_subimage(ctypes.byref(d), w_std_dev.data_ptr(), int(in_block),
                                     int(out_block), _lib.i3(origin), _lib.i3(extent),
                                     int(bool(first)), int(bool(last)),
                                     stream or current_stream_handle()),
               "vxb_conv3d_subimage")


@dataclass
class PackedDeconv:
    w: object
    bias: object
    scale: object
    cin: int
    cout: int
    k: tuple
    stride: tuple
    path: int = 0
    prec: int = 0


def pack_deconv(kernel, bias, *, stride, base_scale=None, force_gather=False,
                device=None, precision="bf16") -> PackedDeconv:
    """Pack a (cout, cin, kx, ky, kz) deconv bank (oracle.py:67-93 orientation)."""
    import torch
    L = _lib.lib()
    w = np.ascontiguousarray(np.asarray(kernel, dtype=np.float32))
    cout, cin = int(w.shape[0]), int(w.shape[1])
    k = tuple(int(v) for v in w.shape[2:])
    stride = tuple(int(s) for s in stride)
    path = _lib.PATH_DIRECT if force_gather else 0
    prec = PRECISIONS[precision]
    nbytes = L.vxb_deconv_weights_bytes3(cin, cout, _lib.i3(k), _lib.i3(stride), path, prec)
    host = np.zeros(nbytes, dtype=np.uint8)
    _lib.check(L.vxb_deconv_pack_weights3(w.ctypes.data, cin, cout, _lib.i3(k), _lib.i3(stride),
                                          path, prec, host.ctypes.data, nbytes),
               "vxb_deconv_pack_weights3")
    dev = device or torch.device("cuda", torch.cuda.current_device())
    scale = None if base_scale is None else device_vector(base_scale, cout, dev)
    return PackedDeconv(torch.from_numpy(host).to(dev), device_vector(bias, cout, dev), scale,
                        cin, cout, k, stride, path, prec)


def deconv3d(x: DTensor, pk: PackedDeconv, out: DTensor, *, base: DTensor = None,
             fused_act=None, stream=None) -> None:
    """Transposed conv (kernels_py.deconv3d, kernels_py.py:162-196), optional fused skip-add."""
    L = _lib.lib()
    d = _lib.VxbDeconvDesc()
    d.in_ = x.vxb()
    d.out = out.vxb()
    d.base = base.vxb() if base is not None else null_tensor()
    d.w_packed = pk.w.data_ptr()
    d.bias = pk.bias.data_ptr()
    d.base_scale = pk.scale.data_ptr() if (pk.scale is not None and base is not None) else None
    d.cin, d.cout = pk.cin, pk.cout
    d.k = _lib.i3(pk.k)
    d.stride = _lib.i3(pk.stride)
    d.act, d.alpha = _act(fused_act)
    d.path = pk.path
    d.prec = pk.prec
    _lib.check(L.vxb_deconv3d(ctypes.byref(d), stream or current_stream_handle()), "vxb_deconv3d")


def pool3d(x: DTensor, out: DTensor, window, stride, mode="max", stream=None) -> None:
    """ops.pool (ops.py:63-86)."""
    L = _lib.lib()
    a, b = x.vxb(), out.vxb()
    _lib.check(L.vxb_pool3d(ctypes.byref(a), ctypes.byref(b), _lib.i3(window), _lib.i3(stride),
                            _lib.POOL_CODE[mode], stream or current_stream_handle()), "vxb_pool3d")


def eltwise(a: DTensor, b: DTensor, out: DTensor, op="add", stream=None) -> None:
    """ops.eltwise (ops.py:50-60)."""
    L = _lib.lib()
    va, vb, vo = a.vxb(), b.vxb(), out.vxb()
    _lib.check(L.vxb_eltwise(ctypes.byref(va), ctypes.byref(vb), ctypes.byref(vo),
                             _lib.ELT_CODE[op], stream or current_stream_handle()), "vxb_eltwise")


def affine_act(x: DTensor, out: DTensor, mult_dev=None, add_dev=None, act=None, alpha=1.0,
               stream=None) -> None:
    """ops.linear_transform / ops.activation (ops.py:89-102), fused."""
    L = _lib.lib()
    a, b = x.vxb(), out.vxb()
    code = _ACT[act] if act is not None else 0
    _lib.check(L.vxb_affine_act(ctypes.byref(a), ctypes.byref(b),
                                mult_dev.data_ptr() if mult_dev is not None else None,
                                add_dev.data_ptr() if add_dev is not None else None,
                                code, float(alpha), stream or current_stream_handle()),
               "vxb_affine_act")


def mergecrop(a: DTensor, b: DTensor, out: DTensor, stream=None) -> None:
    """ops.mergecrop (ops.py:113-136)."""
    L = _lib.lib()
    va, vb, vo = a.vxb(), b.vxb(), out.vxb()
    _lib.check(L.vxb_mergecrop(ctypes.byref(va), ctypes.byref(vb), ctypes.byref(vo),
                               stream or current_stream_handle()), "vxb_mergecrop")


def pad_copy(x: DTensor, out: DTensor, pads, stream=None) -> None:
    """ops.pad_copy (ops.py:105-110)."""
    L = _lib.lib()
    a, b = x.vxb(), out.vxb()
    _lib.check(L.vxb_pad_copy(ctypes.byref(a), ctypes.byref(b), _lib.i3(pads),
                              stream or current_stream_handle()), "vxb_pad_copy")
