"""The B200 kernel module behind the plugin boundary (reference twins:
kernels_cy.py:1-73 and kernels_py.py:1-196).

``ConvInvocation`` / ``SubImageTask`` have the reference's fields.  Their
views may be

* numpy arrays in the reference's blocked layout (B, blocks, X, Y, Z, S) with
  any S in {1,2,4,8,16,32} — what the reference's own ``PlanRunner`` passes
  when this module is registered as one of its backends.
  Operands are moved to HBM, the step runs on the GPU, the result is written
  back into ``out_view`` (interior only, tail lanes zeroed) — so a reference
  runner gets the B200 kernels without any other change;
* ``DTensor`` device views, for callers that keep data resident.

``precision="bf16"`` runs the tensor-core path; ``"fp32"`` runs the fp32
CUDA-core path (reference arithmetic to ~1e-6).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from . import ops as K
from .device import DTensor, empty_blocked, standard
from .errors import ExecutionError


@dataclass
class ConvInvocation:
    """Everything one convolution or deconvolution step needs (kernels_py.py:24-44)."""

    in_view: object
    in_fmaps: int
    kernel: object
    bias: object
    out_view: object
    out_fmaps: int
    stride: tuple = (1, 1, 1)
    additive: bool = False
    base_view: object = None
    base_scale: object = None
    fused_act: tuple = None
    patch_extent: tuple = None


@dataclass(frozen=True)
class SubImageTask:
    """One sub-image application: input block -> patch of an output block (kernels_py.py:47-56)."""

    in_block: int
    out_block: int
    origin: tuple
    extent: tuple
    first: bool
    last: bool


# ------------------------------------------------------------ layout helpers

def blocked_np_to_standard(view: np.ndarray, fmaps: int) -> np.ndarray:
    """(B, blocks, X, Y, Z, S) -> (B, fmaps, X, Y, Z) fp32 (blocked.from_blocked)."""
    b, nb, x, y, z, s = view.shape
    std = np.ascontiguousarray(view).transpose(0, 1, 5, 2, 3, 4).reshape(b, nb * s, x, y, z)
    return np.ascontiguousarray(std[:, :fmaps], dtype=np.float32)


def standard_to_blocked_np(std: np.ndarray, out_view: np.ndarray) -> None:
    """Write a standard image into a blocked (possibly strided) view, tails zero."""
    b, nb, x, y, z, s = out_view.shape
    f = std.shape[1]
    lifted = np.zeros((b, nb * s, x, y, z), dtype=np.float32)
    lifted[:, :f] = std
    out_view[...] = lifted.reshape(b, nb, s, x, y, z).transpose(0, 1, 3, 4, 5, 2)


def standard_kernel(kernel, out_fmaps: int, in_fmaps: int) -> np.ndarray:
    """Accept a BlockedKernel (blocked.py:234-257) or a standard bank."""
    if hasattr(kernel, "view") and hasattr(kernel, "out_blocks"):
        v = np.asarray(kernel.view)          # (OB, IB, kx, ky, kz, S_out, S_in)
        ob, ib, kx, ky, kz, so, si = v.shape
        std = v.transpose(0, 5, 1, 6, 2, 3, 4).reshape(ob * so, ib * si, kx, ky, kz)
        return np.ascontiguousarray(std[:out_fmaps, :in_fmaps], dtype=np.float32)
    return np.ascontiguousarray(np.asarray(kernel, dtype=np.float32)[:out_fmaps, :in_fmaps])


def _is_device(v) -> bool:
    return isinstance(v, DTensor)


def _to_dev(view, fmaps, dtype) -> DTensor:
    from .device import to_device_blocked
    return to_device_blocked(blocked_np_to_standard(view, fmaps), dtype=dtype)


def _packed(inv, precision, transposed):
    key = ("_b200_pack", precision, transposed)
    cache = getattr(inv, "_b200_cache", None)
    if cache is None:
        cache = {}
        inv._b200_cache = cache
    if key not in cache:
        w = standard_kernel(inv.kernel, inv.out_fmaps, inv.in_fmaps)
        bias = np.asarray(inv.bias, dtype=np.float32).reshape(-1)[:inv.out_fmaps]
        scale = None
        if inv.additive and inv.base_scale is not None:
            scale = np.asarray(inv.base_scale, dtype=np.float32).reshape(-1)[:inv.out_fmaps]
        prec = "x3" if precision == "x3" else "bf16"
        if transposed:
            cache[key] = K.pack_deconv(w, bias, stride=inv.stride, base_scale=scale,
                                       force_gather=(precision == "fp32"), precision=prec)
        else:
            path = _lib.PATH_DIRECT if precision == "fp32" else 0
            cache[key] = K.pack_conv(w, bias, stride=inv.stride, base_scale=scale, path=path,
                                     precision=prec)
    return cache[key]


def _run(inv: ConvInvocation, precision: str, transposed: bool) -> None:
    import torch
    if precision not in ("bf16", "fp32", "x3"):
        raise ExecutionError("unknown precision %r" % (precision,))
    pk = _packed(inv, precision, transposed)
    if _is_device(inv.in_view):
        x, out = inv.in_view, inv.out_view
        base = inv.base_view if inv.additive else None
        host_out = None
    else:
        dt = {"fp32": "fp32", "x3": "split"}.get(precision, "bf16")
        x = _to_dev(inv.in_view, inv.in_fmaps, dt)
        base = _to_dev(inv.base_view, inv.out_fmaps, dt) if inv.additive else None
        _, _, ox, oy, oz, _ = inv.out_view.shape
        host_out = inv.out_view
        out = standard(torch.empty((inv.out_view.shape[0], inv.out_fmaps, ox, oy, oz),
                                   dtype=torch.float32, device=x.t.device))
    if transposed:
        K.deconv3d(x, pk, out, base=base, fused_act=inv.fused_act)
    else:
        K.conv3d(x, pk, out, base=base, fused_act=inv.fused_act)
    if host_out is not None:
        standard_to_blocked_np(out.t.cpu().numpy(), host_out)


def conv3d(inv: ConvInvocation, precision: str = "bf16") -> None:
    """Blocked convolution step (kernels_cy.conv3d, kernels_cy.py:49-57)."""
    _run(inv, precision, transposed=False)


def deconv3d(inv: ConvInvocation, precision: str = "bf16") -> None:
    """Transposed convolution step (kernels_py.deconv3d, kernels_py.py:162-196)."""
    _run(inv, precision, transposed=True)


def subimage(task: SubImageTask, inv: ConvInvocation) -> None:
    """One sub-image application through memory (kernels_cy.subimage, kernels_cy.py:60-69).

    Runs in fp32 on the GPU; intermediate accumulators survive the store and
    reload exactly, as in the reference (kernels_py.py:117-124).
    """
    import torch
    from .device import device_vector
    if inv.out_view.shape[5] != 8 or inv.in_view.shape[5] != 8:
        raise ExecutionError("the B200 subimage primitive needs S = 8 lanes")
    w = standard_kernel(inv.kernel, inv.out_fmaps, inv.in_fmaps)
    dev = torch.device("cuda", torch.cuda.current_device())
    x = DTensor(torch.from_numpy(np.ascontiguousarray(inv.in_view, dtype=np.float32)).to(dev),
                inv.in_fmaps, True)
    out_t = torch.from_numpy(np.ascontiguousarray(inv.out_view, dtype=np.float32)).to(dev)
    out = DTensor(out_t, inv.out_fmaps, True)
    base = None
    if inv.additive:
        base = DTensor(torch.from_numpy(np.ascontiguousarray(inv.base_view, dtype=np.float32))
                       .to(dev), inv.out_fmaps, True)
    wd = torch.from_numpy(w).to(dev)
    bias = device_vector(np.asarray(inv.bias, np.float32).reshape(-1)[:inv.out_fmaps], device=dev)
    scale = None
    if inv.additive and inv.base_scale is not None:
        scale = device_vector(np.asarray(inv.base_scale, np.float32).reshape(-1)[:inv.out_fmaps],
                              device=dev)
    K.conv3d_subimage(x, wd, bias, out, cin=inv.in_fmaps, cout=inv.out_fmaps, k=w.shape[2:],
                      stride=inv.stride, in_block=task.in_block, out_block=task.out_block,
                      origin=task.origin, extent=task.extent, first=task.first, last=task.last,
                      base=base, scale_dev=scale, fused_act=inv.fused_act)
    inv.out_view[...] = out_t.cpu().numpy()
