"""Backend registry — the reference's plugin boundary (backend.py:24-61).

A ``Backend`` exposes ``conv3d(inv)``, ``deconv3d(inv)`` and
``subimage(task, inv)`` over a ``ConvInvocation`` (kernels_py.py:24-56),
exactly the three callables the reference runtime binds per conv step
(executor.py:162-164).  Two B200 backends are registered:

* ``b200``       bf16 activations and weights, fp32 accumulate, tcgen05
                 tensor cores (the production path);
* ``b200-x3``    split-bf16 storage (hi + lo planes) and three bf16 tensor-
                 core products per MAC (hi*W_hi + lo*W_hi + hi*W_lo, fp32
                 accumulate): fp32-grade results (~1e-5 relative per conv)
                 at ~3x the MMA work of ``b200``;
* ``b200-fp32``  fp32 everywhere on CUDA cores (verification path; matches
                 the reference's fp32 arithmetic to ~1e-6).

``get_backend(None)`` honours ``VOXPLAN_BACKEND``; ``auto`` picks ``b200``.
Asking for a backend whose native library is not built raises
``ExecutionError`` — there is no CPU fallback (backend.py:56-60 semantics).
"""

from __future__ import annotations

import os

from . import _lib
from .errors import ExecutionError

BACKEND_ENV = "VOXPLAN_BACKEND"
NAMES = ("b200", "b200-x3", "b200-fp32")


class Backend:
    def __init__(self, name, module, precision="bf16"):
        self.name = name
        self.precision = precision
        self.conv3d = lambda inv: module.conv3d(inv, precision=precision)
        self.deconv3d = lambda inv: module.deconv3d(inv, precision=precision)
        self.subimage = lambda task, inv: module.subimage(task, inv)

    def __repr__(self):
        return "Backend(%r)" % self.name


def _cuda_ok() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:  # pragma: no cover - torch missing
        return False


def compiled_available() -> bool:
    return _lib.library_available()


def available_backends() -> tuple:
    if compiled_available() and _cuda_ok():
        return NAMES
    return ()


def get_backend(name=None) -> Backend:
    if name is None:
        name = os.environ.get(BACKEND_ENV, "auto")
    if name in ("auto", ""):
        name = "b200"
    if name not in NAMES:
        raise ExecutionError("unknown backend %r (choose auto, %s)" % (name, ", ".join(NAMES)))
    if not compiled_available():
        raise ExecutionError("%s backend requested but libvxb.so is not built" % name)
    from . import kernels_b200
    return Backend(name, kernels_b200, {"b200-fp32": "fp32", "b200-x3": "x3"}.get(name, "bf16"))


def resolve_device_backend(backend) -> Backend:
    """Accept None / a name / a Backend for the device PlanRunner."""
    if isinstance(backend, Backend):
        return backend
    return get_backend(backend)
