"""ctypes binding of the C ABI in include/vxb.h (libvxb.so, built in-tree).

The product path has no CPU fallback: importing this module succeeds without
the library (so host-only code and CPU tests work), but every entry point
raises ``ExecutionError`` when ``libvxb.so`` is missing or a call fails.
"""

from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_float, c_int, c_int32, c_int64, c_size_t, c_void_p, c_char_p

from .errors import ExecutionError

LIB_NAME = "libvxb.so"
LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), LIB_NAME)

VXB_BF16 = 0
VXB_F32 = 1
VXB_BF16X2 = 2       # split bf16: hi plane + lo plane (s[1]/2 apart)
PREC_BF16 = 0        # VXB_PREC_BF16
PREC_X3 = 1          # VXB_PREC_X3
ACT_CODE = {None: 0, "relu": 1, "elu": 2, "sigmoid": 3}   # kernels_cy.py:19
ABI_VERSION = 5      # include/vxb.h VXB_ABI_VERSION
COPY_INDEPENDENT = 1  # VXB_COPY_INDEPENDENT
PATH_TC = 1
PATH_DIRECT = 2
PATH_TC_UNFOLDED = 3
PATH_TC_N128 = 4
PATH_TC_N64 = 5
PATH_TC_N32 = 6
PATH_TC_N16 = 7
TC_PATHS = (PATH_TC, PATH_TC_UNFOLDED, PATH_TC_N128, PATH_TC_N64, PATH_TC_N32, PATH_TC_N16)
POOL_CODE = {"max": 0, "avg": 1}
ELT_CODE = {"add": 0, "mul": 1, "div": 2}


class VxbTensor(ctypes.Structure):
    _fields_ = [
        ("data", c_void_p),
        ("dtype", c_int32),
        ("blocked", c_int32),
        ("n", c_int32), ("c", c_int32), ("x", c_int32), ("y", c_int32), ("z", c_int32),
        ("pad_", c_int32),
        ("s", c_int64 * 5),
    ]


class VxbConvDesc(ctypes.Structure):
    _fields_ = [
        ("in0", VxbTensor),
        ("in1", VxbTensor),
        ("off0", c_int32 * 3),
        ("off1", c_int32 * 3),
        ("out", VxbTensor),
        ("base", VxbTensor),
        ("w_packed", c_void_p),
        ("bias", c_void_p),
        ("base_scale", c_void_p),
        ("cin", c_int32), ("cout", c_int32),
        ("k", c_int32 * 3),
        ("stride", c_int32 * 3),
        ("pad", c_int32 * 3),
        ("act", c_int32),
        ("alpha", c_float),
        ("path", c_int32),
        ("pool_mode", c_int32),
        ("prec", c_int32),
        ("reserved", c_int32 * 5),
        ("pool_out", VxbTensor),
        ("head_w", c_void_p),
        ("head_b", c_void_p),
        ("head_cout", c_int32),
        ("head_act", c_int32),
        ("head_alpha", c_float),
        ("head_reserved_", c_int32),
        ("head_out", VxbTensor),
    ]


class VxbDeconvDesc(ctypes.Structure):
    _fields_ = [
        ("in_", VxbTensor),
        ("out", VxbTensor),
        ("base", VxbTensor),
        ("w_packed", c_void_p),
        ("bias", c_void_p),
        ("base_scale", c_void_p),
        ("cin", c_int32), ("cout", c_int32),
        ("k", c_int32 * 3),
        ("stride", c_int32 * 3),
        ("act", c_int32),
        ("alpha", c_float),
        ("path", c_int32),
        ("prec", c_int32),
        ("reserved", c_int32 * 6),
    ]


I3 = c_int32 * 3
TP = POINTER(VxbTensor)

# (name, restype, argtypes) for every symbol include/vxb.h declares
SIGNATURES = [
    ("vxb_abi_version", c_int, []),
    ("vxb_last_error", c_char_p, []),
    ("vxb_device_sms", c_int, []),
    ("vxb_debug_read", c_size_t, [c_void_p, c_size_t]),
    ("vxb_conv_select", c_int, [c_int, c_int, I3, I3]),
    ("vxb_set_pdl", c_int, [c_int]),
    ("vxb_conv_select_shape", c_int, [c_int, c_int, I3, I3, I3]),
    ("vxb_conv_select_shape_b", c_int, [c_int, c_int, I3, I3, I3, c_int]),
    ("vxb_conv_weights_bytes", c_size_t, [c_int, c_int, I3, I3, c_int]),
    ("vxb_conv_pack_weights", c_int, [c_void_p, c_int, c_int, I3, I3, c_int, c_void_p, c_size_t]),
    ("vxb_conv_weights_bytes2", c_size_t, [c_int, c_int, c_int, I3, I3, c_int]),
    ("vxb_conv_pack_weights2", c_int,
     [c_void_p, c_int, c_int, c_int, I3, I3, c_int, c_void_p, c_size_t]),
    ("vxb_conv_weights_bytes3", c_size_t, [c_int, c_int, c_int, I3, I3, c_int, c_int]),
    ("vxb_conv_pack_weights3", c_int,
     [c_void_p, c_int, c_int, c_int, I3, I3, c_int, c_int, c_void_p, c_size_t]),
    ("vxb_conv3d", c_int, [POINTER(VxbConvDesc), c_void_p]),
    ("vxb_conv3d_subimage", c_int,
     [POINTER(VxbConvDesc), c_void_p, c_int, c_int, I3, I3, c_int, c_int, c_void_p]),
    ("vxb_deconv_weights_bytes", c_size_t, [c_int, c_int, I3, I3, c_int]),
    ("vxb_deconv_pack_weights", c_int,
     [c_void_p, c_int, c_int, I3, I3, c_int, c_void_p, c_size_t]),
    ("vxb_deconv_weights_bytes3", c_size_t, [c_int, c_int, I3, I3, c_int, c_int]),
    ("vxb_deconv_pack_weights3", c_int,
     [c_void_p, c_int, c_int, I3, I3, c_int, c_int, c_void_p, c_size_t]),
    ("vxb_deconv3d", c_int, [POINTER(VxbDeconvDesc), c_void_p]),
    ("vxb_pool3d", c_int, [TP, TP, I3, I3, c_int, c_void_p]),
    ("vxb_eltwise", c_int, [TP, TP, TP, c_int, c_void_p]),
    ("vxb_affine_act", c_int, [TP, TP, c_void_p, c_void_p, c_int, c_float, c_void_p]),
    ("vxb_mergecrop", c_int, [TP, TP, TP, c_void_p]),
    ("vxb_pad_copy", c_int, [TP, TP, I3, c_void_p]),
    ("vxb_copy", c_int, [TP, TP, c_void_p]),
    ("vxb_copy_windows", c_int, [TP, TP, c_int, c_void_p]),
    ("vxb_pack_zwin_windows", c_int, [TP, c_int, TP, c_int, c_int, c_void_p]),
    ("vxb_copy_ex", c_int, [TP, TP, c_int, c_void_p]),
    ("vxb_pack_zwin", c_int, [TP, TP, c_int, c_int, c_int, c_void_p]),
    ("vxb_zero", c_int, [TP, c_void_p]),
]

_LIB = None


def library_available() -> bool:
    return os.path.exists(LIB_PATH)


def lib():
    """The loaded library; raises ExecutionError when it was not built."""
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise ExecutionError(
                "B200 backend requested but %s is not built "
                "(run __graft_entry__.build())" % LIB_PATH)
        handle = ctypes.CDLL(LIB_PATH)
        for name, res, args in SIGNATURES:
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        if handle.vxb_abi_version() != ABI_VERSION:
            raise ExecutionError("%s has ABI %d, this package needs %d (rebuild it)"
                                 % (LIB_PATH, handle.vxb_abi_version(), ABI_VERSION))
        _LIB = handle
    return _LIB


def check(status: int, what: str) -> None:
    if status != 0:
        msg = lib().vxb_last_error()
        raise ExecutionError("%s failed (%d): %s" % (what, status, msg.decode(errors="replace")))


def i3(v) -> "ctypes.Array":
    a, b, c = (int(t) for t in v)
    return I3(a, b, c)
