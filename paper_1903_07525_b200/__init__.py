"""B200-native (sm_100a) engine for PZnet-style fused 3D-convolution inference.

Drop-in for the reference's public API (voxplan/__init__.py:59-121) on the
conv3d hot path: the same prototxt description, PZNW weights, plan compiler
and ``PlanRunner(plan).run(volume)`` / ``run_tiled`` — executed by
hand-written tcgen05/TMA kernels in ``libvxb.so`` (C ABI: include/vxb.h).
Host-only pieces (parsing, shapes, passes, tiling geometry) import without a
GPU; anything that launches work raises ``ExecutionError`` when the native
library or a CUDA device is missing.
"""

from .backend import (BACKEND_ENV, Backend, available_backends, compiled_available,
                      get_backend)
from .errors import (CycleError, DanglingReferenceError, DuplicateTopError, ExecutionError,
                     FormatError, LayoutError, ModelError, ParseError, PlanError, ShapeError,
                     TileError, UnknownLayerError, VoxplanError)
from .formats import (WeightStore, create_volume, open_volume, read_volume, read_weights,
                      write_volume, write_weights)
from .ir import PassReport, build_ir, optimize
from .netspec import LayerKind, LayerSpec, NetworkSpec
from .plan import (DEFAULT_PATCH_EXTENT, DEFAULT_SIMD_WIDTH, ExecutionPlan, compile_network,
                   dump_plan, parse_plan, read_plan, write_plan)
from .prototxt import parse_network, print_network
from .shapes import validate_shapes
from .tiling import TileGrid, grid_for, plan_tiles


def __getattr__(name):
    # device-side entry points import torch lazily
    if name in ("PlanRunner", "PlanBatch", "execute"):
        from . import runner
        return getattr(runner, name)
    if name in ("run_tiled", "run_tiled_file"):
        from . import tiling
        return getattr(tiling, name)
    if name in ("ConvInvocation", "SubImageTask"):
        from . import kernels_b200
        return getattr(kernels_b200, name)
    raise AttributeError(name)


__version__ = "0.1.0"

__all__ = [
    "BACKEND_ENV", "Backend", "ConvInvocation", "CycleError", "DanglingReferenceError",
    "DEFAULT_PATCH_EXTENT", "DEFAULT_SIMD_WIDTH", "DuplicateTopError", "ExecutionError",
    "ExecutionPlan", "FormatError", "LayerKind", "LayerSpec", "LayoutError", "ModelError",
    "NetworkSpec", "ParseError", "PassReport", "PlanBatch", "PlanError", "PlanRunner", "ShapeError",
    "SubImageTask", "TileError", "TileGrid", "UnknownLayerError", "VoxplanError", "WeightStore",
    "available_backends", "build_ir", "compile_network", "compiled_available", "dump_plan",
    "execute", "get_backend", "grid_for", "optimize", "parse_network", "parse_plan",
    "plan_tiles", "print_network", "read_plan", "read_volume", "open_volume", "create_volume", "read_weights", "run_tiled",
    "run_tiled_file",
    "validate_shapes", "write_plan", "write_volume", "write_weights", "__version__",
]
