"""The reference engine itself (voxplan, built into oracle/_ref by
oracle/build_ref.sh) — TEST INFRASTRUCTURE ONLY.

Used as the CPU baseline ("kind": "reference": BASELINE.md §2 times
``voxplan.PlanRunner(plan, backend="compiled")`` and ``run_tiled``) and by
the reference-side binding tests (the reference's own PlanRunner driving the
B200 Backend).  Networks travel to the reference the way a user's do: as
prototxt text and PZNW bytes (prototxt.py:250-323, formats.py:135-147), so
both engines load identical bytes.
"""

from __future__ import annotations

import os
import sys

REF_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_ref")
_V = None


def available() -> bool:
    return os.path.isfile(os.path.join(REF_DIR, "voxplan", "__init__.py"))


def voxplan():
    """The installed reference package (imported from oracle/_ref)."""
    global _V
    if _V is None:
        if not available():
            raise RuntimeError("oracle/_ref/voxplan not built (run oracle/build_ref.sh)")
        if REF_DIR not in sys.path:
            sys.path.insert(0, REF_DIR)
        import voxplan as V  # noqa: E402
        if not os.path.abspath(V.__file__).startswith(REF_DIR):
            raise RuntimeError("voxplan imported from %s, not oracle/_ref" % V.__file__)
        _V = V
    return _V


def to_reference(spec, store):
    """(NetworkSpec, WeightStore) of this package -> the reference's own
    objects, through the prototxt / PZNW wire formats."""
    from paper_1903_07525_b200 import formats, prototxt
    V = voxplan()
    from voxplan import formats as vf
    rspec = V.parse_network(prototxt.print_network(spec))
    rstore = vf.parse_weights(formats.dump_weights(store))
    return rspec, rstore


def compile_reference(spec, store):
    """The reference compiler (plan.compile_network, plan.py:205-222)."""
    V = voxplan()
    rspec, rstore = to_reference(spec, store)
    plan, _ = V.compile_network(rspec, rstore)
    return plan


def runner(spec, store, backend="compiled"):
    """voxplan.PlanRunner(plan, backend) (executor.py:51-198)."""
    V = voxplan()
    return V.PlanRunner(compile_reference(spec, store), backend=backend)


def run_tiled(plan, volume, workers, overlap=0):
    """voxplan.run_tiled (tiling.py:189-237) with ``workers`` threads."""
    V = voxplan()
    return V.run_tiled(plan, volume, overlap=overlap, backend="compiled", workers=workers)
