"""The reference-side binding, executed: the reference's OWN engine
(voxplan, built into oracle/_ref by oracle/build_ref.sh) drives the B200
kernel module through its plugin boundary.

INTEGRATION.md §1 is one registry entry: ``Backend(name, kernels_b200)``
(backend.py:24-29).  Here that object is handed to the reference's
``PlanRunner(plan, backend=Backend)`` (executor.py:54-59, whose
``_bind_conv`` closures call ``backend.conv3d/deconv3d``, executor.py:
134-164) and to the reference's ``run_tiled`` (tiling.py:189-237), and the
invocations are built with the reference's own ``ConvInvocation`` /
``SubImageTask`` / ``kernel_to_blocked`` / ``to_blocked`` (kernels_py.py:
24-56, blocked.py:209-278) — the objects a reference user's plan produces.
Oracles: the golden outputs of the reference (net*_ref) and the reference's
compiled backend on the same invocation.
"""

import numpy as np
import pytest

from vxb_testutil import cuda_ready

from oracle import ref_voxplan as RV

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not cuda_ready(), reason="needs CUDA + libvxb.so"),
              pytest.mark.skipif(not RV.available(), reason="oracle/_ref not built")]

from oracle import ref_numpy as R  # noqa: E402
from paper_1903_07525_b200 import kernels_b200  # noqa: E402


def _backend(precision):
    """The registry entry of INTEGRATION.md §1, built against the
    reference's own Backend class."""
    V = RV.voxplan()
    from voxplan.backend import Backend
    b = Backend("b200" if precision == "bf16" else "b200-" + precision, kernels_b200)
    b.conv3d = lambda inv: kernels_b200.conv3d(inv, precision=precision)
    b.deconv3d = lambda inv: kernels_b200.deconv3d(inv, precision=precision)
    assert V is not None
    return b


def _ref_net(g, i):
    V = RV.voxplan()
    from voxplan import formats as vf
    spec = V.parse_network(bytes(g["net%d_prototxt" % i]).decode())
    store = vf.parse_weights(bytes(g["net%d_pznw" % i]))
    plan, _ = V.compile_network(spec, store)
    return plan


@pytest.mark.parametrize("i", [0, 1, 2])
@pytest.mark.parametrize("precision", ["fp32", "bf16", "x3"])
def test_reference_planrunner_with_b200_backend(golden_nets, i, precision):
    V = RV.voxplan()
    plan = _ref_net(golden_nets, i)
    runner = V.PlanRunner(plan, backend=_backend(precision))
    assert runner.backend.name.startswith("b200")
    (name, got), = runner.run(golden_nets["net%d_x" % i]).items()
    mx, l2 = R.normalized_error(got, golden_nets["net%d_ref" % i])
    # fp32 CUDA cores / split-bf16: reference arithmetic; bf16 storage: the
    # per-step bf16 rounding of operands (each step round-trips the host here)
    tol = {"fp32": (1e-5, 1e-5), "x3": (5e-5, 3e-5), "bf16": (2e-2, 1e-2)}[precision]
    assert mx < tol[0] and l2 < tol[1], (mx, l2)


def test_reference_run_tiled_with_b200_backend(golden_nets):
    """The reference's thread-pool tiler with two workers, each worker its
    own reference PlanRunner bound to the B200 backend."""
    V = RV.voxplan()
    plan = _ref_net(golden_nets, 0)
    in_dims = plan.inputs[0][2]
    rng = np.random.default_rng(3)
    vol = rng.uniform(-1, 1, tuple(in_dims[:2]) + tuple(2 * d for d in in_dims[2:])
                      ).astype(np.float32)
    got = V.run_tiled(plan, vol, backend=_backend("fp32"), workers=2)
    want = V.run_tiled(plan, vol, backend="compiled", workers=1)
    mx, _ = R.normalized_error(got, want)
    assert got.shape == want.shape and mx < 1e-5, mx


def _make_inv(V, x, k, bias, base=None, out_pads=(0, 0, 0), fused_act=None, simd=8):
    from voxplan.blocked import BlockedTensor, kernel_to_blocked, to_blocked
    from voxplan.kernels_py import ConvInvocation
    fo, fi = k.shape[:2]
    bk = kernel_to_blocked(k, simd)
    bx = to_blocked(x, simd)
    osp = tuple(i - kk + 1 for i, kk in zip(x.shape[2:], k.shape[2:]))
    out = BlockedTensor.zeros(x.shape[0], fo, osp, simd, pads=out_pads)
    lanes = bk.out_blocks * simd
    b = np.zeros(lanes, np.float32)
    b[:fo] = bias
    inv = ConvInvocation(in_view=bx.view, in_fmaps=fi, kernel=bk, bias=b, out_view=out.view,
                         out_fmaps=fo, additive=base is not None,
                         base_view=None if base is None else to_blocked(base, simd).view,
                         fused_act=fused_act)
    return inv, out


@pytest.mark.parametrize("precision", ["fp32", "bf16"])
def test_reference_invocation_known_answers(precision):
    """Known answers (test_kernels.py:80-99, 123-136 of the reference) on
    invocations built by the reference's own helpers."""
    V = RV.voxplan()
    from voxplan.blocked import from_blocked
    b = _backend(precision)
    x = np.ones((1, 1, 3, 3, 3), np.float32)
    inv, out = _make_inv(V, x, np.ones((1, 1, 3, 3, 3), np.float32), [0.0])
    b.conv3d(inv)
    assert from_blocked(out)[0, 0, 0, 0, 0] == 27.0
    inv, out = _make_inv(V, np.zeros_like(x), np.zeros((1, 1, 3, 3, 3), np.float32), [0.5],
                         base=np.full((1, 1, 1, 1, 1), 10.0, np.float32))
    b.conv3d(inv)
    assert from_blocked(out)[0, 0, 0, 0, 0] == 10.5
    # relu epilogue, halo'd output: interior written, halo untouched
    inv, out = _make_inv(V, -x, np.ones((1, 1, 3, 3, 3), np.float32), [0.0],
                         out_pads=(1, 1, 1), fused_act=("relu", 0.0))
    out.data[...] = 7.0
    b.conv3d(inv)
    assert from_blocked(out)[0, 0, 0, 0, 0] == 0.0
    full = out.data.reshape(-1)
    assert np.count_nonzero(full == 7.0) == full.size - 8      # 1 voxel x 8 lanes written


def test_reference_subimage_chain_through_b200():
    """Sub-image tasks (SubImageTask, kernels_py.py:47-56) chained over two
    input blocks equal the reference compiled backend's full conv."""
    V = RV.voxplan()
    from voxplan.backend import get_backend
    from voxplan.blocked import from_blocked
    from voxplan.kernels_py import SubImageTask
    rng = np.random.default_rng(11)
    x = rng.standard_normal((1, 16, 5, 5, 5)).astype(np.float32)
    k = (rng.standard_normal((8, 16, 3, 3, 3)) * 0.2).astype(np.float32)
    bias = rng.standard_normal(8).astype(np.float32)
    inv, out = _make_inv(V, x, k, bias)
    b = _backend("fp32")
    for ib, (first, last) in enumerate([(True, False), (False, True)]):
        b.subimage(SubImageTask(in_block=ib, out_block=0, origin=(0, 0, 0),
                                extent=(3, 3, 3), first=first, last=last), inv)
    inv2, out2 = _make_inv(V, x, k, bias)
    get_backend("compiled").conv3d(inv2)
    np.testing.assert_allclose(from_blocked(out), from_blocked(out2), atol=1e-5, rtol=0)
