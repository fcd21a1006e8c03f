"""Full BASELINE sizes, checked through size-independent properties.

The oracle cannot run a 1x128x32x128x128 conv in seconds, so at full size the
B200 output is compared with a direct fp64 evaluation at sampled output
voxels (all 8 corners, the face centres, and random interior points), using
the same bf16-rounded operands (bf16 storage is the path's stated precision);
plus determinism (two runs bit-identical) and the tail-lane invariant.
Tolerance: |gpu - ref| <= 8e-3 * max|ref over the sample| + 1e-3 (the single
conv bf16 bound of test_gpu_kernels, with slack for the bf16 output store).
"""

import numpy as np
import pytest

from vxb_testutil import cuda_ready

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not cuda_ready(), reason="needs CUDA + libvxb.so")]

import paper_1903_07525_b200 as P  # noqa: E402
from paper_1903_07525_b200 import configs as C, formats  # noqa: E402
from oracle import ref_numpy as R  # noqa: E402


def _samples(shape, n, rng):
    X, Y, Z = shape
    pts = {(x, y, z) for x in (0, X - 1) for y in (0, Y - 1) for z in (0, Z - 1)}
    pts |= {(X // 2, Y // 2, 0), (X // 2, 0, Z // 2), (0, Y // 2, Z // 2),
            (X - 1, Y // 2, Z // 2), (X // 2, Y - 1, Z // 2), (X // 2, Y // 2, Z - 1)}
    while len(pts) < n:
        pts.add(tuple(int(rng.integers(0, s)) for s in shape))
    return sorted(pts)


def _direct(xq, wq, b, pad, pts):
    """fp64 conv (cross-correlation, zero padding) + bias at the given points."""
    cout, cin, kx, ky, kz = wq.shape
    xp = np.pad(xq[0].astype(np.float64), ((0, 0),) + tuple((p, p) for p in pad))
    out = np.empty((len(pts), cout))
    w2 = wq.reshape(cout, -1).astype(np.float64)
    for i, (x, y, z) in enumerate(pts):
        win = xp[:, x:x + kx, y:y + ky, z:z + kz].reshape(-1)
        out[i] = w2 @ win + b
    return out


@pytest.mark.parametrize("c,k", [(128, (3, 3, 3)), (64, (1, 3, 3)), (8, (3, 3, 3))])
def test_config2_full_size_sampled(c, k):
    spec, store = C.config2(c, k)
    plan, _ = P.compile_network(spec, store, fixpoint=True, fuse_deconv_add=True)
    runner = P.PlanRunner(plan)
    x = C.make_input(spec, 11, -1.0, 1.0)
    (name, got), = runner.run(x).items()
    again = runner.run(x)[name]
    np.testing.assert_array_equal(got, again)                    # deterministic
    w = store.tensor("conv", formats.ROLE_KERNEL)
    b = store.tensor("conv", formats.ROLE_BIAS).astype(np.float64)
    pts = _samples(got.shape[2:], 300, np.random.default_rng(c))
    ref = R.activation(_direct(R.bf16_round(x), R.bf16_round(w), b,
                               tuple(v // 2 for v in k), pts).astype(np.float32), "elu")
    g = np.stack([got[0, :, p[0], p[1], p[2]] for p in pts])
    err = np.abs(g - ref)
    assert err.max() <= 8e-3 * np.abs(ref).max() + 1e-3, err.max()


def test_config5_full_patch_invariants():
    """Config 5 at its full 18x192x192 patch (28 convs, the reference's
    14 s-per-patch case): output finite, inside the sigmoid range,
    deterministic, and equal to a one-tile run_tiled over the same volume."""
    spec, store = C.config5()
    plan, _ = P.compile_network(spec, store, fixpoint=True, fuse_deconv_add=True)
    runner = P.PlanRunner(plan)
    x = C.make_input(spec, 12, 0.0, 1.0)
    (name, out), = runner.run(x).items()
    assert out.shape == (1, 3, 18, 192, 192)
    assert np.isfinite(out).all() and out.min() >= 0.0 and out.max() <= 1.0
    np.testing.assert_array_equal(out, runner.run(x)[name])
    np.testing.assert_array_equal(out, P.run_tiled(plan, x))
