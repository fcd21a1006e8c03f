"""Pin the CPU oracle (oracle/ref_numpy.py) before trusting it.

Checks the numpy restatement against golden vectors produced by the
reference itself (tests/golden/make_golden.py -> ops.npz, nets.npz) and
against the reference's known-answer tests (pkg/tests/test_kernels.py:80-136,
268-313, 362-380; pkg/tests/test_oracle.py:57-146).
"""

import numpy as np
import pytest

from oracle import ref_numpy as R


def test_conv_golden(golden_ops):
    g = golden_ops
    for i in range(7):
        s, p = tuple(g["conv%d_meta" % i][:3]), tuple(g["conv%d_meta" % i][3:])
        got = R.conv3d(g["conv%d_x" % i], g["conv%d_w" % i], g["conv%d_b" % i], s, p)
        np.testing.assert_allclose(got, g["conv%d_y" % i], atol=2e-5, rtol=0)


def test_deconv_golden(golden_ops):
    g = golden_ops
    for i in range(3):
        got = R.deconv3d(g["deconv%d_x" % i], g["deconv%d_w" % i], g["deconv%d_b" % i],
                         tuple(g["deconv%d_s" % i]))
        np.testing.assert_allclose(got, g["deconv%d_y" % i], atol=2e-5, rtol=0)


def test_pool_mergecrop_eltwise_golden_exact(golden_ops):
    g = golden_ops
    np.testing.assert_array_equal(R.pool3d(g["pool_x"], 2, 2, "max"), g["pool_max"])
    np.testing.assert_array_equal(R.pool3d(g["pool_x"], 2, 2, "avg"), g["pool_avg"])
    np.testing.assert_array_equal(R.pool3d(g["pool_x"], (1, 2, 2), (1, 2, 2), "max"),
                                  g["pool_aniso"])
    np.testing.assert_array_equal(R.mergecrop(g["mc_a"], g["mc_b"]), g["mc_y"])
    for op in ("add", "mul", "div"):
        np.testing.assert_array_equal(R.eltwise(g["elt_a"], g["elt_b"], op), g["elt_" + op])


def test_linear_and_activations_golden(golden_ops):
    g = golden_ops
    np.testing.assert_array_equal(R.batch_norm(g["bn_x"], g["bn_mean"], g["bn_var"], 1e-5),
                                  g["bn_y"])
    np.testing.assert_array_equal(R.scale(g["bn_x"], g["bn_gamma"], g["bn_beta"]), g["sc_y"])
    np.testing.assert_array_equal(R.activation(g["bn_x"], "relu"), g["relu_y"])
    np.testing.assert_array_equal(R.activation(g["bn_x"], "elu", 0.7), g["elu_y"])
    np.testing.assert_array_equal(R.activation(g["bn_x"], "sigmoid"), g["sig_y"])


def test_known_answers():
    # test_kernels.py:80-87 / test_oracle.py:57-62: all-ones 3^3 -> 27
    one = np.ones((1, 1, 3, 3, 3), np.float32)
    assert R.conv3d(one, one, [0.0])[0, 0, 0, 0, 0] == 27.0
    # test_kernels.py:123-127: identity 1^3 kernel + 2.5
    x = np.random.default_rng(0).standard_normal((1, 1, 4, 4, 4)).astype(np.float32)
    np.testing.assert_array_equal(R.conv3d(x, np.ones((1, 1, 1, 1, 1), np.float32), [2.5]),
                                  x + np.float32(2.5))
    # test_kernels.py:131-136: stride 2 over a constant field -> 9.0 (8 + bias 1)
    got = R.conv3d(np.ones((1, 1, 4, 4, 4), np.float32), np.ones((1, 1, 2, 2, 2), np.float32),
                   [1.0], stride=2)
    np.testing.assert_array_equal(got, np.full((1, 1, 2, 2, 2), 9.0, np.float32))
    # test_kernels.py:268-272: deconv broadcast 3 * 1 + 0.25
    got = R.deconv3d(np.full((1, 1, 1, 1, 1), 3.0, np.float32),
                     np.ones((1, 1, 2, 2, 2), np.float32), [0.25], stride=2)
    np.testing.assert_array_equal(got, np.full((1, 1, 2, 2, 2), 3.25, np.float32))
    # test_kernels.py:310-313 / test_oracle.py:141-146: pooling
    ar = np.arange(1, 9, dtype=np.float32).reshape(1, 1, 2, 2, 2)
    assert R.pool3d(ar, 2, 2, "max").reshape(()) == 8.0
    assert R.pool3d(ar, 2, 2, "avg").reshape(()) == 4.5
    # test_kernels.py:369-374: centre crop [1, 19) of a 20^3 against 18^3
    a = np.random.default_rng(1).standard_normal((1, 2, 20, 20, 20)).astype(np.float32)
    b = np.random.default_rng(2).standard_normal((1, 2, 18, 18, 18)).astype(np.float32)
    np.testing.assert_array_equal(R.mergecrop(a, b),
                                  np.concatenate([a[:, :, 1:19, 1:19, 1:19], b], axis=1))


def test_oracle_vs_fp64_loop(rng):
    # test_oracle.py:26-54 style audit: scalar fp64 loop for a small case
    x = rng.standard_normal((1, 3, 5, 4, 6)).astype(np.float32)
    w = rng.standard_normal((2, 3, 3, 2, 3)).astype(np.float32)
    b = rng.standard_normal(2).astype(np.float32)
    got = R.conv3d(x, w, b, (1, 2, 1), (1, 0, 1))
    xp = np.pad(x.astype(np.float64), ((0, 0), (0, 0), (1, 1), (0, 0), (1, 1)))
    want = np.zeros(got.shape)
    for o in range(2):
        for i in range(got.shape[2]):
            for j in range(got.shape[3]):
                for k in range(got.shape[4]):
                    win = xp[0, :, i:i + 3, 2 * j:2 * j + 2, k:k + 3]
                    want[0, o, i, j, k] = b[o] + (win * w[o]).sum()
    np.testing.assert_allclose(got, want, atol=1e-5, rtol=0)


def test_bf16_round_is_rne():
    v = np.array([1.0, 1.00390625, 1.005859375, -2.0, 3.0e38, np.inf, 0.0], np.float32)
    r = R.bf16_round(v)
    assert r[0] == 1.0
    assert r[1] == 1.0            # exact tie -> even
    assert r[2] == 1.0078125      # above tie -> up
    assert r[3] == -2.0 and np.isinf(r[5]) and r[6] == 0.0


@pytest.mark.parametrize("idx", [0, 1, 2])
def test_ref_run_matches_reference_on_zoo_nets(golden_nets, idx):
    from paper_1903_07525_b200 import formats, prototxt
    g = golden_nets
    spec = prototxt.parse_network(bytes(g["net%d_prototxt" % idx]).decode())
    store = formats.parse_weights(bytes(g["net%d_pznw" % idx]))
    (name, got), = R.ref_run(spec, store, g["net%d_x" % idx]).items()
    np.testing.assert_allclose(got, g["net%d_ref" % idx], atol=1e-5, rtol=1e-5)
