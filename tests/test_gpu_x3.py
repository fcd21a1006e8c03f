"""Split-bf16 ("x3") precision path vs the CPU oracle, through the C ABI.

Backend ``b200-x3`` stores every activation as two bf16 planes (hi = bf16(v),
lo = bf16(v - hi)) and runs each conv as a bf16 tensor-core GEMM over two K
segments, [hi, lo] x bf16(W) and [hi] x bf16(W - bf16(W)), fp32 accumulate.
That reproduces the reference's fp32 arithmetic (_kernels.pyx:44-179) to
~1e-5 relative per conv (``oracle/ref_numpy.run_plan(storage="split")`` is
its emulation).  Tolerances:
  * single conv / deconv vs the fp32 oracle: max-normalised <= 5e-5;
  * storage round trip and pooling: bit-exact against numpy's split_bf16;
  * networks vs ref_run (oracle.py:184-252): per config, stated below.
"""

import numpy as np
import pytest

from vxb_testutil import cuda_ready

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not cuda_ready(), reason="needs CUDA + libvxb.so")]

from oracle import ref_numpy as R  # noqa: E402

X3_TOL = 5e-5


def _dev():
    from paper_1903_07525_b200 import device as D, ops as K
    return D, K


def _conv_x3(x, w, b, pad, act=None, base=None, scale=None, out_dtype="split", path=0):
    import torch
    D, K = _dev()
    xd = D.to_device_blocked(x, dtype="split")
    osp = tuple(s + 2 * p - k + 1 for s, p, k in zip(x.shape[2:], pad, w.shape[2:]))
    out = D.empty_blocked(x.shape[0], w.shape[0], osp, out_dtype)
    bd = D.to_device_blocked(base, dtype="split") if base is not None else None
    pk = K.pack_conv(w, b, base_scale=scale, precision="x3", path=path)
    K.conv3d(xd, pk, out, pad=pad, base=bd, fused_act=(act, 1.0) if act else None)
    torch.cuda.synchronize()
    return D.to_host_standard(out), pk.path


def _ref(x, w, b, pad, act=None, base=None, scale=None):
    y = R.conv3d(x, w, np.zeros_like(b), 1, pad)
    init = b.reshape(1, -1, 1, 1, 1).astype(np.float32)
    if base is not None:
        s = np.ones_like(b) if scale is None else scale
        init = init + s.reshape(1, -1, 1, 1, 1) * base
    y = init + y
    return R.activation(y, act) if act else y


def _split(a):
    hi, lo = R.split_bf16(a)
    return hi + lo


CASES = [
    # cin, cout, spatial, k, pad, act, base
    (16, 16, (4, 16, 8), (3, 3, 3), (1, 1, 1), "relu", False),
    (8, 8, (6, 20, 12), (3, 3, 3), (1, 1, 1), None, False),
    (8, 16, (5, 17, 9), (1, 3, 3), (0, 1, 1), "elu", False),
    (32, 32, (9, 33, 17), (3, 3, 3), (1, 1, 1), "elu", True),
    (64, 64, (5, 19, 23), (3, 3, 3), (1, 1, 1), "elu", False),
    (128, 128, (3, 16, 16), (3, 3, 3), (1, 1, 1), "relu", False),
    (1, 32, (10, 20, 12), (3, 3, 3), (0, 0, 0), "relu", False),
    (36, 28, (6, 20, 19), (3, 3, 3), (1, 1, 1), "elu", True),
    (28, 3, (6, 20, 19), (1, 1, 1), (0, 0, 0), "sigmoid", False),
    (80, 80, (6, 24, 24), (1, 3, 3), (0, 1, 1), "elu", True),
    (5, 7, (8, 8, 8), (3, 3, 3), (0, 0, 0), None, False),
    (24, 40, (21, 7, 9), (1, 3, 3), (0, 1, 1), "relu", True),
]


@pytest.mark.parametrize("case", CASES, ids=lambda c: "c%d-%d_k%s" % (c[0], c[1], c[3]))
def test_x3_conv_matches_fp32_oracle(case):
    cin, cout, sp, k, pad, act, use_base = case
    rng = np.random.default_rng(cin * 1000 + cout + 7)
    x = rng.uniform(-1, 1, (1, cin) + sp).astype(np.float32)
    w = (rng.standard_normal((cout, cin) + k) * np.sqrt(2.0 / (cin * np.prod(k)))).astype(np.float32)
    b = (rng.standard_normal(cout) * 0.1).astype(np.float32)
    osp = tuple(s + 2 * p - kk + 1 for s, p, kk in zip(sp, pad, k))
    base = rng.uniform(-1, 1, (1, cout) + osp).astype(np.float32) if use_base else None
    scale = rng.uniform(0.5, 1.5, cout).astype(np.float32) if use_base else None
    got, path = _conv_x3(x, w, b, pad, act, base, scale)
    assert path != 2  # tensor-core path
    # the reference's fp32 conv on the inputs as stored (split-rounded)
    want = _ref(_split(x), w, b, pad, act, None if base is None else _split(base), scale)
    mx, l2 = R.normalized_error(got, _split(want))
    assert mx < X3_TOL and l2 < 3e-5, (mx, l2)
    # and against the unrounded fp32 oracle: the storage rounding adds ~2^-17
    mx2, _ = R.normalized_error(got, _ref(x, w, b, pad, act, base, scale))
    assert mx2 < 1e-4, mx2


def test_x3_direct_path_matches():
    """Strided convs take the CUDA-core path, reading split inputs as fp32 sums."""
    rng = np.random.default_rng(3)
    x = rng.uniform(-1, 1, (1, 12, 9, 10, 11)).astype(np.float32)
    w = (rng.standard_normal((10, 12, 3, 3, 3)) * 0.1).astype(np.float32)
    b = (rng.standard_normal(10) * 0.1).astype(np.float32)
    got, path = _conv_x3(x, w, b, (1, 1, 1), "elu", path=2)
    assert path == 2
    want = _split(_ref(_split(x), w, b, (1, 1, 1), "elu"))
    mx, _ = R.normalized_error(got, want)
    assert mx < 2e-5, mx


def test_split_storage_round_trip_bit_exact():
    """fp32 NCDHW -> split bf16 blocked -> fp32 NCDHW equals hi + lo of
    numpy's split_bf16, for C multiples of 8 (vectorised pack) and not."""
    import torch
    D, _ = _dev()
    rng = np.random.default_rng(5)
    for c, sp in [(16, (3, 8, 12)), (5, (4, 6, 7)), (28, (2, 9, 16))]:
        x = (rng.standard_normal((2, c) + sp) * 10 ** rng.uniform(-3, 3)).astype(np.float32)
        xd = D.to_device_blocked(x, dtype="split")
        assert xd.split and xd.t.shape[1] == 2 * (-(-c // 8))
        got = D.to_host_standard(xd)
        np.testing.assert_array_equal(got, _split(x))
        # planes: chunk 2j holds hi, 2j+1 lo; tail lanes zero in both
        t = xd.t.float().cpu().numpy()
        hi, lo = R.split_bf16(x)
        j = 0
        np.testing.assert_array_equal(t[:, 0, ..., :min(8, c)],
                                      np.moveaxis(hi[:, :min(8, c)], 1, -1))
        np.testing.assert_array_equal(t[:, 1, ..., :min(8, c)],
                                      np.moveaxis(lo[:, :min(8, c)], 1, -1))
        if c % 8:
            assert not t[:, -2:, ..., c % 8:].any()
        del j
    torch.cuda.synchronize()


def test_split_pool_and_eltwise_exact():
    D, K = _dev()
    rng = np.random.default_rng(9)
    x = rng.standard_normal((1, 12, 4, 8, 10)).astype(np.float32)
    y = rng.standard_normal((1, 12, 4, 8, 10)).astype(np.float32)
    xd = D.to_device_blocked(x, dtype="split")
    yd = D.to_device_blocked(y, dtype="split")
    out = D.empty_blocked(1, 12, (4, 4, 5), "split")
    K.pool3d(xd, out, (1, 2, 2), (1, 2, 2), "max")
    np.testing.assert_array_equal(D.to_host_standard(out),
                                  R.pool3d(_split(x), (1, 2, 2), (1, 2, 2), "max"))
    s = D.empty_blocked(1, 12, (4, 8, 10), "split")
    K.eltwise(xd, yd, s, "add")
    np.testing.assert_array_equal(D.to_host_standard(s), _split(_split(x) + _split(y)))


@pytest.mark.parametrize("cin,cout,k", [(80, 64, (1, 2, 2)), (24, 20, (2, 2, 2)),
                                        (64, 64, (2, 2, 2))])
def test_x3_deconv_matches_fp32_oracle(cin, cout, k):
    import torch
    D, K = _dev()
    rng = np.random.default_rng(cin + cout)
    x = rng.uniform(-1, 1, (1, cin, 3, 6, 8)).astype(np.float32)
    w = (rng.standard_normal((cout, cin) + k) * 0.2).astype(np.float32)
    b = (rng.standard_normal(cout) * 0.1).astype(np.float32)
    osp = tuple((s - 1) * kk + kk for s, kk in zip(x.shape[2:], k))
    base = rng.uniform(-1, 1, (1, cout) + osp).astype(np.float32)
    pk = K.pack_deconv(w, b, stride=k, precision="x3")
    out = D.empty_blocked(1, cout, osp, "split")
    K.deconv3d(D.to_device_blocked(x, dtype="split"), pk, out,
               base=D.to_device_blocked(base, dtype="split"), fused_act=("elu", 1.0))
    torch.cuda.synchronize()
    got = D.to_host_standard(out)
    want = R.activation(R.deconv3d(_split(x), w, b, k) + _split(base), "elu")
    mx, _ = R.normalized_error(got, want)
    assert mx < X3_TOL, mx


def test_precision_mismatch_rejected():
    import paper_1903_07525_b200 as P
    D, K = _dev()
    x = np.zeros((1, 8, 4, 8, 8), np.float32)
    w = np.zeros((8, 8, 3, 3, 3), np.float32)
    b = np.zeros(8, np.float32)
    pk = K.pack_conv(w, b)                      # bf16 weights
    with pytest.raises(P.ExecutionError):
        K.conv3d(D.to_device_blocked(x, dtype="split"), pk,
                 D.empty_blocked(1, 8, (4, 8, 8), "split"), pad=(1, 1, 1))
    pk3 = K.pack_conv(w, b, precision="x3")
    with pytest.raises(P.ExecutionError):
        K.conv3d(D.to_device_blocked(x), pk3, D.empty_blocked(1, 8, (4, 8, 8)), pad=(1, 1, 1))
