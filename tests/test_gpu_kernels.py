"""Device kernels vs the CPU oracle, through the C ABI (libvxb.so).

Tolerances (stated per precision):
  * bf16 tensor-core path: compared with the fp32 oracle run on the same
    bf16-rounded operands, so the only differences are fp32 accumulation
    order and the final bf16 store: max-normalised error <= 8e-3.
  * fp32 CUDA-core path (backend b200-fp32): <= 2e-5 absolute on O(1) data,
    the reference's own 1e-5-class gate (test_kernels.py:140-156).
  * pool / crop / concat / layout copies: bit-exact.
"""

import os

import numpy as np
import pytest

from vxb_testutil import cuda_ready

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not cuda_ready(), reason="needs CUDA + libvxb.so")]

from oracle import ref_numpy as R  # noqa: E402

BF16_TOL = 8e-3


def _dev():
    from paper_1903_07525_b200 import device as D, ops as K
    return D, K


def _conv_bf16(x, w, b, pad, act=None, base=None, scale=None, out_dtype="bf16"):
    import torch
    D, K = _dev()
    xd = D.to_device_blocked(x)
    osp = tuple(s + 2 * p - k + 1 for s, p, k in zip(x.shape[2:], pad, w.shape[2:]))
    if out_dtype == "f32std":   # fp32 NCDHW output written by the conv epilogue
        out = D.standard(torch.empty((x.shape[0], w.shape[0]) + osp, dtype=torch.float32,
                                     device=xd.t.device))
    else:
        out = D.empty_blocked(x.shape[0], w.shape[0], osp, out_dtype)
    bd = D.to_device_blocked(base) if base is not None else None
    pk = K.pack_conv(w, b, base_scale=scale)
    K.conv3d(xd, pk, out, pad=pad, base=bd, fused_act=(act, 1.0) if act else None)
    torch.cuda.synchronize()
    if out_dtype == "f32std":
        return out.t.cpu().numpy(), pk.path
    return D.to_host_standard(out), pk.path


def _ref_bf16(x, w, b, pad, act=None, base=None, scale=None):
    q = R.bf16_round
    y = R.conv3d(q(x), q(w), np.zeros_like(b), 1, pad)
    init = b.reshape(1, -1, 1, 1, 1).astype(np.float32)
    if base is not None:
        s = np.ones_like(b) if scale is None else scale
        init = init + s.reshape(1, -1, 1, 1, 1) * q(base)
    y = init + y
    return R.activation(y, act) if act else y


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
    (256, 512, (3, 11, 11), (3, 3, 3), (0, 0, 0), "relu", False),
    (5, 7, (8, 8, 8), (3, 3, 3), (0, 0, 0), None, False),
    # 1x3x3 folded along y with x > 16 (two partial row tiles) and y < slices
    (24, 40, (21, 7, 9), (1, 3, 3), (0, 1, 1), "relu", True),
    (48, 48, (7, 30, 13), (3, 3, 3), (1, 1, 1), "elu", False),
]


@pytest.mark.parametrize("case", CASES, ids=lambda c: "c%d-%d_k%s" % (c[0], c[1], c[3]))
def test_tc_conv_matches_oracle(case):
    cin, cout, sp, k, pad, act, use_base = case
    rng = np.random.default_rng(cin * 1000 + cout)
    x = rng.uniform(-1, 1, (1, cin) + sp).astype(np.float32)
    w = (rng.standard_normal((cout, cin) + k) * np.sqrt(2.0 / (cin * np.prod(k)))).astype(np.float32)
    b = (rng.standard_normal(cout) * 0.1).astype(np.float32)
    osp = tuple(s + 2 * p - kk + 1 for s, p, kk in zip(sp, pad, k))
    base = rng.uniform(-1, 1, (1, cout) + osp).astype(np.float32) if use_base else None
    scale = rng.uniform(0.5, 1.5, cout).astype(np.float32) if use_base else None
    got, path = _conv_bf16(x, w, b, pad, act, base, scale)
    assert path == 1  # tensor-core path
    want = _ref_bf16(x, w, b, pad, act, base, scale)
    mx, l2 = R.normalized_error(got, want)
    assert mx < BF16_TOL and l2 < 3e-3, (mx, l2)


@pytest.mark.parametrize("k,pad", [((3, 3, 3), (1, 1, 1)), ((1, 3, 3), (0, 1, 1))])
def test_tap_fold_matches_unfolded(k, pad, monkeypatch):
    """Folding the slice-axis taps into N only reorders the fp32 sums."""
    rng = np.random.default_rng(11)
    x = rng.uniform(-1, 1, (2, 16, 9, 21, 10)).astype(np.float32)
    w = (rng.standard_normal((16, 16) + k) * 0.1).astype(np.float32)
    b = rng.standard_normal(16).astype(np.float32)
    folded, _ = _conv_bf16(x, w, b, pad, "elu", out_dtype="fp32")
    monkeypatch.setenv("VXB_TC_FOLD", "0")
    plain, _ = _conv_bf16(x, w, b, pad, "elu", out_dtype="fp32")
    mx, _ = R.normalized_error(folded, plain)
    assert mx < 1e-5, mx


@pytest.mark.parametrize("bx", ["1", "2", "3", "4", "6", "8"])
@pytest.mark.parametrize("c,n,sp", [(8, 1, (18, 20, 12)), (16, 2, (9, 21, 10)),
                                    (28, 1, (18, 33, 12)), (32, 1, (7, 16, 17))])
@pytest.mark.parametrize("k,pad", [((3, 3, 3), (1, 1, 1)), ((1, 3, 3), (0, 1, 1))])
def test_fold_pair_matches_single_cta(bx, c, n, sp, k, pad, monkeypatch):
    """Folded convs with N = 3nt <= 96 run as CTA pairs (cta_group::2, every
    MMA at N = 3nt with scratch slices around the tile); the result differs
    from the single-CTA folded walk only in fp32 summation order.  Covers odd
    tile counts (the pair's padding tile), batch 2, residual operands and all
    tile widths."""
    monkeypatch.setenv("VXB_TC_BX", bx)
    monkeypatch.setenv("VXB_TC_FOLDPAIR", "2")   # every eligible fold pairs
    rng = np.random.default_rng(int(bx) * 100 + c)
    x = rng.uniform(-1, 1, (n, c) + sp).astype(np.float32)
    w = (rng.standard_normal((c, c) + k) * 0.1).astype(np.float32)
    b = rng.standard_normal(c).astype(np.float32)
    base = rng.uniform(-1, 1, (n, c) + sp).astype(np.float32)
    scale = rng.uniform(0.5, 1.5, c).astype(np.float32)
    paired, _ = _conv_bf16(x, w, b, pad, "elu", base, scale, out_dtype="f32std")
    monkeypatch.setenv("VXB_TC_FOLDPAIR", "0")
    single, _ = _conv_bf16(x, w, b, pad, "elu", base, scale, out_dtype="f32std")
    mx, _ = R.normalized_error(paired, single)
    assert mx < 1e-5, mx
    want = _ref_bf16(x, w, b, pad, "elu", base, scale)
    mx, l2 = R.normalized_error(paired, want)
    assert mx < BF16_TOL and l2 < 3e-3, (mx, l2)


@pytest.mark.parametrize("bx", ["3", "6", "8"])
@pytest.mark.parametrize("k,pad", [((3, 3, 3), (1, 1, 1)), ((1, 3, 3), (0, 1, 1))])
def test_fold_tile_widths(bx, k, pad, monkeypatch):
    """Folded tiles of 3/6/8 slices (config 5's 18-deep axis picks 6)."""
    monkeypatch.setenv("VXB_TC_BX", bx)
    rng = np.random.default_rng(int(bx))
    x = rng.uniform(-1, 1, (1, 28, 18, 20, 12)).astype(np.float32)
    w = (rng.standard_normal((28, 28) + k) * 0.1).astype(np.float32)
    b = rng.standard_normal(28).astype(np.float32)
    base = rng.uniform(-1, 1, (1, 28, 18, 20, 12)).astype(np.float32)
    scale = rng.uniform(0.5, 1.5, 28).astype(np.float32)
    got, _ = _conv_bf16(x, w, b, pad, "elu", base, scale)
    want = _ref_bf16(x, w, b, pad, "elu", base, scale)
    mx, l2 = R.normalized_error(got, want)
    assert mx < BF16_TOL and l2 < 3e-3, (mx, l2)


@pytest.mark.parametrize("bx", ["1", "2", "3", "4", "6", "8"])
@pytest.mark.parametrize("c,k,pad,sp", [(28, (1, 3, 3), (0, 1, 1), (18, 33, 20)),
                                        (36, (1, 1, 1), (0, 0, 0), (18, 16, 24)),
                                        (128, (3, 3, 3), (1, 1, 1), (7, 16, 8))])
def test_unfolded_tile_widths_bit_identical(bx, c, k, pad, sp, monkeypatch):
    """Unfolded tiles of 1..8 slices (config 5's 18-deep axis picks 6, three
    full tiles; 8 leaves a last tile of 2 valid slices whose other slices the
    epilogue skips): every output slice accumulates the same K steps in the
    same order, so all widths agree bit for bit and match the oracle."""
    rng = np.random.default_rng(c)
    x = rng.uniform(-1, 1, (2, c) + sp).astype(np.float32)
    w = (rng.standard_normal((c, c) + k) * 0.1).astype(np.float32)
    b = rng.standard_normal(c).astype(np.float32)
    base = rng.uniform(-1, 1, (2, c) + sp).astype(np.float32)
    scale = rng.uniform(0.5, 1.5, c).astype(np.float32)
    monkeypatch.setenv("VXB_TC_FOLD", "0")
    monkeypatch.setenv("VXB_TC_BX", bx)
    got, _ = _conv_bf16(x, w, b, pad, "elu", base, scale)
    monkeypatch.setenv("VXB_TC_BX", "8")
    monkeypatch.setenv("VXB_TC_UNF36", "0")        # power-of-two widths only
    ref, _ = _conv_bf16(x, w, b, pad, "elu", base, scale)
    assert np.array_equal(got, ref)
    want = _ref_bf16(x, w, b, pad, "elu", base, scale)
    mx, l2 = R.normalized_error(got, want)
    assert mx < BF16_TOL and l2 < 3e-3, (mx, l2)


@pytest.mark.parametrize("n,c,sp,pad", [(1, 28, (18, 32, 16), (1, 1, 1)),
                                         (2, 28, (18, 20, 12), (1, 1, 1)),
                                         (1, 32, (32, 16, 16), (1, 1, 1)),
                                         (1, 16, (7, 16, 8), (1, 1, 1)),
                                         (1, 28, (20, 18, 10), (0, 0, 0)),
                                         (3, 8, (5, 33, 9), (1, 1, 1)),
                                         (1, 48, (18, 16, 16), (1, 1, 1))])
@pytest.mark.parametrize("use_base", [False, True])
def test_streamed_fold_matches_oracle(n, c, sp, pad, use_base, monkeypatch):
    """Streamed fold (VXB_TC_STREAM=2, experimental): a CTA walks whole x
    columns slab by slab, the output slices' accumulators live in a TMEM ring
    that the epilogue zeroes after reading.  Same sums as the tiled fold walk
    in another fp32 order: equal to it within fp32 reordering (one bf16 ulp of
    the stored values at most) and within the bf16 bound of the oracle.
    Covers ring wrap-around (18 and 32 slices over 16 / 8 slots), 'valid'
    convolutions (both halo slices real), batches, and residual operands."""
    rng = np.random.default_rng(c + sp[0])
    x = rng.uniform(-1, 1, (n, c) + sp).astype(np.float32)
    w = (rng.standard_normal((c, c, 3, 3, 3)) * 0.1).astype(np.float32)
    b = rng.standard_normal(c).astype(np.float32)
    osp = tuple(s + 2 * p - 2 for s, p in zip(sp, pad))
    base = rng.uniform(-1, 1, (n, c) + osp).astype(np.float32) if use_base else None
    scale = rng.uniform(0.5, 1.5, c).astype(np.float32) if use_base else None
    monkeypatch.setenv("VXB_TC_STREAM", "0")
    tiled, _ = _conv_bf16(x, w, b, pad, "elu", base, scale)
    monkeypatch.setenv("VXB_TC_STREAM", "2")
    got, _ = _conv_bf16(x, w, b, pad, "elu", base, scale)
    assert np.abs(got - tiled).max() <= np.abs(tiled).max() * 2.0 ** -7
    want = _ref_bf16(x, w, b, pad, "elu", base, scale)
    mx, l2 = R.normalized_error(got, want)
    assert mx < BF16_TOL and l2 < 3e-3, (mx, l2)


def test_unfolded_path_for_badly_padded_rows():
    """x = 18 makes y-sliced folding pad 14 of 32 rows: select_shape picks the
    unfolded layout, which must match the oracle (and the folded result)."""
    import torch
    D, K = _dev()
    rng = np.random.default_rng(21)
    x = rng.uniform(-1, 1, (1, 28, 18, 24, 16)).astype(np.float32)
    w = (rng.standard_normal((28, 28, 1, 3, 3)) * 0.1).astype(np.float32)
    b = rng.standard_normal(28).astype(np.float32)
    want = _ref_bf16(x, w, b, (0, 1, 1), "elu")
    xd = D.to_device_blocked(x)
    for out_shape, path in [((18, 24, 16), 3), (None, 1)]:
        out = D.empty_blocked(1, 28, (18, 24, 16))
        pk = K.pack_conv(w, b, out_shape=out_shape)
        assert pk.path == path
        K.conv3d(xd, pk, out, pad=(0, 1, 1), fused_act=("elu", 1.0))
        torch.cuda.synchronize()
        mx, l2 = R.normalized_error(D.to_host_standard(out), want)
        assert mx < BF16_TOL and l2 < 3e-3, (path, mx, l2)


@pytest.mark.parametrize("cin,cout,k,pad,sp,n,out_dtype", [
    (16, 16, (3, 3, 3), (1, 1, 1), (6, 20, 16), 1, "bf16"),
    (1, 28, (1, 3, 3), (0, 1, 1), (5, 18, 12), 1, "bf16"),       # Cin < 8: OOB lanes
    (16, 20, (3, 3, 3), (1, 1, 1), (9, 17, 20), 2, "fp32"),      # batch 2, fp32 NCDHW out
    (13, 20, (3, 3, 3), (1, 1, 1), (9, 17, 20), 1, "bf16"),      # ragged chunk
    (64, 64, (3, 3, 3), (1, 1, 1), (4, 16, 16), 1, "bf16"),
    (128, 128, (3, 3, 3), (1, 1, 1), (4, 16, 8), 1, "bf16"),     # CTA pair (streamed B)
    (32, 32, (3, 3, 3), (0, 0, 0), (8, 20, 12), 1, "bf16"),      # valid padding
])
def test_fp32_input_converted_in_kernel(cin, cout, k, pad, sp, n, out_dtype):
    """The network's fp32 NCDHW input fed straight to the tensor-core conv
    (fp32 TMA boxes + in-kernel bf16 conversion) equals packing first."""
    import torch
    D, K = _dev()
    rng = np.random.default_rng(cin * 7 + cout)
    x = rng.uniform(-1, 1, (n, cin) + sp).astype(np.float32)
    w = (rng.standard_normal((cout, cin) + k) * np.sqrt(2.0 / (cin * np.prod(k)))).astype(np.float32)
    b = (rng.standard_normal(cout) * 0.1).astype(np.float32)
    osp = tuple(s + 2 * p - kk + 1 for s, p, kk in zip(sp, pad, k))
    pk = K.pack_conv(w, b)
    xs = D.standard(torch.from_numpy(x).cuda())
    if out_dtype == "fp32":
        out_t = torch.empty((n, cout) + osp, dtype=torch.float32, device="cuda")
        out = D.standard(out_t)
    else:
        out = D.empty_blocked(n, cout, osp)
    K.conv3d(xs, pk, out, pad=pad, fused_act=("elu", 1.0))
    torch.cuda.synchronize()
    got = out_t.cpu().numpy() if out_dtype == "fp32" else D.to_host_standard(out)
    # same conv from the packed (bf16 blocked) input into the same output layout
    if out_dtype == "fp32":
        ref_t = torch.empty_like(out_t)
        ref = D.standard(ref_t)
    else:
        ref = D.empty_blocked(n, cout, osp)
    K.conv3d(D.to_device_blocked(x), pk, ref, pad=pad, fused_act=("elu", 1.0))
    torch.cuda.synchronize()
    np.testing.assert_array_equal(
        got, ref_t.cpu().numpy() if out_dtype == "fp32" else D.to_host_standard(ref))
    want = _ref_bf16(x, w, b, pad, "elu")
    mx, l2 = R.normalized_error(got, want)
    assert mx < BF16_TOL and l2 < 3e-3, (mx, l2)


def test_fp32_input_unsupported_views_raise():
    """Batch > 1 with a ragged last chunk cannot zero its tail lanes through
    the folded (batch*channel) TMA coordinate: the library refuses it."""
    import torch
    from paper_1903_07525_b200 import ExecutionError
    D, K = _dev()
    pk = K.pack_conv(np.ones((8, 13, 3, 3, 3), np.float32), np.zeros(8, np.float32))
    xs = D.standard(torch.zeros((2, 13, 4, 8, 8), device="cuda"))
    with pytest.raises(ExecutionError):
        K.conv3d(xs, pk, D.empty_blocked(2, 8, (4, 8, 8)), pad=(1, 1, 1))
    xs = D.standard(torch.zeros((1, 13, 4, 8, 6), device="cuda"))   # z rows of 24 B
    with pytest.raises(ExecutionError):
        K.conv3d(xs, pk, D.empty_blocked(1, 8, (4, 8, 6)), pad=(1, 1, 1))


@pytest.mark.parametrize("path", [4, 5])
@pytest.mark.parametrize("cin,cout,k,pad,sp", [
    (96, 256, (3, 3, 3), (0, 0, 0), (6, 20, 12)),      # N-split, unfolded widths
    (40, 80, (1, 3, 3), (0, 1, 1), (5, 18, 12)),       # N-split + fold
])
def test_narrow_n_tiles(path, cin, cout, k, pad, sp):
    """VXB_PATH_TC_N128/_N64 (deep levels): the fmaps are split over N tiles."""
    import torch
    D, K = _dev()
    rng = np.random.default_rng(cout + path)
    x = rng.uniform(-1, 1, (1, cin) + sp).astype(np.float32)
    w = (rng.standard_normal((cout, cin) + k) * np.sqrt(2.0 / (cin * np.prod(k)))).astype(np.float32)
    b = (rng.standard_normal(cout) * 0.1).astype(np.float32)
    osp = tuple(s + 2 * p - kk + 1 for s, p, kk in zip(sp, pad, k))
    pk = K.pack_conv(w, b, path=path)
    assert pk.path == path
    out = D.empty_blocked(1, cout, osp)
    K.conv3d(D.to_device_blocked(x), pk, out, pad=pad, fused_act=("relu", 1.0))
    torch.cuda.synchronize()
    mx, l2 = R.normalized_error(D.to_host_standard(out), _ref_bf16(x, w, b, pad, "relu"))
    assert mx < BF16_TOL and l2 < 3e-3, (mx, l2)


@pytest.mark.parametrize("cin,cout,k,pad,sp,base", [
    (28, 28, (3, 3, 3), (1, 1, 1), (5, 24, 16), True),     # folded, residual
    (13, 20, (3, 3, 3), (1, 1, 1), (4, 19, 13), False),    # odd y/z: floor, ragged chunk
    (64, 80, (1, 1, 1), (0, 0, 0), (3, 16, 8), False),
    (128, 128, (3, 3, 3), (1, 1, 1), (4, 16, 16), False),  # CTA pair
])
def test_fused_maxpool_bit_identical(cin, cout, k, pad, sp, base):
    """Conv with its 1x2x2 MaxPool fused into the epilogue equals conv then
    pool_kernel, bit for bit."""
    import torch
    D, K = _dev()
    rng = np.random.default_rng(cin + cout)
    x = rng.uniform(-1, 1, (1, cin) + sp).astype(np.float32)
    w = (rng.standard_normal((cout, cin) + k) * 0.2).astype(np.float32)
    b = (rng.standard_normal(cout) * 0.1).astype(np.float32)
    osp = tuple(s + 2 * p - kk + 1 for s, p, kk in zip(sp, pad, k))
    bd = D.to_device_blocked(rng.uniform(-1, 1, (1, cout) + osp).astype(np.float32)) if base else None
    pk = K.pack_conv(w, b, base_scale=np.ones(cout, np.float32) if base else None)
    xd = D.to_device_blocked(x)
    out1, out2 = D.empty_blocked(1, cout, osp), D.empty_blocked(1, cout, osp)
    psp = (osp[0], osp[1] // 2, osp[2] // 2)
    p1, p2 = D.empty_blocked(1, cout, psp), D.empty_blocked(1, cout, psp)
    K.conv3d(xd, pk, out1, pad=pad, base=bd, fused_act=("elu", 1.0), pool_out=p1)
    K.conv3d(xd, pk, out2, pad=pad, base=bd, fused_act=("elu", 1.0))
    K.pool3d(out2, p2, (1, 2, 2), (1, 2, 2), "max")
    torch.cuda.synchronize()
    np.testing.assert_array_equal(D.to_host_standard(out1), D.to_host_standard(out2))
    assert torch.equal(p1.t, p2.t)


def test_tc_conv_fp32_output_and_batch2():
    rng = np.random.default_rng(7)
    x = rng.uniform(-1, 1, (2, 16, 4, 18, 10)).astype(np.float32)
    w = (rng.standard_normal((24, 16, 3, 3, 3)) * 0.1).astype(np.float32)
    b = rng.standard_normal(24).astype(np.float32)
    got, _ = _conv_bf16(x, w, b, (1, 1, 1), None, out_dtype="fp32")
    want = _ref_bf16(x, w, b, (1, 1, 1))
    mx, _ = R.normalized_error(got, want)
    assert mx < 1e-5


def test_fused_concat_conv_matches_mergecrop_then_conv():
    import torch
    D, K = _dev()
    rng = np.random.default_rng(3)
    a = rng.uniform(-1, 1, (1, 16, 12, 22, 14)).astype(np.float32)   # skip (larger)
    bb = rng.uniform(-1, 1, (1, 24, 8, 18, 10)).astype(np.float32)   # up
    w = (rng.standard_normal((8, 40, 3, 3, 3)) * 0.1).astype(np.float32)
    bias = rng.standard_normal(8).astype(np.float32)
    m = R.mergecrop(R.bf16_round(a), R.bf16_round(bb))
    want = R.activation(R.conv3d(m, R.bf16_round(w), bias), "relu")
    ad, bd = D.to_device_blocked(a), D.to_device_blocked(bb)
    out = D.empty_blocked(1, 8, (6, 16, 8))
    pk = K.pack_conv(w, bias, cin_split=16)
    K.conv3d(ad, pk, out, x2=bd, off=(2, 2, 2), off2=(0, 0, 0), fused_act=("relu", 1.0))
    torch.cuda.synchronize()
    mx, _ = R.normalized_error(D.to_host_standard(out), want)
    assert mx < BF16_TOL


@pytest.mark.parametrize("stride,pad", [((1, 1, 1), (1, 1, 1)), ((2, 2, 2), (0, 0, 0)),
                                        ((1, 2, 3), (1, 0, 1))])
def test_direct_fp32_path_matches_oracle_1e5(stride, pad):
    """reference gate (test_kernels.py:149-156): strided convs, fp32, 1e-5."""
    import torch
    D, K = _dev()
    from paper_1903_07525_b200 import _lib
    rng = np.random.default_rng(11)
    x = rng.standard_normal((2, 8, 7, 8, 9)).astype(np.float32)
    w = (rng.standard_normal((8, 8, 3, 3, 3)) * 0.2).astype(np.float32)
    b = rng.standard_normal(8).astype(np.float32)
    want = R.conv3d(x, w, b, stride, pad)
    xd = D.to_device_blocked(x, dtype="fp32")
    out = D.empty_blocked(2, 8, want.shape[2:], "fp32")
    pk = K.pack_conv(w, b, stride=stride, path=_lib.PATH_DIRECT)
    K.conv3d(xd, pk, out, pad=pad)
    torch.cuda.synchronize()
    np.testing.assert_allclose(D.to_host_standard(out), want, atol=2e-5, rtol=0)


def test_known_answers_through_backend_api():
    """test_kernels.py:80-136 known answers via Backend.conv3d / subimage."""
    from paper_1903_07525_b200 import get_backend
    from paper_1903_07525_b200.kernels_b200 import ConvInvocation, SubImageTask
    from oracle.ref_engine import to_blocked, from_blocked
    for name in ("b200", "b200-fp32"):
        be = get_backend(name)
        one = np.ones((1, 1, 3, 3, 3), np.float32)
        out = np.zeros((1, 1, 1, 1, 1, 8), np.float32)
        inv = ConvInvocation(to_blocked(one), 1, one, np.zeros(8, np.float32), out, 1)
        be.conv3d(inv)
        assert out[0, 0, 0, 0, 0, 0] == 27.0 and not out[..., 1:].any()
        # bias + base: 10.5 (test_kernels.py:91-99)
        z = np.zeros((1, 1, 3, 3, 3), np.float32)
        base = to_blocked(np.full((1, 1, 1, 1, 1), 10.0, np.float32))
        out = np.zeros((1, 1, 1, 1, 1, 8), np.float32)
        inv = ConvInvocation(to_blocked(z), 1, z, np.array([0.5] + [0] * 7, np.float32), out, 1,
                             additive=True, base_view=base)
        be.conv3d(inv)
        assert out[0, 0, 0, 0, 0, 0] == 10.5
        # epilogue order relu(bias + scale*base) (test_kernels.py:170-181)
        base = to_blocked(np.full((1, 1, 1, 1, 1), -4.0, np.float32))
        for bias, want in ((1.0, 0.0), (3.0, 1.0)):
            out = np.zeros((1, 1, 1, 1, 1, 8), np.float32)
            inv = ConvInvocation(to_blocked(z), 1, z, np.array([bias] + [0] * 7, np.float32), out,
                                 1, additive=True, base_view=base,
                                 base_scale=np.array([0.5] + [0] * 7, np.float32),
                                 fused_act=("relu", 0.0))
            be.conv3d(inv)
            assert out[0, 0, 0, 0, 0, 0] == want
    # sub-image chaining == full conv (test_kernels.py:103-115), fp32 primitive
    rng = np.random.default_rng(5)
    x = rng.standard_normal((1, 16, 5, 5, 5)).astype(np.float32)
    k = (rng.standard_normal((8, 16, 3, 3, 3)) * 0.2).astype(np.float32)
    bias = rng.standard_normal(8).astype(np.float32)
    out = np.zeros((1, 1, 3, 3, 3, 8), np.float32)
    inv = ConvInvocation(to_blocked(x), 16, k, bias, out, 8)
    be = get_backend("b200")
    for ib, (first, last) in enumerate([(True, False), (False, True)]):
        be.subimage(SubImageTask(ib, 0, (0, 0, 0), (3, 3, 3), first, last), inv)
    np.testing.assert_allclose(from_blocked(out, 8), R.conv3d(x, k, bias), atol=1e-5, rtol=0)


def test_tail_lanes_zero_and_halo_clean():
    """test_kernels.py:198-222: sigmoid tails stay 0; writing into a halo
    interior leaves the halo untouched."""
    from paper_1903_07525_b200 import get_backend
    from paper_1903_07525_b200.kernels_b200 import ConvInvocation
    from oracle.ref_engine import to_blocked
    rng = np.random.default_rng(9)
    x = rng.standard_normal((1, 5, 6, 6, 6)).astype(np.float32)
    k = (rng.standard_normal((5, 5, 3, 3, 3)) * 0.2).astype(np.float32)
    b = rng.standard_normal(5).astype(np.float32)
    alloc = np.full((1, 1, 6, 6, 6, 8), 7.0, np.float32)
    interior = alloc[:, :, 1:5, 1:5, 1:5, :]
    inv = ConvInvocation(to_blocked(x), 5, k, np.pad(b, (0, 3)), interior, 5,
                         fused_act=("sigmoid", 0.0))
    get_backend("b200").conv3d(inv)
    assert not interior[..., 5:].any()
    ring = alloc.copy()
    ring[:, :, 1:5, 1:5, 1:5, :] = 7.0
    assert (ring == 7.0).all()
    want = R.activation(R.conv3d(R.bf16_round(x), R.bf16_round(k), b), "sigmoid")
    got = interior.transpose(0, 1, 5, 2, 3, 4).reshape(1, 8, 4, 4, 4)[:, :5]
    assert R.normalized_error(got, want)[0] < BF16_TOL


def test_conv_deterministic():
    rng = np.random.default_rng(2)
    x = rng.uniform(-1, 1, (1, 32, 6, 20, 20)).astype(np.float32)
    w = (rng.standard_normal((32, 32, 3, 3, 3)) * 0.1).astype(np.float32)
    b = np.zeros(32, np.float32)
    a1, _ = _conv_bf16(x, w, b, (1, 1, 1))
    a2, _ = _conv_bf16(x, w, b, (1, 1, 1))
    np.testing.assert_array_equal(a1, a2)


def test_pool_bit_exact_and_avg():
    import torch
    D, K = _dev()
    rng = np.random.default_rng(4)
    x = R.bf16_round(rng.standard_normal((2, 13, 6, 7, 9)).astype(np.float32))
    for win in ((2, 2, 2), (1, 2, 2)):
        want = R.pool3d(x, win, win, "max")
        xd = D.to_device_blocked(x)
        out = D.empty_blocked(2, 13, want.shape[2:])
        K.pool3d(xd, out, win, win, "max")
        torch.cuda.synchronize()
        np.testing.assert_array_equal(D.to_host_standard(out), want)
    want = R.pool3d(x, 2, 2, "avg")
    out = D.empty_blocked(2, 13, want.shape[2:], "fp32")
    K.pool3d(D.to_device_blocked(x, dtype="fp32"), out, (2, 2, 2), (2, 2, 2), "avg")
    torch.cuda.synchronize()
    np.testing.assert_array_equal(D.to_host_standard(out), want)


def test_mergecrop_eltwise_affine_exact(golden_ops):
    import torch
    D, K = _dev()
    g = golden_ops
    a = D.to_device_blocked(g["mc_a"], dtype="fp32")
    b = D.to_device_blocked(g["mc_b"], dtype="fp32")
    out = D.empty_blocked(1, 9, (7, 7, 7), "fp32")
    K.mergecrop(a, b, out)
    for op in ("add", "mul", "div"):
        o = D.empty_blocked(1, 5, (3, 3, 3), "fp32")
        K.eltwise(D.to_device_blocked(g["elt_a"], dtype="fp32"),
                  D.to_device_blocked(g["elt_b"], dtype="fp32"), o, op)
        torch.cuda.synchronize()
        np.testing.assert_array_equal(D.to_host_standard(o), g["elt_" + op])
    torch.cuda.synchronize()
    np.testing.assert_array_equal(D.to_host_standard(out), g["mc_y"])
    x = D.to_device_blocked(g["bn_x"], dtype="fp32")
    o = D.empty_blocked(1, 5, (4, 4, 4), "fp32")
    K.affine_act(x, o, D.device_vector(g["bn_gamma"]), D.device_vector(g["bn_beta"]))
    torch.cuda.synchronize()
    np.testing.assert_array_equal(D.to_host_standard(o), g["sc_y"])
    K.affine_act(x, o, None, None, "elu", 0.7)
    torch.cuda.synchronize()
    np.testing.assert_allclose(D.to_host_standard(o), g["elu_y"], atol=1e-6, rtol=0)


@pytest.mark.parametrize("shape", [(1, 13, 3, 5, 8), (2, 16, 2, 3, 12), (1, 1, 4, 4, 4)])
def test_pack_unpack_vectorized_path_exact(shape, rng):
    """z % 4 == 0 takes the float4 pack/unpack kernels; results bit-exact."""
    D, _ = _dev()
    x = R.bf16_round(rng.standard_normal(shape).astype(np.float32))
    t = D.to_device_blocked(x)
    assert not t.t[:, -1, ..., (shape[1] % 8 or 8):].float().abs().sum().item()
    np.testing.assert_array_equal(D.to_host_standard(t), x)


def test_layout_round_trip_exact(rng):
    D, _ = _dev()
    x = R.bf16_round(rng.standard_normal((2, 11, 3, 5, 7)).astype(np.float32))
    np.testing.assert_array_equal(D.to_host_standard(D.to_device_blocked(x)), x)
    t = D.to_device_blocked(x)
    assert not t.t[:, 1, ..., 3:].float().abs().sum().item()   # tail lanes are zero


@pytest.mark.parametrize("i", [0, 1, 2])
def test_deconv_golden(golden_ops, i):
    import torch
    D, K = _dev()
    g = golden_ops
    x, w, b, s = g["deconv%d_x" % i], g["deconv%d_w" % i], g["deconv%d_b" % i], g["deconv%d_s" % i]
    want_fp32 = g["deconv%d_y" % i]
    # fp32 gather path: reference gate
    pk = K.pack_deconv(w, b, stride=tuple(s), force_gather=True)
    out = D.empty_blocked(1, w.shape[0], want_fp32.shape[2:], "fp32")
    K.deconv3d(D.to_device_blocked(x, dtype="fp32"), pk, out)
    torch.cuda.synchronize()
    np.testing.assert_allclose(D.to_host_standard(out), want_fp32, atol=2e-5, rtol=0)
    # bf16 tensor-core path when k == stride
    if tuple(s) == tuple(w.shape[2:]):
        pk = K.pack_deconv(w, b, stride=tuple(s))
        out = D.empty_blocked(1, w.shape[0], want_fp32.shape[2:])
        K.deconv3d(D.to_device_blocked(x), pk, out)
        torch.cuda.synchronize()
        want = R.deconv3d(R.bf16_round(x), R.bf16_round(w), b, tuple(s))
        assert R.normalized_error(D.to_host_standard(out), want)[0] < BF16_TOL


@pytest.mark.parametrize("k", [(1, 2, 2), (2, 2, 2)])
@pytest.mark.parametrize("cin,cout", [(36, 28), (80, 64), (12, 20)])
def test_deconv_taps_in_n_matches_replicas(k, cin, cout, monkeypatch):
    """k == stride deconvs with taps x round_up(cout,16) <= 256 run as ONE
    1x1x1 GEMM with every tap in N (the epilogue routes each 16-column item
    to its tap's strided output voxels); the sums are the same MMAs as the
    one-replica-per-tap walk, so results are bit-identical, with and without
    the fused skip add + activation."""
    import torch
    D, K = _dev()
    rng = np.random.default_rng(cin + cout + k[0])
    x = rng.uniform(-1, 1, (2, cin, 3, 9, 10)).astype(np.float32)
    w = (rng.standard_normal((cout, cin) + k) * 0.2).astype(np.float32)
    b = rng.standard_normal(cout).astype(np.float32)
    osp = tuple(s * kk for s, kk in zip(x.shape[2:], k))
    base = rng.uniform(-1, 1, (2, cout) + osp).astype(np.float32)
    scale = rng.uniform(0.5, 1.5, cout).astype(np.float32)

    def run(with_base):
        pk = K.pack_deconv(w, b, stride=k, base_scale=scale if with_base else None)
        out = D.empty_blocked(2, cout, osp)
        K.deconv3d(D.to_device_blocked(x), pk, out,
                   base=D.to_device_blocked(base) if with_base else None,
                   fused_act=("elu", 1.0) if with_base else None)
        torch.cuda.synchronize()
        return D.to_host_standard(out)

    for with_base in (False, True):
        monkeypatch.setenv("VXB_DECONV_REPN", "1")
        fused = run(with_base)
        monkeypatch.setenv("VXB_DECONV_REPN", "0")
        plain = run(with_base)
        np.testing.assert_array_equal(fused, plain)
        want = R.deconv3d(R.bf16_round(x), R.bf16_round(w), b, k)
        if with_base:
            want = R.activation(want + scale.reshape(1, -1, 1, 1, 1) * R.bf16_round(base), "elu")
        assert R.normalized_error(fused, want)[0] < BF16_TOL


_FUZZ_N = int(os.environ.get("VXB_FUZZ_N", "12"))   # 300 run clean on a B200 (round 1)


@pytest.mark.parametrize("seed", range(_FUZZ_N))
def test_conv_random_shapes_match_oracle(seed):
    """Seeded random layer shapes (fmap counts 1-160, 3x3x3 / 1x3x3 / 1x1x1 /
    3x1x1 kernels, 'same' or valid padding, batch 1-2, optional residual and
    activation): exercises the tile-shape, fold, CTA-pair, N-split and
    weight-stage choices together against the oracle."""
    rng = np.random.default_rng(1000 + seed)
    cin = int(rng.choice([1, 3, 8, 12, 16, 20, 28, 32, 36, 48, 64, 80, 96, 128, 160]))
    cout = int(rng.choice([3, 8, 16, 24, 28, 32, 40, 64, 96, 128, 160]))
    k = [(3, 3, 3), (1, 3, 3), (1, 1, 1), (3, 1, 1)][int(rng.integers(4))]
    same = bool(rng.integers(2))
    pad = tuple(v // 2 for v in k) if same else (0, 0, 0)
    n = int(rng.integers(1, 3))
    sp = tuple(int(v) for v in rng.integers([3, 5, 5], [13, 40, 40]))
    sp = tuple(max(s, kk) for s, kk in zip(sp, k))
    act = [None, "relu", "elu", "sigmoid"][int(rng.integers(4))]
    use_base = bool(rng.integers(2))
    x = rng.uniform(-1, 1, (n, cin) + sp).astype(np.float32)
    w = (rng.standard_normal((cout, cin) + k) * np.sqrt(2.0 / (cin * np.prod(k)))).astype(np.float32)
    b = (rng.standard_normal(cout) * 0.1).astype(np.float32)
    osp = tuple(s + 2 * p - kk + 1 for s, p, kk in zip(sp, pad, k))
    base = rng.uniform(-1, 1, (n, cout) + osp).astype(np.float32) if use_base else None
    scale = rng.uniform(0.5, 1.5, cout).astype(np.float32) if use_base else None
    got, _ = _conv_bf16(x, w, b, pad, act, base, scale)
    want = _ref_bf16(x, w, b, pad, act, base, scale)
    mx, l2 = R.normalized_error(got, want)
    assert mx < BF16_TOL and l2 < 3e-3, (cin, cout, k, pad, n, sp, act, use_base, mx, l2)


@pytest.mark.parametrize("seed", range(_FUZZ_N))
def test_deconv_random_shapes_match_oracle(seed):
    """Seeded random transposed convs: k == stride (tensor-core replicas or
    taps in N) and k != stride (gather), optional skip add + activation."""
    import torch
    D, K = _dev()
    rng = np.random.default_rng(2000 + seed)
    cin = int(rng.choice([4, 8, 12, 28, 36, 48, 64, 80, 128]))
    cout = int(rng.choice([3, 8, 20, 28, 36, 48, 64, 96]))
    k = [(1, 2, 2), (2, 2, 2), (1, 3, 3), (3, 3, 3)][int(rng.integers(4))]
    stride = k if rng.integers(3) else (1, 2, 2)
    n = int(rng.integers(1, 3))
    sp = tuple(int(v) for v in rng.integers([2, 3, 3], [6, 12, 12]))
    osp = tuple((s - 1) * st + kk for s, st, kk in zip(sp, stride, k))
    act = [None, "relu", "elu"][int(rng.integers(3))]
    use_base = bool(rng.integers(2))
    x = rng.uniform(-1, 1, (n, cin) + sp).astype(np.float32)
    w = (rng.standard_normal((cout, cin) + k) * 0.2).astype(np.float32)
    b = rng.standard_normal(cout).astype(np.float32)
    base = rng.uniform(-1, 1, (n, cout) + osp).astype(np.float32) if use_base else None
    scale = rng.uniform(0.5, 1.5, cout).astype(np.float32) if use_base else None
    pk = K.pack_deconv(w, b, stride=stride, base_scale=scale)
    out = D.empty_blocked(n, cout, osp)
    K.deconv3d(D.to_device_blocked(x), pk, out,
               base=D.to_device_blocked(base) if use_base else None,
               fused_act=(act, 1.0) if act else None)
    torch.cuda.synchronize()
    got = D.to_host_standard(out)
    q = R.bf16_round
    want = R.deconv3d(q(x), q(w), b, stride)
    if use_base:
        want = want + scale.reshape(1, -1, 1, 1, 1) * q(base)
    if act:
        want = R.activation(want, act)
    mx, l2 = R.normalized_error(got, want)
    assert mx < BF16_TOL and l2 < 3e-3, (cin, cout, k, stride, n, sp, act, use_base, mx, l2)


@pytest.mark.parametrize("seed", range(_FUZZ_N))
def test_conv_fused_pool_random_shapes(seed):
    """Seeded random convs with the 1x2x2 max pool fused into the lean
    epilogue (odd and even y / z extents, batch 1-2, residual, activations):
    the stored output equals the unfused conv and the pooled output equals
    the pool kernel on it, bit for bit (ops.py:63-86)."""
    import torch
    D, K = _dev()
    rng = np.random.default_rng(3000 + seed)
    cin = int(rng.choice([3, 8, 16, 28, 36, 48, 64]))
    cout = int(rng.choice([8, 16, 28, 36, 48, 64, 80]))
    k = [(3, 3, 3), (1, 1, 1)][int(rng.integers(2))]
    pad = tuple(v // 2 for v in k)
    n = int(rng.integers(1, 3))
    sp = tuple(int(v) for v in rng.integers([2, 6, 6], [10, 41, 41]))
    act = [None, "relu", "elu"][int(rng.integers(3))]
    use_base = bool(rng.integers(2))
    x = D.to_device_blocked(rng.uniform(-1, 1, (n, cin) + sp).astype(np.float32))
    w = (rng.standard_normal((cout, cin) + k) * np.sqrt(2.0 / (cin * np.prod(k)))).astype(np.float32)
    b = (rng.standard_normal(cout) * 0.1).astype(np.float32)
    base = D.to_device_blocked(rng.uniform(-1, 1, (n, cout) + sp).astype(np.float32)) \
        if use_base else None
    scale = rng.uniform(0.5, 1.5, cout).astype(np.float32) if use_base else None
    pk = K.pack_conv(w, b, base_scale=scale, out_shape=sp)
    fa = (act, 1.0) if act else None
    psp = (sp[0], sp[1] // 2, sp[2] // 2)
    out, ref_out = D.empty_blocked(n, cout, sp), D.empty_blocked(n, cout, sp)
    pooled, ref_pooled = D.empty_blocked(n, cout, psp), D.empty_blocked(n, cout, psp)
    K.conv3d(x, pk, out, pad=pad, base=base, fused_act=fa, pool_out=pooled)
    K.conv3d(x, pk, ref_out, pad=pad, base=base, fused_act=fa)
    K.pool3d(ref_out, ref_pooled, (1, 2, 2), (1, 2, 2), "max")
    torch.cuda.synchronize()
    assert torch.equal(out.t, ref_out.t), (cin, cout, k, n, sp, act, use_base)
    assert torch.equal(pooled.t, ref_pooled.t), (cin, cout, k, n, sp, act, use_base)
