"""The five BASELINE.json workloads as networks + seeded weights.

Each builder returns ``(NetworkSpec, WeightStore)`` in the reference's own
data model (prototxt-printable, PZNW-serialisable), so the same artefacts
drive the reference's CPU engine and the B200 engine.
Weights: He-normal std = sqrt(2 / (cin * kvol)); biases N(0, 0.1); "random
BN" = bn_mean N(0, 0.1), bn_var U[0.5, 1.5], scale_gamma U[0.5, 1.5],
scale_beta N(0, 0.1), bn_eps 1e-5 — all from ``numpy.random.default_rng(seed)``
in declaration order.  Inputs are seeded uniform volumes (``make_input``).
"""

from __future__ import annotations

import numpy as np

from .formats import (DEFAULT_BN_EPS, ROLE_BIAS, ROLE_BN_EPS, ROLE_BN_MEAN, ROLE_BN_VAR,
                      ROLE_KERNEL, ROLE_SCALE_BETA, ROLE_SCALE_GAMMA, WeightStore)
from .netspec import LayerKind, LayerSpec, NetworkSpec
from .shapes import validate_shapes


class _Net:
    def __init__(self, name, seed):
        self.name = name
        self.layers = []
        self.store = WeightStore()
        self.rng = np.random.default_rng(seed)

    def _add(self, name, kind, bottoms, params=None):
        self.layers.append(LayerSpec(name, kind, tuple(bottoms), (name,), dict(params or {})))
        return name

    def input(self, shape):
        return self._add("data", LayerKind.INPUT, (), {"shape": tuple(shape)})

    def conv(self, name, bottom, cin, cout, k, pad=(0, 0, 0), stride=(1, 1, 1),
             kind=LayerKind.CONVOLUTION):
        k = tuple(k)
        self._add(name, kind, (bottom,), {"num_output": cout, "kernel": k,
                                           "stride": tuple(stride), "pad": tuple(pad)})
        std = np.sqrt(2.0 / (cin * int(np.prod(k))))
        self.store.put("%s.%s" % (name, ROLE_KERNEL),
                       self.rng.standard_normal((cout, cin) + k) * std)
        self.store.put("%s.%s" % (name, ROLE_BIAS), self.rng.standard_normal(cout) * 0.1)
        return name

    def bn_scale(self, prefix, bottom, f):
        bn = self._add(prefix + "_bn", LayerKind.BATCH_NORM, (bottom,))
        self.store.put(bn + "." + ROLE_BN_MEAN, self.rng.standard_normal(f) * 0.1)
        self.store.put(bn + "." + ROLE_BN_VAR, self.rng.uniform(0.5, 1.5, f))
        self.store.put(bn + "." + ROLE_BN_EPS, np.float32(DEFAULT_BN_EPS))
        sc = self._add(prefix + "_scale", LayerKind.SCALE, (bn,))
        self.store.put(sc + "." + ROLE_SCALE_GAMMA, self.rng.uniform(0.5, 1.5, f))
        self.store.put(sc + "." + ROLE_SCALE_BETA, self.rng.standard_normal(f) * 0.1)
        return sc

    def act(self, name, bottom, kind, alpha=1.0):
        params = {"alpha": float(alpha)} if kind is LayerKind.ELU else {}
        return self._add(name, kind, (bottom,), params)

    def add(self, name, a, b):
        return self._add(name, LayerKind.ELTWISE, (a, b), {"op": "add"})

    def pool(self, name, bottom, window):
        return self._add(name, LayerKind.POOLING, (bottom,),
                         {"mode": "max", "window": tuple(window), "stride": tuple(window)})

    def merge(self, name, a, b):
        return self._add(name, LayerKind.MERGE_CROP, (a, b))

    def done(self):
        spec = NetworkSpec(self.name, tuple(self.layers))
        validate_shapes(spec, self.store)
        return spec, self.store


def config1(seed=1):
    """PR1 workload: conv 3^3 C16->16 'same' + bias + ReLU on 1x16x32x64x64."""
    n = _Net("cfg1_conv16", seed)
    x = n.input((1, 16, 32, 64, 64))
    c = n.conv("conv", x, 16, 16, (3, 3, 3), pad=(1, 1, 1))
    n.act("relu", c, LayerKind.RELU)
    return n.done()


SWEEP_C = (8, 16, 32, 64, 128)
SWEEP_K = ((3, 3, 3), (1, 3, 3))


def config2(c, k, seed=2):
    """Featuremap sweep layer: conv C->C kernel k 'same' + bias + ELU on 1xCx32x128x128."""
    k = tuple(k)
    n = _Net("cfg2_c%d_k%s" % (c, "x".join(map(str, k))), seed)
    x = n.input((1, c, 32, 128, 128))
    cv = n.conv("conv", x, c, c, k, pad=tuple(v // 2 for v in k))
    n.act("elu", cv, LayerKind.ELU, 1.0)
    return n.done()


def config3(seed=3, spatial=(24, 128, 128), c=64):
    """Residual block: conv-BN-ELU-conv-BN-add(input)-ELU at C=64 on 1x64x24x128x128."""
    n = _Net("cfg3_resblock", seed)
    x = n.input((1, c) + tuple(spatial))
    c1 = n.conv("c1", x, c, c, (3, 3, 3), pad=(1, 1, 1))
    a1 = n.act("c1_elu", n.bn_scale("c1", c1, c), LayerKind.ELU)
    c2 = n.conv("c2", a1, c, c, (3, 3, 3), pad=(1, 1, 1))
    s = n.add("res_add", n.bn_scale("c2", c2, c), x)
    n.act("out_elu", s, LayerKind.ELU)
    return n.done()


def config4(seed=4, spatial=(132, 132, 132), base=32, levels=4, out_ch=3):
    """3D U-net (Cicek et al.): valid 3^3 convs + ReLU, 2^3 maxpool, 2^3 s2
    deconv keeping channels, crop+concat skips, 1^3 head to 3 fmaps.
    Levels l = 0..3 with f = base*2^l: analysis convs f, 2f (bottom 256->512);
    synthesis convs 2f, 2f after concat(skip 2f, up 4f)."""
    n = _Net("cfg4_unet_cicek", seed)
    top, cin = n.input((1, 1) + tuple(spatial)), 1
    skips = []
    for lv in range(levels):
        f = base * 2 ** lv
        top = n.act("d%d_relu1" % lv, n.conv("d%d_conv1" % lv, top, cin, f, (3, 3, 3)),
                    LayerKind.RELU)
        top = n.act("d%d_relu2" % lv, n.conv("d%d_conv2" % lv, top, f, 2 * f, (3, 3, 3)),
                    LayerKind.RELU)
        cin = 2 * f
        if lv < levels - 1:
            skips.append((top, cin))
            top = n.pool("pool%d" % lv, top, (2, 2, 2))
    for lv in range(levels - 2, -1, -1):
        f = base * 2 ** lv
        up = n.conv("u%d_up" % lv, top, cin, cin, (2, 2, 2), stride=(2, 2, 2),
                    kind=LayerKind.DECONVOLUTION)
        skip, sc = skips.pop()
        top = n.merge("u%d_merge" % lv, skip, up)
        top = n.act("u%d_relu1" % lv, n.conv("u%d_conv1" % lv, top, sc + cin, 2 * f, (3, 3, 3)),
                    LayerKind.RELU)
        top = n.act("u%d_relu2" % lv, n.conv("u%d_conv2" % lv, top, 2 * f, 2 * f, (3, 3, 3)),
                    LayerKind.RELU)
        cin = 2 * f
    n.conv("output", top, cin, out_ch, (1, 1, 1))
    return n.done()


# ------------------------------------------------------------------ BN calibration
# Workload generation only (synthetic weights), not an inference path: the
# engine has no CPU execution path.  A trained network's BatchNorm holds the
# running statistics of the activations it normalises; random BN statistics
# (round 1) let config 5's activations grow through 28 unnormalised convs to
# |logit| ~ 600, a degenerate sigmoid output of 0s and 1s in which any
# rounding flips a probability (BASELINE.md §3 note).  Calibrated
# networks keep |logit| ~ 10.

def _np_conv(x, w, b, pad):
    px, py, pz = pad
    x = np.pad(x, ((0, 0), (0, 0), (px, px), (py, py), (pz, pz)))
    co, _, kx, ky, kz = w.shape
    n, _, ix, iy, iz = x.shape
    ox, oy, oz = ix - kx + 1, iy - ky + 1, iz - kz + 1
    out = np.zeros((co, n, ox, oy, oz), np.float32)
    for dx in range(kx):
        for dy in range(ky):
            for dz in range(kz):
                out += np.tensordot(w[:, :, dx, dy, dz],
                                    x[:, :, dx:dx + ox, dy:dy + oy, dz:dz + oz], axes=([1], [1]))
    return np.moveaxis(out, 0, 1) + b.reshape(1, -1, 1, 1, 1)


def _np_deconv_kstride(x, w, b):
    co, _, kx, ky, kz = w.shape
    n, _, ix, iy, iz = x.shape
    out = np.zeros((n, co, ix * kx, iy * ky, iz * kz), np.float32)
    for dx in range(kx):
        for dy in range(ky):
            for dz in range(kz):
                out[:, :, dx::kx, dy::ky, dz::kz] = np.moveaxis(
                    np.tensordot(w[:, :, dx, dy, dz], x, axes=([1], [1])), 0, 1)
    return out + b.reshape(1, -1, 1, 1, 1)


def calibrate_bn(spec, store, x):
    """Set every BatchNorm's (mean, var) to the per-fmap statistics of its own
    input on volume ``x`` (one forward in topological order, each BN applied
    with its calibrated statistics before later layers see it).  Supports the
    layer kinds of the BASELINE U-nets."""
    blobs = {}
    for idx in spec.topological_order():
        lay = spec.layers[idx]
        k, prm = lay.kind, lay.params
        ins = [blobs[b] for b in lay.bottoms]

        def t(role):
            return store.tensor(lay.name, role)
        if k is LayerKind.INPUT:
            out = np.asarray(x, np.float32)
        elif k is LayerKind.CONVOLUTION:
            if tuple(prm.get("stride", (1, 1, 1))) != (1, 1, 1):
                raise ValueError("calibrate_bn: strided conv")
            out = _np_conv(ins[0], t(ROLE_KERNEL), t(ROLE_BIAS), prm["pad"])
        elif k is LayerKind.DECONVOLUTION:
            out = _np_deconv_kstride(ins[0], t(ROLE_KERNEL), t(ROLE_BIAS))
        elif k is LayerKind.POOLING:
            wx, wy, wz = prm["window"]
            a = ins[0]
            n_, c_, X, Y, Z = a.shape
            out = a[:, :, :X // wx * wx, :Y // wy * wy, :Z // wz * wz].reshape(
                n_, c_, X // wx, wx, Y // wy, wy, Z // wz, wz).max(axis=(3, 5, 7))
        elif k is LayerKind.ELTWISE:
            out = ins[0] + ins[1]
        elif k is LayerKind.BATCH_NORM:
            a = ins[0].astype(np.float64)
            mean = a.mean(axis=(0, 2, 3, 4))
            var = a.var(axis=(0, 2, 3, 4))
            store.put(lay.name + "." + ROLE_BN_MEAN, mean)
            store.put(lay.name + "." + ROLE_BN_VAR, var)
            eps = float(np.asarray(store.tensor(lay.name, ROLE_BN_EPS)))
            f = (1.0 / np.sqrt(var + eps)).astype(np.float32)
            out = (ins[0] - mean.astype(np.float32).reshape(1, -1, 1, 1, 1)) * f.reshape(
                1, -1, 1, 1, 1)
        elif k is LayerKind.SCALE:
            out = ins[0] * t(ROLE_SCALE_GAMMA).reshape(1, -1, 1, 1, 1) + \
                t(ROLE_SCALE_BETA).reshape(1, -1, 1, 1, 1)
        elif k is LayerKind.ELU:
            a = ins[0]
            out = np.where(a > 0, a, np.float32(prm.get("alpha", 1.0)) * np.expm1(np.minimum(a, 0)))
        elif k is LayerKind.RELU:
            out = np.maximum(ins[0], 0)
        elif k is LayerKind.SIGMOID:
            out = 1.0 / (1.0 + np.exp(-ins[0]))
        else:
            raise ValueError("calibrate_bn: layer kind %s" % k)
        blobs[lay.tops[0]] = np.asarray(out, np.float32)
    return store


CALIB_PATCH5 = (18, 96, 96)     # calibration volume for config 5 (smaller than a patch)
_CAL_CACHE: dict = {}


def config5(seed=5, patch=(18, 192, 192), feats=(28, 36, 48, 64, 80), out_ch=3, bn="calibrated"):
    """Anisotropic residual symmetric U-net (Lee et al. 2017 style) on one patch.
    Level block: c0 1x3x3 -> BN/Scale/ELU = a0 -> c1 3^3 -> BN/Scale/ELU ->
    c2 3^3 -> add(c2, a0) -> BN/Scale/ELU; 1x2x2 maxpool; 1x2x2 s(1,2,2)
    deconv + summation skip; 1^3 head to 3 fmaps + sigmoid.

    ``bn="calibrated"`` (default): BN statistics measured on a seeded U[0,1)
    calibration volume of min(patch, CALIB_PATCH5) (calibrate_bn), as a
    trained network holds them; ``bn="random"``: round 1's random statistics
    (bn_mean N(0, 0.1), bn_var U[0.5, 1.5])."""
    key = (seed, tuple(patch), tuple(feats), out_ch, bn)
    if key in _CAL_CACHE:
        spec, store = _CAL_CACHE[key]
        return spec, store.copy()
    spec, store = _config5_random(seed, patch, feats, out_ch)
    if bn == "calibrated":
        cp = tuple(min(a, b) for a, b in zip(patch, CALIB_PATCH5))
        xc = np.random.default_rng(55555).uniform(0, 1, (1, 1) + cp).astype(np.float32)
        calibrate_bn(spec, store, xc)
    elif bn != "random":
        raise ValueError("bn must be 'calibrated' or 'random'")
    _CAL_CACHE[key] = (spec, store.copy())
    return spec, store


def _config5_random(seed, patch, feats, out_ch):
    n = _Net("cfg5_unet_aniso", seed)
    top, cin = n.input((1, 1) + tuple(patch)), 1

    def block(pfx, bottom, ci, f):
        c0 = n.conv(pfx + "_c0", bottom, ci, f, (1, 3, 3), pad=(0, 1, 1))
        a0 = n.act(pfx + "_a0", n.bn_scale(pfx + "_c0", c0, f), LayerKind.ELU)
        c1 = n.conv(pfx + "_c1", a0, f, f, (3, 3, 3), pad=(1, 1, 1))
        a1 = n.act(pfx + "_a1", n.bn_scale(pfx + "_c1", c1, f), LayerKind.ELU)
        c2 = n.conv(pfx + "_c2", a1, f, f, (3, 3, 3), pad=(1, 1, 1))
        s = n.add(pfx + "_res", c2, a0)
        return n.act(pfx + "_a2", n.bn_scale(pfx + "_c2", s, f), LayerKind.ELU)

    skips = []
    for lv, f in enumerate(feats):
        top = block("d%d" % lv, top, cin, f)
        cin = f
        if lv < len(feats) - 1:
            skips.append(top)
            top = n.pool("pool%d" % lv, top, (1, 2, 2))
    for lv in range(len(feats) - 2, -1, -1):
        f = feats[lv]
        up = n.conv("u%d_up" % lv, top, cin, f, (1, 2, 2), stride=(1, 2, 2),
                    kind=LayerKind.DECONVOLUTION)
        top = block("u%d" % lv, n.add("u%d_skip" % lv, up, skips.pop()), f, f)
        cin = f
    out = n.conv("output", top, cin, out_ch, (1, 1, 1))
    n.act("prob", out, LayerKind.SIGMOID)
    return n.done()


VOLUME5 = (128, 1024, 1024)


def make_input(spec, seed=0, low=-1.0, high=1.0):
    """Seeded uniform input for the (single) input layer."""
    shape = spec.input_layers()[0].params["shape"]
    return np.random.default_rng(seed).uniform(low, high, shape).astype(np.float32)


def input_range(cfg: int):
    """BASELINE.json input distributions: configs 1-3 U[-1,1], 4-5 U[0,1]."""
    return (-1.0, 1.0) if cfg in (1, 2, 3) else (0.0, 1.0)


def conv_flops(spec) -> float:
    """Algorithmic FLOPs (2 per MAC) of every Convolution/Deconvolution."""
    shapes = validate_shapes(spec)
    total = 0.0
    for lay in spec.layers:
        if lay.kind in (LayerKind.CONVOLUTION, LayerKind.DECONVOLUTION):
            cin = shapes[lay.bottoms[0]][1]
            out = shapes[lay.tops[0]]
            kvol = int(np.prod(lay.params["kernel"]))
            if lay.kind is LayerKind.CONVOLUTION:
                total += 2.0 * cin * kvol * int(np.prod(out[1:])) * out[0]
            else:
                ins = shapes[lay.bottoms[0]]
                total += 2.0 * cin * kvol * out[1] * int(np.prod(ins[2:])) * ins[0]
    return total
