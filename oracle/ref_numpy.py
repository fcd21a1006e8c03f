"""numpy restatement of the reference oracle — TEST INFRASTRUCTURE ONLY.

Every function follows the reference's naive implementation in
pkg/src/voxplan/oracle.py (cited per function): standard (b, f, x, y, z)
arrays, float32 arithmetic, cross-correlation without kernel flip, the same
accumulation order (bias first, then kernel offsets dx, dy, dz ascending).

``run_plan`` is a second oracle at the *plan* level: it executes the steps of
a compiled ExecutionPlan (after fusion) on standard arrays, optionally
rounding every stored tensor and the weights to bf16 the way the B200 path
stores them.  It restates executor.PlanRunner semantics
(pkg/src/voxplan/executor.py:89-198) without the blocked layout.
"""

from __future__ import annotations

import numpy as np

F32 = np.float32


def _t3(v):
    if np.isscalar(v):
        return (int(v),) * 3
    return tuple(int(a) for a in v)


def bf16_round(a) -> np.ndarray:
    """Round-to-nearest-even to bfloat16, returned as float32."""
    a = np.ascontiguousarray(np.asarray(a, dtype=F32))
    u = a.view(np.uint32).astype(np.uint64)
    finite = (u & 0x7F800000) != 0x7F800000
    r = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    r = np.where(finite, r, u & 0xFFFF0000)
    return r.astype(np.uint32).view(F32).reshape(a.shape)


def tf32_trunc(a) -> np.ndarray:
    """The tf32 operand a tcgen05 kind::tf32 MMA reads from fp32: the low 13
    mantissa bits dropped (truncation), returned as float32."""
    a = np.ascontiguousarray(np.asarray(a, dtype=F32))
    return (a.view(np.uint32) & np.uint32(0xFFFFE000)).view(F32).reshape(a.shape)


def split_bf16(a) -> tuple:
    """(hi, lo): hi = bf16(a), lo = bf16(a - hi), both as float32.  hi + lo
    holds a to ~16 mantissa bits; the sum is exact in float32."""
    a = np.asarray(a, dtype=F32)
    hi = bf16_round(a)
    lo = bf16_round(a - hi)
    return hi, lo


def conv3d(image, kernel, bias, stride=1, pad=0):
    """oracle.ref_conv3d (oracle.py:37-64)."""
    x = np.asarray(image, F32)
    w = np.asarray(kernel, F32)
    sx, sy, sz = _t3(stride)
    px, py, pz = _t3(pad)
    x = np.pad(x, ((0, 0), (0, 0), (px, px), (py, py), (pz, pz)))
    n, ci, ix, iy, iz = x.shape
    co, ck, kx, ky, kz = w.shape
    if ck != ci:
        raise ValueError("kernel expects %d input fmaps, image has %d" % (ck, ci))
    ox, oy, oz = (ix - kx) // sx + 1, (iy - ky) // sy + 1, (iz - kz) // sz + 1
    out = np.empty((n, co, ox, oy, oz), F32)
    out[...] = np.asarray(bias, F32).reshape(1, co, 1, 1, 1)
    for dx in range(kx):
        for dy in range(ky):
            for dz in range(kz):
                win = x[:, :, dx:dx + sx * (ox - 1) + 1:sx, dy:dy + sy * (oy - 1) + 1:sy,
                        dz:dz + sz * (oz - 1) + 1:sz]
                # (co, ci) x (n, ci, ...) -> (co, n, ...)
                part = np.tensordot(w[:, :, dx, dy, dz], win, axes=([1], [1]))
                out += np.moveaxis(part, 0, 1)
    return out


def deconv3d(image, kernel, bias, stride=1, pad=0):
    """oracle.ref_deconv3d (oracle.py:67-93): scatter per tap, crop, + bias."""
    x = np.asarray(image, F32)
    w = np.asarray(kernel, F32)
    sx, sy, sz = _t3(stride)
    px, py, pz = _t3(pad)
    n, ci, ix, iy, iz = x.shape
    co, ck, kx, ky, kz = w.shape
    if ck != ci:
        raise ValueError("kernel expects %d input fmaps, image has %d" % (ck, ci))
    full = np.zeros((n, co, (ix - 1) * sx + kx, (iy - 1) * sy + ky, (iz - 1) * sz + kz), F32)
    for dx in range(kx):
        for dy in range(ky):
            for dz in range(kz):
                part = np.moveaxis(np.tensordot(w[:, :, dx, dy, dz], x, axes=([1], [1])), 0, 1)
                full[:, :, dx:dx + sx * (ix - 1) + 1:sx, dy:dy + sy * (iy - 1) + 1:sy,
                     dz:dz + sz * (iz - 1) + 1:sz] += part
    fx, fy, fz = full.shape[2:]
    return full[:, :, px:fx - px, py:fy - py, pz:fz - pz] + np.asarray(bias, F32).reshape(1, co, 1, 1, 1)


def pool3d(image, window, stride, mode="max"):
    """oracle.ref_pool3d (oracle.py:96-122): first window element seeds,
    max / sum in (dx, dy, dz) order, avg divides by the window volume."""
    x = np.asarray(image, F32)
    kx, ky, kz = _t3(window)
    sx, sy, sz = _t3(stride)
    ox, oy, oz = ((x.shape[2] - kx) // sx + 1, (x.shape[3] - ky) // sy + 1,
                  (x.shape[4] - kz) // sz + 1)
    acc = None
    for dx in range(kx):
        for dy in range(ky):
            for dz in range(kz):
                win = x[:, :, dx:dx + sx * (ox - 1) + 1:sx, dy:dy + sy * (oy - 1) + 1:sy,
                        dz:dz + sz * (oz - 1) + 1:sz]
                if acc is None:
                    acc = win.copy()
                elif mode == "max":
                    np.maximum(acc, win, out=acc)
                else:
                    acc += win
    if mode == "avg":
        acc /= F32(kx * ky * kz)
    return acc


def eltwise(a, b, op):
    """oracle.ref_eltwise (oracle.py:125-134)."""
    a, b = np.asarray(a, F32), np.asarray(b, F32)
    with np.errstate(divide="ignore", invalid="ignore"):
        return {"add": np.add, "mul": np.multiply, "div": np.divide}[op](a, b)


def crop_offsets(larger, smaller):
    """shapes.crop_offsets (shapes.py:35-37): floor-centred."""
    return tuple((a - b) // 2 for a, b in zip(larger, smaller))


def mergecrop(a, b):
    """oracle.ref_mergecrop (oracle.py:137-146)."""
    a, b = np.asarray(a, F32), np.asarray(b, F32)
    common = tuple(min(p, q) for p, q in zip(a.shape[2:], b.shape[2:]))

    def crop(t):
        o = crop_offsets(t.shape[2:], common)
        return t[:, :, o[0]:o[0] + common[0], o[1]:o[1] + common[1], o[2]:o[2] + common[2]]
    return np.concatenate([crop(a), crop(b)], axis=1)


def batch_norm(image, mean, var, eps):
    """oracle.ref_batch_norm (oracle.py:149-153): factor in fp64 -> fp32."""
    factor = (1.0 / np.sqrt(np.asarray(var, np.float64) + eps)).astype(F32)
    return ((np.asarray(image, F32) - np.asarray(mean, F32).reshape(1, -1, 1, 1, 1))
            * factor.reshape(1, -1, 1, 1, 1))


def scale(image, gamma, beta):
    """oracle.ref_scale (oracle.py:156-159)."""
    return (np.asarray(image, F32) * np.asarray(gamma, F32).reshape(1, -1, 1, 1, 1)
            + np.asarray(beta, F32).reshape(1, -1, 1, 1, 1))


def activation(image, kind, alpha=1.0):
    """oracle.ref_activation (oracle.py:162-174)."""
    x = np.asarray(image, F32)
    with np.errstate(over="ignore"):
        if kind == "relu":
            return np.maximum(x, F32(0))
        if kind == "elu":
            return np.where(x > 0, x, F32(alpha) * np.expm1(x, dtype=F32))
        if kind == "sigmoid":
            return F32(1) / (F32(1) + np.exp(-x, dtype=F32))
    raise ValueError("unknown activation %r" % kind)


def _kind(layer):
    k = layer.kind
    return getattr(k, "value", k)


def ref_run(spec, store, inputs) -> dict:
    """oracle.ref_run (oracle.py:184-252): naive whole-network forward."""
    inputs_l = [l for l in spec.layers if _kind(l) == "Input"]
    if isinstance(inputs, np.ndarray):
        inputs = {inputs_l[0].tops[0]: inputs}
    blobs = {}
    for idx in spec.topological_order():
        lay = spec.layers[idx]
        k = _kind(lay)
        p = lay.params
        ins = [blobs[b] for b in lay.bottoms]
        t = lambda role: store.tensor(lay.name, role)  # noqa: E731
        if k == "Input":
            out = np.asarray(inputs[lay.tops[0]], F32)
            if tuple(out.shape) != tuple(p["shape"]):
                raise ValueError("input %r has shape %s" % (lay.tops[0], out.shape))
        elif k == "Convolution":
            out = conv3d(ins[0], t("kernel"), t("bias"), p["stride"], p["pad"])
        elif k == "Deconvolution":
            out = deconv3d(ins[0], t("kernel"), t("bias"), p["stride"], p["pad"])
        elif k == "Pooling":
            out = pool3d(ins[0], p["window"], p["stride"], p["mode"])
        elif k == "Eltwise":
            out = eltwise(ins[0], ins[1], p["op"])
        elif k == "MergeCrop":
            out = mergecrop(ins[0], ins[1])
        elif k == "BatchNorm":
            out = batch_norm(ins[0], t("bn_mean"), t("bn_var"), store.bn_eps(lay.name))
        elif k == "Scale":
            out = scale(ins[0], t("scale_gamma"), t("scale_beta"))
        elif k in ("ReLU", "ELU", "Sigmoid"):
            out = activation(ins[0], k.lower(), p.get("alpha", 1.0))
        else:
            raise ValueError("oracle cannot run layer kind %s" % k)
        blobs[lay.tops[0]] = out
    used = {b for l in spec.layers for b in l.bottoms}
    return {tp: blobs[tp] for l in spec.layers for tp in l.tops if tp not in used}


def run_plan(plan, inputs, storage="fp32") -> dict:
    """Execute a compiled plan's steps on standard arrays (executor.py:89-198).

    ``storage`` emulates the B200 backends' roundings (arithmetic stays fp32;
    biases, base scales and BN coefficients stay fp32):
      * "fp32": none (the reference's own arithmetic, in another order);
      * "bf16": network inputs, every step output and every conv/deconv weight
        rounded to bf16 (backend ``b200``);
      * "tf32": fp32 storage, conv/deconv operands truncated to tf32;
      * "split": every stored tensor held as bf16 hi + bf16 lo (backend
        ``b200-x3``), conv(x, W) = conv(x, W_hi) + conv(x_hi, W_lo) with
        W_hi = bf16(W), W_lo = bf16(W - W_hi).
    """
    if storage == "bf16":
        q = bf16_round
    elif storage == "split":
        def q(a):
            hi, lo = split_bf16(a)
            return hi + lo
    else:
        q = lambda a: np.asarray(a, F32)  # noqa: E731
    w = plan.weights
    if isinstance(inputs, np.ndarray):
        inputs = {plan.inputs[0][0]: inputs}
    cur = {}
    for name, bid, dims in plan.inputs:
        cur[bid] = (q(inputs[name]), tuple(dims))

    def read(si):
        arr, dims = cur[si.buffer]
        halo = [(a - b) // 2 for a, b in zip(si.dims[2:], arr.shape[2:])]
        if any(halo):
            arr = np.pad(arr, ((0, 0), (0, 0)) + tuple((h, h) for h in halo))
        return arr

    def contract(fn, x, kern, stride):
        kern = np.asarray(kern, F32)
        zero = np.zeros(kern.shape[0], F32)
        if storage == "bf16":
            return fn(x, bf16_round(kern), zero, stride, 0)
        if storage == "tf32":
            return fn(tf32_trunc(x), tf32_trunc(kern), zero, stride, 0)
        if storage == "split":
            whi, wlo = split_bf16(kern)
            return fn(x, whi, zero, stride, 0) + fn(split_bf16(x)[0], wlo, zero, stride, 0)
        return fn(x, kern, zero, stride, 0)

    for st in plan.steps:
        k = _kind(st)
        p = st.params
        if k == "Pad":
            pads = p["pads"]
            x = read(st.inputs[0])
            cur[st.output.buffer] = (np.pad(x, ((0, 0), (0, 0)) + tuple((v, v) for v in pads)),
                                     None)
            continue
        ins = [read(si) for si in st.inputs]
        if k in ("Convolution", "Deconvolution"):
            kern = w.tensor(st.name, "kernel")
            bias = np.asarray(w.tensor(st.name, "bias"), F32)
            y = contract(conv3d if k == "Convolution" else deconv3d, ins[0], kern, p["stride"])
            init = np.broadcast_to(bias.reshape(1, -1, 1, 1, 1), y.shape).astype(F32)
            if st.additive:
                base = read(st.base)
                sc = (np.ones_like(bias) if st.base_scale is None
                      else np.asarray(st.base_scale, F32))
                init = init + sc.reshape(1, -1, 1, 1, 1) * base
            y = init + y
            if st.fused_act is not None:
                y = activation(y, st.fused_act[0], st.fused_act[1])
        elif k == "Pooling":
            y = pool3d(ins[0], p["window"], p["stride"], p["mode"])
        elif k == "Eltwise":
            y = eltwise(ins[0], ins[1], p["op"])
        elif k == "MergeCrop":
            y = mergecrop(ins[0], ins[1])
        elif k == "BatchNorm":
            f = (1.0 / np.sqrt(np.asarray(w.tensor(st.name, "bn_var"), np.float64)
                               + w.bn_eps(st.name)))
            m = f.astype(F32)
            a = (-np.asarray(w.tensor(st.name, "bn_mean"), np.float64) * f).astype(F32)
            y = ins[0] * m.reshape(1, -1, 1, 1, 1) + a.reshape(1, -1, 1, 1, 1)
        elif k == "Scale":
            y = scale(ins[0], w.tensor(st.name, "scale_gamma"), w.tensor(st.name, "scale_beta"))
        elif k in ("ReLU", "ELU", "Sigmoid"):
            y = activation(ins[0], k.lower(), p.get("alpha", 1.0))
        else:
            raise ValueError("run_plan cannot run step kind %s" % k)
        cur[st.output.buffer] = (q(y), None)
    return {name: cur[bid][0] for name, bid, _ in plan.outputs}


def normalized_error(got, ref) -> tuple:
    """(max|got-ref| / max|ref|, ||got-ref||_2 / ||ref||_2) — the parity
    measures stated per config."""
    got = np.asarray(got, np.float64)
    ref = np.asarray(ref, np.float64)
    d = got - ref
    mx = float(np.abs(d).max() / max(np.abs(ref).max(), 1e-30))
    l2 = float(np.linalg.norm(d.ravel()) / max(np.linalg.norm(ref.ravel()), 1e-30))
    return mx, l2
