"""Shape propagation (reference: shapes.py:1-154).

Shapes are (batch, fmap, x, y, z).  conv/pool: floor((e + 2p - k)/s) + 1;
deconv: (e - 1)s + k - 2p; MergeCrop concatenates fmaps and crops to the
common extent with floor-centred offsets.
"""

from __future__ import annotations

from .errors import ShapeError
from .formats import (ROLE_BIAS, ROLE_BN_MEAN, ROLE_BN_VAR, ROLE_KERNEL, ROLE_SCALE_BETA,
                      ROLE_SCALE_GAMMA)
from .netspec import LayerKind, NetworkSpec

Shape = tuple


def conv_extent(extent: int, kernel: int, stride: int, pad: int) -> int:
    return (extent + 2 * pad - kernel) // stride + 1


def deconv_extent(extent: int, kernel: int, stride: int, pad: int) -> int:
    return (extent - 1) * stride + kernel - 2 * pad


def crop_offsets(larger, smaller) -> tuple:
    """Low-side offsets centring ``smaller`` inside ``larger``, ties floored."""
    return tuple((int(a) - int(b)) // 2 for a, b in zip(larger, smaller))


def _expect(store, layer, role, want):
    key = "%s.%s" % (layer, role)
    if key not in store:
        raise ShapeError("weight store lacks entry %r" % key)
    got = tuple(store.get(key).shape)
    if got != tuple(want):
        raise ShapeError("entry %r has shape %s, expected %s" % (key, got, tuple(want)))


def _layer_shape(lay, ins, store):
    kind, p = lay.kind, lay.params
    if kind is LayerKind.INPUT:
        shape = tuple(int(d) for d in p["shape"])
        if min(shape) < 1:
            raise ShapeError("layer %r declares non-positive input dims %s" % (lay.name, shape))
        return shape
    if kind in (LayerKind.CONVOLUTION, LayerKind.DECONVOLUTION):
        n, f, *sp = ins[0]
        fn = conv_extent if kind is LayerKind.CONVOLUTION else deconv_extent
        out = []
        for axis, (e, k, s, q) in enumerate(zip(sp, p["kernel"], p["stride"], p["pad"])):
            oe = fn(e, k, s, q)
            if oe < 1:
                raise ShapeError(
                    "layer %r produces non-positive extent %d on axis %d "
                    "(input %d, kernel %d, stride %d, pad %d)" % (lay.name, oe, axis, e, k, s, q))
            out.append(oe)
        if store is not None:
            _expect(store, lay.name, ROLE_KERNEL, (p["num_output"], f) + tuple(p["kernel"]))
            _expect(store, lay.name, ROLE_BIAS, (p["num_output"],))
        return (n, p["num_output"]) + tuple(out)
    if kind is LayerKind.POOLING:
        n, f, *sp = ins[0]
        out = []
        for axis, (e, k, s) in enumerate(zip(sp, p["window"], p["stride"])):
            if k > e:
                raise ShapeError("layer %r pooling window %d exceeds extent %d on axis %d"
                                 % (lay.name, k, e, axis))
            out.append((e - k) // s + 1)
        return (n, f) + tuple(out)
    if kind is LayerKind.ELTWISE:
        if ins[0] != ins[1]:
            raise ShapeError("layer %r combines mismatched shapes %s and %s"
                             % (lay.name, ins[0], ins[1]))
        return ins[0]
    if kind is LayerKind.MERGE_CROP:
        (na, fa, *sa), (nb, fb, *sb) = ins
        if na != nb:
            raise ShapeError("layer %r merges different batch sizes" % lay.name)
        if all(a >= b for a, b in zip(sa, sb)):
            common = sb
        elif all(b >= a for a, b in zip(sa, sb)):
            common = sa
        else:
            raise ShapeError("layer %r inputs %s and %s: neither spatial extent contains the other"
                             % (lay.name, tuple(sa), tuple(sb)))
        return (na, fa + fb) + tuple(common)
    if kind in (LayerKind.BATCH_NORM, LayerKind.SCALE) and store is not None:
        f = ins[0][1]
        roles = ((ROLE_BN_MEAN, ROLE_BN_VAR) if kind is LayerKind.BATCH_NORM
                 else (ROLE_SCALE_GAMMA, ROLE_SCALE_BETA))
        for role in roles:
            _expect(store, lay.name, role, (f,))
    return ins[0]


def validate_shapes(spec: NetworkSpec, store=None) -> dict:
    """Propagate shapes; returns blob name -> shape (shapes.py:85-147)."""
    spec.validate()
    shapes: dict = {}
    for idx in spec.topological_order():
        lay = spec.layers[idx]
        out = _layer_shape(lay, [shapes[b] for b in lay.bottoms], store)
        shapes[lay.tops[0]] = tuple(int(d) for d in out)
    return shapes


def network_io(spec: NetworkSpec, shapes: dict):
    inputs = [(lay.tops[0], shapes[lay.tops[0]]) for lay in spec.input_layers()]
    outputs = [(b, shapes[b]) for b in spec.output_blobs()]
    return inputs, outputs
