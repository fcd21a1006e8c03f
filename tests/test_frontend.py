"""Host front end: prototxt, PZNW, shapes, passes, plans — pinned against
artefacts produced by the reference (tests/golden/nets.npz)."""

import numpy as np
import pytest

import paper_1903_07525_b200 as P
from paper_1903_07525_b200 import configs as C
from paper_1903_07525_b200 import formats, plan as vplan, prototxt
from paper_1903_07525_b200.errors import (CycleError, DanglingReferenceError, FormatError,
                                          ModelError, ParseError, PlanError, ShapeError,
                                          UnknownLayerError)
from paper_1903_07525_b200.netspec import LayerKind
from oracle import ref_numpy as R


def _net(g, i):
    spec = prototxt.parse_network(bytes(g["net%d_prototxt" % i]).decode())
    store = formats.parse_weights(bytes(g["net%d_pznw" % i]))
    return spec, store


@pytest.mark.parametrize("i", [0, 1, 2])
def test_prototxt_and_pznw_round_trip_bytes(golden_nets, i):
    spec, store = _net(golden_nets, i)
    assert prototxt.print_network(spec) == bytes(golden_nets["net%d_prototxt" % i]).decode()
    assert formats.dump_weights(store) == bytes(golden_nets["net%d_pznw" % i])


@pytest.mark.parametrize("i", [0, 1, 2])
def test_compiled_plan_matches_reference_plan_bytes(golden_nets, i):
    """Same steps, buffers, fused flags and folded (fp64) weights as the
    reference's compile_network: the serialized plans are byte-identical."""
    spec, store = _net(golden_nets, i)
    plan, report = P.compile_network(spec, store)
    assert vplan.dump_plan(plan) == bytes(golden_nets["net%d_plan" % i])
    assert "\n".join(report.lines()) == bytes(golden_nets["net%d_report" % i]).decode()


@pytest.mark.parametrize("i", [0, 1, 2])
def test_plan_oracle_matches_reference_engine(golden_nets, i):
    spec, store = _net(golden_nets, i)
    plan = vplan.parse_plan(bytes(golden_nets["net%d_plan" % i]))
    (name, got), = R.run_plan(plan, golden_nets["net%d_x" % i]).items()
    np.testing.assert_allclose(got, golden_nets["net%d_engine" % i], atol=2e-5, rtol=1e-5)
    np.testing.assert_allclose(got, golden_nets["net%d_ref" % i], atol=5e-5, rtol=1e-4)


def test_fixpoint_fuses_add_after_bn():
    """one pass round leaves config 3's add + ELU standalone;
    the fixpoint loop fuses them into conv2 and preserves semantics."""
    spec, store = C.config3(spatial=(4, 8, 8), c=16)
    once, _ = P.compile_network(spec, store)
    fix, rep = P.compile_network(spec, store, fixpoint=True)
    kinds_once = [s.kind for s in once.steps]
    kinds_fix = [s.kind for s in fix.steps]
    assert LayerKind.ELTWISE in kinds_once and LayerKind.ELU in kinds_once
    assert LayerKind.ELTWISE not in kinds_fix and LayerKind.ELU not in kinds_fix
    last = [s for s in fix.steps if s.kind is LayerKind.CONVOLUTION][-1]
    assert last.additive and last.fused_act == ("elu", 1.0) and last.base_scale is None
    x = C.make_input(spec, 0)
    ref = R.ref_run(spec, store, x)["out_elu"]
    for p in (once, fix):
        np.testing.assert_allclose(R.run_plan(p, x)["out_elu"], ref, atol=2e-5, rtol=1e-4)


def test_deconv_add_extension_preserves_semantics():
    spec, store = C.config5(patch=(2, 16, 16), feats=(4, 6, 8))
    plan, rep = P.compile_network(spec, store, fixpoint=True, fuse_deconv_add=True)
    assert rep.stat("fuse_deconv_addition").applied == 2
    assert not any(s.kind is LayerKind.ELTWISE for s in plan.steps)
    x = C.make_input(spec, 0, 0, 1)
    ref = R.ref_run(spec, store, x)["prob"]
    np.testing.assert_allclose(R.run_plan(plan, x)["prob"], ref, atol=1e-5, rtol=1e-4)


def test_plan_file_round_trip(tmp_path):
    spec, store = C.config3(spatial=(4, 8, 8), c=8)
    plan, _ = P.compile_network(spec, store, fixpoint=True)
    path = tmp_path / "p.pznp"
    vplan.write_plan(path, plan)
    back = vplan.read_plan(path)
    assert vplan.dump_plan(back) == vplan.dump_plan(plan)
    with pytest.raises(FormatError):
        vplan.parse_plan(b"XXXX" + vplan.dump_plan(plan)[4:])


def test_volume_round_trip(tmp_path, rng):
    x = rng.standard_normal((1, 2, 3, 4, 5)).astype(np.float32)
    formats.write_volume(tmp_path / "v.pznv", x)
    np.testing.assert_array_equal(formats.read_volume(tmp_path / "v.pznv"), x)
    with open(tmp_path / "v.pznv", "ab") as fh:
        fh.write(b"\0")
    with pytest.raises(FormatError):
        formats.read_volume(tmp_path / "v.pznv")


def test_streamed_volume_files_match_read_write(tmp_path, rng):
    """open_volume / create_volume (memory-mapped PZNV, the streamed run_tiled
    path) read and write exactly the bytes of read_volume / write_volume."""
    x = rng.standard_normal((2, 3, 5, 4, 6)).astype(np.float32)
    formats.write_volume(tmp_path / "a.pznv", x)
    m = formats.open_volume(tmp_path / "a.pznv")
    assert m.shape == x.shape
    np.testing.assert_array_equal(np.asarray(m), x)
    out = formats.create_volume(tmp_path / "b.pznv", x.shape)
    out[:, :, 2:] = x[:, :, 2:]          # written in two row blocks, like run_host
    out[:, :, :2] = x[:, :, :2]
    out.flush()
    del out
    assert (tmp_path / "a.pznv").read_bytes() == (tmp_path / "b.pznv").read_bytes()
    with open(tmp_path / "a.pznv", "ab") as fh:
        fh.write(b"\0")
    with pytest.raises(FormatError):
        formats.open_volume(tmp_path / "a.pznv")
    (tmp_path / "c.pznv").write_bytes((tmp_path / "b.pznv").read_bytes()[:-4])
    with pytest.raises(FormatError):
        formats.open_volume(tmp_path / "c.pznv")
    with pytest.raises(FormatError):
        formats.create_volume(tmp_path / "d.pznv", (1, 2, 3))


def test_empty_weight_store_is_12_bytes():
    # test_formats.py:63-68 (the code and tests win over SPEC's 13)
    assert len(formats.dump_weights(formats.WeightStore())) == 12


def test_parse_errors_and_validation():
    with pytest.raises(ParseError):
        prototxt.parse_network('layer { name: "a" type: "Input" input_param { shape { dim: 1 } }')
    with pytest.raises(UnknownLayerError):
        prototxt.parse_network('layer { name: "a" type: "Bogus" top: "a" }')
    with pytest.raises(DanglingReferenceError):
        prototxt.parse_network('layer { name: "r" type: "ReLU" bottom: "x" top: "r" }')
    txt = ('layer { name: "a" type: "ReLU" bottom: "b" top: "a" }\n'
           'layer { name: "b" type: "ReLU" bottom: "a" top: "b" }\n')
    with pytest.raises(CycleError):
        prototxt.parse_network(txt)
    with pytest.raises(ModelError):
        prototxt.parse_network('layer { name: "a" type: "Input" top: "a" top: "b" '
                               'input_param { shape { dim: 1 dim: 1 dim: 1 dim: 1 dim: 1 } } }')


def test_prototxt_grammar_details():
    txt = '''
    name: "t"  # comment
    layer { name: "in" type: "Input" top: "d"
            input_param { shape { dim: 1 dim: 2 dim: 8 dim: 8 dim: 8 } } }
    layer { name: "c" type: "Convolution" bottom: "d" top: "c"
            convolution_param { num_output: 4 kernel_size: 1 kernel_size: 3 kernel_size: 3
                                pad: 0 pad: 1 pad: 1 unknown_field: 3 } }
    layer { name: "p" type: "Pooling" bottom: "c" top: "p"
            pooling_param { pool: AVE kernel_size: 2 } }
    layer { name: "e" type: "ELU" bottom: "p" top: "e" elu_param { alpha: 1 } }
    '''
    spec = prototxt.parse_network(txt)
    c = spec.layer("c")
    assert c.params == {"num_output": 4, "kernel": (1, 3, 3), "stride": (1, 1, 1),
                        "pad": (0, 1, 1)}
    assert spec.layer("p").params == {"mode": "avg", "window": (2, 2, 2), "stride": (2, 2, 2)}
    assert spec.layer("e").params == {"alpha": 1.0}
    assert prototxt.parse_network(prototxt.print_network(spec)) == spec


def test_shape_errors():
    spec, store = C.config1()
    store.put("conv.bias", np.zeros(3, np.float32))
    with pytest.raises(ShapeError):
        P.validate_shapes(spec, store)


def test_deconv_pad_rejected():
    txt = ('layer { name: "in" type: "Input" top: "d" input_param { shape { '
           'dim: 1 dim: 1 dim: 4 dim: 4 dim: 4 } } }\n'
           'layer { name: "u" type: "Deconvolution" bottom: "d" top: "u" '
           'convolution_param { num_output: 1 kernel_size: 2 stride: 2 pad: 1 } }')
    spec = prototxt.parse_network(txt)
    store = formats.WeightStore()
    store.put("u.kernel", np.ones((1, 1, 2, 2, 2), np.float32))
    store.put("u.bias", np.zeros(1, np.float32))
    with pytest.raises(PlanError):
        P.compile_network(spec, store)


@pytest.mark.parametrize("cfg", [1, 3, 4, 5])
def test_config_networks_compile(cfg):
    builders = {1: C.config1, 3: lambda: C.config3(spatial=(4, 8, 8)),
                4: lambda: C.config4(spatial=(44, 44, 44), base=4, levels=3),
                5: lambda: C.config5(patch=(2, 16, 16), feats=(4, 6, 8))}
    spec, store = builders[cfg]()
    plan, _ = P.compile_network(spec, store, fixpoint=True, fuse_deconv_add=True)
    assert plan.steps


def test_full_size_config_shapes():
    assert C.config4()[0].layers[-1].params["num_output"] == 3
    shapes = P.validate_shapes(*C.config4())
    assert shapes["output"] == (1, 3, 44, 44, 44)
    shapes = P.validate_shapes(*C.config5())
    assert shapes["prob"] == (1, 3, 18, 192, 192)
    assert abs(C.conv_flops(C.config5()[0]) / 663552 - 322e3) / 322e3 < 0.05


def test_rebatch_scales_every_batch_dim():
    """plan.rebatch (tiled executor: several patches per launch) sets dims[0]
    of every step input/output/base, plan input and output to the batch,
    scales the buffer table, and keeps everything else (weights, params,
    fused flags) identical; only batch-1 plans are accepted."""
    from paper_1903_07525_b200 import configs as C
    from paper_1903_07525_b200.errors import PlanError
    from paper_1903_07525_b200.plan import rebatch
    spec, store = C.config5(patch=(6, 48, 48), feats=(8, 12, 16, 20))
    plan, _ = P.compile_network(spec, store, fixpoint=True, fuse_deconv_add=True)
    b = rebatch(plan, 3)
    assert [d[2] for d in b.inputs] == [(3,) + tuple(d[2][1:]) for d in plan.inputs]
    assert [d[2] for d in b.outputs] == [(3,) + tuple(d[2][1:]) for d in plan.outputs]
    for s0, s1 in zip(plan.steps, b.steps):
        assert s1.output.dims == (3,) + tuple(s0.output.dims[1:])
        assert [x.dims for x in s1.inputs] == [(3,) + tuple(x.dims[1:]) for x in s0.inputs]
        assert (s1.base is None) == (s0.base is None)
        if s1.base is not None:
            assert s1.base.dims == (3,) + tuple(s0.base.dims[1:])
        assert (s1.kind, s1.name, s1.params, s1.fused_act, s1.additive, s1.base_scale) == \
            (s0.kind, s0.name, s0.params, s0.fused_act, s0.additive, s0.base_scale)
    assert b.arena_elements == 3 * plan.arena_elements
    assert b.weights is plan.weights
    with pytest.raises(PlanError):
        rebatch(b, 2)
