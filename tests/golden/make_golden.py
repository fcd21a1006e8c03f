"""Generate golden vectors from the reference implementation itself.

Run in the build container (where /root/reference exists):
    python tests/golden/make_golden.py
It imports the reference package (voxplan, pkg/src) read-only and writes small
fixtures next to this script.  The GPU box never runs this; tests only read
the committed outputs:

  ops.npz        seeded inputs + reference outputs of oracle.ref_conv3d /
                 ref_deconv3d / ref_pool3d / ref_mergecrop / ref_batch_norm /
                 ref_scale / ref_activation / ref_eltwise (oracle.py:37-174)
  nets.npz       three reference zoo networks (zoo.py) as prototxt text + PZNW
                 bytes, a seeded input, ref_run outputs (oracle.py:184-252),
                 the reference engine's output (executor.PlanRunner, python
                 backend), and the compiled plan (plan.dump_plan bytes) with
                 default passes — pins our front end, compiler and oracle
  tiles.json     plan_tiles geometry for a set of volumes (tiling.py:83-162)
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

REF_SRC = os.environ.get("REF_SRC", "/root/reference/pkg/src")
HERE = os.path.dirname(os.path.abspath(__file__))


def main():
    sys.path.insert(0, REF_SRC)
    import voxplan
    from voxplan import oracle, zoo, plan as vplan, tiling, prototxt, formats

    rng = np.random.default_rng(20261020)
    ops = {}

    def f32(*shape, scale=1.0):
        return (rng.standard_normal(shape) * scale).astype(np.float32)

    conv_cases = [
        # cin, cout, spatial, k, stride, pad
        (5, 7, (8, 8, 8), (3, 3, 3), (1, 1, 1), (0, 0, 0)),
        (8, 8, (7, 8, 9), (3, 3, 3), (2, 2, 2), (1, 1, 1)),
        (8, 8, (7, 8, 9), (3, 3, 3), (1, 2, 3), (0, 1, 1)),
        (16, 16, (6, 10, 12), (3, 3, 3), (1, 1, 1), (1, 1, 1)),
        (12, 20, (5, 9, 11), (1, 3, 3), (1, 1, 1), (0, 1, 1)),
        (1, 16, (9, 9, 9), (3, 3, 3), (1, 1, 1), (0, 0, 0)),
        (24, 3, (4, 6, 8), (1, 1, 1), (1, 1, 1), (0, 0, 0)),
    ]
    for i, (ci, co, sp, k, s, p) in enumerate(conv_cases):
        x = f32(1, ci, *sp)
        w = f32(co, ci, *k, scale=0.2)
        b = f32(co)
        ops["conv%d_x" % i], ops["conv%d_w" % i], ops["conv%d_b" % i] = x, w, b
        ops["conv%d_meta" % i] = np.array(list(s) + list(p), np.int32)
        ops["conv%d_y" % i] = oracle.ref_conv3d(x, w, b, s, p)
    deconv_cases = [(6, 3, (4, 4, 4), (2, 2, 2), (2, 2, 2)),
                    (16, 8, (3, 5, 5), (1, 2, 2), (1, 2, 2)),
                    (4, 4, (3, 3, 3), (3, 3, 3), (2, 2, 2))]
    for i, (ci, co, sp, k, s) in enumerate(deconv_cases):
        x = f32(1, ci, *sp)
        w = f32(co, ci, *k, scale=0.3)
        b = f32(co)
        ops["deconv%d_x" % i], ops["deconv%d_w" % i], ops["deconv%d_b" % i] = x, w, b
        ops["deconv%d_s" % i] = np.array(s, np.int32)
        ops["deconv%d_y" % i] = oracle.ref_deconv3d(x, w, b, s)
    x = f32(2, 5, 6, 7, 8)
    ops["pool_x"] = x
    ops["pool_max"] = oracle.ref_pool3d(x, (2, 2, 2), (2, 2, 2), "max")
    ops["pool_avg"] = oracle.ref_pool3d(x, (2, 2, 2), (2, 2, 2), "avg")
    ops["pool_aniso"] = oracle.ref_pool3d(x, (1, 2, 2), (1, 2, 2), "max")
    a, b2 = f32(1, 6, 9, 7, 9), f32(1, 3, 7, 7, 7)
    ops["mc_a"], ops["mc_b"], ops["mc_y"] = a, b2, oracle.ref_mergecrop(a, b2)
    x = f32(1, 5, 4, 4, 4)
    mean, var = f32(5, scale=0.1), rng.uniform(0.5, 1.5, 5).astype(np.float32)
    gamma, beta = rng.uniform(0.5, 1.5, 5).astype(np.float32), f32(5, scale=0.1)
    ops.update(bn_x=x, bn_mean=mean, bn_var=var, bn_gamma=gamma, bn_beta=beta,
               bn_y=oracle.ref_batch_norm(x, mean, var, 1e-5),
               sc_y=oracle.ref_scale(x, gamma, beta),
               relu_y=oracle.ref_activation(x, "relu"),
               elu_y=oracle.ref_activation(x, "elu", 0.7),
               sig_y=oracle.ref_activation(x, "sigmoid"))
    e1, e2 = f32(1, 5, 3, 3, 3), f32(1, 5, 3, 3, 3)
    ops.update(elt_a=e1, elt_b=e2, elt_add=oracle.ref_eltwise(e1, e2, "add"),
               elt_mul=oracle.ref_eltwise(e1, e2, "mul"),
               elt_div=oracle.ref_eltwise(e1, e2, "div"))
    np.savez_compressed(os.path.join(HERE, "ops.npz"), **ops)

    nets = {}
    cfgs = [zoo.ZooConfig("original", levels=2, base_features=8, input_spatial=(20, 20, 20),
                          seed=3),
            zoo.ZooConfig("symmetric", levels=2, base_features=8, input_spatial=(8, 8, 8), seed=4),
            zoo.ZooConfig("residual", levels=3, base_features=8, input_spatial=(8, 8, 8), seed=5)]
    for i, cfg in enumerate(cfgs):
        spec, store = zoo.generate_zoo(cfg)
        # random (non-identity) BN so folding is exercised
        for name in list(store):
            if name.endswith(".bn_var") or name.endswith(".scale_gamma"):
                store.put(name, rng.uniform(0.5, 1.5, store.get(name).shape))
            elif name.endswith(".bn_mean") or name.endswith(".scale_beta") or name.endswith(".bias"):
                store.put(name, rng.standard_normal(store.get(name).shape) * 0.1)
        x = rng.uniform(0, 1, spec.input_layers()[0].params["shape"]).astype(np.float32)
        ref = oracle.ref_run(spec, store, x)
        plan, report = vplan.compile_network(spec, store)
        eng = voxplan.PlanRunner(plan, backend="python").run(x)
        (oname, yref), = ref.items()
        nets["net%d_prototxt" % i] = np.frombuffer(prototxt.print_network(spec).encode(), np.uint8)
        nets["net%d_pznw" % i] = np.frombuffer(formats.dump_weights(store), np.uint8)
        nets["net%d_x" % i] = x
        nets["net%d_ref" % i] = yref
        nets["net%d_engine" % i] = eng[oname]
        nets["net%d_plan" % i] = np.frombuffer(vplan.dump_plan(plan), np.uint8)
        nets["net%d_report" % i] = np.frombuffer("\n".join(report.lines()).encode(), np.uint8)
    np.savez_compressed(os.path.join(HERE, "nets.npz"), **nets)

    tiles = []
    for vol, pin, pout, ov in [((40, 40, 40), (16, 16, 16), (16, 16, 16), None),
                               ((37, 50, 29), (12, 20, 9), (8, 16, 5), None),
                               ((128, 1024, 1024), (18, 192, 192), (18, 192, 192), 0),
                               ((30, 30, 30), (12, 12, 12), (8, 8, 8), 6)]:
        g = tiling.plan_tiles(vol, pin, pout, ov)
        tiles.append({"volume": vol, "patch_in": pin, "patch_out": pout, "overlap": ov,
                      "counts": g.counts, "volume_out": g.volume_out,
                      "tiles": [[t.index, t.in_lo, t.keep_lo, t.keep_hi, t.out_lo]
                                for t in g.tiles]})
    with open(os.path.join(HERE, "tiles.json"), "w") as fh:
        json.dump(tiles, fh)
    print("wrote", sorted(os.listdir(HERE)))


if __name__ == "__main__":
    main()
