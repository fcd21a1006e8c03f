"""Full-BASELINE-size parity of the B200 backends against the reference oracle
— TEST INFRASTRUCTURE (imported by tests/test_gpu_parity_full.py; also run
standalone on a GPU box to write the per-config table):

    python tests/parity_report.py [out.json]

For every BASELINE config at its full size the network runs
through the reference API (PlanRunner.run on host arrays) with backends
``b200`` (bf16 storage), ``b200-x3`` (split-bf16 storage, fp32-grade) and,
for the single-layer configs, ``b200-fp32``; the output is compared with
``ref_run`` (oracle.py:184-252 restated in oracle/ref_numpy.py) on the same
seeded input: max|gpu - ref| / max|ref| and ||gpu - ref||_2 / ||ref||_2 (the
per-config measures SURVEY §8c asks for).  ``bf16`` is also compared with the
plan-level emulation of its own roundings (run_plan(storage="bf16")), which
isolates kernel errors from the storage precision.
"""

from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

from oracle import ref_numpy as R  # noqa: E402

BACKENDS = ("b200", "b200-x3")


def networks():
    """(name, spec, store, input) at full BASELINE sizes (config 2: every layer)."""
    from paper_1903_07525_b200 import configs as C
    out = [("cfg1",) + C.config1()]
    for k in C.SWEEP_K:
        for c in C.SWEEP_C:
            out.append(("cfg2_c%d_k%s" % (c, "".join(map(str, k))),) + C.config2(c, k))
    out.append(("cfg3",) + C.config3())
    out.append(("cfg4",) + C.config4())
    out.append(("cfg5",) + C.config5())
    out.append(("cfg5_randombn",) + C.config5(bn="random"))
    res = []
    for name, spec, store in out:
        cfg = int(name[3])
        lo, hi = C.input_range(cfg)
        res.append((name, spec, store, C.make_input(spec, 1000 + cfg, lo, hi)))
    return res


_REF_CACHE: dict = {}


def reference(name, spec, store, x):
    if name not in _REF_CACHE:
        ref = R.ref_run(spec, store, x)
        (_, out), = ref.items()
        _REF_CACHE[name] = out
    return _REF_CACHE[name]


def measure(name, spec, store, x, backend):
    import paper_1903_07525_b200 as P
    plan, _ = P.compile_network(spec, store, fixpoint=True, fuse_deconv_add=True)
    runner = P.PlanRunner(plan, backend=backend)
    (_, got), = runner.run(x).items()
    ref = reference(name, spec, store, x)
    mx, l2 = R.normalized_error(got, ref)
    row = {"max_norm": mx, "l2": l2, "max_abs_ref": float(np.abs(ref).max())}
    if backend == "b200":
        (_, emu), = R.run_plan(plan, x, storage="bf16").items()
        row["vs_bf16_emulation"] = dict(zip(("max_norm", "l2"), R.normalized_error(got, emu)))
    del runner
    return row


def report(names=None) -> dict:
    out = {}
    for name, spec, store, x in networks():
        if names and name not in names:
            continue
        out[name] = {}
        for be in BACKENDS:
            t = time.time()
            out[name][be] = measure(name, spec, store, x, be)
            out[name][be]["s"] = round(time.time() - t, 1)
            print(name, be, json.dumps(out[name][be]), flush=True)
    return out


if __name__ == "__main__":
    rep = report()
    path = sys.argv[1] if len(sys.argv) > 1 else None
    if path:
        with open(path, "w") as fh:
            json.dump(rep, fh, indent=1)
