"""Print the conv3d_tc launch index (order within one forward) of a config's
dominant conv, for ncu -k regex:conv3d_tc -s <index> -c 1."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1903_07525_b200 as P  # noqa: E402
from paper_1903_07525_b200 import configs as C, _lib  # noqa: E402
from paper_1903_07525_b200.netspec import LayerKind  # noqa: E402
from bench_util import _dominant  # noqa: E402

cfg = int(sys.argv[1])
spec, store = {1: C.config1, 3: C.config3, 4: C.config4, 5: C.config5}[cfg]()
plan, _ = P.compile_network(spec, store, fixpoint=True, fuse_deconv_add=True)
dom = _dominant(plan)[0]
r = P.PlanRunner(plan)
i = 0
for kind, st, info in r._ops:
    if kind in (LayerKind.CONVOLUTION, LayerKind.DECONVOLUTION):
        if st.name == dom:
            print(i, dom)
            break
        i += 1
