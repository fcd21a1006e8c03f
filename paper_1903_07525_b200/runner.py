"""B200 plan execution (reference: executor.py:51-203).

``PlanRunner(plan).run(inputs)`` keeps the reference's contract: inputs are a
dict name -> standard (batch, fmap, x, y, z) array (or a bare array for a
single-input plan), the result is a dict name -> standard float32 array, and
bad inputs raise ``ExecutionError`` with the reference's messages.

Binding (once):
  * every step is lowered to one device op over ``DTensor`` views in HBM
    (bf16, channel-blocked, S = 8): convolutions get their weights packed
    for the tensor-core or CUDA-core path, BN/Scale coefficients are computed
    in float64 exactly like executor._bn_coefficients (executor.py:44-49);
  * Pad steps and zero-halo buffers (ir.eliminate_padding) become *virtual*
    padding of the consuming convolution (TMA zero fill), so no pad copies
    and no halo storage exist on the device;
  * storage is assigned by liveness from a pool (like the reference arena,
    plan.py:92-127) and allocated once;
  * the whole forward pass (input pack, all steps, output unpack) is captured
    into one CUDA graph.
Running: H2D of the inputs into pinned/static buffers, one graph replay,
D2H of the outputs.  ``run_device`` skips the host copies.
"""

from __future__ import annotations

import os

import numpy as np

from . import _lib
from . import ops as K
from .device import DTensor, LANES, chunks, standard
from .errors import ExecutionError, PlanError
from .formats import (ROLE_BIAS, ROLE_BN_MEAN, ROLE_BN_VAR, ROLE_KERNEL, ROLE_SCALE_BETA,
                      ROLE_SCALE_GAMMA)
from .netspec import DEFAULT_ELU_ALPHA, LayerKind


def _torch():
    import torch
    return torch


def bn_coefficients(mean, var, eps):
    """executor._bn_coefficients (executor.py:44-49): fp64 then fp32."""
    f = 1.0 / np.sqrt(np.asarray(var, np.float64) + eps)
    return f.astype(np.float32), (-np.asarray(mean, np.float64) * f).astype(np.float32)


class _Value:
    """A logical tensor produced by one step (interior dims, no halo)."""

    __slots__ = ("dims", "slot", "readers", "dt", "dtype")

    def __init__(self, dims, dtype="bf16"):
        self.dims = tuple(int(d) for d in dims)
        self.slot = None
        self.readers = 0
        self.dt = None
        self.dtype = dtype

    @property
    def nbytes(self):
        n, c, x, y, z = self.dims
        esz = 2 if self.dtype == "bf16" else 4     # fp32, or split bf16 (hi + lo)
        return n * chunks(c) * x * y * z * LANES * esz


class PlanRunner:
    """Executes one ExecutionPlan on one B200; reusable, deterministic."""

    def __init__(self, plan, backend=None, *, device=None, use_graph=True, fuse_concat=True,
                 fuse_pool=True, fuse_input=False, fuse_head=True, pdl=None, probe=None):
        torch = _torch()
        from .backend import resolve_device_backend
        self.backend = resolve_device_backend(backend)
        if not torch.cuda.is_available():
            raise ExecutionError("the B200 backend needs a CUDA device; none is visible")
        self.plan = plan
        self.device = torch.device(device) if device is not None else torch.device(
            "cuda", torch.cuda.current_device())
        self.use_graph = use_graph
        # programmatic dependent launch for this runner's kernels (None: the
        # VXB_PDL default, on).  Off measured faster for the 12-patch config-5
        # batches (4.65 -> 4.48 ms per batch), on for the single networks of
        # configs 1-4 (config 4 0.82 vs 0.86 ms).
        self.pdl = pdl
        self.precision = self.backend.precision
        # activation storage: bf16, fp32 (CUDA-core path) or split bf16 (x3)
        self.storage = {"x3": "split"}.get(self.precision, self.precision)
        # weight packing precision of the tensor-core paths
        self._prec = "x3" if self.precision == "x3" else "bf16"
        self.fuse_concat = fuse_concat and self.precision == "bf16"
        if os.environ.get("VXB_FUSE_POOL") is not None:     # experiments
            fuse_pool = os.environ["VXB_FUSE_POOL"] == "1"
        self.fuse_pool = fuse_pool and self.precision == "bf16"
        if os.environ.get("VXB_FUSE_INPUT") is not None:    # experiments
            fuse_input = os.environ["VXB_FUSE_INPUT"] == "1"
        self.fuse_input = fuse_input
        self.fuse_head = fuse_head and self.precision in ("bf16", "x3") and \
            os.environ.get("VXB_FUSE_HEAD", "1") == "1"
        self._conv_path = _lib.PATH_DIRECT if self.precision == "fp32" else 0
        self.stream = torch.cuda.Stream(device=self.device)
        # independent input packs (set by PlanBatch while it captures).  A
        # one-element list, not an attribute read through `self`: the call
        # closures must not reference the runner, or runner <-> closure
        # cycles leave dead runners to the cyclic GC, which may then destroy
        # their CUDA graphs in the middle of another runner's stream capture
        # (cudaGraphExecDestroy is illegal during capture and invalidates it).
        self._indep_flag = [False]
        # live timing of one step (bench roofline): external timing events
        # recorded around that step's launch, inside the captured graph
        self.probe = probe
        self._probe_ev = None
        if probe is not None:
            self._probe_ev = (torch.cuda.Event(enable_timing=True, external=True),
                              torch.cuda.Event(enable_timing=True, external=True))
        with torch.cuda.device(self.device):
            self._lower()
            self._allocate()
            self._bind()
        self._graph = None
        self.launches = len(self._calls)

    # ------------------------------------------------------------ lowering
    def _lower(self):
        plan = self.plan
        self._input_dims = {name: tuple(dims) for name, _, dims in plan.inputs}
        cur: dict = {}       # buffer id -> value currently held
        self._values = []
        self._ops = []       # (kind, step, info dict)

        def new_value(dims):
            v = _Value(dims, self.storage)
            self._values.append(v)
            return v

        self._in_values = {}
        for name, bid, dims in plan.inputs:
            v = new_value(dims)
            cur[bid] = v
            self._in_values[name] = v

        def read(si, allow_halo=False):
            v = cur.get(si.buffer)
            if v is None:
                raise PlanError("step reads buffer %d before it is written" % si.buffer)
            halo = tuple((a - b) // 2 for a, b in zip(si.dims[2:], v.dims[2:]))
            if min(halo) < 0 or tuple(si.dims[:2]) != v.dims[:2]:
                raise PlanError("buffer %d read with dims %s, holds %s"
                                % (si.buffer, si.dims, v.dims))
            if any(halo) and not allow_halo:
                raise PlanError("a %s step cannot read a zero-halo view" % "non-conv")
            v.readers += 1
            return v, halo

        for st in plan.steps:
            kind = st.kind
            if kind is LayerKind.PAD:
                v, halo = read(st.inputs[0], allow_halo=True)
                v.readers -= 1  # an alias is not a read; its readers are counted later
                cur[st.output.buffer] = v
                continue
            info = {}
            if kind is LayerKind.CONVOLUTION:
                v, halo = read(st.inputs[0], allow_halo=True)
                info["x"], info["pad"] = v, halo
            elif kind is LayerKind.MERGE_CROP:
                info["a"], _ = read(st.inputs[0])
                info["b"], _ = read(st.inputs[1])
            else:
                info["ins"] = [read(si)[0] for si in st.inputs]
            if st.additive:
                info["base"], _ = read(st.base)
            out = new_value(st.output.dims)
            info["out"] = out
            cur[st.output.buffer] = out
            self._ops.append((kind, st, info))
        self._out_values = {}
        for name, bid, dims in plan.outputs:
            v = cur[bid]
            if v.dims != tuple(dims):
                raise PlanError("output %r dims %s, buffer holds %s" % (name, dims, v.dims))
            v.readers += 1
            self._out_values[name] = v
        if self.fuse_concat:
            self._fuse_mergecrop()
        if self.fuse_pool:
            self._fuse_maxpool()
        if self.fuse_head:
            self._fuse_head()

    def _fuse_mergecrop(self):
        """Zero-copy MergeCrop: a conv whose only input is a MergeCrop of two
        chunk-aligned tensors reads both directly as two K segments (fused
        concat).  The MergeCrop output is never stored."""
        producers = {id(info["out"]): i for i, (_, _, info) in enumerate(self._ops)}
        drop = set()
        for kind, st, info in self._ops:
            if kind is not LayerKind.CONVOLUTION:
                continue
            src = producers.get(id(info["x"]))
            if src is None:
                continue
            mkind, mst, minfo = self._ops[src]
            if mkind is not LayerKind.MERGE_CROP or minfo["out"].readers != 1:
                continue
            if any(info["pad"]) or minfo["a"].dims[1] % LANES:
                continue
            stride = tuple(st.params.get("stride", (1, 1, 1)))
            if stride != (1, 1, 1):
                continue
            a, b, m = minfo["a"], minfo["b"], minfo["out"]
            info["segments"] = (a, b,
                                tuple((sa - sm) // 2 for sa, sm in zip(a.dims[2:], m.dims[2:])),
                                tuple((sb - sm) // 2 for sb, sm in zip(b.dims[2:], m.dims[2:])))
            m.readers = 0
            info["x"] = None
            drop.add(src)
        if drop:
            self._ops = [op for i, op in enumerate(self._ops) if i not in drop]

    def _fuse_head(self):
        """The network's 1x1x1 output conv (<= 4 fmaps, e.g. the U-nets'
        3-fmap head + sigmoid) computed in the epilogue of the conv that
        produces its only input (vxb_conv_desc.head_*): that conv's activated
        output is never stored, the head writes the fp32 network output
        (SURVEY §8f rank 3).  The reference runs the head as its own conv
        step over the stored tensor (executor.py:134-164)."""
        producers = {id(info["out"]): i for i, (_, _, info) in enumerate(self._ops)}
        out_names = {id(v): n for n, v in self._out_values.items()}
        drop = set()
        for i, (kind, st, info) in enumerate(self._ops):
            if kind is not LayerKind.CONVOLUTION or st.additive or "segments" in info:
                continue
            k = self.plan.weights.tensor(st.name, ROLE_KERNEL).shape
            if tuple(k[2:]) != (1, 1, 1) or k[0] > 4 or any(info["pad"]):
                continue
            if tuple(st.params.get("stride", (1, 1, 1))) != (1, 1, 1):
                continue
            hout = info["out"]
            if out_names.get(id(hout)) is None or hout.readers != 1:
                continue
            v = info["x"]
            j = producers.get(id(v))
            if j is None or v.readers != 1:
                continue
            pkind, pst, pinfo = self._ops[j]
            if pkind is not LayerKind.CONVOLUTION or "pool_out" in pinfo or "head" in pinfo:
                continue
            if tuple(pst.params.get("stride", (1, 1, 1))) != (1, 1, 1):
                continue
            pk = self.plan.weights.tensor(pst.name, ROLE_KERNEL).shape
            L = _lib.lib()
            if L.vxb_conv_select(pk[1], pk[0], _lib.i3(pk[2:]), _lib.i3((1, 1, 1))) != \
                    _lib.PATH_TC:
                continue
            pinfo["head"] = (st, hout)
            v.readers = 0
            drop.add(i)
        if drop:
            self._ops = [op for i, op in enumerate(self._ops) if i not in drop]

    def _fuse_maxpool(self):
        """MaxPool 1x2x2 / 1x2x2 (ops.py:63-86) folded into the epilogue of the
        tensor-core conv that produces its input: the conv
        writes its output and the pooled output; the pool step disappears.
        Only x-sliced conv tiles (3-deep x kernels, 1x1x1) pool over their
        (y, z) rows.  On by default since the lean epilogue carries it (round
        1's generic pooled epilogue cost as much as the HBM-bound pool kernel
        it replaced); bit-identical to the pool kernel either way."""
        producers = {id(info["out"]): i for i, (_, _, info) in enumerate(self._ops)}
        drop = set()
        for i, (kind, st, info) in enumerate(self._ops):
            if kind is not LayerKind.POOLING:
                continue
            prm = st.params
            if (prm.get("mode") != "max" or tuple(prm["window"]) != (1, 2, 2)
                    or tuple(prm["stride"]) != (1, 2, 2)):
                continue
            src = info["ins"][0]
            j = producers.get(id(src))
            if j is None:
                continue
            ckind, cst, cinfo = self._ops[j]
            if ckind is not LayerKind.CONVOLUTION or "pool_out" in cinfo:
                continue
            if tuple(cst.params.get("stride", (1, 1, 1))) != (1, 1, 1):
                continue
            k = tuple(int(v) for v in self.plan.weights.tensor(cst.name, ROLE_KERNEL).shape[2:])
            if not (k[0] == 3 or k == (1, 1, 1)):
                continue
            cinfo["pool_out"] = info["out"]
            src.readers -= 1
            drop.add(i)
        if drop:
            self._ops = [op for i, op in enumerate(self._ops) if i not in drop]

    # ------------------------------------------------------------ storage
    def _reads(self, info):
        if "segments" in info:
            rs = [info["segments"][0], info["segments"][1]]
        elif "x" in info:
            rs = [info["x"]]
        else:
            rs = []
        rs += [info[k] for k in ("a", "b", "base") if k in info]
        return rs + list(info.get("ins", []))

    def _allocate(self):
        """Liveness-based slot assignment (best fit by bytes, like the
        reference arena plan.py:92-127), then one allocation per slot."""
        torch = _torch()
        last = {}
        for v in self._in_values.values():
            last[id(v)] = -1
        for i, (_, _, info) in enumerate(self._ops):
            for r in self._reads(info):
                last[id(r)] = i
            last.setdefault(id(info["out"]), i)
            if "pool_out" in info:
                last.setdefault(id(info["pool_out"]), i)
            if "head" in info:
                last.setdefault(id(info["head"][1]), i)
        for v in self._out_values.values():
            last[id(v)] = len(self._ops)
        slots, free = [], []

        def grab(v):
            need = v.nbytes
            fits = [q for q in free if slots[q] >= need]
            if fits:
                q = min(fits, key=lambda k: (slots[k], k))
            elif free:
                q = max(free, key=lambda k: slots[k])
                slots[q] = need
            else:
                slots.append(need)
                return len(slots) - 1
            free.remove(q)
            return q

        for v in self._in_values.values():
            v.slot = grab(v)
        live = list(self._in_values.values())
        for i, (_, _, info) in enumerate(self._ops):
            info["out"].slot = grab(info["out"])
            live.append(info["out"])
            if "pool_out" in info:
                info["pool_out"].slot = grab(info["pool_out"])
                live.append(info["pool_out"])
            if "head" in info:
                info["head"][1].slot = grab(info["head"][1])
                live.append(info["head"][1])
            keep = []
            for v in live:
                if last.get(id(v), -1) <= i:
                    free.append(v.slot)
                else:
                    keep.append(v)
            live = keep
        self._storage = [torch.empty(max(b, 16), dtype=torch.uint8, device=self.device)
                         for b in slots]
        self.device_bytes = sum(slots)
        for v in self._values:
            if v.slot is None:
                continue
            n, c, x, y, z = v.dims
            td = torch.float32 if v.dtype == "fp32" else torch.bfloat16
            planes = 2 if v.dtype == "split" else 1     # split: hi, lo plane per chunk
            numel = n * planes * chunks(c) * x * y * z * LANES
            t = self._storage[v.slot].view(td)[:numel].view(n, planes * chunks(c), x, y, z, LANES)
            v.dt = DTensor(t, c, True, v.dtype == "split")
        # network boundary: fp32 standard staging tensors (device + pinned host)
        self._in_std = {name: torch.empty(self._input_dims[name], dtype=torch.float32,
                                          device=self.device)
                        for name in self._in_values}
        self._out_std = {name: torch.empty(v.dims, dtype=torch.float32, device=self.device)
                         for name, v in self._out_values.items()}
        self._in_pinned = {name: torch.empty(t.shape, dtype=torch.float32, pin_memory=True)
                           for name, t in self._in_std.items()}
        self._out_pinned = {name: torch.empty(t.shape, dtype=torch.float32, pin_memory=True)
                            for name, t in self._out_std.items()}

    # ------------------------------------------------------------ binding
    def _bind(self):
        w = self.plan.weights
        dev = self.device
        calls = []
        # fused input pack (opt-in, fuse_input=True): a network input read only
        # by one tensor-core conv goes to that conv as the fp32 NCDHW tensor
        # itself (converted to bf16 chunks inside the conv, no pack kernel).
        # Off by default: its fp32 TMA boxes have 48-byte rows and the staging
        # + conversion pipeline is slower than the HBM-bound pack kernel
        #
        readers = {}
        for kind, st, info in self._ops:
            if kind is LayerKind.CONVOLUTION and info.get("x") is not None:
                readers.setdefault(id(info["x"]), []).append((st, info))
        fused_in = {}
        self._zwin = {}       # id(conv info) -> (z-window input tensor, kz, pz)
        self.zwin_input = None
        for name, v in self._in_values.items():
            rs = readers.get(id(v), [])
            if v.readers == 1 and len(rs) == 1 and self._f32in_ok(name, *rs[0]):
                fused_in[id(rs[0][1])] = standard(self._in_std[name])
                continue
            src = standard(self._in_std[name])
            zw = self._zwin_plan(v, rs)
            if zw is not None:
                # single-channel input: z taps packed into the chunk lanes
                xz, kz, pz = zw
                self._zwin[id(rs[0][1])] = zw
                self.zwin_input = (name, xz, kz, pz)     # DeviceTiler fuses its gather here
                calls.append(lambda s=src, d=xz, kz=kz, pz=pz, f=self._indep_flag:
                             _pack_zwin(s, d, kz, pz, independent=f[0]))
                continue
            # The pack reads a network input and writes a buffer only this
            # network's later steps read.  Inside a PlanBatch graph the kernel
            # before it is another network's, so it is launched independent
            # (no grid-dependency wait, may run beside that kernel); alone it
            # keeps the ordinary wait, since the input may have just been
            # written by a kernel (a strided torch copy) it must not overtake.
            if os.environ.get("VXB_DEBUG_SKIP_INPUT_PACK") == "1":
                continue        # timing experiments only: inputs never reach the network
            calls.append(lambda s=src, d=v.dt, f=self._indep_flag:
                         _copy(s, d, independent=f[0]))
        n_in = len(calls)
        self._n_in_calls = n_in          # the input packs come first (PlanBatch side stream)
        self.fused_inputs = len(fused_in)
        # fused unpack: a conv/deconv whose result is only a network output
        # writes the fp32 NCDHW output tensor directly from its epilogue
        fused_out = {}
        for name, v in self._out_values.items():
            if v.readers == 1:
                fused_out[id(v)] = name
        self._fused_outputs = set()
        for kind, st, info in self._ops:
            out = info["out"].dt
            oname = fused_out.get(id(info["out"]))
            if oname is not None and kind in (LayerKind.CONVOLUTION, LayerKind.DECONVOLUTION):
                out = standard(self._out_std[oname])
                self._fused_outputs.add(oname)
            if kind is LayerKind.CONVOLUTION:
                base = info["base"].dt if "base" in info else None
                scale = st.base_scale if st.additive else None
                kern = w.tensor(st.name, ROLE_KERNEL)
                stride = tuple(st.params.get("stride", (1, 1, 1)))
                hd = hout = None
                if "head" in info:       # fused 1x1x1 output conv (_fuse_head)
                    hst, hval = info["head"]
                    hname = fused_out[id(hval)]
                    hk = np.asarray(w.tensor(hst.name, ROLE_KERNEL), np.float32)
                    hd = K.make_head(hk.reshape(hk.shape[0], hk.shape[1]),
                                     w.tensor(hst.name, ROLE_BIAS), hst.fused_act, device=dev)
                    hout = standard(self._out_std[hname])
                    self._fused_outputs.add(hname)
                if "segments" in info:
                    a, b, oa, ob = info["segments"]
                    pk = K.pack_conv(kern, w.tensor(st.name, ROLE_BIAS), stride=stride,
                                     base_scale=scale, cin_split=a.dims[1],
                                     out_shape=tuple(info["out"].dims[2:]), batch=int(info["out"].dims[0]), device=dev)
                    pool = info["pool_out"].dt if "pool_out" in info else None
                    calls.append(lambda a=a.dt, b=b.dt, pk=pk, out=out, base=base, oa=oa, ob=ob,
                                 act=st.fused_act, pool=pool, hd=hd, hout=hout:
                                 K.conv3d(a, pk, out, base=base, fused_act=act, x2=b, off=oa,
                                          off2=ob, pool_out=pool, head=hd, head_out=hout))
                elif id(info) in self._zwin:
                    xz, kz, pz = self._zwin[id(info)]
                    # w'(co, l, dx, dy, 0) = w(co, 0, dx, dy, l)
                    kz_w = np.ascontiguousarray(
                        np.transpose(np.asarray(kern, np.float32)[:, 0], (0, 3, 1, 2))[..., None])
                    pk = K.pack_conv(kz_w, w.tensor(st.name, ROLE_BIAS), stride=stride,
                                     base_scale=scale, out_shape=tuple(info["out"].dims[2:]), batch=int(info["out"].dims[0]),
                                     device=dev, precision=self._prec)
                    pool = info["pool_out"].dt if "pool_out" in info else None
                    calls.append(lambda x=xz, pk=pk, out=out, base=base,
                                 pad=(info["pad"][0], info["pad"][1], 0), act=st.fused_act,
                                 pool=pool, hd=hd, hout=hout:
                                 K.conv3d(x, pk, out, pad=pad, base=base, fused_act=act,
                                          pool_out=pool, head=hd, head_out=hout))
                else:
                    pk = K.pack_conv(kern, w.tensor(st.name, ROLE_BIAS), stride=stride,
                                     base_scale=scale, path=self._conv_path,
                                     out_shape=tuple(info["out"].dims[2:]), batch=int(info["out"].dims[0]), device=dev,
                                     precision=self._prec)
                    x = fused_in.get(id(info), info["x"].dt)
                    if id(info) in fused_in and pk.path not in _lib.TC_PATHS:
                        raise ExecutionError("fused fp32 input needs the tensor-core conv path")
                    pool = info["pool_out"].dt if "pool_out" in info else None
                    calls.append(lambda x=x, pk=pk, out=out, base=base,
                                 pad=info["pad"], act=st.fused_act, pool=pool, hd=hd, hout=hout:
                                 K.conv3d(x, pk, out, pad=pad, base=base, fused_act=act,
                                          pool_out=pool, head=hd, head_out=hout))
            elif kind is LayerKind.DECONVOLUTION:
                base = info["base"].dt if "base" in info else None
                scale = st.base_scale if st.additive else None
                pk = K.pack_deconv(w.tensor(st.name, ROLE_KERNEL), w.tensor(st.name, ROLE_BIAS),
                                   stride=tuple(st.params["stride"]), base_scale=scale,
                                   force_gather=self.precision == "fp32", device=dev,
                                   precision=self._prec)
                calls.append(lambda x=info["ins"][0].dt, pk=pk, out=out, base=base,
                             act=st.fused_act: K.deconv3d(x, pk, out, base=base, fused_act=act))
            elif kind is LayerKind.POOLING:
                calls.append(lambda x=info["ins"][0].dt, out=out, p=st.params:
                             K.pool3d(x, out, p["window"], p["stride"], p["mode"]))
            elif kind is LayerKind.ELTWISE:
                a, b = info["ins"]
                calls.append(lambda a=a.dt, b=b.dt, out=out, op=st.params["op"]:
                             K.eltwise(a, b, out, op))
            elif kind is LayerKind.MERGE_CROP:
                calls.append(lambda a=info["a"].dt, b=info["b"].dt, out=out:
                             K.mergecrop(a, b, out))
            elif kind in (LayerKind.BATCH_NORM, LayerKind.SCALE):
                if kind is LayerKind.BATCH_NORM:
                    m, a = bn_coefficients(w.tensor(st.name, ROLE_BN_MEAN),
                                           w.tensor(st.name, ROLE_BN_VAR), w.bn_eps(st.name))
                else:
                    m = w.tensor(st.name, ROLE_SCALE_GAMMA)
                    a = w.tensor(st.name, ROLE_SCALE_BETA)
                from .device import device_vector
                md, ad = device_vector(m, device=dev), device_vector(a, device=dev)
                calls.append(lambda x=info["ins"][0].dt, out=out, md=md, ad=ad:
                             K.affine_act(x, out, md, ad))
            elif kind in (LayerKind.RELU, LayerKind.ELU, LayerKind.SIGMOID):
                act = kind.value.lower()
                alpha = float(st.params.get("alpha", DEFAULT_ELU_ALPHA))
                calls.append(lambda x=info["ins"][0].dt, out=out, act=act, alpha=alpha:
                             K.affine_act(x, out, None, None, act, alpha))
            else:
                raise ExecutionError("plan step %r has unrunnable kind %s" % (st.name, kind))
        self.op_calls = calls[n_in:n_in + len(self._ops)]   # one device call per lowered op
        self.op_names = [st.name for _, st, _ in self._ops]
        if self.probe is not None:
            if self.probe not in self.op_names:
                raise ExecutionError("probe step %r is not a lowered op of this plan" % self.probe)
            i = n_in + self.op_names.index(self.probe)
            ev = self._probe_ev

            def probed(c=calls[i], ev=ev):
                torch = _torch()
                ev[0].record(torch.cuda.current_stream())
                c()
                ev[1].record(torch.cuda.current_stream())
            calls[i] = probed
        for name, v in self._out_values.items():
            if name in self._fused_outputs:
                continue
            dst = standard(self._out_std[name])
            calls.append(lambda s=v.dt, d=dst: _copy(s, d))
        self._calls = calls

    def _zwin_plan(self, v, rs):
        """z-window pack for a 1-channel network input read only by one
        stride-1 tensor-core conv with <= 8 z taps (the U-nets' first layer:
        its 8-lane chunks would otherwise be 7/8 padding).  Returns the
        packed input tensor (n, kz, x, y, oz), kz and the z pad, or None."""
        if self.precision not in ("bf16", "x3") or os.environ.get("VXB_ZWIN", "1") != "1":
            return None
        if v.dims[1] != 1 or v.readers != 1 or len(rs) != 1:
            return None
        st, info = rs[0]
        if "segments" in info or tuple(st.params.get("stride", (1, 1, 1))) != (1, 1, 1):
            return None
        kern = self.plan.weights.tensor(st.name, ROLE_KERNEL)
        k = tuple(int(t) for t in kern.shape[2:])
        pz = int(info["pad"][2])
        if not 1 <= k[2] <= 8 or pz > k[2] - 1:
            return None
        L = _lib.lib()
        if L.vxb_conv_select(k[2], st.output.dims[1], _lib.i3((k[0], k[1], 1)),
                             _lib.i3((1, 1, 1))) != _lib.PATH_TC:
            return None
        n, _, x, y, z = v.dims
        oz = z + 2 * pz - k[2] + 1
        from .device import empty_blocked
        return (empty_blocked(n, k[2], (x, y, oz), self.storage, self.device, zero=True), k[2],
                pz)

    def _f32in_ok(self, name, st, info) -> bool:
        """Can this conv read network input `name` as fp32 NCDHW directly
        (vxb_conv3d's in-kernel conversion: stride 1, one input segment, no
        residual, z rows of 16-byte multiples, whole chunks when batch > 1)?"""
        if not self.fuse_input or self.precision != "bf16":
            return False
        if "segments" in info or "base" in info or st.additive:
            return False
        if tuple(st.params.get("stride", (1, 1, 1))) != (1, 1, 1):
            return False
        n, c, x, y, z = self._input_dims[name]
        k = tuple(int(v) for v in self.plan.weights.tensor(st.name, ROLE_KERNEL).shape[2:])
        if z % 4 or (n > 1 and c % LANES):
            return False
        L = _lib.lib()
        return L.vxb_conv_select(c, st.output.dims[1], _lib.i3(k), _lib.i3((1, 1, 1))) == \
            _lib.PATH_TC

    # ------------------------------------------------------------ running
    def _launch_all(self):
        L = _lib.lib()
        prev = L.vxb_set_pdl(-1 if self.pdl is None else int(bool(self.pdl)))
        try:
            for c in self._calls:
                c()
        finally:
            L.vxb_set_pdl(prev)

    def ensure_graph(self):
        """Capture this runner's graph now if it has not been (the first
        launches also configure the kernels' shared-memory attributes)."""
        torch = _torch()
        if self._graph is None and self.use_graph:
            self._replay()
            self.stream.synchronize()

    def launch_raw(self, skip_inputs=False):
        """Launch the network's kernels on the current stream without the
        graph (for a caller capturing a larger graph around them);
        ``skip_inputs``: the caller has packed the network inputs itself."""
        if not skip_inputs:
            self._launch_all()
            return
        L = _lib.lib()
        prev = L.vxb_set_pdl(-1 if self.pdl is None else int(bool(self.pdl)))
        try:
            for c in self._calls[self._n_in_calls:]:
                c()
        finally:
            L.vxb_set_pdl(prev)

    def _replay(self):
        torch = _torch()
        if not self.use_graph:
            with torch.cuda.stream(self.stream):
                self._launch_all()
            return
        if self._graph is None:
            with torch.cuda.stream(self.stream):
                self._launch_all()          # warm-up (first launches configure kernels)
            # capture from a quiet device, and only this thread's CUDA calls
            # count against the capture (other threads - staging, a clock
            # sampler - may call the runtime meanwhile)
            torch.cuda.synchronize(self.device)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=self.stream, capture_error_mode="thread_local"):
                self._launch_all()
            self._graph = g
        with torch.cuda.stream(self.stream):
            self._graph.replay()

    def _normalize(self, inputs):
        if not isinstance(inputs, dict):
            if len(self._input_dims) != 1:
                raise ExecutionError("plan has %d inputs, pass a dict" % len(self._input_dims))
            inputs = {next(iter(self._input_dims)): inputs}
        for name, want in self._input_dims.items():
            if name not in inputs:
                raise ExecutionError("missing value for input %r" % name)
            got = tuple(inputs[name].shape)
            if got != tuple(want):
                raise ExecutionError("input %r has shape %s, plan wants %s"
                                     % (name, got, tuple(want)))
        return inputs

    def run_device(self, inputs):
        """Device-resident forward: inputs/outputs are CUDA fp32 NCDHW tensors.
        Work is enqueued on ``self.stream``; the returned tensors are the
        runner's static output buffers (valid until the next call)."""
        torch = _torch()
        inputs = self._normalize(inputs)
        cs = torch.cuda.current_stream(self.device)
        self.stream.wait_stream(cs)
        with torch.cuda.stream(self.stream):
            for name, t in inputs.items():
                if t.data_ptr() != self._in_std[name].data_ptr():
                    self._in_std[name].copy_(t, non_blocking=True)
        self._replay()
        cs.wait_stream(self.stream)
        return dict(self._out_std)

    def run_on_stream(self, inputs):
        """``run_device`` without ordering against the caller's current
        stream: the input copies and the graph replay are enqueued on
        ``self.stream`` only (the caller orders producers and consumers of
        the tensors, e.g. several runners pipelining patches)."""
        torch = _torch()
        inputs = self._normalize(inputs)
        if self._graph is None and self.use_graph:
            self._replay()                   # first call: capture (synchronous once)
            self.stream.synchronize()
        with torch.cuda.stream(self.stream):
            for name, t in inputs.items():
                if t.data_ptr() != self._in_std[name].data_ptr():
                    self._in_std[name].copy_(t, non_blocking=True)
        self._replay()
        return dict(self._out_std)

    def run(self, inputs, out=None) -> dict:
        """Reference-compatible forward (executor.py:168-198): host in, host out.
        Inputs go host -> pinned staging -> HBM and outputs the reverse, in
        chunks that overlap the host copies with PCIe (staging.py).  Inputs
        already page-locked (``staging.pinned_empty``) and ``out={name: pinned
        array}`` skip the staging copy: one DMA each way."""
        from . import staging
        inputs = self._normalize(inputs)
        for name, arr in inputs.items():
            staging.upload(arr, self._in_pinned[name], self._in_std[name], self.stream)
        self._replay()
        out = out or {}
        outs = {name: staging.download(t, self._out_pinned[name], self.stream, out.get(name))
                for name, t in self._out_std.items()}
        return outs

    def run_async(self, inputs, out) -> "PendingRun":
        """Non-blocking forward for pipelined serving: page-locked float32
        inputs (``staging.pinned_empty``) and ``out={name: pinned array}``.
        The H2D copies, the graph replay and the D2H copies are enqueued on
        this runner's stream and the call returns at once; ``.wait()`` on the
        result blocks until ``out`` holds the results.  Calls on one runner
        are ordered by its stream; runners on different streams overlap (one
        volume's upload with another's download and compute).  The inputs
        must stay untouched until the run completes."""
        from . import staging
        torch = _torch()
        inputs = self._normalize(inputs)
        for name, arr in inputs.items():
            if not staging.is_pinned(arr):
                raise ExecutionError("run_async needs page-locked float32 inputs "
                                     "(staging.pinned_empty)")
        for name, t in self._out_std.items():
            o = out.get(name) if out else None
            if o is None or tuple(o.shape) != tuple(t.shape) or not staging.is_pinned(o):
                raise ExecutionError("run_async needs a pinned float32 out[%r] of shape %s"
                                     % (name, tuple(t.shape)))
        if self._graph is None and self.use_graph:
            self._replay()              # first call: capture (synchronous once)
            self.stream.synchronize()
        with torch.cuda.stream(self.stream):
            for name, arr in inputs.items():
                self._in_std[name].copy_(torch.from_numpy(arr), non_blocking=True)
            self._graph.replay() if self._graph is not None else self._launch_all()
            for name, t in self._out_std.items():
                torch.from_numpy(out[name]).copy_(t, non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(self.stream)
        return PendingRun(ev, {name: out[name] for name in self._out_std})

    def probe_ms(self) -> float:
        """Duration of the probed step in the last completed run (ms)."""
        if self._probe_ev is None:
            raise ExecutionError("PlanRunner was built without a probe")
        return self._probe_ev[0].elapsed_time(self._probe_ev[1])

    def input_buffers(self) -> dict:
        """The static device input tensors the captured graph reads.  Filling
        them in place and passing them to ``run_device`` skips its copy."""
        return dict(self._in_std)

    @property
    def h2d_bytes(self) -> int:
        return sum(t.numel() * 4 for t in self._in_std.values())

    @property
    def d2h_bytes(self) -> int:
        return sum(t.numel() * 4 for t in self._out_std.values())


class PendingRun:
    """Handle of a ``PlanRunner.run_async`` call."""

    def __init__(self, event, outputs):
        self._event = event
        self.outputs = outputs

    def done(self) -> bool:
        return self._event.query()

    def wait(self) -> dict:
        self._event.synchronize()
        return self.outputs


def _pack_zwin(src: DTensor, dst: DTensor, kz: int, pz: int, independent=False):
    from .device import pack_zwin
    pack_zwin(src, dst, kz, pz, independent=independent)


def _copy(src: DTensor, dst: DTensor, independent=False):
    from .device import copy
    copy(src, dst, independent=independent)


class PlanBatch:
    """Several independent networks (PlanRunners on one device, inputs in
    their static input buffers) replayed back to back as ONE CUDA graph.

    A serving loop over many small volumes, or the config-2 featuremap
    sweep, runs networks whose inputs are all resident: the fp32 -> bf16
    input pack of network i+1 then has no dependency on network i.  Packs are
    launched with VXB_COPY_INDEPENDENT, so inside the graph each one starts as
    soon as the previous network's persistent conv is resident and runs in
    the one CTA slot per SM that conv leaves free (HBM-bound pack beside a
    tensor-bound conv); the next conv still waits for its pack.  Results are
    bit-identical to running the networks one by one.

    The graph holds two streams: the input packs chained on a side stream
    (background launch priority) and each network's body on the main stream
    after its own pack, so the packs stream ahead in the SM slots the convs
    leave free and the convs' CTAs are always dispatched first (config-2
    sweep 0.850 -> 0.832 ms; a side stream without priorities 0.858 ms).

    ``reorder`` (default) runs the networks largest-first by conv FLOPs so
    that each input pack hides behind a conv at least as large as its own
    network's, except that the smallest network goes first (its pack is the
    one nothing hides): config-2 sweep 0.878 ms in listed order, 0.844
    largest-first, 0.842 smallest + largest-first (with the side stream:
    0.837 smallest + largest-first, 0.841 largest-first, 0.861 ascending —
    packs running beside the small memory-bound convs slow them most;
    `tools/batch_timeline.py`).  Outputs are returned in the caller's order."""

    def __init__(self, runners, reorder=True, probe=None):
        torch = _torch()
        if not runners:
            raise ExecutionError("PlanBatch needs at least one runner")
        dev = runners[0].device
        if any(r.device != dev for r in runners):
            raise ExecutionError("PlanBatch runners must share one device")
        self.runners = list(runners)
        order = list(range(len(self.runners)))
        if reorder and len(order) > 2:
            work = [_conv_flops(r.plan) for r in self.runners]
            mode = os.environ.get("VXB_BATCH_ORDER", "small_first")
            if "," in mode:                      # explicit order (experiments)
                order = [int(t) for t in mode.split(",")]
            else:
                order.sort(key=lambda i: work[i] if mode == "asc" else -work[i])
                if mode == "small_first":
                    order = order[-1:] + order[:-1]
        self.order = order
        self.device = dev
        self.stream = torch.cuda.Stream(device=dev)
        self.launches = sum(r.launches for r in runners)
        self._graph = None
        # optional live timing of one network's body inside the graph
        # (external timing events recorded around it at every replay)
        self.probe = probe
        self._probe_ev = None
        if probe is not None:
            self._probe_ev = (torch.cuda.Event(enable_timing=True, external=True),
                              torch.cuda.Event(enable_timing=True, external=True))

    def _capture_two_streams(self):
        """Input packs chained on a side stream (launched at background
        priority), each network's body on the main stream after its own
        pack: the packs stream ahead in the SM slots the convs leave free."""
        torch = _torch()
        side = self._side
        side.wait_stream(self.stream)
        evs = []
        with torch.cuda.stream(side):
            for i in self.order:
                r = self.runners[i]
                for c in r._calls[:r._n_in_calls]:
                    c()
                e = torch.cuda.Event()
                e.record(side)
                evs.append(e)
        for i, e in zip(self.order, evs):
            r = self.runners[i]
            self.stream.wait_event(e)
            if i == self.probe:
                self._probe_ev[0].record(self.stream)
            for c in r._calls[r._n_in_calls:]:
                c()
            if i == self.probe:
                self._probe_ev[1].record(self.stream)
        self.stream.wait_stream(side)

    def replay(self):
        """Enqueue every network once on ``self.stream`` (captured on first use)."""
        torch = _torch()
        two = os.environ.get("VXB_BATCH_SIDE_STREAM", "1") == "1"
        if self._graph is None:
            self._side = torch.cuda.Stream(device=self.device)
            with torch.cuda.device(self.device), torch.cuda.stream(self.stream):
                for i in self.order:
                    self.runners[i]._launch_all()   # warm-up: first launches configure kernels
            torch.cuda.synchronize(self.device)
            indep = os.environ.get("VXB_DEBUG_PACK_DEPENDENT") != "1"
            for r in self.runners:
                r._indep_flag[0] = indep
            try:
                g = torch.cuda.CUDAGraph()
                with torch.cuda.device(self.device), \
                        torch.cuda.graph(g, stream=self.stream, capture_error_mode="thread_local"):
                    if two:
                        self._capture_two_streams()
                    else:
                        for i in self.order:
                            self.runners[i]._launch_all()
            finally:
                for r in self.runners:
                    r._indep_flag[0] = False
            self._graph = g
        with torch.cuda.stream(self.stream):
            self._graph.replay()

    def probe_ms(self) -> float:
        """Duration of the probed network's body in the last replay (ms;
        the replay must have completed)."""
        if self._probe_ev is None:
            raise ExecutionError("PlanBatch was built without a probe")
        return self._probe_ev[0].elapsed_time(self._probe_ev[1])

    def run_device(self):
        """Replay ordered after the caller's current stream; returns each
        runner's static output buffers."""
        torch = _torch()
        cs = torch.cuda.current_stream(self.device)
        self.stream.wait_stream(cs)
        self.replay()
        cs.wait_stream(self.stream)
        return [dict(r._out_std) for r in self.runners]


def _conv_flops(plan) -> float:
    """Multiply-add work of a plan's convolutions (PlanBatch ordering)."""
    f = 0.0
    for st in plan.steps:
        if st.kind is LayerKind.CONVOLUTION:
            k = plan.weights.tensor(st.name, ROLE_KERNEL).shape
            f += 2.0 * float(np.prod(k)) * float(np.prod(st.output.dims[2:])) * st.output.dims[0]
    return f


def execute(plan, inputs, backend=None) -> dict:
    """One-shot convenience (executor.py:201-203)."""
    return PlanRunner(plan, backend=backend).run(inputs)
