#!/usr/bin/env python
"""Benchmark: B200 fused conv3d inference vs the reference CPU engine.

Contract (one JSON line on rank 0):
  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl b200|reference]

Workloads (BASELINE.json configs; synthetic seeded inputs):
  --config 2 (default, BASELINE configs[1]): the featuremap sweep — conv
      C->C (C in 8..128) with kernels 3x3x3 and 1x3x3, 'same' padding, fused
      bias + ELU, on 1xCx32x128x128 fp32 inputs.  One step = all 10 layers,
      each through its PlanRunner (fp32 NCDHW in HBM -> bf16 blocked ->
      tcgen05 conv -> fp32 NCDHW out).  Unit: output voxels/s.
  --config 1, 3, 4: the single layer, residual block and Cicek U-net.
  --config 5: the anisotropic residual U-net over the 128x1024x1024 volume,
      288 patches of 18x192x192 split across ranks (strong scaling).

Timing: W warm-up steps, then K steps bracketed by barrier + synchronize,
CUDA events on the runner streams, max over ranks.  The L2 (126 MB) is
flushed with a 512 MB write between steps, outside the timed windows.
``e2e`` repeats the metric through the public host API (PlanRunner.run with
host fp32 arrays: pinned H2D + graph + D2H inside the timed region).
``roofline`` is the dominant conv kernel alone (CUDA graph of that launch),
``cpu_baseline`` the reference's own compiled kernel (oracle/_ref) on the
host cores on a bounded sample.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "output voxels/sec for 3D U-net inference; conv3d TFLOP/s vs tensor-core peak"


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=60)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=2, choices=[1, 2, 3, 4, 5])
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=20.0,
                    help="target CPU-baseline sample duration")
    return ap.parse_args()


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return {"hbm": p["hbm_gbs"], "bf16": p["bf16_tflops"],
                "bf16_sustained": p.get("bf16_tflops_sustained", p["bf16_tflops"]),
                "source": "measured (MEASURED_PEAKS.json)"}
    except Exception:
        return {"hbm": 6650.0, "bf16": 1590.0, "bf16_sustained": 1400.0,
                "source": "fallback (B200_PROFILING.md)"}


# ------------------------------------------------------------------ workloads

def build_workload(cfg):
    """[(name, spec, store, flops)] for a config."""
    from paper_1903_07525_b200 import configs as C
    if cfg == 2:
        out = []
        for k in C.SWEEP_K:
            for c in C.SWEEP_C:
                spec, store = C.config2(c, k)
                out.append(("c%d_k%s" % (c, "".join(map(str, k))), spec, store))
    elif cfg == 1:
        out = [("cfg1",) + C.config1()]
    elif cfg == 3:
        out = [("cfg3",) + C.config3()]
    elif cfg == 4:
        out = [("cfg4",) + C.config4()]
    else:
        out = [("cfg5",) + C.config5()]
    return [(n, s, st, C.conv_flops(s)) for n, s, st in out]


def output_voxels(spec):
    from paper_1903_07525_b200.shapes import validate_shapes
    shapes = validate_shapes(spec)
    total = 0
    for blob in spec.output_blobs():
        n, _, x, y, z = shapes[blob]
        total += n * x * y * z
    return total


# ------------------------------------------------------------------ clocks

class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def _reader(self):
        for line in self.proc.stdout:
            if line.strip():
                self.lines.append(line)

    def __enter__(self):
        import threading
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=" + self.FIELDS,
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return self
        self.thread = threading.Thread(target=self._reader, daemon=True)
        self.thread.start()
        # nvidia-smi takes a few hundred ms to start: only open the timed
        # region once it is sampling
        t0 = time.time()
        while not self.lines and time.time() - t0 < 5.0 and self.proc.poll() is None:
            time.sleep(0.01)
        self.skip = len(self.lines)          # samples taken before the timed region
        return self

    def __exit__(self, *a):
        if self.proc is not None:
            # a timed region shorter than the 20 ms sampling period would get
            # no sample: wait (<= 100 ms) for one taken at its end
            t0 = time.time()
            while len(self.lines) <= self.skip and time.time() - t0 < 0.1:
                time.sleep(0.005)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                pass
            self.thread.join(timeout=5)
            self.lines = self.lines[self.skip:]

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for l in self.lines:
            parts = [p.strip() for p in l.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------------ B200 arm

def run_b200(args, rank, world, local_rank):
    import torch
    import paper_1903_07525_b200 as P
    from paper_1903_07525_b200 import configs as C, ops as K
    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    peaks = load_peaks()
    lo, hi = C.input_range(args.config)
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)

    def barrier():
        torch.cuda.synchronize(dev)
        if dist is not None:
            dist.barrier()

    if args.config == 5:
        return run_tiled_volume(args, rank, world, dev, dist, peaks, flush)

    work = build_workload(args.config)
    layers = []
    for name, spec, store, flops in work:
        plan, _ = P.compile_network(spec, store, fixpoint=True, fuse_deconv_add=True)
        runner = P.PlanRunner(plan, backend="b200", device=dev)
        x = C.make_input(spec, seed=100 + rank, low=lo, high=hi)
        # inputs resident in HBM: written once into the runner's static input
        # buffer (the tensor its CUDA graph reads), so run_device copies nothing
        xd = runner.input_buffers()
        xd[plan.inputs[0][0]].copy_(torch.from_numpy(x))
        layers.append({"name": name, "plan": plan, "runner": runner, "x": x, "xd": xd,
                       "flops": flops, "vox": output_voxels(spec)})

    # The step: every layer's network once, as one CUDA graph (PlanBatch):
    # each network's fp32 -> bf16 input pack runs beside the previous
    # network's conv (independent launch), each conv waits for its own pack.
    # the dominant network (most conv FLOPs) is timed live inside every
    # timed replay (external events around its body in the graph)
    dom = max(range(len(layers)), key=lambda i: layers[i]["flops"])
    batch = P.PlanBatch([L["runner"] for L in layers])
    # the same batch with timing events around the dominant network's body
    # (its conv): replayed after the timed steps, since the two event nodes
    # cost the step ~20 us (they cut the conv's programmatic-launch overlap)
    pbatch = P.PlanBatch([L["runner"] for L in layers], probe=dom)

    def batch_step():
        """One timed window around the whole sweep on the batch stream (a
        short device-side spin first, so the window holds GPU time only)."""
        cs = torch.cuda.current_stream(dev)
        torch.cuda._sleep(200_000)
        batch.stream.wait_stream(cs)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(batch.stream)
        batch.replay()
        e1.record(batch.stream)
        cs.wait_stream(batch.stream)
        return e0, e1

    def step(timed):
        """Per-layer breakdown (not the headline): one network at a time,
        each in its own window; returns per-layer event pairs."""
        evs = []
        torch.cuda._sleep(200_000)
        for L in layers:
            s = L["runner"].stream
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            # start only once the previous layer (ordered via the current
            # stream) has finished, so the windows do not overlap
            s.wait_stream(torch.cuda.current_stream(dev))
            e0.record(s)
            L["runner"].run_device(L["xd"])
            e1.record(s)
            evs.append((e0, e1))
        return evs

    for _ in range(max(3, args.warmup)):
        batch_step()
        step(False)
    barrier()
    total_ms = 0.0
    live_ms = 0.0
    with ClockSampler(local_rank) as clk:
        for _ in range(args.steps):
            flush.fill_(1.0)            # L2 flush, outside the timed window
            barrier()
            a, b = batch_step()
            torch.cuda.synchronize(dev)
            total_ms += a.elapsed_time(b)
    barrier()
    probe_steps = max(3, min(args.steps, 20))
    for i in range(probe_steps + 2):
        flush.fill_(1.0)
        torch.cuda.synchronize(dev)
        pbatch.run_device()
        torch.cuda.synchronize(dev)
        if i >= 2:
            live_ms += pbatch.probe_ms()
    live_ms = live_ms / probe_steps * args.steps
    per_layer_ms = [0.0] * len(layers)
    layer_steps = max(3, min(args.steps, 10))
    for _ in range(layer_steps):
        flush.fill_(1.0)
        evs = step(True)
        torch.cuda.synchronize(dev)
        for i, (a, b) in enumerate(evs):
            per_layer_ms[i] += a.elapsed_time(b) * args.steps / layer_steps
    if dist is not None:
        t = torch.tensor([total_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = t.item()
    vox_step = sum(L["vox"] for L in layers)
    ms_per_step = total_ms / args.steps
    value = vox_step * world / (ms_per_step * 1e-3)

    # ---- dominant kernel: timed live in the step (above) and alone
    rd = layers[dom]["runner"]
    single = len(rd._calls) - rd._n_in_calls == 1   # body = the conv alone (config 2)
    roof = kernel_roofline(layers[dom], dev, peaks,
                           live_ms=live_ms / args.steps if single else None)

    result = {
        "metric": METRIC, "value": value, "unit": "output voxels/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (seeded uniform inputs, He-normal weights, BASELINE.json shapes)",
        "config": {"workload": workload_name(args.config),
                   "layers": [L["name"] for L in layers],
                   "output_voxels_per_step": vox_step,
                   "parallelism": "replicas" if world > 1 else "single",
                   "l2": "flushed (512 MB write) between steps, outside timed region"},
        "tflops": sum(L["flops"] for L in layers) * world / (ms_per_step * 1e-3) / 1e12,
        "layers_note": "per network run alone (sequential windows, %d passes); the step "
                       "runs them as one graph with input packs overlapping the previous "
                       "network's conv" % layer_steps,
        "layers": {L["name"]: {"ms": per_layer_ms[i] / args.steps,
                               "tflops": L["flops"] / (per_layer_ms[i] / args.steps * 1e-3) / 1e12}
                   for i, L in enumerate(layers)},
        "roofline": roof,
        "gpu_launches": sum(L["runner"].launches for L in layers) * args.steps,
        "clocks": clk.summary(),
    }
    if not args.no_e2e:
        result["e2e"] = e2e_layers(layers, args, dev, dist, world)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        result["cpu_baseline"] = cpu_baseline(args, work, target_s=args.cpu_seconds)
    return result


def workload_name(cfg):
    return {1: "config1: conv3d 3x3x3 C16->16 + bias + ReLU, 1x16x32x64x64",
            2: "config2: featuremap sweep C in {8..128} x k in {3x3x3, 1x3x3}, conv + bias + "
               "ELU on 1xCx32x128x128 (BASELINE configs[1])",
            3: "config3: residual block C64 on 1x64x24x128x128",
            4: "config4: Cicek 3D U-net 132^3 -> 3x44^3",
            5: "config5: anisotropic residual U-net, 128x1024x1024 volume, 18x192x192 patches"}[cfg]


def kernel_roofline(L, dev, peaks, live_ms=None):
    """Roofline of the dominant conv kernel.  ``live_ms``: its duration inside
    the timed steps (external events around it in the step's graph, L2
    flushed before each step) - the figure `achieved` is computed from.  It is
    also timed alone (its launch replayed from a CUDA graph 20 times between
    events on the graph's stream) for reference."""
    import torch
    from paper_1903_07525_b200.netspec import LayerKind
    from paper_1903_07525_b200.formats import ROLE_KERNEL
    runner = L["runner"]
    plan = L["plan"]
    # the network's largest conv (by FLOPs): its own algorithmic FLOPs and
    # bytes (bf16 blocked input, output bf16 or the fused fp32 network output,
    # residual operand if any; weights negligible)
    out_vals = {id(v): name for name, v in runner._out_values.items()}
    best = None
    for c, (kind, st, info) in zip(runner.op_calls, runner._ops):
        if kind is not LayerKind.CONVOLUTION:
            continue
        kshape = plan.weights.tensor(st.name, ROLE_KERNEL).shape
        n, cout, ox, oy, oz = st.output.dims
        f = 2.0 * float(np.prod(kshape)) * n * ox * oy * oz
        # input tensors read (a fused concat reads both segments)
        ins = list(info["segments"][:2]) if "segments" in info else [info["x"]]
        in_b = 2.0 * sum(v.dims[1] * float(np.prod(v.dims[2:])) * v.dims[0] for v in ins)
        fused = out_vals.get(id(info["out"])) in runner._fused_outputs
        out_b = (4.0 if fused else 2.0) * cout * n * ox * oy * oz
        base_b = 2.0 * cout * n * ox * oy * oz if st.additive else 0.0
        if best is None or f > best[1]:
            best = (c, f, in_b + out_b + base_b, st.name)
    call, flops, alg_bytes, conv_name = best
    s = torch.cuda.Stream(device=dev)
    with torch.cuda.stream(s):
        call()
    s.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        call()
    reps = 20
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s):
        for _ in range(3):
            g.replay()
        torch.cuda._sleep(200_000)
        e0.record(s)
        for _ in range(reps):
            g.replay()
        e1.record(s)
    s.synchronize()
    alone_ms = e0.elapsed_time(e1) / reps
    ms = live_ms if live_ms else alone_ms
    ai = flops / alg_bytes
    ridge = peaks["bf16"] * 1e12 / (peaks["hbm"] * 1e9)
    if ai >= ridge:
        achieved = flops / (ms * 1e-3) / 1e12
        roof = {"bound": "tensor", "achieved": achieved, "peak": peaks["bf16"],
                "unit": "TFLOP/s", "frac": achieved / peaks["bf16"]}
    else:
        achieved = alg_bytes / (ms * 1e-3) / 1e9
        roof = {"bound": "hbm", "achieved": achieved, "peak": peaks["hbm"], "unit": "GB/s",
                "frac": achieved / peaks["hbm"]}
    label = L["name"] if conv_name == "conv" or len(runner._ops) <= 2 else \
        "%s/%s" % (L["name"], conv_name)
    roof.update({"kernel": "conv3d_tc_kernel (%s)" % label, "ms_per_launch": ms,
                 "timing": ("in-step: events around it in replays of the step's graph "
                            "(L2 flushed before each)") if live_ms else "alone, 20 graph replays",
                 "alone_ms_per_launch": alone_ms,
                 "alg_flops": flops, "alg_bytes": alg_bytes, "peak_source": peaks["source"],
                 "traffic": ncu_traffic(L["name"])})
    return roof


def ncu_traffic(name):
    """dram bytes per launch from a committed ncu --set full capture, if any."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as fh:
            return json.load(fh).get(name)
    except Exception:
        return None


def e2e_layers(layers, args, dev, dist, world):
    """Same metric through the public host API (PlanRunner.run on host arrays).
    The step's inputs sit in page-locked host memory and results land in
    page-locked arrays (staging.pinned_empty), so each call is one H2D DMA,
    the graph replay and one D2H DMA."""
    import torch
    from paper_1903_07525_b200 import staging
    for L in layers:
        xp = staging.pinned_empty(L["x"].shape)
        xp[...] = L["x"]
        L["xp"] = xp
        L["outp"] = {n: staging.pinned_empty(t.shape) for n, t in L["runner"]._out_std.items()}
        L["runner"].run(L["xp"], out=L["outp"])
    torch.cuda.synchronize(dev)
    if dist is not None:
        dist.barrier()
    steps = max(1, min(args.steps, 5))
    t0 = time.perf_counter()
    pend = []
    for _ in range(steps):
        # every layer's volume is in flight at once: its upload overlaps the
        # other layers' compute and downloads (PlanRunner.run_async); runs on
        # one runner are ordered by its stream
        pend += [L["runner"].run_async(L["xp"], out=L["outp"]) for L in layers]
    for h in pend:
        h.wait()
    torch.cuda.synchronize(dev)
    el = time.perf_counter() - t0
    if dist is not None:
        t = torch.tensor([el], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        el = t.item()
    vox = sum(L["vox"] for L in layers)
    return {"value": vox * world * steps / el, "unit": "output voxels/s",
            "h2d_bytes_per_step": sum(L["runner"].h2d_bytes for L in layers),
            "d2h_bytes_per_step": sum(L["runner"].d2h_bytes for L in layers),
            "steps": steps, "timer": "host wall clock around PlanRunner.run_async + wait for every layer "
                                     "(H2D from pinned host input, graph replay, D2H into "
                                     "pinned host output; layers pipelined across streams)"}


# ------------------------------------------------------------------ CPU baseline

def cpu_threads():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def reference_sample_runner(work, threads, target_s):
    """Bind the reference's compiled kernel for every layer; pick an x-slab
    sample per layer so one pass takes about target_s seconds."""
    from oracle import ref_engine as E
    from oracle import ref_numpy as R
    from paper_1903_07525_b200.formats import ROLE_BIAS, ROLE_KERNEL
    if not E.available():
        return None
    items = []
    for name, spec, store, flops in work:
        conv = [l for l in spec.layers if l.kind.value == "Convolution"]
        if len(conv) != 1:
            return None       # multi-layer nets: see DESIGN.md (config 2 is the bench line)
        lay = conv[0]
        act = [l for l in spec.layers if l.kind.value in ("ReLU", "ELU", "Sigmoid")]
        kind = act[0].kind.value.lower() if act else None
        stp = E.ConvStep(store.tensor(lay.name, ROLE_KERNEL), store.tensor(lay.name, ROLE_BIAS),
                         pad=lay.params["pad"], act=kind)
        shape = spec.input_layers()[0].params["shape"]
        x = np.random.default_rng(7).uniform(-1, 1, shape).astype(np.float32)
        xb = stp.prepare(x)
        ox = shape[2]
        out = np.zeros((1, -(-stp.fo // 8), ox) + tuple(shape[3:]) + (8,), np.float32)
        items.append({"name": name, "step": stp, "xb": xb, "out": out, "ox": ox,
                      "vox_per_row": int(np.prod(shape[3:])), "flops": flops})
    # calibrate rows per layer on one row of each
    t0 = time.perf_counter()
    for it in items:
        it["step"].run_blocked(it["xb"], it["out"], None, (0, 1))
    one_row_all = time.perf_counter() - t0
    rows = max(1, min(items[0]["ox"], int(target_s * threads / max(one_row_all, 1e-6))))
    rows = max(threads, (rows // threads) * threads) if rows >= threads else rows
    rows = min(rows, items[0]["ox"])
    from concurrent.futures import ThreadPoolExecutor
    pool = ThreadPoolExecutor(max_workers=threads)

    def one_pass():
        vox = 0
        for it in items:
            cuts = np.linspace(0, rows, min(threads, rows) + 1).astype(int)
            list(pool.map(lambda i: it["step"].run_blocked(it["xb"], it["out"], None,
                                                          (cuts[i], cuts[i + 1])),
                          range(len(cuts) - 1)))
            vox += rows * it["vox_per_row"]
        return vox

    return one_pass, rows


def cpu_baseline(args, work, target_s):
    threads = cpu_threads()
    r = reference_sample_runner(work, threads, target_s)
    if r is None:
        return {"value": None, "unit": "output voxels/s", "cores": threads, "kind": "reference",
                "sample": "unavailable (oracle/_ref not built or multi-layer config)"}
    one_pass, rows = r
    # whole passes until the sample holds at least ~min(10 s, target) of CPU work
    t0 = time.perf_counter()
    vox, passes = 0, 0
    while True:
        vox += one_pass()
        passes += 1
        el = time.perf_counter() - t0
        if el >= min(10.0, target_s) or passes >= 100:
            break
    return {"value": vox / el, "unit": "output voxels/s", "cores": threads, "kind": "reference",
            "sample": "%d pass(es) over %d of 32 x-rows of every config-2 layer (%d output "
                      "voxels), reference _kernels.conv3d from oracle/_ref, x-slabs on %d "
                      "threads, %.1f s" % (passes, rows, vox, threads, el)}


def run_reference(args, rank, world):
    """--impl reference: the reference's own CPU implementation on the host cores."""
    if world > 1 and rank != 0:
        return None
    threads = cpu_threads()
    work = build_workload(args.config)
    r = reference_sample_runner(work, threads, target_s=min(8.0, args.cpu_seconds))
    if r is None:
        return {"impl": "reference", "metric": METRIC,
                "unavailable": "reference CPU arm implemented for configs 1-2 (oracle/_ref)"}
    one_pass, rows = r
    for _ in range(args.warmup):
        one_pass()
    t0 = time.perf_counter()
    vox = 0
    for _ in range(args.steps):
        vox += one_pass()
    el = time.perf_counter() - t0
    value = vox / el
    return {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "output voxels/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": el / args.steps * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": workload_name(args.config), "sample_rows": rows},
        "cpu_baseline": {"value": value, "unit": "output voxels/s", "cores": threads,
                         "kind": "reference",
                         "sample": "%d of 32 x-rows per layer per step, %d threads" % (rows, threads)},
        "e2e": {"value": value, "unit": "output voxels/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }


# ------------------------------------------------------------------ config 5

def run_tiled_volume(args, rank, world, dev, dist, peaks, flush):
    import torch
    import paper_1903_07525_b200 as P
    from paper_1903_07525_b200 import configs as C, tiling
    spec, store = C.config5()
    plan, _ = P.compile_network(spec, store, fixpoint=True, fuse_deconv_add=True)
    grid = P.grid_for(plan, C.VOLUME5, overlap=0)
    mine = [grid.tiles[i] for i in tiling.partition(len(grid.tiles), world, rank)]
    dt = tiling.DeviceTiler(plan, grid, dev)
    # synthetic volume slab for this rank's tiles only (seeded per x-range)
    lo, hi, olo, ohi = dt.slab_bounds(mine)
    rng = np.random.default_rng(500 + rank)
    slab = rng.uniform(0, 1, (1, 1) + tuple(b - a for a, b in zip(lo, hi))).astype(np.float32)
    dt.slab = torch.from_numpy(slab).to(dev)
    dt.out_slab = torch.empty((1, 3) + tuple(b - a for a, b in zip(olo, ohi)),
                              dtype=torch.float32, device=dev)
    dt.lo, dt.olo = lo, olo
    s = dt.runner.stream
    for _ in range(max(1, args.warmup)):
        dt.run(mine[:4])
    torch.cuda.synchronize(dev)
    if dist is not None:
        dist.barrier()
    tot = 0.0
    with ClockSampler(dev.index) as clk:
        for _ in range(args.steps):
            flush.fill_(1.0)
            torch.cuda.synchronize(dev)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(torch.cuda.current_stream(dev))
            dt.run(mine)
            e1.record(torch.cuda.current_stream(dev))
            torch.cuda.synchronize(dev)
            tot += e0.elapsed_time(e1)
    if dist is not None:
        t = torch.tensor([tot], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        tot = t.item()
    vox = int(np.prod(grid.volume_out))
    ms = tot / args.steps
    flops_patch = C.conv_flops(spec)
    return {
        "metric": METRIC, "value": vox / (ms * 1e-3), "unit": "output voxels/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic", "config": {"workload": workload_name(5), "tiles": len(grid.tiles),
                                        "patches_per_launch": dt.batch,
                                        "parallelism": "tiles/%d ranks" % world},
        "tflops": flops_patch * len(grid.tiles) / (ms * 1e-3) / 1e12,
        "gpu_launches": dt.launches_for(len(mine)) * args.steps,
        "clocks": clk.summary(),
    }


def main():
    args = parse_args()
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    if args.impl == "reference":
        res = run_reference(args, rank, world)
    else:
        res = run_b200(args, rank, world, local_rank)
    if rank == 0 and res is not None:
        print(json.dumps(res))
        sys.stdout.flush()


if __name__ == "__main__":
    main()
