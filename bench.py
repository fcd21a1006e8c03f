#!/usr/bin/env python
"""Benchmark: B200 fused conv3d U-net inference vs the reference CPU engine.

Contract (one JSON line on rank 0):
  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl b200|reference]

Headline (default, --config 5): BASELINE configs[4], the anisotropic
residual U-net over the synthetic 128x1024x1024 volume, tiled into the
reference's (8, 6, 6) grid of 18x192x192 patches (overlap 0).  One step =
the whole volume.  ``value`` = output voxels/s with the volume resident in
HBM (device-timed, max over ranks); ``e2e`` = the same through the public
``run_tiled`` with the host volume in page-locked memory and the result read
back into a page-locked host volume (row-streamed H2D / D2H inside the timed
region).  Under torchrun (N > 1) ranks take contiguous blocks of tiles
(strong scaling, no collective on the data path) and rank 0 gathers the
output volume over NCCL afterwards (timed separately: ``gather_ms``).
``bench.py --gpus N`` without torchrun re-launches itself under torchrun.

At N = 1 the line also carries ``configs``: configs 1-4 (single fused
layer, featuremap sweep, residual block, Cicek U-net), each with its own
value, roofline, e2e and cpu_baseline, and ``x3``: config 5 on the
fp32-grade split-bf16 backend.

Timing rules: W >= 3 warm-up steps; the L2 (126 MB) is flushed with a 512 MB
write before every timed step, outside the timed window; CUDA events on the
launching streams; nvidia-smi clocks sampled during the timed region.
``roofline`` = the dominant conv kernel, timed live by external CUDA events
captured around its launch in the runner's graph (every timed step).
``cpu_baseline`` / ``--impl reference`` = the reference engine itself
(oracle/_ref: voxplan.run_tiled / PlanRunner(backend="compiled")) on the
host cores, on a bounded sample.
"""

from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "output voxels/sec for 3D U-net inference; conv3d TFLOP/s vs tensor-core peak"
DATA = ("synthetic: seeded U[0,1) / U[-1,1) volumes (BASELINE.json shapes and "
        "distributions), He-normal weights, BN statistics calibrated (config 5)")


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=5, choices=[1, 2, 3, 4, 5])
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--backend", default="b200", choices=["b200", "b200-x3"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-subconfigs", action="store_true",
                    help="config 5 only (skip the configs 1-4 sub-lines and x3)")
    ap.add_argument("--cpu-seconds", type=float, default=10.0,
                    help="target CPU-baseline sample duration per config")
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


def cpu_threads():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


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
        t0 = time.time()
        while not self.lines and time.time() - t0 < 5.0 and self.proc.poll() is None:
            time.sleep(0.01)
        self.skip = len(self.lines)
        return self

    def __exit__(self, *a):
        if self.proc is not None:
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
        for line in self.lines:
            parts = [p.strip() for p in line.split(",")]
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


# ------------------------------------------------------------------ algorithmic work

def op_work(plan, storage_bytes=2):
    """Per plan step: (name, kind, flops, bytes) at the plan's batch.
    FLOPs = 2 x MACs of the reference arithmetic; bytes = the step's input
    and output tensors (and residual operand) once each at the storage
    width (no halo re-reads, no padding lanes); a network output
    is written as fp32 by the producing conv's epilogue (4 B)."""
    from paper_1903_07525_b200.formats import ROLE_KERNEL
    from paper_1903_07525_b200.netspec import LayerKind
    out_bids = {bid for _, bid, _ in plan.outputs}
    out = []
    for st in plan.steps:
        if st.kind is LayerKind.PAD:
            continue                  # virtual on the device (TMA zero fill)
        d_out = tuple(st.output.dims)
        n, co = d_out[0], d_out[1]
        vox_out = int(np.prod(d_out[2:]))
        ins = [tuple(si.dims) for si in st.inputs]
        in_elems = sum(d[0] * d[1] * int(np.prod(d[2:])) for d in ins)
        if st.kind is LayerKind.CONVOLUTION:
            k = plan.weights.tensor(st.name, ROLE_KERNEL).shape
            f = 2.0 * float(np.prod(k)) * n * vox_out
        elif st.kind is LayerKind.DECONVOLUTION:
            k = plan.weights.tensor(st.name, ROLE_KERNEL).shape
            vin = int(np.prod(ins[0][2:]))
            f = 2.0 * float(np.prod(k)) * n * vin
        else:
            f = 0.0
        out_b = 4 if (st.output.buffer in out_bids and st.kind in (
            LayerKind.CONVOLUTION, LayerKind.DECONVOLUTION)) else storage_bytes
        b = storage_bytes * in_elems + out_b * n * co * vox_out
        if st.additive and st.base is not None:
            b += storage_bytes * n * co * vox_out
        out.append((st.name, st.kind, f, float(b)))
    return out


def roof_of(flops, nbytes, ms, peaks, peak_key):
    """Roofline dict for one kernel: tensor-bound when its arithmetic
    intensity is past the ridge of the chosen peak."""
    peak_tc = peaks[peak_key]
    ridge = peak_tc * 1e12 / (peaks["hbm"] * 1e9)
    if flops / max(nbytes, 1.0) >= ridge:
        ach = flops / (ms * 1e-3) / 1e12
        return {"bound": "tensor", "achieved": ach, "peak": peak_tc, "unit": "TFLOP/s",
                "frac": ach / peak_tc}
    ach = nbytes / (ms * 1e-3) / 1e9
    return {"bound": "hbm", "achieved": ach, "peak": peaks["hbm"], "unit": "GB/s",
            "frac": ach / peaks["hbm"]}


def network_roofline(work, ms, peaks, peak_key, repeat=1):
    """sum_l max(F_l / P, B_l / BW) / T (SURVEY §8d per-network roofline)."""
    t = sum(max(f / (peaks[peak_key] * 1e12), b / (peaks["hbm"] * 1e9)) for _, _, f, b in work)
    t *= repeat
    return {"frac": t / (ms * 1e-3), "roofline_ms": t * 1e3,
            "peak_tflops": peaks[peak_key], "peak_hbm_gbs": peaks["hbm"]}


def ncu_traffic(name):
    """dram bytes per launch from a committed ncu --set full capture, if any."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as fh:
            return json.load(fh).get(name)
    except Exception:
        return None


# ------------------------------------------------------------------ reference CPU arm

def ref_volume_sample(spec, store, threads, patch=None):
    """The reference engine on `threads` config-5 tiles: voxplan.run_tiled
    (tiling.py:189-237, backend "compiled", workers = threads) over a
    (1, 1, 18, 192, 192 * threads) slice of the synthetic volume (overlap 0:
    exactly `threads` disjoint 18x192x192 tiles, each costing what a tile of
    the full 288-tile grid costs).  ``patch``: the same U-net compiled for a
    smaller patch (the engine's per-voxel rate does not depend on the patch:
    0.076 / 0.081 / 0.077 M voxels/s single-threaded at 18x192x192 /
    18x192x96 / 18x96x96).  Returns (run, voxels per run, tiles)."""
    from oracle import ref_voxplan as RV
    if patch is not None:
        from paper_1903_07525_b200 import configs as C
        spec, store = C.config5(patch=tuple(patch))
    plan = RV.compile_reference(spec, store)
    patch = spec.input_layers()[0].params["shape"][2:]
    vol = np.random.default_rng(77).uniform(
        0, 1, (1, 1, patch[0], patch[1], patch[2] * threads)).astype(np.float32)

    def run():
        RV.run_tiled(plan, vol, workers=threads)
    return run, threads * int(np.prod(patch)), threads


def ref_network_sample(spec, store, x, threads):
    """The reference engine's PlanRunner(plan, "compiled") (executor.py:51-198)
    on `threads` independent copies of the volume, one runner per host
    thread (the reference's only parallelism: independent volumes/patches per
    worker, tiling.py:211-225).  Returns (run, output voxels per run)."""
    import psutil
    from concurrent.futures import ThreadPoolExecutor
    from oracle import ref_voxplan as RV
    V = RV.voxplan()
    plan = RV.compile_reference(spec, store)
    arena = plan.arena_bytes
    avail = psutil.virtual_memory().available
    n = max(1, min(threads, int(avail * 0.5 // max(arena, 1))))
    runners = [V.PlanRunner(plan, backend="compiled") for _ in range(n)]
    pool = ThreadPoolExecutor(max_workers=n)
    from bench_util import output_voxels
    vox = output_voxels(spec)

    def run():
        list(pool.map(lambda r: r.run(x), runners))
    return run, vox * n, n


def ref_sweep_sample(work, threads, target_s):
    """Config 2: the reference's compiled _kernels.conv3d (oracle/_ref) on
    x-slabs of each layer across the host threads (round-1 arm)."""
    from concurrent.futures import ThreadPoolExecutor
    from oracle import ref_engine as E
    from paper_1903_07525_b200.formats import ROLE_BIAS, ROLE_KERNEL
    if not E.available():
        return None
    items = []
    for name, spec, store, _ in work:
        lay = [layer for layer in spec.layers if layer.kind.value == "Convolution"][0]
        act = [layer for layer in spec.layers if layer.kind.value in ("ReLU", "ELU", "Sigmoid")]
        kind = act[0].kind.value.lower() if act else None
        stp = E.ConvStep(store.tensor(lay.name, ROLE_KERNEL), store.tensor(lay.name, ROLE_BIAS),
                         pad=lay.params["pad"], act=kind)
        shape = spec.input_layers()[0].params["shape"]
        x = np.random.default_rng(7).uniform(-1, 1, shape).astype(np.float32)
        xb = stp.prepare(x)
        ox = shape[2]
        out = np.zeros((1, -(-stp.fo // 8), ox) + tuple(shape[3:]) + (8,), np.float32)
        items.append({"step": stp, "xb": xb, "out": out, "ox": ox,
                      "vox_per_row": int(np.prod(shape[3:]))})
    t0 = time.perf_counter()
    for it in items:
        it["step"].run_blocked(it["xb"], it["out"], None, (0, 1))
    one_row_all = time.perf_counter() - t0
    rows = max(1, min(items[0]["ox"], int(target_s * threads / max(one_row_all, 1e-6))))
    rows = max(threads, (rows // threads) * threads) if rows >= threads else rows
    rows = min(rows, items[0]["ox"])
    pool = ThreadPoolExecutor(max_workers=threads)

    def run():
        for it in items:
            cuts = np.linspace(0, rows, min(threads, rows) + 1).astype(int)
            list(pool.map(lambda i: it["step"].run_blocked(it["xb"], it["out"], None,
                                                          (cuts[i], cuts[i + 1])),
                          range(len(cuts) - 1)))
    return run, rows * sum(it["vox_per_row"] for it in items), rows


def timed_passes(run, min_s, max_passes=100):
    t0 = time.perf_counter()
    n = 0
    while True:
        run()
        n += 1
        el = time.perf_counter() - t0
        if el >= min_s or n >= max_passes:
            return n, el


def cpu_baseline(cfg, nets, target_s):
    """The reference engine on this box's host cores, bounded sample."""
    threads = cpu_threads()
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    try:
        if cfg == 5:
            spec, store = nets[0][1], nets[0][2]
            run, vox, tiles = ref_volume_sample(spec, store, threads)
            passes, el = timed_passes(run, min(target_s, 1.0))
            return {"value": vox * passes / el, "unit": "output voxels/s", "cores": threads,
                    "kind": "reference",
                    "sample": "%d pass(es) of %d config-5 tiles through voxplan.run_tiled("
                              "backend='compiled', workers=%d) (oracle/_ref), %.1f s; the "
                              "288-tile volume rate is the same per tile" %
                              (passes, tiles, threads, el)}
        if cfg == 2:
            r = ref_sweep_sample(nets, threads, target_s)
            if r is None:
                raise RuntimeError("oracle/_ref not built")
            run, vox, rows = r
            passes, el = timed_passes(run, min(target_s, 10.0))
            return {"value": vox * passes / el, "unit": "output voxels/s", "cores": threads,
                    "kind": "reference",
                    "sample": "%d pass(es) over %d of 32 x-rows of every config-2 layer, the "
                              "reference's _kernels.conv3d (oracle/_ref) on x-slabs, %d threads, "
                              "%.1f s" % (passes, rows, threads, el)}
        name, spec, store, x = nets[0]
        run, vox, n = ref_network_sample(spec, store, x, threads)
        passes, el = timed_passes(run, min(target_s, 3.0))
        return {"value": vox * passes / el, "unit": "output voxels/s", "cores": n,
                "kind": "reference",
                "sample": "%d pass(es) of %d concurrent volumes, one voxplan.PlanRunner(plan, "
                          "'compiled') per thread (oracle/_ref), %.1f s" % (passes, n, el)}
    except Exception as exc:  # the baseline is reported, not required
        return {"value": None, "unit": "output voxels/s", "cores": threads, "kind": "reference",
                "sample": "unavailable: %s" % exc}


def run_reference(args, rank, world):
    """--impl reference: the reference's own CPU engine on the host cores,
    on the same config / metric; each step a bounded sample."""
    if world > 1 and rank != 0:
        return None
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    threads = cpu_threads()
    from bench_util import build_nets, workload_name
    nets = build_nets(args.config)
    if args.config == 5:
        # a full 18x192x192 tile takes ~14 s per worker on the GPU hosts; with
        # more than a handful of steps each worker takes an 18x96x96 quarter
        # patch per step instead, so the whole arm stays within a few minutes
        quarter = (args.steps + args.warmup) > 8
        run, vox, tiles = ref_volume_sample(nets[0][1], nets[0][2], threads,
                                            patch=(18, 96, 96) if quarter else None)
        sample = ("%d %s per step (one per worker) through voxplan.run_tiled(backend="
                  "'compiled', workers=%d), oracle/_ref%s" % (
                      tiles, "18x96x96 quarter patches" if quarter else "18x192x192 tiles",
                      threads, "; the same network per voxel (single-threaded 0.077 vs "
                      "0.076 M vox/s at 18x96x96 vs 18x192x192), but with every core busy the "
                      "engine runs ~1.5x faster per voxel on quarter patches (cache locality), "
                      "so this sample favours the reference" if quarter else ""))
    elif args.config == 2:
        r = ref_sweep_sample(nets, threads, min(8.0, args.cpu_seconds))
        if r is None:
            return {"impl": "reference", "metric": METRIC,
                    "unavailable": "oracle/_ref not built"}
        run, vox, rows = r
        sample = "%d of 32 x-rows of every sweep layer per step, %d threads" % (rows, threads)
    else:
        name, spec, store, x = nets[0]
        run, vox, n = ref_network_sample(spec, store, x, threads)
        threads = n
        sample = "%d concurrent volumes per step, one voxplan.PlanRunner per thread" % n
    for _ in range(args.warmup):
        run()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        run()
    el = time.perf_counter() - t0
    value = vox * args.steps / el
    return {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "output voxels/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": el / args.steps * 1e3, "higher_is_better": True,
        "scaling": "strong" if args.config == 5 else "weak", "vs_baseline": None,
        "dtype": "f32", "data": DATA,
        "config": {"workload": workload_name(args.config), "sample": sample},
        "cpu_baseline": {"value": value, "unit": "output voxels/s", "cores": threads,
                         "kind": "reference", "sample": sample},
        "e2e": {"value": value, "unit": "output voxels/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }


# ------------------------------------------------------------------ B200 arm

def run_b200(args, rank, world, local_rank):
    import torch
    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    peaks = load_peaks()
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    import bench_util as U
    if args.config == 5:
        res = U.bench_volume(args, rank, world, dev, dist, peaks, flush, backend=args.backend)
        if rank == 0 and world == 1 and not args.no_subconfigs:
            sub = {}
            for c in (1, 2, 3, 4):
                sub["config%d" % c] = U.bench_network(c, args, dev, peaks, flush,
                                                      with_cpu=not args.no_cpu_baseline,
                                                      with_e2e=not args.no_e2e,
                                                      cpu_fn=cpu_baseline)
            res["configs"] = sub
            if args.backend == "b200":
                res["x3"] = U.bench_volume(args, rank, world, dev, None, peaks, flush,
                                           backend="b200-x3", light=True)
        if rank == 0 and world == 1 and not args.no_cpu_baseline:
            res["cpu_baseline"] = cpu_baseline(5, U.build_nets(5), args.cpu_seconds)
    else:
        res = U.bench_network(args.config, args, dev, peaks, flush,
                              with_cpu=(rank == 0 and world == 1 and not args.no_cpu_baseline),
                              with_e2e=not args.no_e2e, headline=True, world=world, dist=dist,
                              cpu_fn=cpu_baseline)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()
    return res


def spawn(args):
    """bench.py --gpus N without torchrun: re-launch under torchrun, one
    rank per GPU (127.0.0.1 rendezvous), and pass rank 0's line through."""
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           "--nproc-per-node", str(args.gpus), "--master-addr", "127.0.0.1",
           "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    args = parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn(args))
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
