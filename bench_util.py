"""GPU-side measurement helpers of bench.py (device timing, rooflines, e2e).

Nothing here touches oracle/: the CPU reference arm lives in bench.py.
"""

from __future__ import annotations

import json
import os
import time

import numpy as np

from bench import METRIC, DATA, ClockSampler, network_roofline, ncu_traffic, op_work, roof_of

ROOT = os.path.dirname(os.path.abspath(__file__))


def workload_name(cfg):
    return {1: "config1: conv3d 3x3x3 C16->16 + bias + ReLU, 1x16x32x64x64 (BASELINE configs[0])",
            2: "config2: featuremap sweep C in {8..128} x k in {3x3x3, 1x3x3}, conv + bias + "
               "ELU on 1xCx32x128x128 (BASELINE configs[1])",
            3: "config3: residual block C64 on 1x64x24x128x128 (BASELINE configs[2])",
            4: "config4: Cicek 3D U-net 132^3 -> 3x44^3 (BASELINE configs[3])",
            5: "config5: anisotropic residual U-net, 128x1024x1024 volume, 288 tiles of "
               "18x192x192 (BASELINE configs[4])"}[cfg]


def build_nets(cfg):
    """[(name, spec, store, input)] of a config (config 2: its 10 layers)."""
    from paper_1903_07525_b200 import configs as C
    lo, hi = C.input_range(cfg)
    if cfg == 2:
        out = []
        for k in C.SWEEP_K:
            for c in C.SWEEP_C:
                spec, store = C.config2(c, k)
                out.append(("c%d_k%s" % (c, "".join(map(str, k))), spec, store))
    else:
        spec, store = {1: C.config1, 3: C.config3, 4: C.config4, 5: C.config5}[cfg]()
        out = [("cfg%d" % cfg, spec, store)]
    return [(n, s, st, C.make_input(s, 100 + i, lo, hi)) for i, (n, s, st) in enumerate(out)]


def output_voxels(spec):
    from paper_1903_07525_b200.shapes import validate_shapes
    shapes = validate_shapes(spec)
    total = 0
    for blob in spec.output_blobs():
        n, _, x, y, z = shapes[blob]
        total += n * x * y * z
    return total


def _dominant(plan):
    """(name, flops, bytes) of the plan's largest conv (by FLOPs)."""
    from paper_1903_07525_b200.netspec import LayerKind
    best = None
    for name, kind, f, b in op_work(plan):
        if kind is LayerKind.CONVOLUTION and (best is None or f > best[1]):
            best = (name, f, b)
    return best


def _sync_barrier(dev, dist):
    import torch
    torch.cuda.synchronize(dev)
    if dist is not None:
        dist.barrier()


def _max_over_ranks(v, dev, dist):
    if dist is None:
        return v
    import torch
    t = torch.tensor([v], device=dev, dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def _parity(name, backend):
    try:
        with open(os.path.join(ROOT, "profiles", "r02_parity.json")) as fh:
            r = json.load(fh)[name][backend]
        return {"max_norm": r["max_norm"], "l2": r["l2"],
                "source": "profiles/r02_parity.json (tests/parity_report.py vs ref_run)"}
    except Exception:
        return None


# ------------------------------------------------------------------ config 5 volume

def bench_volume(args, rank, world, dev, dist, peaks, flush, backend="b200", light=False):
    """Config 5: the 128x1024x1024 volume through DeviceTiler (resident) and
    run_tiled (host volume in / out, e2e)."""
    import torch
    import paper_1903_07525_b200 as P
    from paper_1903_07525_b200 import configs as C, staging, tiling
    spec, store = C.config5()
    plan, _ = P.compile_network(spec, store, fixpoint=True, fuse_deconv_add=True)
    grid = P.grid_for(plan, C.VOLUME5, overlap=0)
    mine = [grid.tiles[i] for i in tiling.partition(len(grid.tiles), world, rank)]
    dom = _dominant(plan)
    dt = tiling.DeviceTiler(plan, grid, dev, backend=backend, probe=dom[0])
    # the synthetic volume (seeded; every rank holds the same one)
    vol = staging.pinned_empty((1, 1) + tuple(C.VOLUME5))
    rng = np.random.default_rng(500)
    for x0 in range(0, C.VOLUME5[0], 16):
        vol[0, 0, x0:x0 + 16] = rng.uniform(0, 1, (min(16, C.VOLUME5[0] - x0),) +
                                            tuple(C.VOLUME5[1:])).astype(np.float32)
    lo, hi, olo, ohi = dt.slab_bounds(mine)
    with torch.cuda.device(dev):
        slab = torch.from_numpy(vol)[(slice(None), slice(None)) +
                                     tuple(slice(a, b) for a, b in zip(lo, hi))].to(dev)
        out_slab = torch.empty((1, dt.out_fmaps) + tuple(b - a for a, b in zip(olo, ohi)),
                               dtype=torch.float32, device=dev)
    dt.bind_slabs(slab, lo, out_slab, olo)
    steps = args.steps if not light else max(1, min(args.steps, 5))
    for _ in range(max(3, args.warmup) if not light else 1):
        dt.run(mine)
    _sync_barrier(dev, dist)
    tot, probe = 0.0, []
    cs = torch.cuda.current_stream(dev)
    with ClockSampler(dev.index) as clk:
        for _ in range(steps):
            flush.fill_(1.0)                       # L2 flush, outside the timed window
            _sync_barrier(dev, dist)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(cs)
            dt.run(mine)
            e1.record(cs)
            torch.cuda.synchronize(dev)
            tot += e0.elapsed_time(e1)
            probe.append(dt.runner.probe_ms())     # the dominant conv, last replay of the step
    tot = _max_over_ranks(tot, dev, dist)
    ms = tot / steps
    vox = int(np.prod(grid.volume_out))
    flops_tile = sum(f for _, _, f, _ in op_work(plan))
    res = {
        "metric": METRIC, "value": vox / (ms * 1e-3), "unit": "output voxels/s",
        "n_gpus": world, "steps": steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "bf16" if backend == "b200" else "bf16x3 (split-bf16 storage, 3 bf16 MMAs)",
        "data": DATA,
        "config": {"workload": workload_name(5), "backend": backend,
                   "tiles": len(grid.tiles), "tiles_this_rank": len(mine),
                   "patches_per_launch": dt.batch, "streams": len(dt.runners),
                   "parallelism": "tiles/%d ranks (contiguous blocks, no collective)" % world,
                   "l2": "flushed (512 MB write) before every step, outside the timed region",
                   "inputs": "volume slab resident in HBM before the timed region"},
        "tflops": flops_tile * len(grid.tiles) / (ms * 1e-3) / 1e12,
        "gpu_launches": dt.launches_for(len(mine)) * steps,
        "clocks": clk.summary(),
    }
    if light:
        res["parity"] = _parity("cfg5", backend)
        return {k: res[k] for k in ("value", "unit", "ms_per_step", "steps", "tflops", "dtype",
                                    "parity", "clocks")}
    # ---- roofline of the dominant conv, timed live inside the steps
    bwork = op_work(dt.runner.plan)
    dname, dflops, dbytes = [(n, f, b) for n, _, f, b in bwork if n == dom[0]][0]
    pms = statistics_mean(probe)
    roof = roof_of(dflops, dbytes, pms, peaks, "bf16_sustained")
    roof.update({"kernel": "conv3d_tc_kernel (config5 %s, %d patches per launch)" %
                           (dname, dt.batch),
                 "ms_per_launch": pms, "alg_flops": dflops, "alg_bytes": dbytes,
                 "timing": "in-step: external CUDA events captured around the launch in the "
                           "runner's graph; last replay of every timed step (%d samples)" % steps,
                 "peak_source": peaks["source"] + ", sustained (kernel inside a long step)",
                 "traffic": ncu_traffic("cfg5_" + dname)})
    res["roofline"] = roof
    res["network_roofline"] = network_roofline(op_work(plan), ms, peaks, "bf16_sustained",
                                               repeat=len(grid.tiles))
    res["parity"] = _parity("cfg5", backend)
    # ---- end to end through the public API (host volume in, host volume out)
    if not args.no_e2e:
        out = staging.pinned_empty((1, dt.out_fmaps) + tuple(grid.volume_out))
        if world == 1:
            run = lambda: P.run_tiled(plan, vol, grid=grid, devices=[dev], out=out,  # noqa: E731
                                      backend=backend)
        else:
            run = lambda: dt.run_host(vol, out, mine)  # noqa: E731
        run()
        _sync_barrier(dev, dist)
        n_e2e = max(1, min(steps, 3))
        t0 = time.perf_counter()
        for _ in range(n_e2e):
            run()
        el = _max_over_ranks(time.perf_counter() - t0, dev, dist)
        h2d = sum(int(np.prod([b - a for a, b in zip(*dt.slab_bounds(r)[:2])])) * 4
                  for r in dt.rows(mine))
        d2h = sum(int(np.prod([b - a for a, b in zip(*dt.slab_bounds(r)[2:])])) * 4 *
                  dt.out_fmaps for r in dt.rows(mine))
        res["e2e"] = {"value": vox * n_e2e / el, "unit": "output voxels/s",
                      "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "steps": n_e2e,
                      "timer": "host wall clock around run_tiled(plan, host volume, out=host "
                               "volume): x-rows streamed H2D / computed / D2H on separate "
                               "streams, page-locked host arrays"}
    # ---- final gather of the output volume to rank 0 (NCCL), multi-GPU
    if dist is not None:
        res["gather_ms"] = gather_volume(dt, mine, grid, dev, dist, rank, world)
    return res


def statistics_mean(v):
    return float(sum(v) / max(1, len(v)))


def gather_volume(dt, mine, grid, dev, dist, rank, world):
    """Rank 0 receives every rank's output slab into one device volume over
    NCCL (tiling.gather_volume, point-to-point); max-over-ranks device time
    in ms."""
    import torch
    from paper_1903_07525_b200 import tiling
    _sync_barrier(dev, dist)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    cs = torch.cuda.current_stream(dev)
    e0.record(cs)
    tiling.gather_volume(dt.out_slab, grid, rank, world, dist)
    e1.record(cs)
    torch.cuda.synchronize(dev)
    return _max_over_ranks(e0.elapsed_time(e1), dev, dist)


# ------------------------------------------------------------------ configs 1-4

def bench_network(cfg, args, dev, peaks, flush, *, with_cpu, with_e2e, headline=False, world=1,
                  dist=None, cpu_fn=None):
    """Configs 1-4: every network resident in HBM, one CUDA graph per step
    (config 2: the 10 sweep layers as one PlanBatch graph)."""
    import torch
    import paper_1903_07525_b200 as P
    nets = build_nets(cfg)
    runners, plans, probed = [], [], []
    for name, spec, store, x in nets:
        plan, _ = P.compile_network(spec, store, fixpoint=True, fuse_deconv_add=True)
        plans.append(plan)
        r = P.PlanRunner(plan, backend="b200", device=dev)
        r.input_buffers()[plan.inputs[0][0]].copy_(torch.from_numpy(x))
        runners.append(r)
        if cfg != 2:
            # the same plan with external timing events around its dominant
            # conv: the event nodes split the graph (config 1: 20 -> 35 us per
            # step), so `value` is timed on the plain runner and the roofline
            # kernel in a second pass of probed steps
            rp = P.PlanRunner(plan, backend="b200", device=dev, probe=_dominant(plan)[0])
            rp.input_buffers()[plan.inputs[0][0]].copy_(torch.from_numpy(x))
            probed.append(rp)
    batch = batch_probe = None
    if cfg == 2:
        doms = [(_dominant(p)[1], i) for i, p in enumerate(plans)]
        dom_i = max(doms)[1]
        batch = P.PlanBatch(runners)
        batch_probe = P.PlanBatch(runners, probe=dom_i)
    steps = args.steps if headline else max(3, min(args.steps, 20))
    cs = torch.cuda.current_stream(dev)

    def step(with_probe=False):
        if batch is not None:
            (batch_probe if with_probe else batch).run_device()
        else:
            r = probed[0] if with_probe else runners[0]
            r.run_device(r.input_buffers())

    def timed(with_probe):
        for _ in range(max(3, args.warmup)):
            step(with_probe)
        _sync_barrier(dev, dist)
        tot, probe = 0.0, []
        with ClockSampler(dev.index) as clk:
            for _ in range(steps):
                flush.fill_(1.0)
                _sync_barrier(dev, dist)
                torch.cuda._sleep(200_000)               # keep the window device-bound
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record(cs)
                step(with_probe)
                e1.record(cs)
                torch.cuda.synchronize(dev)
                tot += e0.elapsed_time(e1)
                if with_probe:
                    probe.append(batch_probe.probe_ms() if batch is not None
                                 else probed[0].probe_ms())
        return tot, probe, clk

    tot, _, clk = timed(False)
    tot_probed, probe, _ = timed(True)
    tot = _max_over_ranks(tot, dev, dist)
    ms = tot / steps
    vox = sum(output_voxels(s) for _, s, _, _ in nets)
    flops = sum(sum(f for _, _, f, _ in op_work(p)) for p in plans)
    # dominant conv: live per-step timing (probe) and its algorithmic work
    if batch is not None:
        dplan = plans[dom_i]
        dname = nets[dom_i][0]
    else:
        dplan = plans[0]
        dname = "cfg%d" % cfg
    dn, df, db = _dominant(dplan)
    pms = statistics_mean(probe)
    roof = roof_of(df, db, pms, peaks, "bf16")
    roof.update({"kernel": "conv3d_tc_kernel (%s/%s)" % (dname, dn), "ms_per_launch": pms,
                 "alg_flops": df, "alg_bytes": db,
                 "timing": "in-step: external CUDA events captured around the launch in the "
                           "graph, in a second pass of %d flushed steps (%.4f ms per step with "
                           "the event nodes; `value` is timed on the same graph without "
                           "them)" % (steps, tot_probed / steps),
                 "peak_source": peaks["source"] + ", burst",
                 "traffic": ncu_traffic("%s/%s" % (dname, dn)) or ncu_traffic(dname)})
    res = {"value": vox * world / (ms * 1e-3), "unit": "output voxels/s", "ms_per_step": ms,
           "steps": steps, "tflops": flops * world / (ms * 1e-3) / 1e12,
           "workload": workload_name(cfg), "roofline": roof,
           "network_roofline": network_roofline(
               [w for p in plans for w in op_work(p)], ms, peaks, "bf16"),
           "gpu_launches": sum(r.launches for r in runners) * steps,
           "clocks": clk.summary(), "parity": _parity("cfg%d" % cfg if cfg != 2 else
                                                      "cfg2_c128_k333", "b200")}
    if cfg == 2:
        res["layers"] = sweep_layers(nets, plans, dev, peaks, flush)
    if with_e2e:
        res["e2e"] = e2e_runners(runners, nets, steps, dev, dist, world)
    if with_cpu and cpu_fn is not None:
        res["cpu_baseline"] = cpu_fn(cfg, nets, args.cpu_seconds)
    if headline:
        res.update({"metric": METRIC, "n_gpus": world, "warmup": args.warmup,
                    "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
                    "dtype": "bf16", "data": DATA,
                    "config": {"workload": workload_name(cfg),
                               "parallelism": "replicas" if world > 1 else "single",
                               "l2": "flushed (512 MB write) before every step, outside the "
                                     "timed region"}})
        res["metric"] = METRIC
    return res


def sweep_layers(nets, plans, dev, peaks, flush, reps=8):
    """Config 2, layer by layer: each network (input pack + conv) replayed
    alone after an L2 flush, its conv timed by external events inside the
    graph; roofline fraction of every layer (tensor or HBM bound)."""
    import torch
    import paper_1903_07525_b200 as P
    out = []
    cs = torch.cuda.current_stream(dev)
    for (name, _, _, x), plan in zip(nets, plans):
        dn, df, db = _dominant(plan)
        r = P.PlanRunner(plan, backend="b200", device=dev, probe=dn)
        r.input_buffers()[plan.inputs[0][0]].copy_(torch.from_numpy(x))
        for _ in range(3):
            r.run_device(r.input_buffers())
        torch.cuda.synchronize(dev)
        t = []
        for _ in range(reps):
            flush.fill_(1.0)
            torch.cuda.synchronize(dev)
            torch.cuda._sleep(200_000)
            r.run_device(r.input_buffers())
            cs.synchronize()
            torch.cuda.synchronize(dev)
            t.append(r.probe_ms())
        ms = float(np.median(t))
        roof = roof_of(df, db, ms, peaks, "bf16")
        out.append({"layer": name, "us": ms * 1e3, "bound": roof["bound"],
                    "achieved": roof["achieved"], "unit": roof["unit"], "frac": roof["frac"]})
        del r
    return out


def e2e_runners(runners, nets, steps, dev, dist, world):
    """The metric through the public host API: PlanRunner.run_async with
    page-locked host input and output arrays (H2D, graph replay, D2H)."""
    import torch
    from paper_1903_07525_b200 import staging
    items = []
    for r, (_, spec, _, x) in zip(runners, nets):
        xp = staging.pinned_empty(x.shape)
        xp[...] = x
        outp = {n: staging.pinned_empty(t.shape) for n, t in r._out_std.items()}
        r.run(xp, out=outp)
        items.append((r, xp, outp))
    torch.cuda.synchronize(dev)
    if dist is not None:
        dist.barrier()
    n = max(1, min(steps, 5))
    t0 = time.perf_counter()
    pend = []
    for _ in range(n):
        pend += [r.run_async(xp, out=outp) for r, xp, outp in items]
    for h in pend:
        h.wait()
    torch.cuda.synchronize(dev)
    el = _max_over_ranks(time.perf_counter() - t0, dev, dist)
    vox = sum(output_voxels(s) for _, s, _, _ in nets)
    return {"value": vox * world * n / el, "unit": "output voxels/s",
            "h2d_bytes_per_step": sum(r.h2d_bytes for r in runners),
            "d2h_bytes_per_step": sum(r.d2h_bytes for r in runners), "steps": n,
            "timer": "host wall clock around PlanRunner.run_async + wait (H2D from page-locked "
                     "host input, graph replay, D2H into page-locked host output; networks "
                     "pipelined across streams)"}
