"""Turn a profiles/run_profiles.sh capture (gpurun_out/prof) into the
tracked round summaries under profiles/.  Usage: python profiles/summarize.py r01"""
import csv
import json
import os
import re
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "gpurun_out", "prof")
DST = os.path.join(ROOT, "profiles")
TAG = sys.argv[1] if len(sys.argv) > 1 else "r01"

METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "sm__cycles_elapsed.avg", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32_sparsity_off.avg.pct_of_peak_sustained_elapsed",
    "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum",
    "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
    "launch__shared_mem_per_block_dynamic", "smsp__inst_executed.sum",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
]
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "usecond": 1e-6, "us": 1e-6,
        "nsecond": 1e-9, "ns": 1e-9, "msecond": 1e-3}


def ncu_raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, u, v = rows[0], rows[1], rows[2]
    res = {"kernel": v[h.index("Kernel Name")]}
    for m in METRICS:
        if m in h:
            i = h.index(m)
            try:
                val = float(v[i].replace(",", ""))
            except ValueError:
                continue
            res[m] = {"value": val, "unit": u[i]}
    return res


def to_bytes(e):
    return e["value"] * UNIT.get(e["unit"], 1)


def launches(path):
    rows = list(csv.reader(open(path)))
    i = [k for k, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[i]
    ki, mi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    return [(r[ki].split("(")[0].replace("void ", "").replace("vxb::", ""),
             float(r[mi].replace(",", "")) * UNIT.get(r[ui], 1e-9) * 1e6) for r in rows[i + 1:]]


def main():
    summary = {}
    b = json.load(open(os.path.join(SRC, "bench.json")))
    json.dump(b, open(os.path.join(DST, "%s_bench.json" % TAG), "w"), indent=1)
    for name in ("launches_config2.csv", "launches_cfg5_patch.csv"):
        shutil.copy(os.path.join(SRC, name), os.path.join(DST, "%s_%s" % (TAG, name)))
    traffic = {}
    for layer in ("c128_k333", "c16_k333"):
        rep = os.path.join(SRC, "ncu_%s.ncu-rep" % layer)
        if os.path.exists(rep):
            r = ncu_raw(rep)
            json.dump(r, open(os.path.join(DST, "%s_ncu_%s.json" % (TAG, layer)), "w"), indent=1)
            traffic[layer] = to_bytes(r["dram__bytes_read.sum"]) + to_bytes(r["dram__bytes_write.sum"])
            summary["ncu_" + layer] = {
                "us": r["gpu__time_duration.sum"]["value"],
                "dram_bytes_per_launch": traffic[layer],
                "tensor_pipe_active_pct": r.get(
                    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", {}).get("value"),
                "smem_tc_wavefronts_pct": r.get(
                    "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
                    {}).get("value")}
    json.dump(traffic, open(os.path.join(DST, "ncu_traffic.json"), "w"), indent=1)
    # config 2 step: the last run of 10 (pack, conv) pairs = the last timed step
    # (the dominant-kernel replays that follow are conv-only)
    seq = launches(os.path.join(SRC, "launches_config2.csv"))
    step = []
    for i in range(len(seq) - 19, -1, -1):
        w = seq[i:i + 20]
        if all(w[2 * k][0].startswith("pack") and w[2 * k + 1][0].startswith("conv3d_tc")
               for k in range(10)):
            step = w
            break
    tot = sum(t for _, t in step)
    summary["config2_step_from_launch_list"] = {
        "launches": [(n, round(t, 2)) for n, t in step], "total_us": tot,
        "conv_share": sum(t for n, t in step if n.startswith("conv3d_tc")) / tot if tot else None}
    ops = [l.split()[2] for l in open(os.path.join(SRC, "cfg5_ops.txt")).read().splitlines()[1:]
           if len(l.split()) > 2]
    seq5 = launches(os.path.join(SRC, "launches_cfg5_patch.csv"))[-(len(ops) + 1):]
    summary["config5_patch_launches_us"] = [(nm, k, round(t, 1)) for nm, (k, t) in
                                            zip(["pack"] + ops, seq5)]
    summary["config5_patch_total_us"] = sum(t for _, t in seq5)
    kb = {}
    for line in open(os.path.join(SRC, "kbench.txt")):
        m = re.match(r"(c\d+_k\d+) (\{.*\})", line.strip())
        if m:
            kb[m.group(1)] = json.loads(m.group(2))
    summary["kernel_only_us_config2_layers (bf16 blocked in/out, 20 graph replays, L2 flushed)"] = kb
    summary["bench"] = {k: b.get(k) for k in ("value", "ms_per_step", "tflops", "roofline", "e2e",
                                               "cpu_baseline", "clocks", "layers")}
    json.dump(summary, open(os.path.join(DST, "%s_summary.json" % TAG), "w"), indent=1)
    print(json.dumps({k: v for k, v in summary.items() if k != "config5_patch_launches_us"},
                     indent=1)[:3000])


if __name__ == "__main__":
    main()
