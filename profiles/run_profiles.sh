#!/usr/bin/env bash
# Round profile capture (run on the GPU box via gpurun from the repo root).
# Every ncu pass runs only after the same command exited 0 without ncu.
set -u
OUT=gpurun_out/prof
mkdir -p "$OUT"
# 1. the bench line (no profiler)
timeout 900 python bench.py > "$OUT/bench.json" 2> "$OUT/bench.err"; echo "bench rc=$?"
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > "$OUT/bench_short.json" 2>/dev/null; echo "short rc=$?"
# 2. launch list of the same (short) command: per-launch durations, cold + serialised
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file "$OUT/launches_config2.csv" python bench.py --steps 2 --warmup 3 --no-cpu-baseline \
  --no-e2e > /dev/null 2>&1; echo "launches rc=$?"
# 3. full capture of the dominant kernel: c128_k333, the 2nd conv launch (PlanBatch warm-up
#    order: smallest network first, then largest-first by FLOPs; c16_k333 is the 8th)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:conv3d_tc -s 1 -c 1 \
  -o "$OUT/ncu_c128_k333" -f python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e \
  > /dev/null 2>&1; echo "full rc=$?"
# 4. one low-fmap conv (c16_k333) and the config-5 patch launch list
timeout 900 ncu --set full --clock-control none --import-source on -k regex:conv3d_tc -s 7 -c 1 \
  -o "$OUT/ncu_c16_k333" -f python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e \
  > /dev/null 2>&1; echo "full16 rc=$?"
timeout 300 python tools/cfg5_patch.py > "$OUT/cfg5_ops.txt" 2>&1
ITERS=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file "$OUT/launches_cfg5_patch.csv" python tools/cfg5_patch.py > /dev/null 2>&1; echo "cfg5 rc=$?"
REPS=20 timeout 300 python tools/kbench.py > "$OUT/kbench.txt" 2>&1; echo "kbench rc=$?"
