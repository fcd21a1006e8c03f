#!/usr/bin/env bash
# Round-2 profile capture (run on the GPU box via gpurun from the repo root).
# Every ncu pass runs only after the same command exited 0 without ncu.
set -u
OUT=gpurun_out/prof2
mkdir -p "$OUT"
# config-5 batch of 4 patches (the bench's launch unit): timing + op order
BATCH=4 timeout 300 python tools/cfg5_patch.py > "$OUT/cfg5_b4_ops.txt" 2>&1; echo "cfg5 rc=$?"
# launch list of the same command (cold, serialised per-launch durations)
BATCH=4 ITERS=1 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none --csv --log-file "$OUT/launches_cfg5_b4.csv" python tools/cfg5_patch.py \
  > /dev/null 2>&1; echo "cfg5 launches rc=$?"
# full capture of the config-5 dominant conv (d0_c1 = 2nd conv launch) and two others
for spec in "1 d0_c1" "0 d0_c0" "2 d0_c2"; do
  set -- $spec
  BATCH=4 ITERS=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:conv3d_tc \
    -s $1 -c 1 -o "$OUT/ncu_cfg5_$2" -f python tools/cfg5_patch.py > /dev/null 2>&1; echo "full $2 rc=$?"
done
