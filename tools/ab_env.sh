# A/B of an env knob on the config-5 launch list (batch 12): AB="VAR=a VAR=b"
set -u
OUT=gpurun_out/ab; mkdir -p $OUT
for kv in ${AB}; do
  env $kv BATCH=12 ITERS=1 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $OUT/launches_$kv.csv python tools/cfg5_patch.py > /dev/null 2>&1; echo "$kv rc=$?"
  env $kv BATCH=12 timeout 300 python tools/cfg5_patch.py 2>&1 | grep "patch ms"
done
