# config-5 launch lists (batch 12) under conv debug modes (timing only: results are wrong)
set -u
OUT=gpurun_out/dbg; mkdir -p $OUT
for m in ${MODES:-0 256 512 1}; do
  VXB_TC_DBGMODE=$m BATCH=12 ITERS=1 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $OUT/launches_$m.csv python tools/cfg5_patch.py > /dev/null 2>&1; echo "mode $m rc=$?"
done
