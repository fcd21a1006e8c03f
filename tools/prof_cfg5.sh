set -u
OUT=gpurun_out/prof2; mkdir -p $OUT
BATCH=4 VXB_PRINT=1 timeout 300 python tools/cfg5_patch.py > $OUT/cfg5_b4_ops.txt 2>&1; echo "cfg5 rc=$?"
BATCH=1 timeout 300 python tools/cfg5_patch.py > $OUT/cfg5_b1_ops.txt 2>&1; echo "cfg5 b1 rc=$?"
BATCH=4 ITERS=1 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $OUT/launches_cfg5_b4.csv python tools/cfg5_patch.py > /dev/null 2>&1; echo "launches rc=$?"
BATCH=4 ITERS=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:conv3d_tc -s 1 -c 1 -o $OUT/ncu_cfg5_d0_c1 -f python tools/cfg5_patch.py > /dev/null 2>&1; echo "full rc=$?"
