# full ncu captures of chosen config-5 conv launches (index among conv3d_tc launches)
set -u
OUT=gpurun_out/ncu5; mkdir -p $OUT
B=${BATCH:-12}
for spec in ${SPECS:-"30 head 2 d0_c2 27 u0_up 0 d0_c0 28 u0_c0"}; do :; done
set -- ${SPECS:-30 head 2 d0_c2 27 u0_up 0 d0_c0 28 u0_c0}
while [ $# -ge 2 ]; do
  BATCH=$B ITERS=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:conv3d_tc \
    -s $1 -c 1 -o $OUT/ncu_$2 -f python tools/cfg5_patch.py > /dev/null 2>&1; echo "full $2 rc=$?"
  shift 2
done
# text summaries (the reports themselves can exceed gpurun's 64 MiB return limit)
for f in $OUT/*.ncu-rep; do
  b=${f%.ncu-rep}
  ncu -i $f --page details --csv > $b.details.csv 2>/dev/null
  ncu -i $f --page raw --csv > $b.raw.csv 2>/dev/null
  ncu -i $f --page source --csv --print-source cuda > $b.src_cuda.csv 2>/dev/null
  ncu -i $f --page source --csv --print-source sass > $b.src_sass.csv 2>/dev/null
  [ -n "${KEEP_REP:-}" ] || rm -f $f
done
