# ncu --set full of kbench layers (kernel alone), text summaries only
OUT=gpurun_out/ncukb; mkdir -p $OUT
for L in ${LAYERS:-c64_k133 c32_k333}; do
  ONLY=$L REPS=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:conv3d_tc -s 3 -c 1 -o $OUT/$L -f python tools/kbench.py > /dev/null 2>&1; echo "$L rc=$?"
  ncu -i $OUT/$L.ncu-rep --page raw --csv > $OUT/$L.raw.csv 2>/dev/null
  ncu -i $OUT/$L.ncu-rep --page details --csv > $OUT/$L.details.csv 2>/dev/null
  rm -f $OUT/$L.ncu-rep
done
