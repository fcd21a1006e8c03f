# ncu --set full of each config's dominant conv (the bench roofline kernel);
# writes DRAM bytes and duration per launch to gpurun_out/ncudom/traffic.json
set -u
OUT=gpurun_out/ncudom; mkdir -p $OUT
echo "{" > $OUT/traffic.json
for cfg in 1 3 4; do
  set -- $(python tools/conv_index.py $cfg 2>/dev/null | tail -1)
  idx=$1; name=$2
  CFG=$cfg ITERS=1 timeout 600 ncu --set full --clock-control none -k regex:conv3d_tc -s $idx -c 1 -o $OUT/cfg$cfg -f python tools/cfg_launches.py > /dev/null 2>&1
  ncu -i $OUT/cfg$cfg.ncu-rep --page raw --csv > $OUT/cfg$cfg.raw.csv 2>/dev/null; rm -f $OUT/cfg$cfg.ncu-rep
  python -c "
import csv; r=list(csv.reader(open('$OUT/cfg$cfg.raw.csv'))); d=dict(zip(r[0], r[2])); u=dict(zip(r[0], r[1]))
sc={'byte':1,'Kbyte':1e3,'Mbyte':1e6,'Gbyte':1e9}
b=sum(float(d[m].replace(',',''))*sc[u[m]] for m in ('dram__bytes_read.sum','dram__bytes_write.sum'))
print('  \"cfg$cfg/$name\": %.1f,' % b)" >> $OUT/traffic.json
done
BATCH=36 ITERS=1 VXB_PDL=0 timeout 600 ncu --set full --clock-control none -k regex:conv3d_tc -s 1 -c 1 -o $OUT/cfg5 -f python tools/cfg5_patch.py > /dev/null 2>&1
ncu -i $OUT/cfg5.ncu-rep --page raw --csv > $OUT/cfg5.raw.csv 2>/dev/null
ncu -i $OUT/cfg5.ncu-rep --page details --csv > $OUT/cfg5.details.csv 2>/dev/null; rm -f $OUT/cfg5.ncu-rep
python -c "
import csv; r=list(csv.reader(open('$OUT/cfg5.raw.csv'))); d=dict(zip(r[0], r[2])); u=dict(zip(r[0], r[1]))
sc={'byte':1,'Kbyte':1e3,'Mbyte':1e6,'Gbyte':1e9}
b=sum(float(d[m].replace(',',''))*sc[u[m]] for m in ('dram__bytes_read.sum','dram__bytes_write.sum'))
print('  \"cfg5_d0_c1\": %.1f' % b)" >> $OUT/traffic.json
echo "}" >> $OUT/traffic.json
cat $OUT/traffic.json
