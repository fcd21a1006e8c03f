# full GPU tests + config-5 patch timing + launch list (batch 12)
set -u
OUT=gpurun_out/chk; mkdir -p $OUT
timeout 1200 python -m pytest tests -m gpu -x -q > $OUT/pt.log 2>&1; echo "pytest rc=$?"; tail -3 $OUT/pt.log
BATCH=12 timeout 300 python tools/cfg5_patch.py 2>&1 | grep "patch ms"
BATCH=12 ITERS=1 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $OUT/launches.csv python tools/cfg5_patch.py > /dev/null 2>&1; echo "launches rc=$?"
[ -n "${BENCH:-}" ] && { timeout 300 python bench.py --config 5 --no-subconfigs --no-cpu-baseline --steps 5 > $OUT/b5.json 2>$OUT/b5.err; echo "bench rc=$?"; python -c "import json; d=json.loads(open('$OUT/b5.json').read().splitlines()[-1]); print('cfg5 ms', d['ms_per_step'], 'e2e Gvox/s', d['e2e']['value']/1e9)"; }
true
