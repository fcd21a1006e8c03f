# config-5 volume: patches per launch x runner streams (device-timed value only)
for s in 2 1; do for b in 4 6 8 12 16; do
  r=$(VOXPLAN_PATCH_BATCH=$b VOXPLAN_STREAMS=$s timeout 300 python bench.py --config 5 --no-subconfigs --no-cpu-baseline --no-e2e --steps 5 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'])")
  echo "streams $s batch $b ms $r"
done; done
