# A/B of env settings on the config-5 volume bench (device value only): AB="A=1 A=2"
for kv in ${AB}; do
  r=$(env $kv timeout 300 python bench.py --config 5 --no-subconfigs --no-cpu-baseline --no-e2e --steps 5 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'])")
  echo "$kv ms $r"
done
