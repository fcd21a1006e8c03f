#!/usr/bin/env bash
# Config-5 volume step under environment variants (bench.py, headline only).
# Usage: tools/env_sweep.sh "VAR=a VAR2=b" "VAR=c" ...
for v in "$@"; do
  r=$(env $v timeout 600 python bench.py --no-subconfigs --no-cpu-baseline --no-e2e --steps 5 --warmup 3 2>/dev/null \
      | python -c "import json,sys; r=json.loads(sys.stdin.read()); print('%.2f ms  roof %.3f  dom %.1f us' % (r['ms_per_step'], r['network_roofline']['frac'], r['roofline']['ms_per_launch']*1e3))")
  echo "[$v] $r"
done
