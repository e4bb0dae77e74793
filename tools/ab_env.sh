#!/bin/bash
# A/B of environment switches: tools/ab_env.sh "A=1 B=0|A=0" "c1 c5w" [steps]
IFS='|' read -ra envs <<< "$1"; cfgs="$2"; steps="${3:-5}"
for e in "${envs[@]}"; do for c in $cfgs; do
  env $e python bench.py --config $c --steps $steps --warmup 3 --no-cpu 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.readlines()[-1])
print('[$e] $c', round(d['value'],1), round(d['ms_per_step'],3), d['solve']['syncs_to_tol'], d['solve']['total_iters'], {k: round(v,2) for k,v in d['roofline']['kernel_ms'].items()})"
done; done
