# Device iter/s of every bench config under a list of environments (GPU box):
#   ENVS="SSCG_ZM=0 SSCG_ZM=1" bash tools/configs_sweep.sh
for cfg in ${CONFIGS:-c1 c2 c3 c4}; do
  for e in ${ENVS:-""}; do
    r=$(env $(echo "$e" | tr ',' ' ') timeout 900 python bench.py --config $cfg --steps 3 --warmup 3 --no-cpu 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print(round(d['value'],1), round(d['ms_per_step'],2), d['config']['syncs_to_tol'], d['config']['total_iters'], d['roofline']['mpk_schedule'].get('form'), d['roofline']['kernel_ms'])" 2>&1)
    echo "$cfg [$e] $r"
  done
done
