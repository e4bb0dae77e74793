#!/bin/bash
# A/B of side builds: tools/ab_libs.sh "lib1.so lib2.so" "c1 c5w" [steps]
libs="$1"; cfgs="$2"; steps="${3:-5}"
for lib in $libs; do for c in $cfgs; do
  SSCG_LIB=$PWD/paper_1908_04081_b200/_lib/$lib python bench.py --config $c --steps $steps --warmup 3 --no-cpu 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.readlines()[-1])
print('$lib $c', round(d['value'],1), round(d['ms_per_step'],3), d['solve']['syncs_to_tol'], d['solve']['total_iters'], {k: round(v,2) for k,v in d['roofline']['kernel_ms'].items()}, d['roofline'].get('small_phases_us_per_call'))"
done; done
