# A/B of matrix-powers schedules over side-built libraries (GPU box):
#   LIBS="libsscg.so libsscg_x.so" ENVS="SSCG_ZM=1 SSCG_ZM=0" bash tools/sweep_libs.sh
fmt() { python -c "
import sys,json
for l in sys.stdin:
  try: d=json.loads(l)
  except Exception: print(l.strip()[:200]); continue
  print(d['env'], d['sched']['ctas'], d['sched']['passes'][:1], round(d['ms_per_outer'],3), round(d['mpk_ms_per_outer'],3), d.get('dbg') or '')
"; }
for lib in ${LIBS:-libsscg.so}; do
  echo "== $lib"
  SSCG_LIB=paper_1908_04081_b200/_lib/$lib timeout 600 python tools/ab_sweep.py --config ${CONFIG:-c5w} --outer ${OUTER:-10} ${ENVS:-SSCG_ZM=1} 2>&1 | fmt
done
