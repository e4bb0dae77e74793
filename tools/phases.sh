for cfg in c1 c2 c3; do
  timeout 600 python bench.py --config $cfg --steps 2 --warmup 3 --no-cpu 2>/dev/null | tail -1 > gpurun_out/ph_$cfg.json
done
