set -x
python bench.py --steps 1 --warmup 0 --no-cpu --no-secondary > gpurun_out/r2d_bench_plain.json 2> gpurun_out/r2d_bench_plain.err || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/r2d_c5w_launches.csv python bench.py --steps 1 --warmup 0 --no-cpu --no-secondary > gpurun_out/r2d_ncu1.log 2>&1
python tools/ncu_target.py 3 c5w > gpurun_out/r2d_target.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:k_small -s 1 -c 2 -o gpurun_out/r2d_small -f python tools/ncu_target.py 3 c5w > gpurun_out/r2d_ncu2.log 2>&1
python tools/ncu_target.py 6 c1 > gpurun_out/r2d_target_c1.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/r2d_c1_launches.csv python tools/ncu_target.py 6 c1 > gpurun_out/r2d_ncu3.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_leja_ -s 20 -c 4 -o gpurun_out/r2d_leja -f python tools/ncu_target.py 6 c1 > gpurun_out/r2d_ncu4.log 2>&1
ls -la gpurun_out | tail
