# Round-2 final captures (r2c: dynamic strips + PDL weight packs): launch list of the bench (plain run first, then ncu),
# and ncu --set full of the rows kernels of the stack (one launch each).
set -e
timeout 400 python bench.py > gpurun_out/r2c_bench_default.json 2> gpurun_out/r2c_bench_default.err
timeout 300 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-parity > gpurun_out/plain_bench.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2c_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-parity > gpurun_out/ncu_launch.log 2>&1 || true
for spec in "1 fwd rows_walk_kernel" "1 dI rows_walk_kernel" "1 dK rows_wgrad_kernel" "2 fwd rows_walk_kernel" "2 dI rows_conv_kernel" "2 dK rows_wgrad_kernel" "3 fwd rows_conv_kernel" "3 dI rows_walk_kernel" "3 dK rows_wgrad_kernel" "4 fwd rows_fc_kernel" "4 dI rows_fc_kernel" "4 dK rows_fc_kernel"; do
  set -- $spec
  timeout 120 python tests/probe/run_rows_layer.py $1 $2 3 > gpurun_out/plain_$1$2.log 2>&1
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$3 -s 2 -c 1 -o gpurun_out/r2c_L$1_$2 python tests/probe/run_rows_layer.py $1 $2 3 > gpurun_out/ncu_$1$2.log 2>&1 || true
done
ls gpurun_out/r2c_*.ncu-rep
