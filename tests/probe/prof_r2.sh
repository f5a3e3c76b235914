set -e
python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/plain_bench.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1 || true
for spec in "1 dI rows_conv_kernel" "1 fwd rows_conv_kernel" "1 dK rows_wgrad_kernel" "3 dI rows_conv_kernel" "4 dI rows_fc_kernel" "2 fwd rows_conv_kernel"; do
  set -- $spec
  python tests/probe/run_rows_layer.py $1 $2 3 > gpurun_out/plain_$1$2.log 2>&1
  ncu --set full --clock-control none --import-source on -k regex:$3 -s 2 -c 1 -o gpurun_out/r2_L$1_$2 python tests/probe/run_rows_layer.py $1 $2 3 > gpurun_out/ncu_$1$2.log 2>&1 || true
done
ls gpurun_out/*.ncu-rep
