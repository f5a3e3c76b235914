# Round 2: ncu captures of the training step's tensor-core primary kernels
# (one launch each, --set full) and the launch list of the training step.
timeout 300 python bench.py --config pcapsnet_train --steps 2 --warmup 1 --no-cpu-baseline --no-parity > gpurun_out/plain_train.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:primary_tc_fwd -c 1 -o gpurun_out/r2_P_fwd python bench.py --config pcapsnet_train --steps 1 --warmup 1 --no-cpu-baseline --no-parity --eager > gpurun_out/ncu_pf.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:primary_tc_dk -c 1 -o gpurun_out/r2_P_dK python bench.py --config pcapsnet_train --steps 1 --warmup 1 --no-cpu-baseline --no-parity --eager > gpurun_out/ncu_pd.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_train_launches.csv python bench.py --config pcapsnet_train --steps 2 --warmup 1 --no-cpu-baseline --no-parity > gpurun_out/ncu_tl.log 2>&1
ls gpurun_out/r2_P_*.ncu-rep
