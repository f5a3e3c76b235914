# Round-2 final measurements: default bench line, training step, fp32 stack,
# configs 2-4, reference arms, GPU tests, smoke
set -x
timeout 400 python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err
timeout 400 python bench.py --config pcapsnet_train > gpurun_out/final_train.json 2> gpurun_out/final_train.err
timeout 300 python bench.py --dtype fp32 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/final_fp32.json 2> gpurun_out/final_fp32.err
rm -f gpurun_out/final_cfg.jsonl
for c in layer_s1 layer_s2 fc; do timeout 300 python bench.py --config $c --no-cpu-baseline >> gpurun_out/final_cfg.jsonl 2>> gpurun_out/final_cfg.err; done
timeout 400 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/final_ref.json 2> gpurun_out/final_ref.err
timeout 400 python bench.py --impl reference --config pcapsnet_train --steps 2 --warmup 1 > gpurun_out/final_ref_train.json 2> gpurun_out/final_ref_train.err
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/final_gpu_tests.log 2>&1; tail -2 gpurun_out/final_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/final_smoke.log 2>&1; tail -1 gpurun_out/final_smoke.log
