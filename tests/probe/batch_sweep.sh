# Single-GPU batch sweep: one rank's share of the batch-1024
# stack at 8/4/2/1 GPUs, graph replay vs eager launches.
for b in 128 256 512 1024; do
  for e in "" "--eager"; do
    timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-parity --batch $b $e | tail -1
  done
done
