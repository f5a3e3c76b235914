#!/bin/bash
# graph-timed passes of the conv stack layers (run_layer.py, 20 iterations each)
for cfg in "fwd 1024,24,24,8,8,3,3,1" "dI 1024,24,24,8,8,3,3,1" "fwd 1024,22,22,8,16,3,3,2" "dI 1024,22,22,8,16,3,3,2" "fwd 1024,10,10,16,32,3,3,1" "dI 1024,10,10,16,32,3,3,1"; do
  echo "$cfg: $(timeout 60 python tests/probe/run_layer.py $cfg 20 | tail -1 | sed 's/.*graph/graph/')"
done
