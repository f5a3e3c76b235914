#!/bin/bash
# MMA-only skeletons: dbg 101 = no loads/repack/stores/epilogue (MMAs only), 103 = nothing
for cfg in "fwd 1024,24,24,8,8,3,3,1" "fwd 1024,22,22,8,16,3,3,2" "dI 1024,22,22,8,16,3,3,2" "fwd 1024,10,10,16,32,3,3,1" "dI 1024,10,10,16,32,3,3,1"; do
  for d in 0 101 103 69; do echo "$cfg dbg=$d: $(CAPSCONV_MMA_DBG=$d timeout 60 python tests/probe/run_layer.py $cfg 20 | tail -1 | sed 's/.*graph/graph/')"; done
done
