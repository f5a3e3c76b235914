#!/bin/bash
# conv_mma_kernel component sweep (CAPSCONV_MMA_DBG bits: 1 loads, 2 MMAs, 4 stores, 32 epilogue units)
for cfg in "fwd 1024,22,22,8,16,3,3,2" "fwd 1024,10,10,16,32,3,3,1" "dI 1024,22,22,8,16,3,3,2" "dI 1024,10,10,16,32,3,3,1"; do
  for d in 0 1 2 4 36 3 7 39; do echo "$cfg dbg=$d: $(CAPSCONV_MMA_DBG=$d timeout 60 python tests/probe/run_layer.py $cfg 20 | tail -1 | sed 's/.*graph/graph/')"; done
done
