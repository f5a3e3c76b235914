#!/bin/bash
# wgrad component sweep (CAPSCONV_WG_DBG bits: 1 transpose, 2 MMAs, 4 B repack, 16 A build)
for cfg in "dK 1024,24,24,8,8,3,3,1" "dK 1024,22,22,8,16,3,3,2" "dK 1024,10,10,16,32,3,3,1"; do
  for d in 0 2 21 23 1 4 16; do echo "$cfg dbg=$d: $(CAPSCONV_WG_DBG=$d timeout 60 python tests/probe/run_layer.py $cfg 20 | tail -1 | sed 's/.*graph/graph/')"; done
done
