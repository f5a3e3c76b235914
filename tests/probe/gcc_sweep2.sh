#!/bin/bash
# (G, CC) sweep of the conv MMA planner for the L2 / L3 passes
for spec in "fwd 1024,22,22,8,16,3,3,2" "fwd 1024,10,10,16,32,3,3,1" "dI 1024,10,10,16,32,3,3,1" "dI 1024,22,22,8,16,3,3,2"; do
 set -- $spec
 for g in 1 2 3 4 6 8; do for c in 4 8 16; do
  r=$(CAPSCONV_FORCE_G=$g CAPSCONV_FORCE_CC=$c CAPSCONV_DEBUG=1 timeout 60 python tests/probe/run_layer.py $1 $2 10 2>&1)
  echo "$r" | grep -q "mma plan" || continue
  echo "$1 $2 G=$g CC=$c $(echo "$r" | grep -o 'G=[0-9]* mtiles') $(echo "$r" | grep -o 'CC=[0-9]*' | head -1) $(echo "$r" | grep -o 'stages=[0-9]*') $(echo "$r" | grep -o 'nstg=[0-9]*') $(echo "$r" | grep -o 'h_box=[0-9]*') $(echo "$r" | grep -o 'graph.*')"
 done; done
done
