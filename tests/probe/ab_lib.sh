#!/bin/bash
# A/B two builds of libcapsconv (ab/lib_old.so vs ab/lib_new.so) on the given passes, alternating
for round in 1 2; do
  for cfg in "$@"; do
    for v in old new; do
      echo "$v $cfg: $(CAPSCONV_LIB=ab/lib_$v.so timeout 60 python tests/probe/run_layer.py $cfg 20 | tail -1 | sed 's/.*graph/graph/')"
    done
  done
done
