#!/bin/bash
# FC dK probe: the kernel with copies / MMAs disabled (CAPSCONV_FC_DBG bits 1 / 2)
for d in 0 1 2 3; do CAPSCONV_FC_DBG=$d python tests/probe/run_layer.py dK 1024,8,8,32,10,8,8,1 1; done
