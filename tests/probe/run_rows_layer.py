"""Probe: run one pass of one config-5 stack layer in the rows layout (for
ncu captures).  Usage: python tests/probe/run_rows_layer.py <layer 1-4> <fwd|dI|dK> [reps]"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import capsinputs  # noqa: E402
import paper_2104_02621_b200 as pkg  # noqa: E402


def main():
    li = int(sys.argv[1]) - 1
    op = sys.argv[2]
    reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
    pkg.load_library()
    dev = "cuda:0"
    L = capsinputs.stack_layers(capsinputs.STACK_BATCH, pkg.output_dims)[li]
    Ho, Wo = pkg.output_dims(L.H, L.W, L.KH, L.KW, L.stride)
    I = capsinputs.make_input(L, dtype=torch.bfloat16, layer_idx=li).to(dev).permute(0, 1, 2, 4, 3, 5).contiguous()
    K = capsinputs.make_kernel(L, dtype=torch.bfloat16, layer_idx=li).to(dev)
    dO = capsinputs.make_grad_output(L.o_shape(Ho, Wo), dtype=torch.bfloat16, layer_idx=li).to(dev)
    dO = dO.permute(0, 1, 2, 4, 3, 5).contiguous()
    for _ in range(reps):
        if op == "fwd":
            pkg.fwd(I, K, L.stride, layout="rows")
        elif op == "dI":
            pkg.bwd_data(dO, K, L.stride, L.H, L.W, layout="rows")
        else:
            pkg.bwd_kernel(I, dO, L.stride, L.KH, L.KW, layout="rows")
    torch.cuda.synchronize()
    print("ok")


if __name__ == "__main__":
    main()
