"""Probe: run each pass of one BASELINE config in the rows layout, synchronising
after each (to find a hanging or failing pass).  Usage: run_cfg.py <cfg> [batch]"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import capsinputs  # noqa: E402
import paper_2104_02621_b200 as pkg  # noqa: E402


def main():
    L = capsinputs.CONFIGS[sys.argv[1]]
    if len(sys.argv) > 2:
        L = L.with_batch(int(sys.argv[2]))
    pkg.load_library()
    dev = "cuda:0"
    Ho, Wo = pkg.output_dims(L.H, L.W, L.KH, L.KW, L.stride)
    I = capsinputs.make_input(L, dtype=torch.bfloat16).to(dev).permute(0, 1, 2, 4, 3, 5).contiguous()
    K = capsinputs.make_kernel(L, dtype=torch.bfloat16).to(dev)
    dO = capsinputs.make_grad_output(L.o_shape(Ho, Wo), dtype=torch.bfloat16).to(dev).permute(0, 1, 2, 4, 3, 5).contiguous()
    ext = (L.B, L.H, L.W, L.C, L.Cout, L.KH, L.KW, L.D1, L.D2, L.D3, L.stride)
    for name, op, f in (("fwd", pkg.OP_FWD, lambda: pkg.fwd(I, K, L.stride, layout="rows")),
                        ("dI", pkg.OP_BWD_DATA, lambda: pkg.bwd_data(dO, K, L.stride, L.H, L.W, layout="rows")),
                        ("dK", pkg.OP_BWD_KERNEL, lambda: pkg.bwd_kernel(I, dO, L.stride, L.KH, L.KW, layout="rows"))):
        print(name, "path", pkg.select_path(op, torch.bfloat16, ext, "rows"), flush=True)
        f()
        torch.cuda.synchronize()
        print(name, "ok", flush=True)


if __name__ == "__main__":
    main()
