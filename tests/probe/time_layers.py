"""Probe: per-pass device time of the config-5 stack layers, natural vs rows
layout (CUDA events, L2 flushed before every rep, median of reps).
Usage: python tests/probe/time_layers.py [reps] [ops]   (ops: e.g. fwd,dI,dK)"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import capsinputs  # noqa: E402
import paper_2104_02621_b200 as pkg  # noqa: E402

HBM = 6553.6e9


def main():
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
    ops = sys.argv[2].split(",") if len(sys.argv) > 2 else ["fwd", "dI", "dK"]
    layouts = sys.argv[3].split(",") if len(sys.argv) > 3 else ["natural", "rows"]
    if os.environ.get("PROBE"):
        from paper_2104_02621_b200 import _build
        lib = _build.PROBE_LIB
        if os.environ.get("PROBE_LIB"):
            lib = os.path.join(os.path.dirname(_build.PROBE_LIB), os.environ["PROBE_LIB"])
        pkg.load_library(lib)   # diagnostic flavour (-DCAPSCONV_PROBES)
    else:
        pkg.load_library()
    dev = "cuda:0"
    layers = capsinputs.stack_layers(capsinputs.STACK_BATCH, pkg.output_dims)
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    for li, L in enumerate(layers):
        Ho, Wo = pkg.output_dims(L.H, L.W, L.KH, L.KW, L.stride)
        I = capsinputs.make_input(L, dtype=torch.bfloat16, layer_idx=li).to(dev)
        K = capsinputs.make_kernel(L, dtype=torch.bfloat16, layer_idx=li).to(dev)
        dO = capsinputs.make_grad_output(L.o_shape(Ho, Wo), dtype=torch.bfloat16, layer_idx=li).to(dev)
        flops = 2 * L.B * Ho * Wo * 4 * L.Cout * 4 * L.KH * L.KW * L.C * 4
        nI, nO, nK = I.numel() * 2, dO.numel() * 2, K.numel()
        byts = {"fwd": nI + nO + 2 * nK, "dI": nI + nO + 2 * nK, "dK": nI + nO + 4 * nK}
        for lay in layouts:
            Il = I.permute(0, 1, 2, 4, 3, 5).contiguous() if lay == "rows" else I
            dOl = dO.permute(0, 1, 2, 4, 3, 5).contiguous() if lay == "rows" else dO
            fns = {
                "fwd": lambda: pkg.fwd(Il, K, L.stride, layout=lay),
                "dI": lambda: pkg.bwd_data(dOl, K, L.stride, L.H, L.W, layout=lay),
                "dK": lambda: pkg.bwd_kernel(Il, dOl, L.stride, L.KH, L.KW, layout=lay),
            }
            for op in ops:
                f = fns[op]
                for _ in range(3):
                    f()
                ts = []
                for _ in range(reps):
                    flush.fill_(1.0)
                    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    a.record()
                    f()
                    b.record()
                    torch.cuda.synchronize()
                    ts.append(a.elapsed_time(b) * 1e-3)
                ts.sort()
                t = ts[len(ts) // 2]
                roof = max(byts[op] / HBM, flops / 1401e12)
                print("L%d %-3s %-7s %8.1f us  %6.1f TFLOP/s  %6.0f GB/s  roof %.3f" % (
                    li + 1, op, lay, t * 1e6, flops / t / 1e12, byts[op] / t / 1e9, roof / t), flush=True)


if __name__ == "__main__":
    main()
