"""Probe: event-time one pass of one config-5 stack layer (rows layout) with
either library flavour, L2 flushed between reps; knobs come from the
environment (read once per process when the plan is built).
Usage: [CAPSCONV_PROBE_LIB=1] [DTYPE=fp32] python tests/probe/time_layer.py <layer 1-4> <fwd|dI|dK> [reps]"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import capsinputs  # noqa: E402
import paper_2104_02621_b200 as pkg  # noqa: E402
import paper_2104_02621_b200.capsconv as cc  # noqa: E402
from paper_2104_02621_b200 import _build  # noqa: E402


def main():
    li = int(sys.argv[1]) - 1
    op = sys.argv[2]
    reps = int(sys.argv[3]) if len(sys.argv) > 3 else 20
    cc.load_library(_build.PROBE_LIB if os.environ.get("CAPSCONV_PROBE_LIB") else None)
    dev = "cuda:0"
    L = capsinputs.stack_layers(capsinputs.STACK_BATCH, pkg.output_dims)[li]
    dt = torch.float32 if os.environ.get("DTYPE") == "fp32" else torch.bfloat16
    Ho, Wo = pkg.output_dims(L.H, L.W, L.KH, L.KW, L.stride)
    I = capsinputs.make_input(L, dtype=dt, layer_idx=li).to(dev).permute(0, 1, 2, 4, 3, 5).contiguous()
    K = capsinputs.make_kernel(L, dtype=dt, layer_idx=li).to(dev)
    dO = capsinputs.make_grad_output(L.o_shape(Ho, Wo), dtype=dt, layer_idx=li).to(dev)
    dO = dO.permute(0, 1, 2, 4, 3, 5).contiguous()
    if op == "fwd":
        f = lambda: pkg.fwd(I, K, L.stride, layout="rows")  # noqa: E731
    elif op == "dI":
        f = lambda: pkg.bwd_data(dO, K, L.stride, L.H, L.W, layout="rows")  # noqa: E731
    else:
        f = lambda: pkg.bwd_kernel(I, dO, L.stride, L.KH, L.KW, layout="rows")  # noqa: E731
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    f()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        flush.fill_(1)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        f()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    ts.sort()
    tag = os.environ.get("TAG", "")
    print("L%d %s %s median %.1f us min %.1f" % (li + 1, op, tag, ts[len(ts) // 2], ts[0]), flush=True)


if __name__ == "__main__":
    main()
