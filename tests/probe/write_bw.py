"""Probe: device write / copy bandwidth for buffers the size of the FC layer's
dI (67 MB) and of the L2 flush, and a read-only reduction, timed with CUDA events (warm, back to back)."""
import torch

dev = "cuda:0"
for mb in (16, 67, 134, 256):
    n = mb << 20
    x = torch.empty(n, dtype=torch.uint8, device=dev)
    y = torch.empty(n, dtype=torch.uint8, device=dev)
    xf = x.view(torch.float32)
    for name, f in (("fill", lambda: x.fill_(3)), ("copy", lambda: y.copy_(x)), ("read(sum)", lambda: xf.sum())):
        for _ in range(3):
            f()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(20):
            f()
        b.record()
        torch.cuda.synchronize()
        t = a.elapsed_time(b) / 20 * 1e-3
        byts = 2 * n if name == "copy" else n
        print("%s %4d MB: %.1f us  %.0f GB/s" % (name, mb, t * 1e6, byts / t / 1e9), flush=True)
