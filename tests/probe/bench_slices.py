"""Time the S-slice capsule calls (fwd, dI, dK) with CUDA events on a
CapsNet-sized layer; report useful TFLOP/s (the slice-wise flops), next to the
matrix-capsule (S = 1) calls on one slice's shape in both layouts, scaled by S
(the grouped form's target: within 20% of those).  python tests/probe/bench_slices.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2104_02621_b200.capsconv as cc

cc.load_library()
for (B, H, W, C, Co, KH, KW, S, D, s) in [(256, 24, 24, 8, 8, 3, 3, 2, 4, 1), (256, 24, 24, 4, 4, 3, 3, 3, 4, 1)]:
    Ho, Wo = cc.output_dims(H, W, KH, KW, s)
    I = torch.randn(B, H, W, C, S, D, D, device="cuda").bfloat16()
    K = (torch.randn(KH, KW, C, Co, S, D, D, device="cuda") * 0.1).bfloat16()
    dO = torch.randn(B, Ho, Wo, Co, S, D, D, device="cuda").bfloat16()
    flops = 2 * B * Ho * Wo * D * Co * D * KH * KW * C * D * S     # slice-wise, per pass
    fl = {"fwd": lambda: cc.fwd_slices(I, K, s), "dI": lambda: cc.bwd_data_slices(dO, K, s, H, W),
          "dK": lambda: cc.bwd_kernel_slices(I, dO, s, KH, KW)}
    res = []
    for name, f in fl.items():
        for _ in range(3):
            f()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(20):
            f()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 20
        res.append("%s %.3f ms %.1f useful TFLOP/s" % (name, ms, flops / ms / 1e9))
    # the S = 1 path: one slice's problem (C -> Co matrix capsules), S times
    I1 = torch.randn(B, H, W, C, D, D, device="cuda").bfloat16()
    K1 = (torch.randn(KH, KW, C, Co, D, D, device="cuda") * 0.1).bfloat16()
    dO1 = torch.randn(B, Ho, Wo, Co, D, D, device="cuda").bfloat16()
    for lay in ("natural", "rows"):
        Il = I1.permute(0, 1, 2, 4, 3, 5).contiguous() if lay == "rows" else I1
        dOl = dO1.permute(0, 1, 2, 4, 3, 5).contiguous() if lay == "rows" else dO1
        f1 = {"fwd": lambda: cc.fwd(Il, K1, s, layout=lay), "dI": lambda: cc.bwd_data(dOl, K1, s, H, W, layout=lay),
              "dK": lambda: cc.bwd_kernel(Il, dOl, s, KH, KW, layout=lay)}
        for name, f in f1.items():
            for _ in range(3):
                f()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record()
            for _ in range(20):
                f()
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / 20 * S
            res.append("S=1 %s %s x%d %.3f ms %.1f TFLOP/s" % (lay, name, S, ms, flops / ms / 1e9))
    print("B=%d %dx%d C=%d Cout=%d %dx%d S=%d D=%d s=%d:" % (B, H, W, C, Co, KH, KW, S, D, s), "; ".join(res))
