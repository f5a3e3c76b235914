"""Run each pass once (for one ncu --set full capture of several kernels):
   python tests/probe/capture_ops.py OP:B,H,W,C,Cout,KH,KW,s [...]"""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch
import capsinputs
import paper_2104_02621_b200.capsconv as cc
cc.load_library()
for spec in sys.argv[1:]:
    op, shape = spec.split(":")
    B, H, W, C, Co, KH, KW, s = map(int, shape.split(","))
    L = capsinputs.Layer(B, H, W, C, Co, KH, KW, 4, 4, 4, s)
    I = capsinputs.make_input(L, dtype=torch.bfloat16).cuda()
    K = capsinputs.make_kernel(L, dtype=torch.bfloat16).cuda()
    Ho, Wo = cc.output_dims(H, W, KH, KW, s)
    dO = capsinputs.make_grad_output(L.o_shape(Ho, Wo), dtype=torch.bfloat16).cuda()
    {"fwd": lambda: cc.fwd(I, K, s), "dI": lambda: cc.bwd_data(dO, K, s, H, W),
     "dK": lambda: cc.bwd_kernel(I, dO, s, KH, KW)}[op]()
    torch.cuda.synchronize()
