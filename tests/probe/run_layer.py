"""Run one capsule-conv pass repeatedly (for ncu / timing).  Usage:
   python tests/probe/run_layer.py OP B,H,W,C,Cout,KH,KW,s [iters] [dtype]   OP in fwd,dI,dK"""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch
import capsinputs
import paper_2104_02621_b200.capsconv as cc
cc.load_library(os.environ.get("CAPSCONV_LIB"))   # A/B: an alternative build
op = sys.argv[1]
B, H, W, C, Co, KH, KW, s = map(int, sys.argv[2].split(","))
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 5
dt = torch.bfloat16 if (len(sys.argv) <= 4 or sys.argv[4] == "bf16") else torch.float32
L = capsinputs.Layer(B, H, W, C, Co, KH, KW, 4, 4, 4, s)
I = capsinputs.make_input(L, dtype=dt).cuda()
K = capsinputs.make_kernel(L, dtype=dt).cuda()
Ho, Wo = cc.output_dims(H, W, KH, KW, s)
dO = capsinputs.make_grad_output(L.o_shape(Ho, Wo), dtype=dt).cuda()
fn = {"fwd": lambda: cc.fwd(I, K, s), "dI": lambda: cc.bwd_data(dO, K, s, H, W),
      "dK": lambda: cc.bwd_kernel(I, dO, s, KH, KW)}[op]
for _ in range(2):
    fn()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(iters):
    fn()
e1.record()
torch.cuda.synchronize()
eager = e0.elapsed_time(e1) / iters
g = torch.cuda.CUDAGraph()
cs = torch.cuda.Stream()
cs.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(cs):
    fn()
    torch.cuda.synchronize()
    with torch.cuda.graph(g, stream=cs):
        for _ in range(iters):
            fn()
torch.cuda.synchronize()
g.replay()
torch.cuda.synchronize()
e0.record()
g.replay()
e1.record()
torch.cuda.synchronize()
print("%s %s: eager %.4f ms/iter, graph %.4f ms/iter" % (op, sys.argv[2], eager, e0.elapsed_time(e1) / iters))
