import os, sys, torch
sys.path.insert(0, "/root/repo")
import capsinputs
import paper_2104_02621_b200 as pkg
from paper_2104_02621_b200 import _build
from paper_2104_02621_b200.stack import CapsStack, LayerSpec
pkg.load_library(_build.PROBE_LIB)
dev = torch.device("cuda:0")
specs = [LayerSpec(*l) for l in capsinputs.STACK_LAYERS]
si = capsinputs.STACK_INPUT
B = 1024
layers = capsinputs.stack_layers(B, pkg.output_dims)
Ks = [capsinputs.make_kernel(L, dtype=torch.bfloat16, layer_idx=i) for i, L in enumerate(layers)]
st = CapsStack(specs, si["H"], si["W"], 4, B, Ks, dev, layout="rows")
X = capsinputs.make_input(layers[0], dtype=torch.bfloat16).permute(0,1,2,4,3,5).contiguous().to(dev)
dY = torch.randn(B, 1, 1, 4, 10, 4, device=dev).to(torch.bfloat16)
st.step(X, dY); torch.cuda.synchronize()
g = st.grads[2]
print("g", g.shape, g.stride(), g.is_contiguous(), g.data_ptr() % 16)
for _ in range(2):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); pkg.bwd_data(g, st.K[1], 2, 22, 22, out=st.grads[1], layout="rows"); b.record(); torch.cuda.synchronize()
    print("L2 dI from stack grads", a.elapsed_time(b))
g2 = torch.randn_like(g.float()).to(torch.bfloat16)
for _ in range(2):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); pkg.bwd_data(g2, st.K[1], 2, 22, 22, out=st.grads[1], layout="rows"); b.record(); torch.cuda.synchronize()
    print("L2 dI random", a.elapsed_time(b))

# full step with per-call events (eager), as bench.py times it
import time
class T:
    def __init__(self): self.p = []; self.o = {}
    def begin(self, li, k):
        e = torch.cuda.Event(enable_timing=True); e.record(); self.o[(li, k)] = e
    def end(self, li, k):
        e = torch.cuda.Event(enable_timing=True); e.record(); self.p.append(((li, k), self.o.pop((li, k)), e))
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
res = {}
for it in range(5):
    tm = T()
    flush.zero_()
    st.step(X, dY, timer=tm)
    torch.cuda.synchronize()
    for k, a, b in tm.p:
        res.setdefault(k, []).append(a.elapsed_time(b))
for k in sorted(res):
    print("step L%d %-3s %.1f us" % (k[0] + 1, k[1], 1000 * sorted(res[k])[2]))
