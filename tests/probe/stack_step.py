"""Run N steps of the config-5 stack (global batch 1024, bf16) -- for ncu."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch
import capsinputs
import paper_2104_02621_b200 as pkg
from paper_2104_02621_b200.stack import CapsStack, LayerSpec
pkg.load_library()
steps = int(sys.argv[1]) if len(sys.argv) > 1 else 2
dev = torch.device("cuda", 0)
specs = [LayerSpec(*l) for l in capsinputs.STACK_LAYERS]
si = capsinputs.STACK_INPUT
B = capsinputs.STACK_BATCH
layers = capsinputs.stack_layers(B, pkg.output_dims)
Ks = [capsinputs.make_kernel(L, dtype=torch.bfloat16, layer_idx=i) for i, L in enumerate(layers)]
X = torch.empty(layers[0].i_shape(), dtype=torch.bfloat16, device=dev).uniform_(-1, 1)
h, w = si["H"], si["W"]
for s in specs:
    h, w = pkg.output_dims(h, w, s.KH, s.KW, s.stride)
dY = torch.empty((B, h, w, specs[-1].Cout, 4, 4), dtype=torch.bfloat16, device=dev).uniform_(-1, 1)
st = CapsStack(specs, si["H"], si["W"], 4, B, Ks, dev)
for _ in range(steps):
    st.step(X, dY)
torch.cuda.synchronize()
print("ok", steps, "steps")
