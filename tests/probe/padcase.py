import sys, os, numpy as np, torch
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import capsinputs, oracle
import paper_2104_02621_b200.capsconv as cc
cc.load_library()
for case in [(2, 7, 7, 16, 32, 3, 3, 1, 2), (2, 7, 7, 16, 32, 3, 3, 1, 1), (2, 9, 9, 16, 32, 3, 3, 1, 2), (2, 7, 7, 8, 8, 3, 3, 1, 2), (2,7,7,16,16,3,3,1,2)]:
    B, H, W, C, Co, KH, KW, s, pad = case
    L = capsinputs.Layer(B, H, W, C, Co, KH, KW, 4, 4, 4, s)
    I = capsinputs.make_input(L, "int1", torch.bfloat16); K = capsinputs.make_kernel(L, "int1", torch.bfloat16)
    Ho, Wo = oracle.output_dims(H, W, KH, KW, s, pad)
    dO = capsinputs.make_grad_output(L.o_shape(Ho, Wo), "int1", torch.bfloat16)
    dK = cc.bwd_kernel(I.cuda(), dO.cuda(), s, KH, KW, pad=pad).cpu().numpy()
    r, _ = oracle.bwd_kernel(I.double().numpy(), dO.double().numpy(), s, KH, KW, pad)
    bad = np.argwhere(dK != r)
    print(case, "maxerr", np.abs(dK - r).max(), "nbad", len(bad), "first bad (p,q,c,co)", bad[:3, :4].tolist() if len(bad) else None)
