"""Quick GPU check of the MMA path against the SIMT path and the oracle."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import capsinputs, oracle
import paper_2104_02621_b200.capsconv as cc
from helpers import rel_err, to_np
cc.load_library()
cases = [tuple(map(int, a.split(","))) for a in sys.argv[1:]] or [
    (1, 12, 40, 8, 8, 3, 3, 4, 4, 4, 1), (2, 9, 11, 4, 5, 3, 3, 4, 4, 4, 1), (3, 10, 9, 8, 8, 3, 3, 4, 4, 4, 2),
    (2, 8, 8, 32, 10, 8, 8, 4, 4, 4, 1), (5, 7, 7, 16, 32, 3, 3, 4, 4, 4, 2), (64, 32, 32, 8, 8, 3, 3, 4, 4, 4, 1),
    (128, 16, 16, 16, 32, 3, 3, 4, 4, 4, 2), (256, 8, 8, 32, 10, 8, 8, 4, 4, 4, 1)]
for case in cases:
    L = capsinputs.Layer(*case)
    I = capsinputs.make_input(L, dtype=torch.bfloat16); K = capsinputs.make_kernel(L, dtype=torch.bfloat16)
    Ho, Wo = oracle.output_dims(L.H, L.W, L.KH, L.KW, L.stride)
    dO = capsinputs.make_grad_output(L.o_shape(Ho, Wo), dtype=torch.bfloat16)
    Id, Kd, dOd = I.cuda(), K.cuda(), dO.cuda()
    paths = [cc.select_path(op, torch.bfloat16, (L.B, L.H, L.W, L.C, L.Cout, L.KH, L.KW, 4, 4, 4, L.stride)) for op in (0, 1, 2)]
    O = cc.fwd(Id, Kd, L.stride); dI = cc.bwd_data(dOd, Kd, L.stride, L.H, L.W); dK = cc.bwd_kernel(Id, dOd, L.stride, L.KH, L.KW); torch.cuda.synchronize()
    rdK, adK = oracle.bwd_kernel(to_np(I), to_np(dO), L.stride, L.KH, L.KW)
    rO, aO = oracle.fwd(to_np(I), to_np(K), L.stride)
    rdI, adI = oracle.bwd_data(to_np(dO), to_np(K), L.stride, L.H, L.W)
    print(case, "paths", paths, "fwd err %.2e" % rel_err(to_np(O), rO, aO), "dI err %.2e" % rel_err(to_np(dI), rdI, adI), "dK err %.2e" % rel_err(to_np(dK), rdK, adK), flush=True)
