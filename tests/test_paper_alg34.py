"""The paper-faithful comparison arm (bench.py --impl paper-alg34: Algorithms
3/4 with materialised im2col / extends and batched 4x4 matmuls) computes the
same O, dI, dK as the oracle (run here in fp64 on the CPU)."""
import sys
import os

import numpy as np
import pytest
import torch

import capsinputs

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402


@pytest.mark.parametrize("case", [(2, 7, 6, 3, 2, 3, 2, 1), (2, 9, 8, 2, 3, 3, 3, 2), (3, 4, 4, 4, 2, 4, 4, 1)])
def test_alg34_matches_oracle(oracle_mod, case):
    B, H, W, C, Co, KH, KW, s = case
    L = capsinputs.Layer(B=B, H=H, W=W, C=C, Cout=Co, KH=KH, KW=KW, D1=4, D2=4, D3=4, stride=s)
    I = capsinputs.make_input(L).double()
    K = capsinputs.make_kernel(L).double()
    Ho, Wo = oracle_mod.output_dims(H, W, KH, KW, s)
    dO = capsinputs.make_grad_output(L.o_shape(Ho, Wo)).double()
    O = bench.alg34_layer(I, K, s)
    dI, dK = bench.alg34_layer(I, K, s, dO)
    rO, _ = oracle_mod.fwd(I.numpy(), K.numpy(), s)
    rdI, _ = oracle_mod.bwd_data(dO.numpy(), K.numpy(), s, H, W)
    rdK, _ = oracle_mod.bwd_kernel(I.numpy(), dO.numpy(), s, KH, KW)
    np.testing.assert_allclose(O.numpy(), rO, rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(dI.numpy(), rdI, rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(dK.double().numpy(), rdK, rtol=1e-5, atol=1e-6)
