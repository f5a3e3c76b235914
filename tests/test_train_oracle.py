"""CPU pins of the training-step oracle: the primary layer as
a capsule convolution with C = Cout = D1 = D2 = 1 equals a plain conv2d
(torch, fp64), the channel mapping between the primary output and the capsule
map is the rows order (reading R25) and inverts, and the SGD step matches a
hand-computed one.  No GPU."""
import numpy as np
import torch

import capsinputs


def test_primary_layer_is_conv2d(oracle_mod):
    """Plain convolution of a one-channel image to 128 channels, as torch
    computes it (cross-correlation, NCHW): the oracle's capsule convolution
    with D = (1, 1, 128) must equal it -- an independent definition."""
    L = capsinputs.Layer(B=2, H=9, W=8, C=1, Cout=1, KH=5, KW=4, D1=1, D2=1, D3=128, stride=1)
    img = capsinputs.make_input(L, dtype=torch.float64)
    K = capsinputs.make_kernel(L, dtype=torch.float64)
    O, _ = oracle_mod.fwd(img.numpy(), K.numpy(), 1)
    x = img.reshape(2, 9, 8).unsqueeze(1)                                      # (B, 1, H, W)
    w = K.reshape(5, 4, 128).permute(2, 0, 1).unsqueeze(1).contiguous()       # (128, 1, KH, KW)
    ref = torch.nn.functional.conv2d(x, w)                                     # (B, 128, Ho, Wo)
    np.testing.assert_allclose(O.reshape(2, 5, 5, 128), ref.permute(0, 2, 3, 1).numpy(), rtol=0, atol=1e-13)


def test_primary_layer_dk_is_conv2d_weight_grad(oracle_mod):
    """dK of the primary layer = torch autograd's conv2d weight gradient."""
    L = capsinputs.Layer(B=3, H=8, W=7, C=1, Cout=1, KH=3, KW=3, D1=1, D2=1, D3=16, stride=1)
    img = capsinputs.make_input(L, dtype=torch.float64)
    dO = capsinputs.make_grad_output((3, 6, 5, 1, 1, 16), dtype=torch.float64)
    dK, _ = oracle_mod.bwd_kernel(img.numpy(), dO.numpy(), 1, 3, 3)
    w = torch.zeros(16, 1, 3, 3, dtype=torch.float64, requires_grad=True)
    y = torch.nn.functional.conv2d(img.reshape(3, 8, 7).unsqueeze(1), w)
    y.backward(dO.reshape(3, 6, 5, 16).permute(0, 3, 1, 2))
    np.testing.assert_allclose(dK.reshape(3, 3, 16), w.grad.permute(2, 3, 0, 1).reshape(3, 3, 16).numpy(),
                               rtol=0, atol=1e-12)


def test_primary_channel_order(oracle_mod):
    """Channel o = (d1*C + c)*D + d2 lands on capsule (c, d1, d2) (one-hot),
    and the two maps invert each other."""
    C, D = 8, 4
    for (c, d1, d2) in [(0, 0, 0), (3, 1, 2), (7, 3, 3), (5, 0, 1)]:
        prim = np.zeros((1, 2, 2, 1, 1, C * D * D))
        prim[0, 1, 0, 0, 0, (d1 * C + c) * D + d2] = 1.0
        caps = oracle_mod.primary_to_caps(prim, C, D)
        assert caps.shape == (1, 2, 2, C, D, D)
        assert caps[0, 1, 0, c, d1, d2] == 1.0 and caps.sum() == 1.0
        np.testing.assert_array_equal(oracle_mod.caps_to_primary(caps), prim)


def test_sgd_update_hand_example(oracle_mod):
    w = np.array([1.0, 2.0, -0.5, 0.0])
    g = np.array([10.0, -4.0, 0.0, 3.0])
    np.testing.assert_array_equal(oracle_mod.sgd_update(w, g, 0.25), [-1.5, 3.0, -0.5, -0.75])
    np.testing.assert_array_equal(oracle_mod.sgd_update(w, g, 0.0), w)


def test_train_step_reduces_to_its_parts(oracle_mod):
    """With lr = 0 the weights are unchanged, and the returned dKs are the
    stack's dKs plus the primary dK of the stack's dX (composition check on a
    tiny stack)."""
    from paper_2104_02621_b200.stack import LayerSpec  # shapes only
    specs = [LayerSpec(2, 2, 3, 3, 1), LayerSpec(2, 3, 2, 2, 1)]
    B, D = 2, 4
    P = capsinputs.Layer(B=B, H=9, W=9, C=1, Cout=1, KH=3, KW=3, D1=1, D2=1, D3=2 * D * D, stride=1)
    img = capsinputs.make_input(P, dtype=torch.float64).numpy()
    Kp = capsinputs.make_kernel(P, dtype=torch.float64).numpy()
    Ks, h = [], 7
    for i, sp in enumerate(specs):
        L = capsinputs.Layer(B=B, H=h, W=h, C=sp.C, Cout=sp.Cout, KH=sp.KH, KW=sp.KW, D1=D, D2=D, D3=D, stride=1)
        Ks.append(capsinputs.make_kernel(L, dtype=torch.float64, layer_idx=i).numpy())
        h = h - sp.KH + 1
    dY = capsinputs.make_grad_output((B, h, h, 3, D, D), dtype=torch.float64).numpy()
    new, dKs, _ = oracle_mod.train_step(img, Kp, Ks, [1, 1], dY, 0.0, False)
    for a, b in zip(new, [Kp] + Ks):
        np.testing.assert_array_equal(a, b)
    prim, _ = oracle_mod.fwd(img, Kp, 1)
    acts, dX, sdK, _ = oracle_mod.stack_fwd_bwd(oracle_mod.primary_to_caps(prim, 2, D), Ks, [1, 1], dY, False)
    for a, b in zip(dKs[1:], sdK):
        np.testing.assert_array_equal(a, b)
    dKp, _ = oracle_mod.bwd_kernel(img, oracle_mod.caps_to_primary(dX), 1, 3, 3)
    np.testing.assert_array_equal(dKs[0], dKp)
