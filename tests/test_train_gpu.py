"""GPU parity of the routing-free P-CapsNet training step (SURVEY NEXT-4,
paper_2104_02621_b200/train.py): primary layer + the config-5 stack + one SGD
step, through libcapsconv, against oracle.train_step (bf16 layer boundaries,
reading R13; primary layer reading R25).  Checks every dK (normalised error,
bf16 bar), every fp32 master after the step (= w - lr*dK with the device's
own dK, one fp32 rounding: within 1 ulp) and every bf16 working copy (= the
RNE bf16 of its master, exactly)."""
import numpy as np
import pytest
import torch

import capsinputs
from helpers import TOL, assert_close, to_np

pytestmark = pytest.mark.gpu

DEV = "cuda:0"


@pytest.fixture(scope="module")
def cc():
    from paper_2104_02621_b200 import _build
    _build.build()
    import paper_2104_02621_b200.capsconv as cc
    cc.load_library()
    return cc


def _setup(B, oracle_mod):
    from paper_2104_02621_b200.stack import LayerSpec
    specs = [LayerSpec(*l) for l in capsinputs.STACK_LAYERS]
    layers = capsinputs.stack_layers(B, oracle_mod.output_dims)
    Ks = [capsinputs.make_kernel(L, dtype=torch.bfloat16, layer_idx=i) for i, L in enumerate(layers)]
    P = capsinputs.primary_layer(B)
    img = capsinputs.make_input(P, dtype=torch.bfloat16, layer_idx=capsinputs.PRIMARY_SEED_LAYER)
    Kp = capsinputs.make_kernel(P, dtype=torch.bfloat16, layer_idx=capsinputs.PRIMARY_SEED_LAYER)
    h, w = capsinputs.STACK_INPUT["H"], capsinputs.STACK_INPUT["W"]
    for s in specs:
        h, w = oracle_mod.output_dims(h, w, s.KH, s.KW, s.stride)
    dY = capsinputs.make_grad_output((B, h, w, specs[-1].Cout, 4, 4), dtype=torch.bfloat16, layer_idx=len(specs))
    return specs, Ks, img, Kp, dY


@pytest.mark.parametrize("B", [3, 32])
@pytest.mark.parametrize("graph", [False, True], ids=["eager", "graph"])
def test_train_step_matches_oracle(cc, oracle_mod, B, graph):
    from paper_2104_02621_b200.train import CapsTrainer
    specs, Ks, img, Kp, dY = _setup(B, oracle_mod)
    si = capsinputs.STACK_INPUT
    lr = capsinputs.TRAIN_LR
    tr = CapsTrainer(specs, si["H"], si["W"], 4, B, Kp, Ks, DEV, lr)
    img_d = img.to(DEV)
    dY_rows = dY.permute(0, 1, 2, 4, 3, 5).contiguous().to(DEV)      # the stack runs in the rows layout
    w0 = [m.clone() for m in [tr.masterP] + tr.masters]
    if graph:
        g, cs = torch.cuda.CUDAGraph(), torch.cuda.Stream()
        cs.wait_stream(torch.cuda.current_stream())
        snap = [m.clone() for m in [tr.masterP] + tr.masters]
        ksnap = [k.clone() for k in [tr.KP] + tr.stack.K]
        with torch.cuda.stream(cs):
            tr.step(img_d, dY_rows)                 # warm-up (workspaces), then restore the weights
            torch.cuda.synchronize()
            for m, s0 in zip([tr.masterP] + tr.masters, snap):
                m.copy_(s0)
            for k, s0 in zip([tr.KP] + tr.stack.K, ksnap):
                k.copy_(s0)
            torch.cuda.synchronize()
            with torch.cuda.graph(g, stream=cs):
                tr.step(img_d, dY_rows)
        for m, s0 in zip([tr.masterP] + tr.masters, snap):
            m.copy_(s0)
        for k, s0 in zip([tr.KP] + tr.stack.K, ksnap):
            k.copy_(s0)
        torch.cuda.synchronize()
        g.replay()
    else:
        tr.step(img_d, dY_rows)
    torch.cuda.synchronize()
    new, rdK, den = oracle_mod.train_step(to_np(img), to_np(Kp), [to_np(k) for k in Ks], [s.stride for s in specs],
                                          to_np(dY), lr, True)
    dks = [tr.dKP] + list(tr.stack.dK)
    names = ["primary"] + ["L%d" % (i + 1) for i in range(len(specs))]
    for name, got, ref, a in zip(names, dks, rdK, den):
        assert_close(to_np(got), ref, a, torch.bfloat16, "dK " + name)
    for name, m, m0, g_, k in zip(names, [tr.masterP] + tr.masters, w0, dks, [tr.KP] + tr.stack.K):
        # the update itself: one fp32 rounding of w - lr*g, with the device's own g
        # and the learning rate as the ABI passes it (an fp32 value)
        want = (to_np(m0) - float(np.float32(lr)) * to_np(g_)).astype(np.float32)
        np.testing.assert_array_max_ulp(m.cpu().numpy(), want, maxulp=1)
        assert torch.equal(k, m.to(torch.bfloat16)), name
    # and the updated weights against the oracle's step: off by lr times the
    # dK error (bounded by the bf16 bar times its abs-sum) plus fp32 rounding
    for name, m, ref, a in zip(names, [tr.masterP] + tr.masters, new, den):
        diff = np.abs(to_np(m) - ref)
        bound = lr * TOL[torch.bfloat16] * np.asarray(a) + 1e-6 * (1 + np.abs(ref))
        assert np.all(diff <= bound), "%s: weights off the oracle's step" % name


def test_sgd_update_exact(cc):
    """capsconv_sgd_update on ragged lengths: master = fp32(w - lr*g) (one
    rounding), bf16 copy = RNE(master), fp32 in place."""
    gen = torch.Generator().manual_seed(5)
    for n in (1, 3, 4, 1001, 4096):
        w = (torch.rand(n, generator=gen) * 4 - 2).to(DEV)
        g = (torch.rand(n, generator=gen) * 4 - 2).to(DEV)
        w0 = w.clone()
        out = torch.empty(n, dtype=torch.bfloat16, device=DEV)
        cc.sgd_update(w, g, 0.125, out)
        torch.cuda.synchronize()
        want = (w0.double() - 0.125 * g.double()).float()
        np.testing.assert_array_max_ulp(w.cpu().numpy(), want.cpu().numpy(), maxulp=1)
        assert torch.equal(out, w.to(torch.bfloat16))
        w2 = w0.clone()
        cc.sgd_update(w2, g, 0.125)               # fp32 working copy = the master itself
        torch.cuda.synchronize()
        assert torch.equal(w2, w)


PRIMARY_CASES = [
    # B, H, W, K, N (= Cout * D3), Cout
    (3, 28, 28, 5, 128, 1),
    (2, 11, 9, 3, 32, 1),
    (2, 13, 17, 7, 64, 2),
    (1, 9, 12, 5, 256, 4),
    (2, 15, 14, 7, 128, 1),      # tensor-core dK with 49 taps; CUDA-core forward (49 > 32 taps)
    (3, 10, 12, 3, 128, 2),      # tensor-core fwd and dK with 9 taps, Cout = 2
]


@pytest.mark.parametrize("case", PRIMARY_CASES, ids=lambda c: "x".join(map(str, c)))
@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32], ids=["bf16", "f32"])
def test_primary_layer_kernels(cc, oracle_mod, case, dtype):
    """The one-channel plain-convolution kernels (csrc/primary.cu: C = D1 = D2
    = 1; tcgen05 for bf16 with 128 channels, CUDA cores otherwise) against the
    oracle, fwd and dK, random data; also exact-integer data bitwise (sums of
    at most 49 products of small integers; ragged last 128-pixel tiles)."""
    B, H, W, K, N, Cout = case
    L = capsinputs.Layer(B=B, H=H, W=W, C=1, Cout=Cout, KH=K, KW=K, D1=1, D2=1, D3=N // Cout, stride=1)
    Ho, Wo = H - K + 1, W - K + 1
    for kind in ("uniform", "int"):
        img = capsinputs.make_input(L, kind, dtype)
        Kp = capsinputs.make_kernel(L, kind, dtype)
        dO = capsinputs.make_grad_output(L.o_shape(Ho, Wo), kind, dtype)
        O = cc.fwd(img.to(DEV), Kp.to(DEV), 1)
        dK = cc.bwd_kernel(img.to(DEV), dO.to(DEV), 1, K, K)
        torch.cuda.synchronize()
        rO, aO = oracle_mod.fwd(to_np(img), to_np(Kp), 1)
        rdK, adK = oracle_mod.bwd_kernel(to_np(img), to_np(dO), 1, K, K)
        if kind == "int":
            want = oracle_mod.round_bf16(rO) if dtype == torch.bfloat16 else rO
            np.testing.assert_array_equal(to_np(O), want)
            np.testing.assert_array_equal(to_np(dK), rdK)
        else:
            assert_close(to_np(O), rO, aO, dtype, "primary fwd")
            assert_close(to_np(dK), rdK, adK, torch.float32, "primary dK")
