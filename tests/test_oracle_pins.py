"""Pins for the CPU oracle against things other than itself (no GPU needed).

Each test names the passage or the mathematical fact it relies on.  A
plausible mistake in the oracle (dropped term, wrong sign or index,
transposed operand, wrong stride placement) fails at least one of them:
  * Fig 2 golden value and its backward closed forms (symmetric: catch sum
    length / shape law only);
  * an independent pure-Python brute force (dI in *scatter* form, the
    opposite of the oracle's gather form);
  * the F1 identity with torch.nn.functional.conv2d (fp64) and its autograd
    (catches transposes, orientation and stride errors);
  * the FC degenerate case as an einsum;
  * one-hot placement, the scalar Alg-1 case, the identity kernel;
  * linearity, adjointness, finite differences, and the |term| pass.
"""
import itertools
import os

import numpy as np
import pytest
import torch

import capsinputs

pytestmark = pytest.mark.filterwarnings("ignore")

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _read_golden(name):
    out = {}
    lines = [l.strip() for l in open(os.path.join(GOLDEN, name)) if l.strip() and not l.startswith("#")]
    i = 0
    while i < len(lines):
        parts = lines[i].split()
        key = parts[0]
        if key == "dI_plane":
            rows = [list(map(float, lines[i + 1 + r].split())) for r in range(5)]
            out[key] = np.array(rows)
            i += 6
            continue
        vals = [float(v) for v in parts[1:]]
        out[key] = vals
        i += 1
    return out


def rnd(shape, seed, lo=-1.0, hi=1.0):
    g = np.random.default_rng(seed)
    return g.uniform(lo, hi, size=shape)


# ---------------------------------------------------------------- shape law

def test_shape_law_examples(oracle_mod):
    # PAPER.md:53 (5x5 input, 4x4 kernel -> 2x2); forced cases from the formula
    assert oracle_mod.output_dims(5, 5, 4, 4, 1) == (2, 2)
    assert oracle_mod.output_dims(7, 7, 1, 1, 1) == (7, 7)
    assert oracle_mod.output_dims(28, 28, 3, 3, 2) == (13, 13)
    assert oracle_mod.output_dims(16, 16, 3, 3, 2) == (7, 7)
    assert oracle_mod.output_dims(8, 8, 8, 8, 1) == (1, 1)
    for bad in [(4, 4, 5, 1, 1), (4, 4, 1, 5, 1), (4, 4, 1, 1, 0), (0, 4, 1, 1, 1)]:
        with pytest.raises(oracle_mod.OracleError):
            oracle_mod.output_dims(*bad)


# ---------------------------------------------------------------- Fig 2

def test_fig2_forward_golden(oracle_mod):
    g = _read_golden("fig2_forward.txt")
    I = np.ones([int(v) for v in g["input_shape"]])
    K = np.ones([int(v) for v in g["kernel_shape"]])
    O, A = oracle_mod.fwd(I, K, int(g["stride"][0]))
    assert list(O.shape) == [int(v) for v in g["output_shape"]]
    assert np.all(O == g["output_all"][0])
    assert np.all(A == g["output_all"][0])


def test_fig2_backward_closed_forms(oracle_mod):
    g = _read_golden("fig2_backward.txt")
    I = np.ones((1, 5, 5, 1, 3, 3))
    K = np.ones((4, 4, 1, 1, 3, 3))
    dO = np.ones((1, 2, 2, 1, 3, 3))
    dK, _ = oracle_mod.bwd_kernel(I, dO, 1, 4, 4)
    assert np.all(dK == g["dK_all"][0])
    dI, _ = oracle_mod.bwd_data(dO, K, 1, 5, 5)
    for c, d1, d2 in itertools.product(range(1), range(3), range(3)):
        np.testing.assert_array_equal(dI[0, :, :, c, d1, d2], g["dI_plane"])


# ---------------------------------------------------------------- brute force

def _brute_fwd(I, K, s):
    B, H, W, C, D1, D2 = I.shape
    KH, KW, _, Co, _, D3 = K.shape
    Ho, Wo = (H - KH) // s + 1, (W - KW) // s + 1
    O = np.zeros((B, Ho, Wo, Co, D1, D3))
    for b in range(B):
        for x in range(Ho):
            for y in range(Wo):
                for co in range(Co):
                    for p in range(KH):
                        for q in range(KW):
                            for c in range(C):
                                # (D1 x D2) @ (D2 x D3), PAPER.md:84 / :107
                                a = I[b, x * s + p, y * s + q, c]
                                k = K[p, q, c, co]
                                for i in range(D1):
                                    for j in range(D3):
                                        acc = 0.0
                                        for t in range(D2):
                                            acc += a[i, t] * k[t, j]
                                        O[b, x, y, co, i, j] += acc
    return O


def _brute_bwd(I, K, dO, s):
    """Scatter-form backward: walk every forward term and add its partial
    derivatives (the opposite traversal to the oracle's gather form)."""
    B, H, W, C, D1, D2 = I.shape
    KH, KW, _, Co, _, D3 = K.shape
    _, Ho, Wo, _, _, _ = dO.shape
    dI = np.zeros_like(I)
    dK = np.zeros_like(K)
    for b, x, y, co, p, q, c in itertools.product(range(B), range(Ho), range(Wo), range(Co),
                                                  range(KH), range(KW), range(C)):
        h, w = x * s + p, y * s + q
        for i, j, t in itertools.product(range(D1), range(D3), range(D2)):
            g = dO[b, x, y, co, i, j]
            dI[b, h, w, c, i, t] += g * K[p, q, c, co, t, j]
            dK[p, q, c, co, t, j] += g * I[b, h, w, c, i, t]
    return dI, dK


BRUTE_CASES = [
    # B, H, W, C, Co, KH, KW, D1, D2, D3, s
    (2, 4, 5, 2, 3, 2, 2, 2, 2, 2, 1),
    (1, 5, 5, 1, 2, 3, 2, 3, 2, 1, 2),
    (1, 6, 4, 2, 1, 3, 1, 1, 3, 2, 2),
    (2, 3, 3, 1, 1, 3, 3, 2, 3, 4, 1),
]


@pytest.mark.parametrize("case", BRUTE_CASES)
def test_bruteforce(oracle_mod, case):
    B, H, W, C, Co, KH, KW, D1, D2, D3, s = case
    I = rnd((B, H, W, C, D1, D2), 1)
    K = rnd((KH, KW, C, Co, D2, D3), 2)
    O, _ = oracle_mod.fwd(I, K, s)
    Ob = _brute_fwd(I, K, s)
    np.testing.assert_allclose(O, Ob, rtol=1e-13, atol=1e-13)
    dO = rnd(O.shape, 3)
    dI, _ = oracle_mod.bwd_data(dO, K, s, H, W)
    dK, _ = oracle_mod.bwd_kernel(I, dO, s, KH, KW)
    dIb, dKb = _brute_bwd(I, K, dO, s)
    np.testing.assert_allclose(dI, dIb, rtol=1e-13, atol=1e-13)
    np.testing.assert_allclose(dK, dKb, rtol=1e-13, atol=1e-13)


# ---------------------------------------------------------------- F1: conv2d identity

def _conv2d_view(I, K, s):
    """Capsule conv == conv2d with D1 folded into the batch, C_in=(c,d2),
    C_out=(c',d3).  Library routine in fp64; autograd gives the
    adjoints."""
    B, H, W, C, D1, D2 = I.shape
    KH, KW, _, Co, _, D3 = K.shape
    It = torch.tensor(I, requires_grad=True)
    Kt = torch.tensor(K, requires_grad=True)
    x = It.permute(0, 4, 3, 5, 1, 2).reshape(B * D1, C * D2, H, W)
    wgt = Kt.permute(3, 5, 2, 4, 0, 1).reshape(Co * D3, C * D2, KH, KW)
    y = torch.nn.functional.conv2d(x, wgt, stride=s)
    Ho, Wo = y.shape[-2:]
    O = y.reshape(B, D1, Co, D3, Ho, Wo).permute(0, 4, 5, 2, 1, 3)
    return It, Kt, O


CONV_CASES = [
    (2, 6, 7, 2, 3, 3, 2, 2, 3, 4, 1),
    (1, 7, 7, 3, 2, 3, 3, 4, 4, 4, 2),
    (2, 5, 5, 1, 1, 5, 5, 3, 2, 1, 1),
    (3, 9, 8, 2, 2, 2, 3, 4, 4, 4, 3),
    (1, 8, 8, 4, 2, 8, 8, 4, 4, 4, 1),
]


@pytest.mark.parametrize("case", CONV_CASES)
def test_conv2d_identity(oracle_mod, case):
    B, H, W, C, Co, KH, KW, D1, D2, D3, s = case
    I = rnd((B, H, W, C, D1, D2), 11)
    K = rnd((KH, KW, C, Co, D2, D3), 12)
    It, Kt, Ot = _conv2d_view(I, K, s)
    O, _ = oracle_mod.fwd(I, K, s)
    np.testing.assert_allclose(O, Ot.detach().numpy(), rtol=1e-12, atol=1e-12)
    dO = rnd(O.shape, 13)
    Ot.backward(torch.tensor(dO))
    dI, _ = oracle_mod.bwd_data(dO, K, s, H, W)
    dK, _ = oracle_mod.bwd_kernel(I, dO, s, KH, KW)
    np.testing.assert_allclose(dI, It.grad.numpy(), rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(dK, Kt.grad.numpy(), rtol=1e-12, atol=1e-12)


# ---------------------------------------------------------------- degenerate cases

def test_fc_is_einsum(oracle_mod):
    # FC capsule layer == full-extent capsule conv (reading R18)
    I = rnd((3, 4, 4, 2, 2, 3), 21)
    K = rnd((4, 4, 2, 5, 3, 2), 22)
    O, _ = oracle_mod.fwd(I, K, 1)
    ref = np.einsum("bpqcik,pqcokn->boin", I, K)
    np.testing.assert_allclose(O[:, 0, 0], ref, rtol=1e-12, atol=1e-12)


def test_scalar_case_is_alg1(oracle_mod):
    # D1=D2=D3=1: capsule conv degenerates to scalar convolution (Alg 1,
    # PAPER.md:62-81, read as cross-correlation, R8).  Independent loop:
    I = rnd((2, 6, 5, 3, 1, 1), 31)
    K = rnd((3, 2, 3, 4, 1, 1), 32)
    for s in (1, 2):
        O, _ = oracle_mod.fwd(I, K, s)
        Ho, Wo = (6 - 3) // s + 1, (5 - 2) // s + 1
        ref = np.zeros((2, Ho, Wo, 4))
        for b in range(2):
            for i in range(Ho):
                for j in range(Wo):
                    for m in range(4):
                        ref[b, i, j, m] = sum(I[b, i * s + x, j * s + y, n, 0, 0] * K[x, y, n, m, 0, 0]
                                              for x in range(3) for y in range(2) for n in range(3))
        np.testing.assert_allclose(O[..., 0, 0], ref, rtol=1e-13, atol=1e-13)


def test_identity_kernel(oracle_mod):
    # 1x1 kernel whose capsule is the identity: O == I
    I = rnd((2, 3, 4, 1, 3, 4), 41)
    K = np.eye(4).reshape(1, 1, 1, 1, 4, 4)
    O, _ = oracle_mod.fwd(I, K, 1)
    np.testing.assert_array_equal(O, I)


def test_zero_kernel(oracle_mod):
    I = rnd((1, 5, 5, 2, 2, 2), 42)
    K = np.zeros((3, 3, 2, 3, 2, 2))
    O, _ = oracle_mod.fwd(I, K, 1)
    assert O.shape == (1, 3, 3, 3, 2, 2) and np.all(O == 0)


@pytest.mark.parametrize("s", [1, 2, 3])
def test_one_hot_placement(oracle_mod, s):
    # one-hot I at (b0,h0,w0,c0,i0,t0) and one-hot K at (p0,q0,c0,o0,t0,j0):
    # exactly one nonzero output, at (b0,(h0-p0)/s,(w0-q0)/s,o0,i0,j0)
    B, H, W, C, Co, KH, KW, D1, D2, D3 = 2, 9, 8, 3, 2, 3, 2, 3, 2, 4
    b0, c0, i0, t0, o0, j0 = 1, 2, 1, 1, 1, 3
    Ho, Wo = (H - KH) // s + 1, (W - KW) // s + 1
    for (x0, y0, p0, q0) in [(1, 2, 2, 1), (0, 0, 0, 0), (Ho - 1, Wo - 1, KH - 1, KW - 1)]:
        h0, w0 = x0 * s + p0, y0 * s + q0
        I = np.zeros((B, H, W, C, D1, D2))
        I[b0, h0, w0, c0, i0, t0] = 1.0
        K = np.zeros((KH, KW, C, Co, D2, D3))
        K[p0, q0, c0, o0, t0, j0] = 2.0
        O, _ = oracle_mod.fwd(I, K, s)
        nz = np.argwhere(O != 0)
        assert nz.tolist() == [[b0, x0, y0, o0, i0, j0]]
        assert O[b0, x0, y0, o0, i0, j0] == 2.0
    # an input position between strided windows meets no tap with a matching K
    if s > 1:
        I = np.zeros((B, H, W, C, D1, D2))
        I[0, 1, 1, 0, 0, 0] = 1.0
        K = np.zeros((KH, KW, C, Co, D2, D3))
        K[0, 0, 0, 0, 0, 0] = 1.0
        O, _ = oracle_mod.fwd(I, K, s)
        assert np.all(O == 0)


# ---------------------------------------------------------------- invariants

def test_linearity(oracle_mod):
    I = rnd((2, 6, 6, 2, 3, 2), 51)
    K1 = rnd((3, 3, 2, 2, 2, 3), 52)
    K2 = rnd((3, 3, 2, 2, 2, 3), 53)
    O, _ = oracle_mod.fwd(I, K1, 1)
    for a in (-1.0, 0.5, 3.0):
        Oa, _ = oracle_mod.fwd(a * I, K1, 1)
        np.testing.assert_allclose(Oa, a * O, rtol=1e-12, atol=1e-12)
        Ob, _ = oracle_mod.fwd(I, a * K1, 1)
        np.testing.assert_allclose(Ob, a * O, rtol=1e-12, atol=1e-12)
    O12, _ = oracle_mod.fwd(I, K1 + K2, 1)
    O2, _ = oracle_mod.fwd(I, K2, 1)
    np.testing.assert_allclose(O12, O + O2, rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("s", [1, 2])
def test_adjoint_identity(oracle_mod, s):
    # <O, dO> = <I, dI> = <K, dK> = sum I*K*dO
    I = rnd((2, 7, 6, 3, 2, 3), 61)
    K = rnd((3, 2, 3, 2, 3, 2), 62)
    O, _ = oracle_mod.fwd(I, K, s)
    dO = rnd(O.shape, 63)
    dI, _ = oracle_mod.bwd_data(dO, K, s, 7, 6)
    dK, _ = oracle_mod.bwd_kernel(I, dO, s, 3, 2)
    a = np.sum(O * dO)
    assert abs(np.sum(I * dI) - a) <= 1e-11 * max(1.0, abs(a))
    assert abs(np.sum(K * dK) - a) <= 1e-11 * max(1.0, abs(a))


def test_finite_differences(oracle_mod):
    # L = sum O^2 / 2, dO = O, central differences, h = 1e-5
    B, H, W, C, Co, KH, KW, D1, D2, D3, s = 1, 4, 4, 2, 2, 2, 2, 2, 2, 2, 1
    I = rnd((B, H, W, C, D1, D2), 71)
    K = rnd((KH, KW, C, Co, D2, D3), 72)

    def loss(I_, K_):
        O_, _ = oracle_mod.fwd(I_, K_, s)
        return 0.5 * np.sum(O_ * O_)

    O, _ = oracle_mod.fwd(I, K, s)
    dI, _ = oracle_mod.bwd_data(O, K, s, H, W)
    dK, _ = oracle_mod.bwd_kernel(I, O, s, KH, KW)
    h = 1e-5
    g = np.random.default_rng(7)
    for _ in range(12):
        idx = tuple(int(g.integers(n)) for n in I.shape)
        Ip, Im = I.copy(), I.copy()
        Ip[idx] += h
        Im[idx] -= h
        fd = (loss(Ip, K) - loss(Im, K)) / (2 * h)
        assert abs(fd - dI[idx]) <= 1e-6 * max(1.0, abs(fd))
        idx = tuple(int(g.integers(n)) for n in K.shape)
        Kp, Km = K.copy(), K.copy()
        Kp[idx] += h
        Km[idx] -= h
        fd = (loss(I, Kp) - loss(I, Km)) / (2 * h)
        assert abs(fd - dK[idx]) <= 1e-6 * max(1.0, abs(fd))


def test_abs_pass_is_conv_of_abs(oracle_mod):
    # sum |a*b| = sum |a|*|b|: the abs pass equals the value pass on |inputs|
    I = rnd((2, 6, 5, 2, 3, 2), 81)
    K = rnd((2, 3, 2, 3, 2, 2), 82)
    O, A = oracle_mod.fwd(I, K, 2)
    Oa, _ = oracle_mod.fwd(np.abs(I), np.abs(K), 2)
    np.testing.assert_allclose(A, Oa, rtol=1e-13)
    dO = rnd(O.shape, 83)
    _, dIa = oracle_mod.bwd_data(dO, K, 2, 6, 5)
    dIv, _ = oracle_mod.bwd_data(np.abs(dO), np.abs(K), 2, 6, 5)
    np.testing.assert_allclose(dIa, dIv, rtol=1e-13)
    _, dKa = oracle_mod.bwd_kernel(I, dO, 2, 2, 3)
    dKv, _ = oracle_mod.bwd_kernel(np.abs(I), np.abs(dO), 2, 2, 3)
    np.testing.assert_allclose(dKa, dKv, rtol=1e-13)


def test_round_bf16_matches_ieee_cast(oracle_mod):
    # torch's fp32 -> bf16 cast is IEEE round-to-nearest-even
    g = torch.Generator().manual_seed(5)
    x = (torch.randn(20000, generator=g) * torch.exp2(torch.randint(-30, 30, (20000,), generator=g).float()))
    ties = torch.tensor([1.0 + 2.0 ** -8, 1.0 + 3 * 2.0 ** -8, -(1.0 + 2.0 ** -8), 0.0, 2.0 ** -130])
    x = torch.cat([x, ties])
    ref = x.to(torch.bfloat16).double().numpy()
    got = oracle_mod.round_bf16(x.double().numpy())
    np.testing.assert_array_equal(got, ref)


def test_integer_inputs_are_exact(oracle_mod):
    # exact-integer inputs (capsinputs kind="int") give integer outputs
    L = capsinputs.Layer(B=2, H=6, W=6, C=3, Cout=2, KH=3, KW=3, D1=4, D2=4, D3=4, stride=1)
    I = capsinputs.make_input(L, "int").numpy()
    K = capsinputs.make_kernel(L, "int").numpy()
    O, _ = oracle_mod.fwd(I, K, 1)
    assert np.all(O == np.round(O))


def test_stack_depth1_and_fd(oracle_mod):
    # depth-1 stack == the layer; tiny 2-layer stack passes finite differences
    I = rnd((1, 5, 5, 2, 2, 2), 91)
    K1 = rnd((2, 2, 2, 2, 2, 2), 92)
    K2 = rnd((2, 2, 2, 1, 2, 2), 93)
    O1, _ = oracle_mod.fwd(I, K1, 1)
    dY = rnd(O1.shape, 94)
    acts, dX, dKs, _ = oracle_mod.stack_fwd_bwd(I, [K1], [1], dY, False)
    np.testing.assert_array_equal(acts[1], O1)
    dI1, _ = oracle_mod.bwd_data(dY, K1, 1, 5, 5)
    np.testing.assert_array_equal(dX, dI1)

    def loss(I_, K1_, K2_):
        a, _ = oracle_mod.fwd(I_, K1_, 1)
        b, _ = oracle_mod.fwd(a, K2_, 2)
        return 0.5 * np.sum(b * b)

    a1, _ = oracle_mod.fwd(I, K1, 1)
    y, _ = oracle_mod.fwd(a1, K2, 2)
    _, dX, dKs, _ = oracle_mod.stack_fwd_bwd(I, [K1, K2], [1, 2], y, False)
    h = 1e-5
    for idx in [(0, 1, 2, 1, 0, 1), (0, 4, 4, 0, 1, 0)]:
        Ip, Im = I.copy(), I.copy()
        Ip[idx] += h
        Im[idx] -= h
        fd = (loss(Ip, K1, K2) - loss(Im, K1, K2)) / (2 * h)
        assert abs(fd - dX[idx]) <= 1e-6 * max(1.0, abs(fd))
    for idx in [(1, 0, 1, 1, 0, 1), (0, 1, 0, 0, 1, 1)]:
        Kp, Km = K1.copy(), K1.copy()
        Kp[idx] += h
        Km[idx] -= h
        fd = (loss(I, Kp, K2) - loss(I, Km, K2)) / (2 * h)
        assert abs(fd - dKs[0][idx]) <= 1e-6 * max(1.0, abs(fd))


def test_stack_bf16_boundaries_chain(oracle_mod):
    """Reading R13: with bf16_boundaries the oracle stack rounds each layer's
    forward output and each propagated dI to bf16 (RNE) -- and nothing else.
    Pinned against a hand-composed 2-layer chain built from independent
    pieces: torch conv2d in fp64 on the F1 view (autograd for dI, dK) and
    torch's IEEE bfloat16 cast.  Inputs are small dyadic rationals (multiples
    of 1/4, dY of 1/64), so every fp64 sum is exact and the roundings are the
    only inexact steps."""
    g = np.random.default_rng(2024)
    q = lambda shape: g.integers(-4, 5, size=shape) / 4.0
    X = q((2, 9, 9, 3, 4, 4))
    K1 = q((3, 3, 3, 5, 4, 4))
    K2 = q((3, 3, 5, 2, 4, 4))
    bf = lambda t: t.detach().to(torch.bfloat16).to(torch.float64)

    def layer(I, K, s, dO=None):
        It, Kt, O = _conv2d_view(I, K, s)
        if dO is None:
            return O.detach()
        O.backward(torch.as_tensor(dO))
        return It.grad, Kt.grad

    a1 = bf(layer(X, K1, 1))                       # rounded activation
    y = bf(layer(a1.numpy(), K2, 2))
    dY = g.integers(-100, 101, size=tuple(y.shape)) / 64.0   # more significant bits than bf16 keeps
    dI2, dK2 = layer(a1.numpy(), K2, 2, dY)        # dK from the rounded activation
    dI2 = bf(dI2)                                  # rounded propagated gradient
    dX, dK1 = layer(X, K1, 1, dI2.numpy())
    dX = bf(dX)

    acts, rdX, rdKs, _ = oracle_mod.stack_fwd_bwd(X, [K1, K2], [1, 2], dY, True)
    np.testing.assert_array_equal(acts[1], a1.numpy())
    np.testing.assert_array_equal(acts[2], y.numpy())
    np.testing.assert_array_equal(rdX, dX.numpy())
    np.testing.assert_array_equal(rdKs[1], dK2.numpy())   # dK itself is NOT rounded (fp32 output)
    np.testing.assert_array_equal(rdKs[0], dK1.numpy())
    # non-vacuous: the roundings change the activation, the gradients and dK1
    acts0, rdX0, rdKs0, _ = oracle_mod.stack_fwd_bwd(X, [K1, K2], [1, 2], dY, False)
    assert not np.array_equal(acts0[1], acts[1])
    assert not np.array_equal(rdX0, rdX)
    assert not np.array_equal(rdKs0[0], rdKs[0])


# ---------------------------------------------------------------- zero padding
# Pinned to the (already pinned) unpadded oracle run on an explicitly
# zero-padded input -- numpy's pad, not the oracle's own index arithmetic --
# plus the adjoint identities of the padded linear map.
PAD_CASES = [
    # B, H, W, C, Cout, KH, KW, D1, D2, D3, s, pad
    (2, 5, 6, 2, 3, 3, 3, 2, 3, 2, 1, 1),
    (1, 7, 7, 3, 2, 3, 3, 4, 4, 4, 2, 1),
    (2, 4, 5, 1, 2, 2, 3, 3, 2, 4, 1, 2),
    (1, 6, 6, 2, 2, 5, 5, 2, 2, 2, 2, 2),
]


def _pad_inputs(case):
    B, H, W, C, Co, KH, KW, D1, D2, D3, s, pad = case
    rng = np.random.default_rng(hash(case) & 0xffff)
    I = rng.uniform(-1, 1, (B, H, W, C, D1, D2))
    K = rng.uniform(-1, 1, (KH, KW, C, Co, D2, D3))
    Ho, Wo = (H + 2 * pad - KH) // s + 1, (W + 2 * pad - KW) // s + 1
    dO = rng.uniform(-1, 1, (B, Ho, Wo, Co, D1, D3))
    return I, K, dO


def _zero_pad(I, pad):
    return np.pad(I, ((0, 0), (pad, pad), (pad, pad), (0, 0), (0, 0), (0, 0)))


@pytest.mark.parametrize("case", PAD_CASES)
def test_pad_shape_law(oracle_mod, case):
    B, H, W, C, Co, KH, KW, D1, D2, D3, s, pad = case
    assert oracle_mod.output_dims(H, W, KH, KW, s, pad) == ((H + 2 * pad - KH) // s + 1, (W + 2 * pad - KW) // s + 1)
    # "same" capsule convolution: 3x3, stride 1, pad 1 keeps the spatial size
    assert oracle_mod.output_dims(9, 7, 3, 3, 1, 1) == (9, 7)


@pytest.mark.parametrize("case", PAD_CASES)
def test_pad_equals_unpadded_on_zero_padded_input(oracle_mod, case):
    B, H, W, C, Co, KH, KW, D1, D2, D3, s, pad = case
    I, K, dO = _pad_inputs(case)
    Ip = _zero_pad(I, pad)
    O, _ = oracle_mod.fwd(I, K, s, pad)
    Or, _ = oracle_mod.fwd(Ip, K, s)
    np.testing.assert_allclose(O, Or, rtol=0, atol=1e-13)
    # dK of the padded conv = dK of the plain conv on the padded input
    dK, _ = oracle_mod.bwd_kernel(I, dO, s, KH, KW, pad)
    dKr, _ = oracle_mod.bwd_kernel(Ip, dO, s, KH, KW)
    np.testing.assert_allclose(dK, dKr, rtol=0, atol=1e-12)
    # dI of the padded conv = the interior of dI of the plain conv on the padded grid
    dI, _ = oracle_mod.bwd_data(dO, K, s, H, W, pad)
    dIr, _ = oracle_mod.bwd_data(dO, K, s, H + 2 * pad, W + 2 * pad)
    np.testing.assert_allclose(dI, dIr[:, pad:pad + H, pad:pad + W], rtol=0, atol=1e-12)


@pytest.mark.parametrize("case", PAD_CASES)
def test_pad_adjoint_identities(oracle_mod, case):
    """<fwd(I), dO> = <I, dI(dO)> = <K, dK(I, dO)> for the padded map."""
    B, H, W, C, Co, KH, KW, D1, D2, D3, s, pad = case
    I, K, dO = _pad_inputs(case)
    O, _ = oracle_mod.fwd(I, K, s, pad)
    dI, _ = oracle_mod.bwd_data(dO, K, s, H, W, pad)
    dK, _ = oracle_mod.bwd_kernel(I, dO, s, KH, KW, pad)
    a = float(np.sum(O * dO))
    assert abs(a - float(np.sum(I * dI))) <= 1e-10 * max(1.0, abs(a))
    assert abs(a - float(np.sum(K * dK))) <= 1e-10 * max(1.0, abs(a))


# ---------------------------------------------------------------- S-slice capsules
SLICE_CASES = [
    # B, H, W, C, Cout, KH, KW, S, D1, D2, D3, s
    (2, 5, 6, 2, 3, 3, 3, 2, 2, 3, 2, 1),
    (1, 7, 7, 3, 2, 3, 3, 3, 3, 3, 3, 2),
    (2, 4, 5, 1, 2, 2, 3, 1, 4, 4, 4, 1),
]


def _slice_inputs(case):
    B, H, W, C, Co, KH, KW, S, D1, D2, D3, s = case
    rng = np.random.default_rng(sum(case))
    Ho, Wo = (H - KH) // s + 1, (W - KW) // s + 1
    return (rng.uniform(-1, 1, (B, H, W, C, S, D1, D2)), rng.uniform(-1, 1, (KH, KW, C, Co, S, D2, D3)),
            rng.uniform(-1, 1, (B, Ho, Wo, Co, S, D1, D3)))


@pytest.mark.parametrize("case", SLICE_CASES)
def test_slices_are_independent_matrix_convolutions(oracle_mod, case):
    """Slice s of every result is the (pinned) matrix-capsule oracle applied to
    slice s of the operands (numpy slicing, not the oracle's own indexing)."""
    B, H, W, C, Co, KH, KW, S, D1, D2, D3, s = case
    I, K, dO = _slice_inputs(case)
    O, _ = oracle_mod.fwd_slices(I, K, s)
    dI, _ = oracle_mod.bwd_data_slices(dO, K, s, H, W)
    dK, _ = oracle_mod.bwd_kernel_slices(I, dO, s, KH, KW)
    for sl in range(S):
        Or, _ = oracle_mod.fwd(I[:, :, :, :, sl], K[:, :, :, :, sl], s)
        dIr, _ = oracle_mod.bwd_data(dO[:, :, :, :, sl], K[:, :, :, :, sl], s, H, W)
        dKr, _ = oracle_mod.bwd_kernel(I[:, :, :, :, sl], dO[:, :, :, :, sl], s, KH, KW)
        np.testing.assert_allclose(O[:, :, :, :, sl], Or, rtol=0, atol=1e-12)
        np.testing.assert_allclose(dI[:, :, :, :, sl], dIr, rtol=0, atol=1e-12)
        np.testing.assert_allclose(dK[:, :, :, :, sl], dKr, rtol=0, atol=1e-12)


def test_slices_fig2_rank3_reading(oracle_mod):
    """PAPER.md:44-53 with 3x3x3 capsules read as S = 3 slices of 3x3: all-ones
    5x5 input, all-ones 4x4 kernel -> 2x2 output of 48s (16 taps x inner dim 3)."""
    I = np.ones((1, 5, 5, 1, 3, 3, 3))
    K = np.ones((4, 4, 1, 1, 3, 3, 3))
    O, _ = oracle_mod.fwd_slices(I, K, 1)
    assert O.shape == (1, 2, 2, 1, 3, 3, 3)
    assert np.all(O == 48.0)


@pytest.mark.parametrize("case", SLICE_CASES)
def test_slices_adjoint_identities(oracle_mod, case):
    B, H, W, C, Co, KH, KW, S, D1, D2, D3, s = case
    I, K, dO = _slice_inputs(case)
    O, _ = oracle_mod.fwd_slices(I, K, s)
    dI, _ = oracle_mod.bwd_data_slices(dO, K, s, H, W)
    dK, _ = oracle_mod.bwd_kernel_slices(I, dO, s, KH, KW)
    a = float(np.sum(O * dO))
    assert abs(a - float(np.sum(I * dI))) <= 1e-10 * max(1.0, abs(a))
    assert abs(a - float(np.sum(K * dK))) <= 1e-10 * max(1.0, abs(a))
