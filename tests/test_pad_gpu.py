"""GPU parity of zero padding (reading R21) through
the C ABI's *_pad entry points, against the oracle's padded functions
(themselves pinned to the unpadded oracle on a numpy-padded input,
tests/test_oracle_pins.py).  Every case runs on the library's own path choice
and on the SIMT path; exact-integer cases are compared bit for bit."""
import numpy as np
import pytest
import torch

import capsinputs
from helpers import assert_close, to_np

pytestmark = pytest.mark.gpu
DEV = "cuda:0"

# B, H, W, C, Cout, KH, KW, s, pad
CASES = [
    (3, 9, 9, 8, 8, 3, 3, 1, 1),        # "same" 3x3
    (2, 10, 11, 8, 16, 3, 3, 2, 1),     # stride 2
    (2, 7, 7, 16, 32, 3, 3, 1, 2),      # pad > (K-1)/2
    (2, 6, 5, 4, 4, 5, 5, 1, 2),        # "same" 5x5, ragged C
    (1, 5, 5, 3, 2, 3, 3, 2, 1),        # odd channels
    (34, 12, 12, 8, 8, 3, 3, 1, 1),     # several M tiles, ragged tail
    (2, 9, 9, 16, 32, 3, 3, 1, 2),      # windows starting/ending inside padding rows
    (2, 10, 11, 8, 16, 3, 3, 2, 2),     # stride 2, pad 2
]


@pytest.fixture(scope="module")
def cc():
    from paper_2104_02621_b200 import _build
    _build.build()
    import paper_2104_02621_b200.capsconv as cc
    cc.load_library()
    yield cc
    cc.set_path_override(cc.PATH_AUTO)


@pytest.fixture(params=["auto", "simt"])
def path(request, cc):
    cc.set_path_override(cc.PATH_AUTO if request.param == "auto" else cc.PATH_SIMT)
    yield request.param
    cc.set_path_override(cc.PATH_AUTO)


def _tensors(case, kind, dtype):
    B, H, W, C, Co, KH, KW, s, pad = case
    L = capsinputs.Layer(B, H, W, C, Co, KH, KW, 4, 4, 4, s)
    I = capsinputs.make_input(L, kind, dtype)
    K = capsinputs.make_kernel(L, kind, dtype)
    Ho, Wo = (H + 2 * pad - KH) // s + 1, (W + 2 * pad - KW) // s + 1
    dO = capsinputs.make_grad_output(L.o_shape(Ho, Wo), kind, dtype)
    return I, K, dO


@pytest.mark.parametrize("case", CASES)
@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16], ids=["f32", "bf16"])
def test_pad_parity(cc, oracle_mod, path, case, dtype):
    B, H, W, C, Co, KH, KW, s, pad = case
    I, K, dO = _tensors(case, "uniform", dtype)
    assert cc.output_dims(H, W, KH, KW, s, pad) == oracle_mod.output_dims(H, W, KH, KW, s, pad)
    Id, Kd, dOd = I.to(DEV), K.to(DEV), dO.to(DEV)
    O = cc.fwd(Id, Kd, s, pad=pad)
    dI = cc.bwd_data(dOd, Kd, s, H, W, pad=pad)
    dK = cc.bwd_kernel(Id, dOd, s, KH, KW, pad=pad)
    torch.cuda.synchronize()
    rO, aO = oracle_mod.fwd(to_np(I), to_np(K), s, pad)
    rdI, adI = oracle_mod.bwd_data(to_np(dO), to_np(K), s, H, W, pad)
    rdK, adK = oracle_mod.bwd_kernel(to_np(I), to_np(dO), s, KH, KW, pad)
    assert_close(to_np(O), rO, aO, dtype, "fwd")
    assert_close(to_np(dI), rdI, adI, dtype, "bwd_data")
    assert_close(to_np(dK), rdK, adK, torch.float32, "bwd_kernel")


@pytest.mark.parametrize("case", CASES)
def test_pad_exact(cc, oracle_mod, path, case):
    """Exact-integer inputs: bitwise equal to the (bf16-rounded) oracle."""
    B, H, W, C, Co, KH, KW, s, pad = case
    I, K, dO = _tensors(case, "int1", torch.bfloat16)
    Id, Kd, dOd = I.to(DEV), K.to(DEV), dO.to(DEV)
    O = cc.fwd(Id, Kd, s, pad=pad)
    dI = cc.bwd_data(dOd, Kd, s, H, W, pad=pad)
    dK = cc.bwd_kernel(Id, dOd, s, KH, KW, pad=pad)
    torch.cuda.synchronize()
    rO, _ = oracle_mod.fwd(to_np(I), to_np(K), s, pad)
    rdI, _ = oracle_mod.bwd_data(to_np(dO), to_np(K), s, H, W, pad)
    rdK, _ = oracle_mod.bwd_kernel(to_np(I), to_np(dO), s, KH, KW, pad)
    np.testing.assert_array_equal(to_np(O), oracle_mod.round_bf16(rO))
    np.testing.assert_array_equal(to_np(dI), oracle_mod.round_bf16(rdI))
    np.testing.assert_array_equal(to_np(dK), rdK)
    if path == "auto" and KH <= 3 and C % 4 == 0 and Co % 4 == 0:
        # bf16 4x4 capsules with padding run on the tensor-core kernels (the tiny
        # odd-channel and 5x5-over-4-channel cases take SIMT for dK, as unpadded)
        ext = (B, H, W, C, Co, KH, KW, 4, 4, 4, s, pad)
        assert [cc.select_path(op, torch.bfloat16, ext) for op in (0, 1, 2)] == [cc.PATH_MMA] * 3


def test_pad_zero_is_unpadded(cc):
    """pad = 0 through the *_pad entry points is the unpadded call, bit for bit."""
    case = (2, 9, 9, 8, 8, 3, 3, 1, 0)
    I, K, dO = _tensors(case, "uniform", torch.bfloat16)
    Id, Kd = I.to(DEV), K.to(DEV)
    a = cc.fwd(Id, Kd, 1, pad=0)
    b = cc.fwd(Id, Kd, 1)
    torch.cuda.synchronize()
    assert torch.equal(a, b)


def test_pad_autograd(cc, oracle_mod):
    """caps_conv2d with padding: gradients are the padded adjoints."""
    case = (2, 8, 8, 8, 8, 3, 3, 1, 1)
    B, H, W, C, Co, KH, KW, s, pad = case
    I, K, dO = _tensors(case, "int1", torch.float32)
    Id = I.to(DEV).requires_grad_(True)
    Kd = K.to(DEV).requires_grad_(True)
    O = cc.caps_conv2d(Id, Kd, s, pad)
    O.backward(dO.to(DEV))
    rdI, _ = oracle_mod.bwd_data(to_np(dO), to_np(K), s, H, W, pad)
    rdK, _ = oracle_mod.bwd_kernel(to_np(I), to_np(dO), s, KH, KW, pad)
    np.testing.assert_array_equal(to_np(Id.grad), rdI)
    np.testing.assert_array_equal(to_np(Kd.grad), rdK)


def test_pad_validation(cc):
    """Negative padding and a kernel larger than the padded input are rejected."""
    with pytest.raises(cc.CapsConvError):
        cc.output_dims(5, 5, 3, 3, 1, -1)
    with pytest.raises(cc.CapsConvError):
        cc.output_dims(2, 2, 7, 7, 1, 2)
    assert cc.output_dims(2, 2, 5, 5, 1, 2) == (2, 2)


def _same_stack_layers(oracle_mod, batch):
    si = capsinputs.STACK_INPUT
    h, w = si["H"], si["W"]
    out = []
    for (C, Co, KH, KW, s, pad) in capsinputs.STACK_SAME_LAYERS:
        out.append((batch, h, w, C, Co, KH, KW, s, pad))
        h, w = oracle_mod.output_dims(h, w, KH, KW, s, pad)
    return out


@pytest.mark.parametrize("li", range(len(capsinputs.STACK_SAME_LAYERS)))
def test_same_stack_layers_full_batch_exact(cc, oracle_mod, li):
    """Each layer of the zero-padded stack (bench.py --config stack_same) at
    global batch 1024, exact-integer inputs: bitwise equal to the oracle, on
    the tensor-core path."""
    case = _same_stack_layers(oracle_mod, capsinputs.STACK_BATCH)[li]
    B, H, W, C, Co, KH, KW, s, pad = case
    L = capsinputs.Layer(B, H, W, C, Co, KH, KW, 4, 4, 4, s)
    I = capsinputs.make_input(L, "int1", torch.bfloat16, layer_idx=li)
    K = capsinputs.make_kernel(L, "int1", torch.bfloat16, layer_idx=li)
    Ho, Wo = oracle_mod.output_dims(H, W, KH, KW, s, pad)
    dO = capsinputs.make_grad_output(L.o_shape(Ho, Wo), "int1", torch.bfloat16, layer_idx=li)
    ext = (B, H, W, C, Co, KH, KW, 4, 4, 4, s, pad)
    assert [cc.select_path(op, torch.bfloat16, ext) for op in (0, 1, 2)] == [cc.PATH_MMA] * 3
    Id, Kd, dOd = I.to(DEV), K.to(DEV), dO.to(DEV)
    O = cc.fwd(Id, Kd, s, pad=pad)
    dI = cc.bwd_data(dOd, Kd, s, H, W, pad=pad)
    dK = cc.bwd_kernel(Id, dOd, s, KH, KW, pad=pad)
    torch.cuda.synchronize()
    rO, _ = oracle_mod.fwd(to_np(I), to_np(K), s, pad)
    rdI, _ = oracle_mod.bwd_data(to_np(dO), to_np(K), s, H, W, pad)
    rdK, _ = oracle_mod.bwd_kernel(to_np(I), to_np(dO), s, KH, KW, pad)
    np.testing.assert_array_equal(to_np(O), oracle_mod.round_bf16(rO))
    np.testing.assert_array_equal(to_np(dI), oracle_mod.round_bf16(rdI))
    np.testing.assert_array_equal(to_np(dK), rdK)
