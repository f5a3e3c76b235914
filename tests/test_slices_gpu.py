"""GPU parity of S-slice capsules (reading R22)
through the C ABI's *_slices entry points against the oracle's slice-wise
functions (pinned to the matrix oracle per slice, tests/test_oracle_pins.py).
Both kernel paths: 4x4 capsules in bf16 take the tensor-core kernels on the
channel-expanded problem, 3x3 / fp32 the SIMT kernels."""
import numpy as np
import pytest
import torch

from helpers import assert_close, to_np

pytestmark = pytest.mark.gpu
DEV = "cuda:0"

# B, H, W, C, Cout, KH, KW, S, D, s
CASES = [
    (2, 9, 9, 4, 4, 3, 3, 2, 4, 1),
    (2, 10, 10, 4, 8, 3, 3, 3, 4, 2),
    (3, 7, 7, 2, 3, 3, 3, 3, 3, 1),      # rank-3 3x3x3 capsules (Fig 2's kind)
    (20, 5, 5, 8, 4, 5, 5, 2, 4, 1),     # full extent (FC view) with slices
]


@pytest.fixture(scope="module")
def cc():
    from paper_2104_02621_b200 import _build
    _build.build()
    import paper_2104_02621_b200.capsconv as cc
    cc.load_library()
    return cc


def _tensors(case, dtype, kind):
    B, H, W, C, Co, KH, KW, S, D, s = case
    g = torch.Generator().manual_seed(sum(case))
    Ho, Wo = (H - KH) // s + 1, (W - KW) // s + 1
    def draw(shape):
        if kind == "int":
            return torch.randint(-1, 2, shape, generator=g).to(dtype)
        return (torch.rand(shape, generator=g) * 2 - 1).to(dtype)
    return (draw((B, H, W, C, S, D, D)), draw((KH, KW, C, Co, S, D, D)), draw((B, Ho, Wo, Co, S, D, D)))


@pytest.mark.parametrize("case", CASES)
@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16], ids=["f32", "bf16"])
def test_slices_parity(cc, oracle_mod, case, dtype):
    B, H, W, C, Co, KH, KW, S, D, s = case
    I, K, dO = _tensors(case, dtype, "uniform")
    O = cc.fwd_slices(I.to(DEV), K.to(DEV), s)
    dI = cc.bwd_data_slices(dO.to(DEV), K.to(DEV), s, H, W)
    dK = cc.bwd_kernel_slices(I.to(DEV), dO.to(DEV), s, KH, KW)
    torch.cuda.synchronize()
    rO, aO = oracle_mod.fwd_slices(to_np(I), to_np(K), s)
    rdI, adI = oracle_mod.bwd_data_slices(to_np(dO), to_np(K), s, H, W)
    rdK, adK = oracle_mod.bwd_kernel_slices(to_np(I), to_np(dO), s, KH, KW)
    assert_close(to_np(O), rO, aO, dtype, "fwd_slices")
    assert_close(to_np(dI), rdI, adI, dtype, "bwd_data_slices")
    assert_close(to_np(dK), rdK, adK, torch.float32, "bwd_kernel_slices")


@pytest.mark.parametrize("case", CASES)
def test_slices_exact(cc, oracle_mod, case):
    B, H, W, C, Co, KH, KW, S, D, s = case
    I, K, dO = _tensors(case, torch.bfloat16, "int")
    O = cc.fwd_slices(I.to(DEV), K.to(DEV), s)
    dI = cc.bwd_data_slices(dO.to(DEV), K.to(DEV), s, H, W)
    dK = cc.bwd_kernel_slices(I.to(DEV), dO.to(DEV), s, KH, KW)
    torch.cuda.synchronize()
    rO, _ = oracle_mod.fwd_slices(to_np(I), to_np(K), s)
    rdI, _ = oracle_mod.bwd_data_slices(to_np(dO), to_np(K), s, H, W)
    rdK, _ = oracle_mod.bwd_kernel_slices(to_np(I), to_np(dO), s, KH, KW)
    np.testing.assert_array_equal(to_np(O), oracle_mod.round_bf16(rO))
    np.testing.assert_array_equal(to_np(dI), oracle_mod.round_bf16(rdI))
    np.testing.assert_array_equal(to_np(dK), rdK)


def test_slices_fig2(cc):
    """PAPER.md:44-53 with 3x3x3 capsules as S = 3 slices: all-ones -> 48s."""
    I = torch.ones((1, 5, 5, 1, 3, 3, 3), dtype=torch.float32, device=DEV)
    K = torch.ones((4, 4, 1, 1, 3, 3, 3), dtype=torch.float32, device=DEV)
    O = cc.fwd_slices(I, K, 1)
    torch.cuda.synchronize()
    assert O.shape == (1, 2, 2, 1, 3, 3, 3) and bool(torch.all(O == 48.0))
