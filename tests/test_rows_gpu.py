"""GPU parity of the D1-outer ("rows") layout: libcapsconv through its C ABI
(capsconv_*_ex, layout CAPSCONV_LAYOUT_ROWS) against the CPU oracle.

Inputs are generated in the natural layout (capsinputs), permuted to
(B, H, W, D1, C, D2) for the call and the results permuted back, so the
oracle is untouched.  The rows layout runs its own TMA-fed tensor-core
kernels where they apply (bf16, 4x4 capsules) and the natural path between
two permutations otherwise; both are covered.  Full-size stack layers are
checked bit-exactly on exact-integer inputs (every sum is an integer below
2^24, bf16 outputs must equal RNE_bf16(exact))."""
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
    yield cc
    cc.set_path_override(cc.PATH_AUTO)


def to_rows(t):      # natural (B,H,W,C,D1,D2) -> rows (B,H,W,D1,C,D2)
    return t.permute(0, 1, 2, 4, 3, 5).contiguous()


def from_rows(t):    # rows -> natural
    return t.permute(0, 1, 2, 4, 3, 5).contiguous()


def run_rows(cc, L, I, K, dO):
    Id, Kd, dOd = to_rows(I.to(DEV)), K.to(DEV), to_rows(dO.to(DEV))
    O = cc.fwd(Id, Kd, L.stride, layout="rows")
    dI = cc.bwd_data(dOd, Kd, L.stride, L.H, L.W, layout="rows")
    dK = cc.bwd_kernel(Id, dOd, L.stride, L.KH, L.KW, layout="rows")
    torch.cuda.synchronize()
    return from_rows(O), from_rows(dI), dK


def ext_of(L):
    return (L.B, L.H, L.W, L.C, L.Cout, L.KH, L.KW, L.D1, L.D2, L.D3, L.stride)


SMALL = [
    # B, H, W, C, Cout, KH, KW, D1, D2, D3, s
    (2, 9, 11, 4, 8, 3, 3, 4, 4, 4, 1),
    (3, 10, 9, 8, 8, 3, 3, 4, 4, 4, 2),
    (2, 8, 8, 32, 12, 8, 8, 4, 4, 4, 1),
    (1, 12, 40, 8, 8, 3, 3, 4, 4, 4, 1),
    (5, 7, 7, 16, 32, 3, 3, 4, 4, 4, 2),
    (3, 13, 6, 4, 16, 2, 3, 4, 4, 4, 3),
    (2, 6, 5, 2, 3, 2, 3, 2, 3, 5, 1),
    (4, 11, 11, 8, 16, 1, 1, 4, 4, 4, 1),
    (2, 34, 17, 8, 8, 3, 3, 4, 4, 4, 1),
    (3, 12, 12, 16, 16, 5, 5, 4, 4, 4, 1),
    (2, 9, 9, 8, 4, 3, 3, 4, 4, 4, 1),
]


@pytest.mark.parametrize("case", SMALL, ids=lambda c: "x".join(map(str, c)))
@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32], ids=["bf16", "f32"])
def test_rows_small_random(cc, oracle_mod, case, dtype):
    L = capsinputs.Layer(*case)
    I = capsinputs.make_input(L, "uniform", dtype)
    K = capsinputs.make_kernel(L, "uniform", dtype)
    Ho, Wo = oracle_mod.output_dims(L.H, L.W, L.KH, L.KW, L.stride)
    dO = capsinputs.make_grad_output(L.o_shape(Ho, Wo), "uniform", dtype)
    O, dI, dK = run_rows(cc, L, I, K, dO)
    rO, aO = oracle_mod.fwd(to_np(I), to_np(K), L.stride)
    rdI, adI = oracle_mod.bwd_data(to_np(dO), to_np(K), L.stride, L.H, L.W)
    rdK, adK = oracle_mod.bwd_kernel(to_np(I), to_np(dO), L.stride, L.KH, L.KW)
    assert_close(to_np(O), rO, aO, dtype, "rows fwd")
    assert_close(to_np(dI), rdI, adI, dtype, "rows bwd_data")
    assert_close(to_np(dK), rdK, adK, torch.float32, "rows bwd_kernel")


@pytest.mark.parametrize("case", SMALL[:6], ids=lambda c: "x".join(map(str, c)))
def test_rows_small_exact(cc, oracle_mod, case):
    """Exact-integer bf16 inputs: bitwise (order-independent sums)."""
    L = capsinputs.Layer(*case)
    dt = torch.bfloat16
    I = capsinputs.make_input(L, "int", dt)
    K = capsinputs.make_kernel(L, "int", dt)
    Ho, Wo = oracle_mod.output_dims(L.H, L.W, L.KH, L.KW, L.stride)
    dO = capsinputs.make_grad_output(L.o_shape(Ho, Wo), "int", dt)
    O, dI, dK = run_rows(cc, L, I, K, dO)
    rO, _ = oracle_mod.fwd(to_np(I), to_np(K), L.stride)
    rdI, _ = oracle_mod.bwd_data(to_np(dO), to_np(K), L.stride, L.H, L.W)
    rdK, _ = oracle_mod.bwd_kernel(to_np(I), to_np(dO), L.stride, L.KH, L.KW)
    np.testing.assert_array_equal(to_np(O), oracle_mod.round_bf16(rO))
    np.testing.assert_array_equal(to_np(dI), oracle_mod.round_bf16(rdI))
    np.testing.assert_array_equal(to_np(dK), rdK)


def _stack_layers():
    import oracle
    return capsinputs.stack_layers(capsinputs.STACK_BATCH, oracle.output_dims)


@pytest.mark.parametrize("li", [0, 1, 2, 3], ids=["L1", "L2", "L3", "FC"])
def test_rows_stack_layers_full_batch_exact(cc, oracle_mod, li):
    """Each config-5 stack layer at batch 1024 in the rows layout (the launch
    configuration bench.py times), exact-integer inputs in {-1, 0, 1}."""
    L = _stack_layers()[li]
    dt = torch.bfloat16
    I = capsinputs.make_input(L, "int1", dt, layer_idx=li)
    K = capsinputs.make_kernel(L, "int1", dt, layer_idx=li)
    Ho, Wo = oracle_mod.output_dims(L.H, L.W, L.KH, L.KW, L.stride)
    dO = capsinputs.make_grad_output(L.o_shape(Ho, Wo), "int1", dt, layer_idx=li)
    O, dI, dK = run_rows(cc, L, I, K, dO)
    rO, _ = oracle_mod.fwd(to_np(I), to_np(K), L.stride)
    rdI, _ = oracle_mod.bwd_data(to_np(dO), to_np(K), L.stride, L.H, L.W)
    rdK, _ = oracle_mod.bwd_kernel(to_np(I), to_np(dO), L.stride, L.KH, L.KW)
    assert np.abs(rdK).max() < 2 ** 24
    # every layer runs the rows-layout tensor-core kernels on every pass
    for op in (cc.OP_FWD, cc.OP_BWD_DATA, cc.OP_BWD_KERNEL):
        assert cc.select_path(op, dt, ext_of(L), "rows") == cc.PATH_MMA, op
    np.testing.assert_array_equal(to_np(O), oracle_mod.round_bf16(rO))
    np.testing.assert_array_equal(to_np(dI), oracle_mod.round_bf16(rdI))
    np.testing.assert_array_equal(to_np(dK), rdK)


@pytest.mark.parametrize("cfg", ["layer_s1", "layer_s2", "fc"])
def test_rows_configs_full_exact(cc, oracle_mod, cfg):
    """BASELINE.json configs 2-4 at their full batch in the rows layout (the
    launch configuration of bench.py --config), exact-integer inputs."""
    L = capsinputs.CONFIGS[cfg]
    dt = torch.bfloat16
    I = capsinputs.make_input(L, "int1", dt)
    K = capsinputs.make_kernel(L, "int1", dt)
    Ho, Wo = oracle_mod.output_dims(L.H, L.W, L.KH, L.KW, L.stride)
    dO = capsinputs.make_grad_output(L.o_shape(Ho, Wo), "int1", dt)
    for op in (cc.OP_FWD, cc.OP_BWD_DATA, cc.OP_BWD_KERNEL):
        assert cc.select_path(op, dt, ext_of(L), "rows") == cc.PATH_MMA, op
    O, dI, dK = run_rows(cc, L, I, K, dO)
    rO, _ = oracle_mod.fwd(to_np(I), to_np(K), L.stride)
    rdI, _ = oracle_mod.bwd_data(to_np(dO), to_np(K), L.stride, L.H, L.W)
    rdK, _ = oracle_mod.bwd_kernel(to_np(I), to_np(dO), L.stride, L.KH, L.KW)
    assert np.abs(rdK).max() < 2 ** 24
    np.testing.assert_array_equal(to_np(O), oracle_mod.round_bf16(rO))
    np.testing.assert_array_equal(to_np(dI), oracle_mod.round_bf16(rdI))
    np.testing.assert_array_equal(to_np(dK), rdK)


FC_CASES = [
    # B, S (= H = W = KH = KW), C, Cout: full-extent (fully-connected) layers on
    # the rows-layout GEMMs -- ragged batch tiles, several pixels, Cout < 16
    (64, 8, 32, 10),
    (37, 4, 32, 16),
    (96, 2, 64, 10),
    (32, 3, 32, 4),
]


@pytest.mark.parametrize("case", FC_CASES, ids=lambda c: "x".join(map(str, c)))
def test_rows_fc_exact(cc, oracle_mod, case):
    B, S, C, Co = case
    L = capsinputs.Layer(B, S, S, C, Co, S, S, 4, 4, 4, 1)
    dt = torch.bfloat16
    I = capsinputs.make_input(L, "int1", dt)
    K = capsinputs.make_kernel(L, "int1", dt)
    dO = capsinputs.make_grad_output(L.o_shape(1, 1), "int1", dt)
    assert cc.select_path(cc.OP_FWD, dt, ext_of(L), "rows") == cc.PATH_MMA
    O, dI, dK = run_rows(cc, L, I, K, dO)
    rO, _ = oracle_mod.fwd(to_np(I), to_np(K), 1)
    rdI, _ = oracle_mod.bwd_data(to_np(dO), to_np(K), 1, S, S)
    rdK, _ = oracle_mod.bwd_kernel(to_np(I), to_np(dO), 1, S, S)
    np.testing.assert_array_equal(to_np(O), oracle_mod.round_bf16(rO))
    np.testing.assert_array_equal(to_np(dI), oracle_mod.round_bf16(rdI))
    np.testing.assert_array_equal(to_np(dK), rdK)


WALK_CASES = [
    # B, H, W, C, Cout, KH, KW, D1, D2, D3, s: the row-walk kernel (rows_walk.cu) --
    # G = 2 and 4 images per tile with a ragged last group, 32-pixel x tiles,
    # more output rows than accumulator slots (ring wrap), KW = 2 / 4, two
    # source chunks, 16-column rows, stride-2 phase planes
    (3, 10, 12, 8, 8, 3, 3, 4, 4, 4, 1),
    (2, 20, 40, 8, 8, 3, 3, 4, 4, 4, 1),
    (5, 9, 6, 8, 4, 3, 2, 4, 4, 4, 1),
    (2, 23, 23, 8, 16, 3, 3, 4, 4, 4, 2),
    (2, 14, 70, 8, 8, 3, 3, 4, 4, 4, 2),
    (2, 12, 12, 16, 16, 3, 4, 4, 4, 4, 1),
    (1, 30, 9, 32, 16, 2, 3, 4, 4, 4, 1),
    (2, 12, 12, 8, 4, 5, 3, 4, 4, 4, 1),
    (2, 32, 32, 8, 8, 3, 3, 4, 4, 4, 1),    # dI rows read 34 source pixels, one 32-pixel tile
    (3, 16, 16, 16, 32, 3, 3, 4, 4, 4, 2),  # config 3's layer at a small batch
]


@pytest.mark.parametrize("case", WALK_CASES, ids=lambda c: "x".join(map(str, c)))
def test_rows_walk_exact(cc, oracle_mod, case):
    """Exact-integer bf16 inputs through the row-walk forward / dI kernel."""
    L = capsinputs.Layer(*case)
    dt = torch.bfloat16
    I = capsinputs.make_input(L, "int", dt)
    K = capsinputs.make_kernel(L, "int", dt)
    Ho, Wo = oracle_mod.output_dims(L.H, L.W, L.KH, L.KW, L.stride)
    dO = capsinputs.make_grad_output(L.o_shape(Ho, Wo), "int", dt)
    assert cc.select_path(cc.OP_FWD, dt, ext_of(L), "rows") == cc.PATH_MMA
    O, dI, dK = run_rows(cc, L, I, K, dO)
    rO, _ = oracle_mod.fwd(to_np(I), to_np(K), L.stride)
    rdI, _ = oracle_mod.bwd_data(to_np(dO), to_np(K), L.stride, L.H, L.W)
    rdK, _ = oracle_mod.bwd_kernel(to_np(I), to_np(dO), L.stride, L.KH, L.KW)
    np.testing.assert_array_equal(to_np(O), oracle_mod.round_bf16(rO))
    np.testing.assert_array_equal(to_np(dI), oracle_mod.round_bf16(rdI))
    np.testing.assert_array_equal(to_np(dK), rdK)


def test_rows_deterministic(cc):
    L = _stack_layers()[0]
    I = to_rows(capsinputs.make_input(L, dtype=torch.bfloat16).to(DEV))
    dO = torch.randn(L.B, 22, 22, 4, L.Cout, 4, device=DEV).to(torch.bfloat16)
    a = cc.bwd_kernel(I, dO, 1, 3, 3, layout="rows")
    b = cc.bwd_kernel(I, dO, 1, 3, 3, layout="rows")
    assert torch.equal(a, b)


@pytest.mark.parametrize("second", ["fwd", "dI"])
def test_rows_k_is_previous_output(cc, oracle_mod, second):
    """A call whose K is the output of the immediately preceding call on the
    same stream (no synchronisation between them): the library sees the
    overlap and packs K fully ordered instead of beside the previous kernel's
    tail (include/capsconv.h, "Streams").  Exact-integer data, bitwise."""
    dt = torch.bfloat16
    L1 = capsinputs.Layer(16, 12, 12, 8, 8, 3, 3, 4, 4, 4, 1)        # walk fwd, O: 16x10x10 x 8 caps
    L2 = capsinputs.Layer(4, 10, 10, 8, 8, 3, 3, 4, 4, 4, 1)         # K: 3x3 x 8 x 8 caps
    I1 = to_rows(capsinputs.make_input(L1, "int1", dt).to(DEV))
    K1 = capsinputs.make_kernel(L1, "int1", dt).to(DEV)
    n1 = 16 * 10 * 10 * 4 * 8 * 4
    nk2 = 3 * 3 * 8 * 8 * 16
    buf = torch.zeros(n1, dtype=dt, device=DEV)
    O1 = buf.view(16, 10, 10, 4, 8, 4)
    K2 = buf[:nk2].view(3, 3, 8, 8, 4, 4)
    I2 = capsinputs.make_input(L2, "int1", dt)
    dO2 = capsinputs.make_grad_output(L2.o_shape(8, 8), "int1", dt)
    torch.cuda.synchronize()
    cc.fwd(I1, K1, 1, out=O1, layout="rows")
    if second == "fwd":
        R = cc.fwd(to_rows(I2.to(DEV)), K2, 1, layout="rows")
    else:
        R = cc.bwd_data(to_rows(dO2.to(DEV)), K2, 1, L2.H, L2.W, layout="rows")
    torch.cuda.synchronize()
    k2 = to_np(K2)
    assert np.abs(k2).max() > 0
    if second == "fwd":
        ref, _ = oracle_mod.fwd(to_np(I2), k2, 1)
    else:
        ref, _ = oracle_mod.bwd_data(to_np(dO2), k2, 1, L2.H, L2.W)
    np.testing.assert_array_equal(to_np(from_rows(R)), oracle_mod.round_bf16(ref))
