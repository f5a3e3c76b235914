"""GPU parity: libcapsconv (through its C ABI) against the CPU oracle.

Small cases span several tiles and ragged tails; full BASELINE.json sizes
are checked bit-exactly on exact-integer inputs (every product and partial
sum is an integer below 2^24, so any summation order gives the exact value;
bf16 outputs must equal RNE_bf16(exact)) and within tolerance on uniform
inputs.  Both kernel paths are exercised: the library's own choice (AUTO)
and the SIMT path forced.
"""
import numpy as np
import pytest
import torch

import capsinputs
from helpers import TOL, assert_close, rel_err, to_np

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


@pytest.fixture(params=["auto", "simt"])
def path(request, cc):
    cc.set_path_override(cc.PATH_AUTO if request.param == "auto" else cc.PATH_SIMT)
    yield request.param
    cc.set_path_override(cc.PATH_AUTO)


def run_all(cc, L, I, K, dO):
    Id, Kd, dOd = I.to(DEV), K.to(DEV), dO.to(DEV)
    O = cc.fwd(Id, Kd, L.stride)
    dI = cc.bwd_data(dOd, Kd, L.stride, L.H, L.W)
    dK = cc.bwd_kernel(Id, dOd, L.stride, L.KH, L.KW)
    torch.cuda.synchronize()
    return O, dI, dK


def check_layer(cc, oracle_mod, L, dtype, kind="uniform"):
    I = capsinputs.make_input(L, kind, dtype)
    K = capsinputs.make_kernel(L, kind, dtype)
    Ho, Wo = oracle_mod.output_dims(L.H, L.W, L.KH, L.KW, L.stride)
    dO = capsinputs.make_grad_output(L.o_shape(Ho, Wo), kind, dtype)
    O, dI, dK = run_all(cc, L, I, K, dO)
    rO, aO = oracle_mod.fwd(to_np(I), to_np(K), L.stride)
    rdI, adI = oracle_mod.bwd_data(to_np(dO), to_np(K), L.stride, L.H, L.W)
    rdK, adK = oracle_mod.bwd_kernel(to_np(I), to_np(dO), L.stride, L.KH, L.KW)
    assert O.dtype == dtype and dI.dtype == dtype and dK.dtype == torch.float32
    e = (assert_close(to_np(O), rO, aO, dtype, "fwd"),
         assert_close(to_np(dI), rdI, adI, dtype, "bwd_data"),
         # dK is accumulated and stored in fp32 from exactly representable
         # products (bf16 x bf16 is exact in fp32): the fp32 bar applies
         assert_close(to_np(dK), rdK, adK, torch.float32, "bwd_kernel"))
    return e


SMALL = [
    # B, H, W, C, Cout, KH, KW, D1, D2, D3, s
    (2, 9, 11, 3, 5, 3, 3, 4, 4, 4, 1),
    (3, 10, 9, 8, 8, 3, 3, 4, 4, 4, 2),
    (2, 8, 8, 32, 10, 8, 8, 4, 4, 4, 1),
    (1, 12, 40, 8, 8, 3, 3, 4, 4, 4, 1),
    (5, 7, 7, 16, 32, 3, 3, 4, 4, 4, 2),
    (3, 13, 6, 4, 16, 2, 3, 4, 4, 4, 3),
    (2, 6, 5, 2, 3, 2, 3, 2, 3, 5, 1),
    (1, 5, 5, 1, 1, 4, 4, 3, 3, 3, 1),
    (2, 7, 7, 3, 2, 3, 3, 1, 1, 1, 3),
    (1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1),
    (4, 11, 11, 8, 16, 1, 1, 4, 4, 4, 1),
    (2, 34, 17, 8, 8, 3, 3, 4, 4, 4, 1),
]


@pytest.mark.parametrize("case", SMALL, ids=lambda c: "x".join(map(str, c)))
@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16], ids=["f32", "bf16"])
def test_small_random(cc, oracle_mod, path, case, dtype):
    L = capsinputs.Layer(*case)
    check_layer(cc, oracle_mod, L, dtype)


def test_fig2_golden_through_abi(cc, oracle_mod, path):
    # all-ones 5x5 input of 3x3 capsules, all-ones 4x4 kernel -> 48s
    L = capsinputs.CONFIGS["fig2"]
    I = capsinputs.make_input(L, "ones").to(DEV)
    K = capsinputs.make_kernel(L, "ones").to(DEV)
    O = cc.fwd(I, K, 1)
    assert tuple(O.shape) == (1, 2, 2, 1, 3, 3)
    assert torch.all(O == 48.0)
    dO = torch.ones_like(O)
    dK = cc.bwd_kernel(I, dO, 1, 4, 4)
    assert torch.all(dK == 12.0)
    dI = cc.bwd_data(dO, K, 1, 5, 5)
    plane = torch.tensor([[3, 6, 6, 6, 3]] + [[6, 12, 12, 12, 6]] * 3 + [[3, 6, 6, 6, 3]], dtype=torch.float32)
    for d1 in range(3):
        for d2 in range(3):
            assert torch.equal(dI[0, :, :, 0, d1, d2].cpu(), plane)


FULL = [("layer_s1", torch.float32), ("layer_s1", torch.bfloat16), ("layer_s2", torch.bfloat16),
        ("fc", torch.bfloat16), ("fc", torch.float32)]


@pytest.mark.parametrize("name,dtype", FULL, ids=lambda v: str(v).replace("torch.", ""))
def test_full_size_exact_integers(cc, oracle_mod, name, dtype):
    """Bitwise at BASELINE.json's full sizes (the launch configuration bench
    times): exact-integer inputs make the result order independent."""
    L = capsinputs.CONFIGS[name]
    I = capsinputs.make_input(L, "int", dtype)
    K = capsinputs.make_kernel(L, "int", dtype)
    Ho, Wo = oracle_mod.output_dims(L.H, L.W, L.KH, L.KW, L.stride)
    dO = capsinputs.make_grad_output(L.o_shape(Ho, Wo), "int", dtype)
    O, dI, dK = run_all(cc, L, I, K, dO)
    rO, _ = oracle_mod.fwd(to_np(I), to_np(K), L.stride)
    rdI, _ = oracle_mod.bwd_data(to_np(dO), to_np(K), L.stride, L.H, L.W)
    rdK, _ = oracle_mod.bwd_kernel(to_np(I), to_np(dO), L.stride, L.KH, L.KW)
    assert np.abs(rdK).max() < 2 ** 24 and np.abs(rO).max() < 2 ** 24
    if dtype == torch.bfloat16:
        rO, rdI = oracle_mod.round_bf16(rO), oracle_mod.round_bf16(rdI)
    np.testing.assert_array_equal(to_np(O), rO)
    np.testing.assert_array_equal(to_np(dI), rdI)
    np.testing.assert_array_equal(to_np(dK), rdK)


@pytest.mark.parametrize("name,dtype", FULL, ids=lambda v: str(v).replace("torch.", ""))
def test_full_size_uniform(cc, oracle_mod, name, dtype):
    L = capsinputs.CONFIGS[name]
    check_layer(cc, oracle_mod, L, dtype)


def test_misaligned_pointers_take_a_correct_path(cc, oracle_mod):
    L = capsinputs.Layer(2, 9, 9, 8, 8, 3, 3, 4, 4, 4, 1)
    I = capsinputs.make_input(L, "uniform", torch.bfloat16)
    K = capsinputs.make_kernel(L, "uniform", torch.bfloat16)
    # offset by one element so the data pointers are only 2-byte aligned
    Ib = torch.empty(I.numel() + 1, dtype=torch.bfloat16, device=DEV)
    Ib[1:].copy_(I.reshape(-1))
    Iv = Ib[1:].view(I.shape)
    O = cc.fwd(Iv, K.to(DEV), 1)
    rO, aO = oracle_mod.fwd(to_np(I), to_np(K), 1)
    assert_close(to_np(O), rO, aO, torch.bfloat16, "fwd misaligned")


def test_overwrites_output(cc):
    L = capsinputs.Layer(2, 8, 8, 4, 4, 3, 3, 4, 4, 4, 1)
    I = capsinputs.make_input(L).to(DEV)
    K = capsinputs.make_kernel(L).to(DEV)
    O1 = cc.fwd(I, K, 1)
    O2 = torch.full_like(O1, float("nan"))
    cc.fwd(I, K, 1, out=O2)
    assert torch.equal(O1, O2)


def test_deterministic(cc):
    L = capsinputs.CONFIGS["layer_s1"]
    I = capsinputs.make_input(L, dtype=torch.bfloat16).to(DEV)
    dO = torch.randn(64, 30, 30, 8, 4, 4, device=DEV).to(torch.bfloat16)
    a = cc.bwd_kernel(I, dO, 1, 3, 3)
    b = cc.bwd_kernel(I, dO, 1, 3, 3)
    assert torch.equal(a, b)


def test_autograd_function(cc, oracle_mod):
    L = capsinputs.Layer(2, 7, 7, 4, 4, 3, 3, 4, 4, 4, 2)
    I = capsinputs.make_input(L).to(DEV).requires_grad_(True)
    K = capsinputs.make_kernel(L).to(DEV).requires_grad_(True)
    O = cc.caps_conv2d(I, K, 2)
    g = torch.randn_like(O)
    O.backward(g)
    rdI, adI = oracle_mod.bwd_data(to_np(g), to_np(K), 2, 7, 7)
    rdK, adK = oracle_mod.bwd_kernel(to_np(I), to_np(g), 2, 3, 3)
    assert_close(to_np(I.grad), rdI, adI, torch.float32)
    assert_close(to_np(K.grad), rdK, adK, torch.float32)


def test_launch_counter_moves(cc):
    L = capsinputs.Layer(1, 6, 6, 2, 2, 3, 3, 4, 4, 4, 1)
    n0 = cc.launch_count()
    cc.fwd(capsinputs.make_input(L).to(DEV), capsinputs.make_kernel(L).to(DEV), 1)
    torch.cuda.synchronize()
    assert cc.launch_count() > n0


def _stack_layers():
    import oracle
    return capsinputs.stack_layers(capsinputs.STACK_BATCH, oracle.output_dims)


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32], ids=["bf16", "f32"])
@pytest.mark.parametrize("li", [0, 1, 2, 3], ids=["L1", "L2", "L3", "FC"])
def test_stack_layers_full_batch_exact(cc, oracle_mod, li, dtype):
    """Each layer of the config-5 stack at global batch 1024 (the sizes bench.py
    times), exact-integer inputs in {-1, 0, 1}: bitwise equal to the oracle --
    bf16 on the tensor-core path, fp32 on the exact-fp32 (SIMT) path."""
    L = _stack_layers()[li]
    I = capsinputs.make_input(L, "int1", dtype, layer_idx=li)
    K = capsinputs.make_kernel(L, "int1", dtype, layer_idx=li)
    Ho, Wo = oracle_mod.output_dims(L.H, L.W, L.KH, L.KW, L.stride)
    dO = capsinputs.make_grad_output(L.o_shape(Ho, Wo), "int1", dtype, layer_idx=li)
    O, dI, dK = run_all(cc, L, I, K, dO)
    rO, _ = oracle_mod.fwd(to_np(I), to_np(K), L.stride)
    rdI, _ = oracle_mod.bwd_data(to_np(dO), to_np(K), L.stride, L.H, L.W)
    rdK, _ = oracle_mod.bwd_kernel(to_np(I), to_np(dO), L.stride, L.KH, L.KW)
    assert np.abs(rdK).max() < 2 ** 24
    # the benchmarked configuration runs on the tensor-core path, every pass
    ext = (L.B, L.H, L.W, L.C, L.Cout, L.KH, L.KW, L.D1, L.D2, L.D3, L.stride)
    want = cc.PATH_MMA if dtype == torch.bfloat16 else cc.PATH_SIMT
    assert [cc.select_path(op, dtype, ext) for op in (0, 1, 2)] == [want] * 3
    rnd = oracle_mod.round_bf16 if dtype == torch.bfloat16 else (lambda x: x)
    np.testing.assert_array_equal(to_np(O), rnd(rO))
    np.testing.assert_array_equal(to_np(dI), rnd(rdI))
    np.testing.assert_array_equal(to_np(dK), rdK)


def test_stack_step_small_batch(cc, oracle_mod):
    """The product stack (CapsStack over libcapsconv) against the oracle stack
    with bf16 rounding at the layer boundaries (reading R13), batch 6."""
    from paper_2104_02621_b200.stack import CapsStack, LayerSpec
    specs = [LayerSpec(*l) for l in capsinputs.STACK_LAYERS]
    si = capsinputs.STACK_INPUT
    B = 6
    layers = capsinputs.stack_layers(B, oracle_mod.output_dims)
    Ks = [capsinputs.make_kernel(L, dtype=torch.bfloat16, layer_idx=i) for i, L in enumerate(layers)]
    X = capsinputs.make_input(layers[0], dtype=torch.bfloat16)
    h, w = si["H"], si["W"]
    for s in specs:
        h, w = oracle_mod.output_dims(h, w, s.KH, s.KW, s.stride)
    dY = capsinputs.make_grad_output((B, h, w, specs[-1].Cout, 4, 4), dtype=torch.bfloat16, layer_idx=len(specs))
    st = CapsStack(specs, si["H"], si["W"], 4, B, Ks, DEV)
    dKs = st.step(X.to(DEV), dY.to(DEV))
    torch.cuda.synchronize()
    acts, dX, rdKs, den = oracle_mod.stack_fwd_bwd(to_np(X), [to_np(k) for k in Ks], [s.stride for s in specs],
                                                   to_np(dY), True)
    assert_close(to_np(st.out), acts[-1], den["fwd"][-1], torch.bfloat16, "stack output")
    assert_close(to_np(st.grads[0]), dX, den["dI"][0], torch.bfloat16, "stack dX")
    for li in range(len(specs)):
        assert_close(to_np(dKs[li]), rdKs[li], den["dK"][li], torch.bfloat16, "stack dK L%d" % (li + 1))


def test_stack_step_graph_matches_serialised(cc):
    """The config-5 stack step as bench.py times it -- captured once in a CUDA
    graph (kernels chained by programmatic-dependent-launch edges, no host
    synchronisation) and replayed -- against the same chain run op by op with
    a device synchronisation after every call, global batch 1024.  Every
    kernel is deterministic, so any ordering hazard between consecutive
    kernels shows up as a bitwise difference."""
    from paper_2104_02621_b200.stack import CapsStack, LayerSpec
    specs = [LayerSpec(*l) for l in capsinputs.STACK_LAYERS]
    si = capsinputs.STACK_INPUT
    B = capsinputs.STACK_BATCH
    layers = capsinputs.stack_layers(B, cc.output_dims)
    Ks = [capsinputs.make_kernel(L, dtype=torch.bfloat16, layer_idx=i).to(DEV) for i, L in enumerate(layers)]
    X = capsinputs.make_input(layers[0], dtype=torch.bfloat16).to(DEV)
    hw = [(si["H"], si["W"])]
    for s in specs:
        hw.append(cc.output_dims(hw[-1][0], hw[-1][1], s.KH, s.KW, s.stride))
    dY = capsinputs.make_grad_output((B, hw[-1][0], hw[-1][1], specs[-1].Cout, 4, 4), dtype=torch.bfloat16,
                                     layer_idx=len(specs)).to(DEV)
    # serialised reference
    acts = [X]
    for li, s in enumerate(specs):
        acts.append(cc.fwd(acts[-1], Ks[li], s.stride))
        torch.cuda.synchronize()
    g, rdK = dY, [None] * len(specs)
    for li in range(len(specs) - 1, -1, -1):
        s = specs[li]
        rdK[li] = cc.bwd_kernel(acts[li], g, s.stride, s.KH, s.KW)
        torch.cuda.synchronize()
        g = cc.bwd_data(g, Ks[li], s.stride, hw[li][0], hw[li][1])
        torch.cuda.synchronize()
    # graph-captured product step
    st = CapsStack(specs, si["H"], si["W"], 4, B, Ks, DEV)
    graph, cs = torch.cuda.CUDAGraph(), torch.cuda.Stream()
    cs.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(cs):
        st.step(X, dY)
        torch.cuda.synchronize()
        with torch.cuda.graph(graph, stream=cs):
            st.step(X, dY)
    torch.cuda.synchronize()
    for t in [st.out] + st.grads + st.dK:
        t.fill_(float("nan"))
    graph.replay()
    graph.replay()
    torch.cuda.synchronize()
    assert torch.equal(st.out, acts[-1])
    assert torch.equal(st.grads[0], g)
    for li in range(len(specs)):
        assert torch.equal(st.dK[li], rdK[li]), li


FC_RAGGED = [
    # B, H=W=KH=KW, C, Cout: full-extent (FC) layers on the mma.sync kernels --
    # ragged batch (split-K / image-slice tails, partial stages), flattened
    # channel counts that are not multiples of 4 or 64, odd and small Cout
    (37, 3, 5, 3),
    (130, 2, 12, 16),
    (1, 1, 7, 1),
    (257, 4, 9, 10),
    (64, 8, 32, 10),
]


@pytest.mark.parametrize("case", FC_RAGGED, ids=lambda c: "x".join(map(str, c)))
def test_fc_ragged_exact(cc, oracle_mod, case):
    """Full-extent capsule layers with ragged extents, exact-integer bf16
    inputs: bitwise equal to the oracle on the library's own path."""
    B, S, C, Co = case
    L = capsinputs.Layer(B, S, S, C, Co, S, S, 4, 4, 4, 1)
    I = capsinputs.make_input(L, "int1", torch.bfloat16)
    K = capsinputs.make_kernel(L, "int1", torch.bfloat16)
    dO = capsinputs.make_grad_output(L.o_shape(1, 1), "int1", torch.bfloat16)
    O, dI, dK = run_all(cc, L, I, K, dO)
    rO, _ = oracle_mod.fwd(to_np(I), to_np(K), 1)
    rdI, _ = oracle_mod.bwd_data(to_np(dO), to_np(K), 1, S, S)
    rdK, _ = oracle_mod.bwd_kernel(to_np(I), to_np(dO), 1, S, S)
    np.testing.assert_array_equal(to_np(O), oracle_mod.round_bf16(rO))
    np.testing.assert_array_equal(to_np(dI), oracle_mod.round_bf16(rdI))
    np.testing.assert_array_equal(to_np(dK), rdK)
