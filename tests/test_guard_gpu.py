"""Out-of-bounds write guard for every kernel family (compute-sanitizer is
closed on this GPU pool, so this is the bounds check of our own): each output
and the workspace are views into larger buffers whose guard regions hold a
random canary; after every call the canaries must be intact and the result
must equal the same call into a plain tensor.  Inputs sit at the very end of
their allocation (a read past them would fault or read the next guard).
Hangs surface as the probe build's mbarrier watchdog trap elsewhere
(umma.cuh); here every call runs under the product library."""
import numpy as np
import pytest
import torch

import capsinputs

pytestmark = pytest.mark.gpu
DEV = "cuda:0"
GUARD = 64 * 1024   # bytes of canary on each side

CASES = [
    # B, H, W, C, Cout, KH, KW, D1, D2, D3, s
    (2, 10, 12, 8, 8, 3, 3, 4, 4, 4, 1),     # walk fwd / dI, rows dK
    (3, 11, 11, 8, 16, 3, 3, 4, 4, 4, 2),    # walk fwd s2, rows_conv dI s2
    (2, 9, 9, 16, 32, 3, 3, 4, 4, 4, 1),     # rows_conv fwd (N = 128), walk dI
    (37, 4, 4, 32, 10, 4, 4, 4, 4, 4, 1),    # rows FC GEMMs, ragged batch tile
    (2, 34, 17, 8, 8, 3, 3, 4, 4, 4, 1),     # several x tiles / ring wraps
    (2, 6, 5, 2, 3, 2, 3, 2, 3, 5, 1),       # generic shapes: natural path between permutations
    (3, 28, 28, 1, 1, 5, 5, 1, 1, 128, 1),   # training-step primary layer: tcgen05 fwd / dK (bf16)
    (2, 13, 17, 1, 2, 7, 7, 1, 1, 32, 1),    # primary layer on CUDA cores (N = 64, 7x7)
]


@pytest.fixture(scope="module")
def cc():
    from paper_2104_02621_b200 import _build
    _build.build()
    import paper_2104_02621_b200.capsconv as cc
    cc.load_library()
    return cc


def guarded(shape, dtype, gen):
    """A tensor of `shape` inside a buffer with GUARD canary bytes on both sides."""
    n = int(np.prod(shape)) * torch.empty((), dtype=dtype).element_size()
    buf = torch.randint(0, 256, (GUARD + n + GUARD,), dtype=torch.uint8, generator=gen).to(DEV)
    ref = buf.clone()
    view = buf[GUARD:GUARD + n].view(dtype).view(shape)
    return buf, ref, view


def tail_input(t):
    """t copied to the end of a larger allocation (16-byte aligned)."""
    n = t.numel() * t.element_size()
    pad = (256 - n % 256) % 256 + 256
    buf = torch.zeros(n + pad, dtype=torch.uint8, device=DEV)
    v = buf[pad:].view(t.dtype).view(t.shape)
    v.copy_(t)
    return v


def rows(t):
    return t.permute(0, 1, 2, 4, 3, 5).contiguous()


@pytest.mark.parametrize("case", CASES, ids=lambda c: "x".join(map(str, c)))
@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32], ids=["bf16", "f32"])
@pytest.mark.parametrize("layout", ["natural", "rows"])
def test_guards(cc, case, dtype, layout, monkeypatch):
    L = capsinputs.Layer(*case)
    gen = torch.Generator().manual_seed(hash(case) & 0xffff)
    Ho, Wo = cc.output_dims(L.H, L.W, L.KH, L.KW, L.stride)
    I = capsinputs.make_input(L, dtype=dtype).to(DEV)
    K = capsinputs.make_kernel(L, dtype=dtype).to(DEV)
    dO = capsinputs.make_grad_output(L.o_shape(Ho, Wo), dtype=dtype).to(DEV)
    if layout == "rows":
        I, dO = rows(I), rows(dO)
    I, K, dO = tail_input(I), tail_input(K), tail_input(dO)
    # guarded workspace
    wsb = {}

    def ws(nbytes, device, stream_handle):
        if nbytes == 0:
            return None
        b, r, v = guarded((nbytes,), torch.uint8, gen)
        wsb["buf"], wsb["ref"], wsb["n"] = b, r, nbytes
        return v
    monkeypatch.setattr(cc, "_workspace", ws)
    calls = [
        ("fwd", lambda out: cc.fwd(I, K, L.stride, out=out, layout=layout), cc.fwd(I, K, L.stride, layout=layout)),
        ("dI", lambda out: cc.bwd_data(dO, K, L.stride, L.H, L.W, out=out, layout=layout),
         cc.bwd_data(dO, K, L.stride, L.H, L.W, layout=layout)),
        ("dK", lambda out: cc.bwd_kernel(I, dO, L.stride, L.KH, L.KW, out=out, layout=layout),
         cc.bwd_kernel(I, dO, L.stride, L.KH, L.KW, layout=layout)),
    ]
    torch.cuda.synchronize()
    for name, f, plain in calls:
        buf, ref, view = guarded(plain.shape, plain.dtype, gen)
        f(view)
        torch.cuda.synchronize()
        assert torch.equal(buf[:GUARD], ref[:GUARD]), name + ": write before the output"
        assert torch.equal(buf[-GUARD:], ref[-GUARD:]), name + ": write past the output"
        if "buf" in wsb:
            b, r = wsb["buf"], wsb["ref"]
            assert torch.equal(b[:GUARD], r[:GUARD]), name + ": write before the workspace"
            assert torch.equal(b[-GUARD:], r[-GUARD:]), name + ": write past the workspace"
        assert torch.equal(view, plain), name + ": result differs from the unguarded call"


def test_guard_sgd_update(cc):
    """capsconv_sgd_update writes exactly n masters and n working copies."""
    gen = torch.Generator().manual_seed(11)
    for n in (5, 4096 + 6):   # ragged tails of the 4-wide vectors
        wb, wr, w = guarded((n,), torch.float32, gen)
        w.copy_(torch.rand(n, generator=gen).to(DEV))
        wr = wb.clone()
        g = torch.rand(n, generator=gen).to(DEV)
        ob, orf, o = guarded((n,), torch.bfloat16, gen)
        cc.sgd_update(w, g, 0.5, o)
        torch.cuda.synchronize()
        assert torch.equal(wb[:GUARD], wr[:GUARD]) and torch.equal(wb[-GUARD:], wr[-GUARD:]), "master guards"
        assert torch.equal(ob[:GUARD], orf[:GUARD]) and torch.equal(ob[-GUARD:], orf[-GUARD:]), "copy guards"
        assert torch.equal(o, w.to(torch.bfloat16))
