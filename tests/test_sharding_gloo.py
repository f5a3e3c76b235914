"""Multi-rank logic of the stack driver (paper_2104_02621_b200/stack.py) on
CPU with the gloo backend, world size 2.

The product's CapsStack runs unchanged (batch sharding, per-layer dK
all-reduce, reverse layer order); only its compute backend is swapped for an
oracle-backed shim, because there is no GPU here.  Invariant checked: the sum
over ranks of the shard dK equals the full-batch dK (reading R16: SUM, not
mean), and every rank ends with the same dK.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_2104_02621_b200.stack import CapsStack, LayerSpec, shard_range

SPECS = [LayerSpec(2, 3, 3, 3, 1), LayerSpec(3, 2, 2, 2, 2), LayerSpec(2, 2, 2, 2, 1)]
H = W = 7
D = 2
GB = 5   # odd: shards of 2 and 3


class OracleOps:
    """Compute backend shim with the binding's signatures (test only)."""

    @staticmethod
    def output_dims(H, W, KH, KW, s, pad=0):
        return oracle.output_dims(H, W, KH, KW, s, pad)

    @staticmethod
    def fwd(I, K, stride, out=None, pad=0):
        O, _ = oracle.fwd(I.numpy(), K.numpy(), stride, pad)
        out.copy_(torch.from_numpy(O))
        return out

    @staticmethod
    def bwd_data(dO, K, stride, H, W, out=None, pad=0):
        dI, _ = oracle.bwd_data(dO.numpy(), K.numpy(), stride, H, W, pad)
        out.copy_(torch.from_numpy(dI))
        return out

    @staticmethod
    def bwd_kernel(I, dO, stride, KH, KW, out=None, pad=0):
        dK, _ = oracle.bwd_kernel(I.numpy(), dO.numpy(), stride, KH, KW, pad)
        out.copy_(torch.from_numpy(dK))
        return out


def make_data():
    g = torch.Generator().manual_seed(7)
    weights = [torch.rand((s.KH, s.KW, s.C, s.Cout, D, D), generator=g, dtype=torch.float64) - 0.5 for s in SPECS]
    X = torch.rand((GB, H, W, SPECS[0].C, D, D), generator=g, dtype=torch.float64) - 0.5
    h, w = H, W
    for s in SPECS:
        h, w = oracle.output_dims(h, w, s.KH, s.KW, s.stride)
    dY = torch.rand((GB, h, w, SPECS[-1].Cout, D, D), generator=g, dtype=torch.float64) - 0.5
    return weights, X, dY


def _worker(rank, world, port, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        weights, X, dY = make_data()
        lo, hi = shard_range(GB, rank, world)
        st = CapsStack(SPECS, H, W, D, hi - lo, weights, "cpu", ops=OracleOps)
        dKs = st.step(X[lo:hi], dY[lo:hi])
        out_q.put((rank, [k.numpy().copy() for k in dKs], st.out.numpy().copy(), st.grads[0].numpy().copy()))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_shard_range_partitions():
    for gb in (1, 5, 1024):
        for world in (1, 2, 3, 8):
            spans = [shard_range(gb, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == gb
            assert all(spans[i][1] == spans[i + 1][0] for i in range(world - 1))
            assert max(b - a for a, b in spans) - min(b - a for a, b in spans) <= 1


def test_world2_dK_allreduce_equals_full_batch():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict()
    for _ in range(2):
        r, dks, out, dx = q.get(timeout=300)
        res[r] = (dks, out, dx)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # full-batch reference through the oracle stack (no sharding)
    weights, X, dY = make_data()
    acts, dX, dKs, _ = oracle.stack_fwd_bwd(X.numpy(), [w.numpy() for w in weights], [s.stride for s in SPECS],
                                            dY.numpy(), False)
    for li in range(len(SPECS)):
        np.testing.assert_allclose(res[0][0][li], dKs[li], rtol=1e-12, atol=1e-12)
        np.testing.assert_array_equal(res[0][0][li], res[1][0][li])
    # forward output and dX are per-shard (no collective): concatenated == full batch
    lo1 = shard_range(GB, 1, 2)[0]
    np.testing.assert_allclose(np.concatenate([res[0][1], res[1][1]]), acts[-1], rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(np.concatenate([res[0][2], res[1][2]]), dX, rtol=1e-12, atol=1e-12)
    assert lo1 == 2


def test_single_process_stack_matches_oracle():
    weights, X, dY = make_data()
    st = CapsStack(SPECS, H, W, D, GB, weights, "cpu", ops=OracleOps)
    dKs = st.step(X, dY)
    acts, dX, rdKs, _ = oracle.stack_fwd_bwd(X.numpy(), [w.numpy() for w in weights], [s.stride for s in SPECS],
                                             dY.numpy(), False)
    for li in range(len(SPECS)):
        np.testing.assert_allclose(dKs[li].numpy(), rdKs[li], rtol=1e-12, atol=1e-12)
    assert st.step_flops() == 3 * sum(st.layer_flops(i) for i in range(len(SPECS)))


def test_single_process_padded_stack_matches_oracle():
    """The stack driver threads each layer's zero padding."""
    specs = [LayerSpec(2, 3, 3, 3, 1, 1), LayerSpec(3, 2, 3, 3, 2, 1), LayerSpec(2, 2, 4, 4, 1, 0)]
    g = torch.Generator().manual_seed(11)
    weights = [torch.rand((s.KH, s.KW, s.C, s.Cout, D, D), generator=g, dtype=torch.float64) - 0.5 for s in specs]
    X = torch.rand((GB, H, W, specs[0].C, D, D), generator=g, dtype=torch.float64) - 0.5
    h, w = H, W
    for s in specs:
        h, w = oracle.output_dims(h, w, s.KH, s.KW, s.stride, s.pad)
    dY = torch.rand((GB, h, w, specs[-1].Cout, D, D), generator=g, dtype=torch.float64) - 0.5
    st = CapsStack(specs, H, W, D, GB, weights, "cpu", ops=OracleOps)
    dKs = st.step(X, dY)
    acts, dX, rdKs, _ = oracle.stack_fwd_bwd(X.numpy(), [w_.numpy() for w_ in weights], [s.stride for s in specs],
                                             dY.numpy(), False, pads=[s.pad for s in specs])
    np.testing.assert_allclose(st.out.numpy(), acts[-1], rtol=1e-12, atol=1e-12)
    for li in range(len(specs)):
        np.testing.assert_allclose(dKs[li].numpy(), rdKs[li], rtol=1e-12, atol=1e-12)


# ---------------------------------------------------------------- training step
class OracleTrainOps(OracleOps):
    """OracleOps plus the rows layout (permuted around the oracle) and SGD,
    for the product CapsTrainer on CPU (test only)."""

    @staticmethod
    def _nat(t, layout):
        return t.permute(0, 1, 2, 4, 3, 5).contiguous() if layout == "rows" else t

    @staticmethod
    def fwd(I, K, stride, out=None, pad=0, layout="natural"):
        O, _ = oracle.fwd(OracleTrainOps._nat(I, layout).numpy(), K.numpy(), stride, pad)
        out.copy_(OracleTrainOps._nat(torch.from_numpy(O), layout))
        return out

    @staticmethod
    def bwd_data(dO, K, stride, H, W, out=None, pad=0, layout="natural"):
        dI, _ = oracle.bwd_data(OracleTrainOps._nat(dO, layout).numpy(), K.numpy(), stride, H, W, pad)
        out.copy_(OracleTrainOps._nat(torch.from_numpy(dI), layout))
        return out

    @staticmethod
    def bwd_kernel(I, dO, stride, KH, KW, out=None, pad=0, layout="natural"):
        dK, _ = oracle.bwd_kernel(OracleTrainOps._nat(I, layout).numpy(), OracleTrainOps._nat(dO, layout).numpy(),
                                  stride, KH, KW, pad)
        out.copy_(torch.from_numpy(dK))
        return out

    @staticmethod
    def sgd_update(w, g, lr, out=None):
        w.copy_(torch.from_numpy(oracle.sgd_update(w.numpy(), g.numpy(), lr)))
        if out is not None:
            out.copy_(w)
        return out


TSPECS = [LayerSpec(2, 2, 3, 3, 1), LayerSpec(2, 2, 2, 2, 1)]
TLR = 0.05


def make_train_data():
    g = torch.Generator().manual_seed(9)
    weights = [torch.rand((s.KH, s.KW, s.C, s.Cout, D, D), generator=g, dtype=torch.float64) - 0.5 for s in TSPECS]
    Kp = torch.rand((3, 3, 1, 1, 1, TSPECS[0].C * D * D), generator=g, dtype=torch.float64) - 0.5
    img = torch.rand((GB, H + 2, W + 2, 1, 1, 1), generator=g, dtype=torch.float64) - 0.5
    h, w = H, W
    for s in TSPECS:
        h, w = oracle.output_dims(h, w, s.KH, s.KW, s.stride)
    dY = torch.rand((GB, h, w, D, TSPECS[-1].Cout, D), generator=g, dtype=torch.float64) - 0.5   # rows layout
    return weights, Kp, img, dY


def _train_worker(rank, world, port, out_q):
    from paper_2104_02621_b200.train import CapsTrainer
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        weights, Kp, img, dY = make_train_data()
        lo, hi = shard_range(GB, rank, world)
        tr = CapsTrainer(TSPECS, H, W, D, hi - lo, Kp, weights, "cpu", TLR, ops=OracleTrainOps)
        new = tr.step(img[lo:hi], dY[lo:hi])
        out_q.put((rank, [m.numpy().copy() for m in new]))
    finally:
        dist.destroy_process_group()


def test_world2_training_step_equals_full_batch():
    """Data-parallel training step: every rank ends with the same updated
    weights -- the primary layer's included -- and they equal the full-batch
    step (dK is a sum over the batch, so the SUM all-reduce of the shard dKs
    is the full-batch dK)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_train_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict()
    for _ in range(2):
        r, ws = q.get(timeout=300)
        res[r] = ws
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    from paper_2104_02621_b200.train import CapsTrainer
    weights, Kp, img, dY = make_train_data()
    full = CapsTrainer(TSPECS, H, W, D, GB, Kp, weights, "cpu", TLR, ops=OracleTrainOps)
    ref = [m.numpy().copy() for m in full.step(img, dY)]
    assert len(ref) == len(TSPECS) + 1
    for i in range(len(ref)):
        np.testing.assert_array_equal(res[0][i], res[1][i])
        np.testing.assert_allclose(res[0][i], ref[i], rtol=1e-6, atol=1e-6)
        assert not np.array_equal(ref[i], ([Kp] + weights)[i].numpy().astype(np.float32))   # the step moved it
