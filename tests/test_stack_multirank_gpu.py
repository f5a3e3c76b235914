"""The production multi-rank branch of the stack driver on the GPU: two
processes on cuda:0, each the real CapsStack over libcapsconv with
overlap=True, joined by a gloo process group on CUDA tensors.  Each layer's
dK is all-reduced on the side stream (event -> comm_stream.wait_event ->
all_reduce -> current_stream.wait_stream), which is the code path the N>1
bench takes with NCCL (BJ:5 item (3)).

Exact-integer inputs ({-1, 0, 1}) keep every fp32 sum exact, so the checks
are bitwise: Sigma over ranks of the shard dK == the full-batch oracle dK
(reading R16: SUM), both ranks hold the same dK, and each rank's output and
dX equal the oracle stack (bf16 boundaries, R13) on its shard.  No kernel
waits on another process: the collective is host-side (gloo)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

import capsinputs

pytestmark = pytest.mark.gpu

GB = 6   # global batch; shards of 3 and 3 images


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _data():
    import oracle
    layers = capsinputs.stack_layers(GB, oracle.output_dims)
    Ks = [capsinputs.make_kernel(L, "int1", torch.bfloat16, layer_idx=i) for i, L in enumerate(layers)]
    X = capsinputs.make_input(layers[0], "int1", torch.bfloat16)
    last = layers[-1]
    Ho, Wo = oracle.output_dims(last.H, last.W, last.KH, last.KW, last.stride)
    dY = capsinputs.make_grad_output(last.o_shape(Ho, Wo), "int1", torch.bfloat16, layer_idx=len(layers))
    return Ks, X, dY


def _worker(rank, world, port, q):
    import torch.distributed as dist
    sys_path = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    import sys
    if sys_path not in sys.path:
        sys.path.insert(0, sys_path)
    from paper_2104_02621_b200.stack import CapsStack, LayerSpec, shard_range
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        Ks, X, dY = _data()
        specs = [LayerSpec(*l) for l in capsinputs.STACK_LAYERS]
        si = capsinputs.STACK_INPUT
        lo, hi = shard_range(GB, rank, world)
        st = CapsStack(specs, si["H"], si["W"], 4, hi - lo, Ks, "cuda:0")
        assert st.overlap and st.world == world and st.comm_stream is not None
        dKs = st.step(X[lo:hi].cuda(), dY[lo:hi].cuda())
        torch.cuda.synchronize()
        q.put((rank, [k.cpu().double().numpy() for k in dKs], st.out.cpu().double().numpy(),
               st.grads[0].cpu().double().numpy()))
    except BaseException as e:  # report instead of hanging the parent
        q.put((rank, repr(e), None, None))
        raise
    finally:
        dist.destroy_process_group()


def test_world2_overlapped_allreduce_on_gpu(oracle_mod):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(2):
        r, dks, out, dx = q.get(timeout=600)
        assert not isinstance(dks, str), "rank %d failed: %s" % (r, dks)
        res[r] = (dks, out, dx)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    Ks, X, dY = _data()
    strides = [l[4] for l in capsinputs.STACK_LAYERS]
    f64 = lambda t: t.to(torch.float64).numpy()
    acts, dX, dKs, _ = oracle_mod.stack_fwd_bwd(f64(X), [f64(k) for k in Ks], strides, f64(dY), True)
    for li in range(len(Ks)):
        assert np.abs(dKs[li]).max() < 2 ** 24
        np.testing.assert_array_equal(res[0][0][li], dKs[li])
        np.testing.assert_array_equal(res[1][0][li], dKs[li])
    np.testing.assert_array_equal(np.concatenate([res[0][1], res[1][1]]), acts[-1])
    np.testing.assert_array_equal(np.concatenate([res[0][2], res[1][2]]), dX)
