"""Probe of the tcgen05 descriptor conventions (csrc/umma.cuh) on the GPU:
D = A * B^T through shared-memory operands in canonical no-swizzle layouts,
compared with a float64 matmul of the same bf16 / fp32 values."""
import ctypes
import os
import subprocess

import pytest
import torch

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
PROBE = os.path.join(HERE, "probe")
LIB = os.path.join(PROBE, "libumma_probe.so")
SRC = os.path.join(PROBE, "umma_probe.cu")
CSRC = os.path.join(os.path.dirname(HERE), "paper_2104_02621_b200", "csrc")


@pytest.fixture(scope="module")
def probe():
    if not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC) or \
            os.path.getmtime(LIB) < os.path.getmtime(os.path.join(CSRC, "umma.cuh")):
        subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O2", "-std=c++17", "-Xcompiler",
                        "-fPIC", "-shared", "-I", CSRC, "-I", os.path.join(os.path.dirname(HERE), "include"),
                        "-o", LIB, SRC], check=True)
    lib = ctypes.CDLL(LIB)
    lib.umma_probe.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p] + [ctypes.c_int] * 8
    lib.umma_probe.restype = ctypes.c_int
    return lib


CASES = [
    # tf32, a_mn, b_mn, N, K, shift, swz
    (0, 0, 0, 32, 64, 0, 1),
    (0, 0, 0, 32, 64, 4, 1),
    (0, 0, 0, 64, 64, 3, 1),
    (0, 0, 0, 32, 64, 8, 1),
    (0, 0, 0, 32, 32, 0, 0),
    (0, 0, 0, 32, 32, 4, 0),
    (0, 0, 0, 32, 32, 1, 0),
    (0, 0, 0, 32, 64, 12, 0),
    (0, 0, 0, 48, 32, 0, 0),
    (0, 0, 0, 128, 48, 8, 0),
    (0, 0, 0, 256, 16, 0, 0),
    (0, 1, 0, 32, 32, 0, 0),
    (0, 1, 0, 64, 32, 4, 0),
    (0, 0, 1, 32, 32, 0, 0),
    (0, 1, 1, 32, 64, 0, 0),
    (1, 0, 0, 32, 32, 0, 0),
    (1, 0, 0, 64, 32, 4, 0),
]


@pytest.mark.parametrize("case", CASES, ids=lambda c: "tf32%d_amn%d_bmn%d_N%d_K%d_sh%d_swz%d" % c)
def test_umma_layouts(probe, case):
    tf32, a_mn, b_mn, N, K, shift, swz = case
    dt = torch.float32 if tf32 else torch.bfloat16
    g = torch.Generator().manual_seed(1)
    if a_mn:
        RA, KA = 128, K + shift       # shift along K (k rows)
    else:
        RA, KA = 128 + shift, K       # shift along M (rows)
    A = (torch.randint(-4, 5, (RA, KA), generator=g).float() / 4).to(dt)
    B = (torch.randint(-4, 5, (N, K), generator=g).float() / 4).to(dt)
    Ad, Bd = A.cuda(), B.cuda()
    D = torch.zeros(128, N, dtype=torch.float32, device="cuda")
    rc = probe.umma_probe(tf32, Ad.data_ptr(), Bd.data_ptr(), D.data_ptr(), RA, KA, N, K, a_mn, b_mn, shift, swz)
    assert rc == 0, "CUDA error %d" % rc
    if a_mn:
        Aeff = A[:, shift:shift + K]
    else:
        Aeff = A[shift:shift + 128, :]
    ref = Aeff.double() @ B.double().T
    torch.testing.assert_close(D.cpu().double(), ref, rtol=0, atol=0)


@pytest.mark.parametrize("N,K", [(32, 16), (32, 64), (48, 32), (128, 32)])
def test_umma_ts_tmem_a(probe, N, K):
    """A operand in TMEM written by tcgen05.st (lane = row, 32-bit column j =
    elements 2j, 2j+1), B in shared memory; kind::f16 TS MMA."""
    probe.umma_probe_ts.argtypes = [ctypes.c_void_p] * 3 + [ctypes.c_int] * 2
    probe.umma_probe_ts.restype = ctypes.c_int
    g = torch.Generator().manual_seed(3)
    A = (torch.randint(-4, 5, (128, K), generator=g).float() / 4).to(torch.bfloat16)
    B = (torch.randint(-4, 5, (N, K), generator=g).float() / 4).to(torch.bfloat16)
    Ad, Bd = A.cuda(), B.cuda()
    D = torch.zeros(128, N, dtype=torch.float32, device="cuda")
    assert probe.umma_probe_ts(Ad.data_ptr(), Bd.data_ptr(), D.data_ptr(), N, K) == 0
    ref = A.double() @ B.double().T
    torch.testing.assert_close(D.cpu().double(), ref, rtol=0, atol=0)
