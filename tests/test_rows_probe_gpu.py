"""Probe of the descriptor conventions the D1-outer ("rows") capsule layout
relies on (tests/probe/rows_probe.cu): TMA-swizzled row-major operands read
by tcgen05.mma as K-major with whole-row start shifts (forward / dI tap
shifts) and as MN-major with atoms at arbitrary row strides (dK slot and
column shifts).  Compared bit-exactly with a float64 matmul of the same
exactly-representable bf16 values."""
import ctypes
import os
import subprocess

import pytest
import torch

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
PROBE = os.path.join(HERE, "probe")
LIB = os.path.join(PROBE, "librows_probe.so")
SRC = os.path.join(PROBE, "rows_probe.cu")
CSRC = os.path.join(os.path.dirname(HERE), "paper_2104_02621_b200", "csrc")


def load_probe():
    if not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC) or \
            os.path.getmtime(LIB) < os.path.getmtime(os.path.join(CSRC, "umma.cuh")):
        subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O2", "-std=c++17", "-Xcompiler",
                        "-fPIC", "-shared", "-I", CSRC, "-I", os.path.join(os.path.dirname(HERE), "include"),
                        "-o", LIB, SRC], check=True)
    lib = ctypes.CDLL(LIB)
    lib.rows_probe.argtypes = [ctypes.c_void_p] * 3 + [ctypes.c_int] * 10
    lib.rows_probe.restype = ctypes.c_int
    lib.rows_bench.argtypes = [ctypes.c_int] * 8
    lib.rows_bench.restype = ctypes.c_double
    lib.sync_bench.argtypes = [ctypes.c_int] * 3
    lib.sync_bench.restype = ctypes.c_double
    lib.tile_bench.argtypes = [ctypes.c_int] * 7
    lib.tile_bench.restype = ctypes.c_double
    lib.tmem_bw.argtypes = [ctypes.c_int] * 2
    lib.tmem_bw.restype = ctypes.c_double
    lib.queue_bench.argtypes = [ctypes.c_int] * 4
    lib.queue_bench.restype = ctypes.c_double
    return lib


@pytest.fixture(scope="module")
def probe():
    return load_probe()


def _rup(x, m):
    return (x + m - 1) // m * m


def run_case(probe, mode, E, swz, N, K, a_shift, b_shift=0, a_k0=0, seed=0):
    g = torch.Generator().manual_seed(seed)
    if mode == 0:
        RA, RB = a_shift + 128, N
    else:
        RA, RB = a_k0 + K + (128 // E - 1) * a_shift, K + (N // E - 1) * b_shift
    RA, RB = _rup(RA, 64), _rup(RB, 64)
    A = (torch.randint(-4, 5, (RA, E), generator=g).float() / 4).to(torch.bfloat16)
    B = (torch.randint(-4, 5, (RB, E), generator=g).float() / 4).to(torch.bfloat16)
    Ad, Bd = A.cuda(), B.cuda()
    D = torch.zeros(128, N, dtype=torch.float32, device="cuda")
    rc = probe.rows_probe(Ad.data_ptr(), Bd.data_ptr(), D.data_ptr(), RA, RB, E, swz, mode, N, K, a_shift, b_shift,
                          a_k0)
    assert rc == 0, "probe rc %d" % rc
    Af, Bf = A.double(), B.double()
    if mode == 0:
        ref = Af[a_shift:a_shift + 128] @ Bf[:N].T
    else:
        # A^T atoms: m = j*E + e -> A[a_k0 + k + j*a_shift, e]; B atoms likewise
        Aop = torch.cat([Af[a_k0 + j * a_shift: a_k0 + j * a_shift + K] for j in range(128 // E)], dim=1)  # K x 128
        Bop = torch.cat([Bf[j * b_shift: j * b_shift + K] for j in range(N // E)], dim=1)                 # K x N
        ref = Aop.T @ Bop
    return D.cpu().double(), ref


CASES = [
    # mode, E, swz, N, K, a_shift, b_shift, a_k0
    (0, 32, 64, 32, 32, 0, 0, 0),
    (0, 32, 64, 32, 32, 4, 0, 0),
    (0, 32, 64, 96, 32, 5, 0, 0),
    (0, 32, 64, 32, 32, 13, 0, 0),
    (0, 64, 128, 128, 64, 4, 0, 0),
    (0, 64, 128, 64, 64, 11, 0, 0),
    (1, 32, 64, 96, 64, 96, 4, 0),
    (1, 32, 64, 96, 32, 44, 4, 8),
    (1, 32, 64, 32, 16, 4, 0, 4),
    (1, 32, 64, 64, 48, 40, 8, 16),
    (1, 64, 128, 192, 32, 40, 4, 0),
    (1, 64, 128, 128, 64, 44, 8, 4),
]


@pytest.mark.parametrize("case", CASES, ids=lambda c: "m%d_E%d_sw%d_N%d_K%d_a%d_b%d_k%d" % c)
def test_rows_layout(probe, case):
    mode, E, swz, N, K, a_shift, b_shift, a_k0 = case
    got, ref = run_case(probe, mode, E, swz, N, K, a_shift, b_shift, a_k0)
    torch.testing.assert_close(got, ref, rtol=0, atol=0)


if __name__ == "__main__":
    import sys
    lib = load_probe()
    if "--sync" in sys.argv:
        for mode, name in ((0, "commit->wait round trip"), (1, "commit issue"), (2, "mbarrier hand-off x2")):
            for nb in (1, 148):
                print("sync %-24s blocks %3d: %.1f cycles" % (name, nb, lib.sync_bench(mode, 2000, nb)))
        sys.exit(0)
    if "--queue" in sys.argv:
        for N in (96, 192):
            for K in (1, 2, 4, 8):
                row = []
                for spin in (0, 100, 200, 400, 800):
                    row.append("spin %3d: %6.0f" % (spin, lib.queue_bench(N, K, spin, 200)))
                print("queue N %3d K %d  " % (N, K) + "  ".join(row), flush=True)
        sys.exit(0)
    if "--tmem" in sys.argv:
        for nw in (1, 4, 8, 16):
            print("tmem read nwarps %2d: %.1f bytes/cycle/SM" % (nw, lib.tmem_bw(nw, 2000)))
        sys.exit(0)
    if "--tile" in sys.argv:
        for N in (96, 128):
            for per in (6, 24):
                for bmode in (0, 4):
                    cyc = lib.tile_bench(N, 400, per, 4, 1, 1, bmode)
                    print("tile N %3d per %2d bmode %d: %.1f cycles/MMA" % (N, per, bmode, cyc))
        sys.exit(0)
    if "--align" in sys.argv:
        for mode, swz in ((0, 64), (2, 64), (2, 128), (1, 64)):
            for N in (96, 192):
                for aoff in (0, 256):
                    for walk in (0, 256):
                        cyc = lib.rows_bench(mode, swz, N, 4096, 1, 148, aoff, walk)
                        print("align mode %d swz %3d N %3d aoff %4d walk %4d: %.1f cycles/MMA" % (
                            mode, swz, N, aoff, walk, cyc))
        sys.exit(0)
    for c in CASES:
        got, ref = run_case(lib, *c)
        print("case", c, "max |diff| = %.3g" % float((got - ref).abs().max()))
    for mode, swz in ((0, 64), (0, 128), (1, 64), (1, 128)):
        for N in (32, 64, 96, 128, 192, 256):
            for nacc in (1, 2):
                cyc = lib.rows_bench(mode, swz, N, 4096, nacc, 148, 0, 0)
                print("bench mode %d swz %d N %3d nacc %d: %.1f cycles/MMA" % (mode, swz, N, nacc, cyc))
