"""The C-ABI library loads, exports every symbol include/capsconv.h declares,
and validates arguments (host logic only; no compute calls without a GPU)."""
import ctypes
import os
import re

import pytest
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "capsconv.h")


@pytest.fixture(scope="module")
def cc():
    from paper_2104_02621_b200 import _build
    _build.build()
    import paper_2104_02621_b200.capsconv as cc
    cc.load_library()
    return cc


def declared_symbols():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"CAPSCONV_API\s+[^;(]*?\b(capsconv_\w+)\s*\(", src)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for s in ("capsconv_fwd", "capsconv_bwd_data", "capsconv_bwd_kernel", "capsconv_output_dims",
              "capsconv_workspace_bytes", "capsconv_status_string", "capsconv_last_error"):
        assert s in syms


def test_library_exports_every_declared_symbol(cc):
    lib = ctypes.CDLL(cc.LIB_PATH)
    for s in declared_symbols():
        assert hasattr(lib, s), "libcapsconv.so does not export %s" % s


def test_exports_only_the_c_abi(cc):
    import subprocess
    out = subprocess.run(["nm", "-D", "--defined-only", cc.LIB_PATH], capture_output=True, text=True).stdout
    exported = {l.split()[-1] for l in out.splitlines() if " T " in l}
    assert exported == set(declared_symbols())


def test_version(cc):
    assert re.match(r"^\d+\.\d+\.\d+$", cc.version())


@pytest.mark.parametrize("args,expect", [
    ((5, 5, 4, 4, 1), (2, 2)),
    ((32, 32, 3, 3, 1), (30, 30)),
    ((16, 16, 3, 3, 2), (7, 7)),
    ((22, 22, 3, 3, 2), (10, 10)),
    ((8, 8, 8, 8, 1), (1, 1)),
    ((28, 28, 3, 3, 2), (13, 13)),
])
def test_output_dims(cc, args, expect):
    assert cc.output_dims(*args) == expect


def test_output_dims_errors(cc):
    for bad in [(4, 4, 5, 1, 1), (4, 4, 1, 1, 0), (0, 4, 1, 1, 1), (4, 4, 0, 1, 1)]:
        with pytest.raises(cc.CapsConvError):
            cc.output_dims(*bad)


def _raw(cc):
    return cc.load_library()


EXT_OK = (2, 8, 8, 2, 3, 3, 3, 4, 4, 4, 1)


def test_validation_before_any_launch(cc):
    lib = _raw(cc)
    vp = ctypes.c_void_p
    fake = vp(0x1000)
    # null tensor pointer
    st = lib.capsconv_fwd(0, *EXT_OK, None, fake, fake, None, 0, None)
    assert st == 1 and b"NULL" in lib.capsconv_last_error()
    # bad extents / stride / dtype
    bad_shape = (2, 8, 8, 2, 3, 9, 3, 4, 4, 4, 1)
    assert lib.capsconv_fwd(0, *bad_shape, fake, fake, fake, None, 0, None) == 2
    zero_ext = (2, 8, 8, 0, 3, 3, 3, 4, 4, 4, 1)
    assert lib.capsconv_bwd_data(0, *zero_ext, fake, fake, fake, None, 0, None) == 2
    bad_stride = EXT_OK[:-1] + (0,)
    assert lib.capsconv_bwd_kernel(1, *bad_stride, fake, fake, fake, None, 0, None) == 3
    assert lib.capsconv_fwd(7, *EXT_OK, fake, fake, fake, None, 0, None) == 4
    # status strings
    for s in range(9):
        assert lib.capsconv_status_string(s).startswith(b"CAPSCONV_")


def test_overflow_is_rejected(cc):
    lib = _raw(cc)
    fake = ctypes.c_void_p(0x1000)
    huge = (1 << 40, 8, 8, 2, 3, 3, 3, 4, 4, 4, 1)
    assert lib.capsconv_fwd(0, *huge, fake, fake, fake, None, 0, None) == 6


def test_workspace_query_and_insufficient_workspace(cc):
    lib = _raw(cc)
    ext = (64, 32, 32, 8, 8, 3, 3, 4, 4, 4, 1)
    need = cc.workspace_bytes(cc.OP_BWD_KERNEL, torch.float32, ext)
    assert need >= 0
    assert cc.workspace_bytes(cc.OP_FWD, torch.float32, (1, 5, 5, 1, 1, 4, 4, 3, 3, 3, 1)) == 0
    if need > 0:
        fake = ctypes.c_void_p(0x1000)
        st = lib.capsconv_bwd_kernel(0, *ext, fake, fake, fake, fake, need - 1, None)
        assert st == 5


def test_select_path_is_total(cc):
    # every valid problem has a path; fig2 (D=3, C=1) must take SIMT
    assert cc.select_path(cc.OP_FWD, torch.float32, (1, 5, 5, 1, 1, 4, 4, 3, 3, 3, 1)) == cc.PATH_SIMT
    for op in (cc.OP_FWD, cc.OP_BWD_DATA, cc.OP_BWD_KERNEL):
        for dt in (torch.float32, torch.bfloat16):
            for ext in [(64, 32, 32, 8, 8, 3, 3, 4, 4, 4, 1), (128, 16, 16, 16, 32, 3, 3, 4, 4, 4, 2),
                        (256, 8, 8, 32, 10, 8, 8, 4, 4, 4, 1), (3, 7, 5, 3, 2, 2, 3, 2, 5, 3, 3)]:
                assert cc.select_path(op, dt, ext) in (cc.PATH_SIMT, cc.PATH_MMA)


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-device error on a CPU-only host")
def test_no_device_error(cc):
    lib = _raw(cc)
    fake = ctypes.c_void_p(0x1000)
    # a workspace of the required size, so that the device check is what fails
    need = ctypes.c_size_t()
    assert lib.capsconv_workspace_bytes(0, 0, *EXT_OK, ctypes.byref(need)) == 0
    st = lib.capsconv_fwd(0, *EXT_OK, fake, fake, fake, fake if need.value else None, need.value, None)
    assert st == 7


def test_python_binding_refuses_cpu_tensors(cc):
    I = torch.zeros(1, 5, 5, 1, 3, 3)
    K = torch.zeros(4, 4, 1, 1, 3, 3)
    with pytest.raises(ValueError):
        cc.fwd(I, K, 1)


def test_layout_argument(cc):
    """capsconv_*_ex: an unknown layout is CAPSCONV_ERR_DTYPE before anything
    else; both layouts have a path for every valid problem, and the rows
    layout's fallback reserves workspace for its two permuted copies."""
    lib = _raw(cc)
    fake = ctypes.c_void_p(0x1000)
    ext12 = EXT_OK + (0,)
    for fn in (lib.capsconv_fwd_ex, lib.capsconv_bwd_data_ex, lib.capsconv_bwd_kernel_ex):
        fn.argtypes = [ctypes.c_int, ctypes.c_int] + [ctypes.c_int64] * 12 + [ctypes.c_void_p] * 4 + \
            [ctypes.c_size_t, ctypes.c_void_p]
        assert fn(1, 2, *ext12, fake, fake, fake, None, 0, None) == 4
        assert b"layout" in lib.capsconv_last_error()
    for op in (cc.OP_FWD, cc.OP_BWD_DATA, cc.OP_BWD_KERNEL):
        for dt in (torch.float32, torch.bfloat16):
            for ext in [(64, 32, 32, 8, 8, 3, 3, 4, 4, 4, 1), (3, 7, 5, 3, 2, 2, 3, 2, 5, 3, 3)]:
                assert cc.select_path(op, dt, ext, "rows") in (cc.PATH_SIMT, cc.PATH_MMA)
    # fp32 rows problems run the natural path between permutations
    ext = (2, 9, 9, 3, 5, 3, 3, 4, 4, 4, 1)
    nat = cc.workspace_bytes(cc.OP_FWD, torch.float32, ext)
    rows = cc.workspace_bytes(cc.OP_FWD, torch.float32, ext, "rows")
    n_in, n_out = 2 * 9 * 9 * 3 * 16 * 4, 2 * 7 * 7 * 5 * 16 * 4
    assert rows >= nat + n_in + n_out
    with pytest.raises(ValueError):
        cc.workspace_bytes(cc.OP_FWD, torch.float32, ext, "columns")


def test_sgd_update_validation(cc):
    """capsconv_sgd_update validates before any launch (no device needed):
    unknown dtype (4), n < 0 or a non-finite lr (2), NULL pointers (1); n = 0
    is a no-op that returns OK even with NULL pointers."""
    lib = cc.load_library()
    f = lib.capsconv_sgd_update
    buf = (ctypes.c_float * 8)()
    p = ctypes.cast(buf, ctypes.c_void_p)
    lr = ctypes.c_float(0.1)
    assert f(7, 4, lr, p, p, p, None) == 4 and b"dtype" in lib.capsconv_last_error()
    assert f(0, -1, lr, p, p, p, None) == 2
    assert f(0, 4, ctypes.c_float(float("nan")), p, p, p, None) == 2 and b"learning rate" in lib.capsconv_last_error()
    assert f(0, 4, lr, None, p, p, None) == 1 and b"NULL" in lib.capsconv_last_error()
    assert f(1, 0, lr, None, None, None, None) == 0
