"""ctypes wrapper around oracle/capsconv_oracle.c (TEST INFRASTRUCTURE ONLY).

Arrays are numpy float64, C-contiguous, in the layouts of DESIGN.md §2:
  I, dI : (B, H, W, C, D1, D2)
  K, dK : (KH, KW, C, Cout, D2, D3)
  O, dO : (B, Ho, Wo, Cout, D1, D3)
Each compute function returns (value, abs_sum) where abs_sum is
sum |term| over the same terms (the error-metric denominator, reading R19).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "capsconv_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None


class OracleError(ValueError):
    pass


def lib_path() -> str:
    return _LIB


def build(force: bool = False) -> str:
    """Compile the oracle with gcc -O2 -fopenmp (no -ffast-math, no SIMD flags)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + ".tmp.%d" % os.getpid()
        cmd = ["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-std=c11", "-fno-fast-math",
               "-o", tmp, _SRC, "-lm"]
        subprocess.run(cmd, check=True)
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    with _lock:
        if _lib is None:
            build()
            lib = ctypes.CDLL(_LIB)
            i64 = ctypes.c_int64
            dp = ctypes.POINTER(ctypes.c_double)
            lib.oracle_output_dims.argtypes = [i64] * 5 + [ctypes.POINTER(i64)] * 2
            lib.oracle_output_dims.restype = ctypes.c_int
            for name in ("oracle_fwd", "oracle_bwd_data", "oracle_bwd_kernel"):
                fn = getattr(lib, name)
                fn.argtypes = [i64] * 11 + [dp] * 4
                fn.restype = ctypes.c_int
                fp = getattr(lib, name + "_pad")
                fp.argtypes = [i64] * 12 + [dp] * 4
                fp.restype = ctypes.c_int
            for name in ("oracle_fwd_slices", "oracle_bwd_data_slices", "oracle_bwd_kernel_slices"):
                fn = getattr(lib, name)
                fn.argtypes = [i64] * 12 + [dp] * 4
                fn.restype = ctypes.c_int
            lib.oracle_output_dims_pad.argtypes = [i64] * 6 + [ctypes.POINTER(i64)] * 2
            lib.oracle_output_dims_pad.restype = ctypes.c_int
            lib.oracle_round_bf16_array.argtypes = [dp, i64]
            lib.oracle_round_bf16_array.restype = None
            lib.oracle_num_threads.argtypes = []
            lib.oracle_num_threads.restype = ctypes.c_int
            lib.oracle_set_num_threads.argtypes = [ctypes.c_int]
            lib.oracle_set_num_threads.restype = None
            _lib = lib
    return _lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _f64(a) -> np.ndarray:
    a = np.asarray(a)
    return np.ascontiguousarray(a, dtype=np.float64)


def num_threads() -> int:
    return int(_load().oracle_num_threads())


def set_num_threads(n: int) -> None:
    """OpenMP thread count of the oracle loops (timing only)."""
    _load().oracle_set_num_threads(int(n))


def output_dims(H, W, KH, KW, stride, pad=0):
    lib = _load()
    ho, wo = ctypes.c_int64(), ctypes.c_int64()
    if pad:
        rc = lib.oracle_output_dims_pad(H, W, KH, KW, stride, pad, ctypes.byref(ho), ctypes.byref(wo))
    else:
        rc = lib.oracle_output_dims(H, W, KH, KW, stride, ctypes.byref(ho), ctypes.byref(wo))
    if rc:
        raise OracleError("oracle_output_dims: status %d" % rc)
    return ho.value, wo.value


def fwd(I, K, stride, pad=0):
    """O = I (*) K  (Algorithm 2); pad > 0: symmetric zero
    padding (oracle_fwd_pad)."""
    I, K = _f64(I), _f64(K)
    B, H, W, C, D1, D2 = I.shape
    KH, KW, C2, Cout, D2b, D3 = K.shape
    if C2 != C or D2b != D2:
        raise OracleError("channel / inner capsule dims disagree")
    Ho, Wo = output_dims(H, W, KH, KW, stride, pad)
    O = np.empty((B, Ho, Wo, Cout, D1, D3))
    A = np.empty_like(O)
    if pad:
        rc = _load().oracle_fwd_pad(B, H, W, C, Cout, KH, KW, D1, D2, D3, stride, pad,
                                    _ptr(I), _ptr(K), _ptr(O), _ptr(A))
    else:
        rc = _load().oracle_fwd(B, H, W, C, Cout, KH, KW, D1, D2, D3, stride,
                                _ptr(I), _ptr(K), _ptr(O), _ptr(A))
    if rc:
        raise OracleError("oracle_fwd: status %d" % rc)
    return O, A


def bwd_data(dO, K, stride, H, W, pad=0):
    """dI, the adjoint of fwd in I (Algorithm 4 read as in R10/R11)."""
    dO, K = _f64(dO), _f64(K)
    B, Ho, Wo, Cout, D1, D3 = dO.shape
    KH, KW, C, Cout2, D2, D3b = K.shape
    if Cout2 != Cout or D3b != D3:
        raise OracleError("output channel / capsule dims disagree")
    if output_dims(H, W, KH, KW, stride, pad) != (Ho, Wo):
        raise OracleError("dO spatial shape does not follow the shape law")
    dI = np.empty((B, H, W, C, D1, D2))
    A = np.empty_like(dI)
    if pad:
        rc = _load().oracle_bwd_data_pad(B, H, W, C, Cout, KH, KW, D1, D2, D3, stride, pad,
                                         _ptr(dO), _ptr(K), _ptr(dI), _ptr(A))
    else:
        rc = _load().oracle_bwd_data(B, H, W, C, Cout, KH, KW, D1, D2, D3, stride,
                                     _ptr(dO), _ptr(K), _ptr(dI), _ptr(A))
    if rc:
        raise OracleError("oracle_bwd_data: status %d" % rc)
    return dI, A


def bwd_kernel(I, dO, stride, KH, KW, pad=0):
    """dK, the adjoint of fwd in K (Algorithm 4 read as in R10/R11)."""
    I, dO = _f64(I), _f64(dO)
    B, H, W, C, D1, D2 = I.shape
    B2, Ho, Wo, Cout, D1b, D3 = dO.shape
    if B2 != B or D1b != D1:
        raise OracleError("batch / D1 disagree")
    if output_dims(H, W, KH, KW, stride, pad) != (Ho, Wo):
        raise OracleError("dO spatial shape does not follow the shape law")
    dK = np.empty((KH, KW, C, Cout, D2, D3))
    A = np.empty_like(dK)
    if pad:
        rc = _load().oracle_bwd_kernel_pad(B, H, W, C, Cout, KH, KW, D1, D2, D3, stride, pad,
                                           _ptr(I), _ptr(dO), _ptr(dK), _ptr(A))
    else:
        rc = _load().oracle_bwd_kernel(B, H, W, C, Cout, KH, KW, D1, D2, D3, stride,
                                       _ptr(I), _ptr(dO), _ptr(dK), _ptr(A))
    if rc:
        raise OracleError("oracle_bwd_kernel: status %d" % rc)
    return dK, A


def fwd_slices(I, K, stride):
    """S-slice capsules: I (B,H,W,C,S,D1,D2),
    K (KH,KW,C,Cout,S,D2,D3) -> O (B,Ho,Wo,Cout,S,D1,D3), slice-wise products."""
    I, K = _f64(I), _f64(K)
    B, H, W, C, S, D1, D2 = I.shape
    KH, KW, C2, Cout, S2, D2b, D3 = K.shape
    if C2 != C or S2 != S or D2b != D2:
        raise OracleError("channel / slice / inner capsule dims disagree")
    Ho, Wo = output_dims(H, W, KH, KW, stride)
    O = np.empty((B, Ho, Wo, Cout, S, D1, D3))
    A = np.empty_like(O)
    rc = _load().oracle_fwd_slices(B, H, W, C, Cout, KH, KW, S, D1, D2, D3, stride, _ptr(I), _ptr(K), _ptr(O), _ptr(A))
    if rc:
        raise OracleError("oracle_fwd_slices: status %d" % rc)
    return O, A


def bwd_data_slices(dO, K, stride, H, W):
    dO, K = _f64(dO), _f64(K)
    B, Ho, Wo, Cout, S, D1, D3 = dO.shape
    KH, KW, C, Cout2, S2, D2, D3b = K.shape
    if Cout2 != Cout or S2 != S or D3b != D3 or output_dims(H, W, KH, KW, stride) != (Ho, Wo):
        raise OracleError("shapes disagree")
    dI = np.empty((B, H, W, C, S, D1, D2))
    A = np.empty_like(dI)
    rc = _load().oracle_bwd_data_slices(B, H, W, C, Cout, KH, KW, S, D1, D2, D3, stride, _ptr(dO), _ptr(K), _ptr(dI),
                                        _ptr(A))
    if rc:
        raise OracleError("oracle_bwd_data_slices: status %d" % rc)
    return dI, A


def bwd_kernel_slices(I, dO, stride, KH, KW):
    I, dO = _f64(I), _f64(dO)
    B, H, W, C, S, D1, D2 = I.shape
    B2, Ho, Wo, Cout, S2, D1b, D3 = dO.shape
    if B2 != B or S2 != S or D1b != D1 or output_dims(H, W, KH, KW, stride) != (Ho, Wo):
        raise OracleError("shapes disagree")
    dK = np.empty((KH, KW, C, Cout, S, D2, D3))
    A = np.empty_like(dK)
    rc = _load().oracle_bwd_kernel_slices(B, H, W, C, Cout, KH, KW, S, D1, D2, D3, stride, _ptr(I), _ptr(dO),
                                          _ptr(dK), _ptr(A))
    if rc:
        raise OracleError("oracle_bwd_kernel_slices: status %d" % rc)
    return dK, A


def round_bf16(x) -> np.ndarray:
    """Round every element to the nearest bfloat16 (ties to even), in float64."""
    x = _f64(x).copy()
    _load().oracle_round_bf16_array(_ptr(x), x.size)
    return x


def stack_fwd_bwd(X, Ks, strides, dY, bf16_boundaries: bool, pads=None):
    """Config-5 stack: layers composed with the identity between them
    (reading R17), forward then backward in reverse order.

    When ``bf16_boundaries`` is set, each layer's forward output and each
    propagated dI is rounded to bf16 where the GPU path stores bf16
    (reading R13).  Returns (outputs, dX, dKs, abs-sums dict).
    """
    pads = list(pads) if pads is not None else [0] * len(Ks)
    acts = [_f64(X)]
    fabs_ = []
    for K, s, pd in zip(Ks, strides, pads):
        O, A = fwd(acts[-1], K, s, pd)
        if bf16_boundaries:
            O = round_bf16(O)
        acts.append(O)
        fabs_.append(A)
    g = _f64(dY)
    dKs = [None] * len(Ks)
    dKabs = [None] * len(Ks)
    dIabs = [None] * len(Ks)
    for li in range(len(Ks) - 1, -1, -1):
        K, s, pd = Ks[li], strides[li], pads[li]
        x = acts[li]
        dK, dKa = bwd_kernel(x, g, s, K.shape[0], K.shape[1], pd)
        dKs[li], dKabs[li] = dK, dKa
        dI, dIa = bwd_data(g, K, s, x.shape[1], x.shape[2], pd)
        if bf16_boundaries:
            dI = round_bf16(dI)
        dIabs[li] = dIa
        g = dI
    return acts, g, dKs, {"fwd": fabs_, "dK": dKabs, "dI": dIabs}


def sgd_update(w, g, lr):
    """One SGD step (plain gradient descent, no momentum):
    w - lr * g, exact in float64 (the device computes it with one fp32 fma)."""
    return _f64(w) - float(lr) * _f64(g)


def primary_to_caps(prim, C, D):
    """Primary-layer output (B, H, W, 1, 1, C*D*D), channel o = (d1*C + c)*D + d2
    (the rows order, reading R25) -> the natural capsule map (B, H, W, C, D, D)."""
    p = _f64(prim)
    B, H, W = p.shape[:3]
    return np.ascontiguousarray(p.reshape(B, H, W, D, C, D).transpose(0, 1, 2, 4, 3, 5))


def caps_to_primary(x):
    """Inverse of primary_to_caps: (B, H, W, C, D, D) -> (B, H, W, 1, 1, C*D*D)."""
    x = _f64(x)
    B, H, W, C, D1, D2 = x.shape
    return np.ascontiguousarray(x.transpose(0, 1, 2, 4, 3, 5).reshape(B, H, W, 1, 1, C * D1 * D2))


def train_step(img, Kp, Ks, strides, dY, lr, bf16_boundaries: bool):
    """The routing-free P-CapsNet training step:
    primary layer (the capsule convolution with C = Cout = D1 = D2 = 1, reading
    R25) -> the stack (stack_fwd_bwd) -> primary dK from the stack's dX -> one
    SGD step on every weight.  dY is the stack output gradient in the natural
    layout.  Returns (new weights [Kp, K_0, ...] in float64, dKs [dKp, dK_0, ...],
    abs-sums [of dKp, dK_0, ...])."""
    C0, D = Ks[0].shape[2], Ks[0].shape[4]
    prim, _ = fwd(img, Kp, 1)
    if bf16_boundaries:
        prim = round_bf16(prim)
    X = primary_to_caps(prim, C0, D)
    acts, dX, dKs, absd = stack_fwd_bwd(X, Ks, strides, dY, bf16_boundaries)
    dprim = caps_to_primary(dX)
    dKp, dKp_abs = bwd_kernel(img, dprim, 1, Kp.shape[0], Kp.shape[1])
    new = [sgd_update(Kp, dKp, lr)] + [sgd_update(K, g, lr) for K, g in zip(Ks, dKs)]
    return new, [dKp] + list(dKs), [dKp_abs] + list(absd["dK"])
