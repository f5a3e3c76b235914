"""Thin Python binding of libcapsconv (include/capsconv.h).

Argument marshalling only: shapes are read from the tensors, pointers and the
current CUDA stream are passed to the C ABI, and every step of the capsule
convolution runs inside libcapsconv's kernels.  PyTorch provides device
memory and streams (plumbing).  There is no CPU fallback: if the library is
missing or the tensors are not CUDA tensors, these functions raise.

Layouts (Algorithm 2), chosen per call with
``layout=``:
  "natural" I, dI : (B, H, W, C, D1, D2)   O, dO : (B, Ho, Wo, Cout, D1, D3)
  "rows"    I, dI : (B, H, W, D1, C, D2)   O, dO : (B, Ho, Wo, D1, Cout, D3)
  K : (KH, KW, C, Cout, D2, D3) and dK (always float32) in both.
"""
from __future__ import annotations

import ctypes
import os
import threading
from typing import Optional, Tuple

import torch

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "libcapsconv.so")

OP_FWD, OP_BWD_DATA, OP_BWD_KERNEL = 0, 1, 2
PATH_AUTO, PATH_SIMT, PATH_MMA = 0, 1, 2
LAYOUT_NATURAL, LAYOUT_ROWS = 0, 1
_LAYOUTS = {"natural": LAYOUT_NATURAL, "rows": LAYOUT_ROWS, LAYOUT_NATURAL: LAYOUT_NATURAL, LAYOUT_ROWS: LAYOUT_ROWS}
_DT = {torch.float32: 0, torch.bfloat16: 1}

_lock = threading.Lock()
_lib = None


class CapsConvError(RuntimeError):
    """A non-OK status from libcapsconv."""


def load_library(path: Optional[str] = None):
    """Load libcapsconv.so (built in-tree by __graft_entry__.build()).  Raises
    if it is missing: there is no fallback implementation."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        p = path or LIB_PATH
        if not os.path.exists(p):
            raise ImportError("libcapsconv.so not found at %s; run `python -c 'import __graft_entry__ as g; "
                              "g.build()'` (nvcc, sm_100a) first" % p)
        lib = ctypes.CDLL(p)
        i64, sz = ctypes.c_int64, ctypes.c_size_t
        vp = ctypes.c_void_p
        ext = [i64] * 11
        lib.capsconv_output_dims.argtypes = [i64] * 5 + [ctypes.POINTER(i64)] * 2
        lib.capsconv_workspace_bytes.argtypes = [ctypes.c_int, ctypes.c_int] + ext + [ctypes.POINTER(sz)]
        lib.capsconv_select_path.argtypes = [ctypes.c_int, ctypes.c_int] + ext + [ctypes.POINTER(ctypes.c_int)]
        lib.capsconv_set_path_override.argtypes = [ctypes.c_int]
        for name in ("capsconv_fwd", "capsconv_bwd_data", "capsconv_bwd_kernel"):
            getattr(lib, name).argtypes = [ctypes.c_int] + ext + [vp, vp, vp, vp, sz, vp]
        ext12 = [i64] * 12
        lib.capsconv_output_dims_pad.argtypes = [i64] * 6 + [ctypes.POINTER(i64)] * 2
        lib.capsconv_workspace_bytes_pad.argtypes = [ctypes.c_int, ctypes.c_int] + ext12 + [ctypes.POINTER(sz)]
        lib.capsconv_select_path_pad.argtypes = [ctypes.c_int, ctypes.c_int] + ext12 + [ctypes.POINTER(ctypes.c_int)]
        for name in ("capsconv_fwd_pad", "capsconv_bwd_data_pad", "capsconv_bwd_kernel_pad"):
            getattr(lib, name).argtypes = [ctypes.c_int] + ext12 + [vp, vp, vp, vp, sz, vp]
        ci = ctypes.c_int
        lib.capsconv_workspace_bytes_ex.argtypes = [ci, ci, ci] + ext12 + [ctypes.POINTER(sz)]
        lib.capsconv_select_path_ex.argtypes = [ci, ci, ci] + ext12 + [ctypes.POINTER(ci)]
        for name in ("capsconv_fwd_ex", "capsconv_bwd_data_ex", "capsconv_bwd_kernel_ex"):
            getattr(lib, name).argtypes = [ci, ci] + ext12 + [vp, vp, vp, vp, sz, vp]
        for name in ("capsconv_workspace_bytes_ex", "capsconv_select_path_ex", "capsconv_fwd_ex",
                     "capsconv_bwd_data_ex", "capsconv_bwd_kernel_ex"):
            getattr(lib, name).restype = ci
        lib.capsconv_sgd_update.argtypes = [ctypes.c_int, i64, ctypes.c_float, vp, vp, vp, vp]
        lib.capsconv_sgd_update.restype = ctypes.c_int
        lib.capsconv_workspace_bytes_slices.argtypes = [ctypes.c_int, ctypes.c_int] + [i64] * 12 + [ctypes.POINTER(sz)]
        for name in ("capsconv_fwd_slices", "capsconv_bwd_data_slices", "capsconv_bwd_kernel_slices"):
            getattr(lib, name).argtypes = [ctypes.c_int] + [i64] * 12 + [vp, vp, vp, vp, sz, vp]
            getattr(lib, name).restype = ctypes.c_int
        lib.capsconv_workspace_bytes_slices.restype = ctypes.c_int
        for name in ("capsconv_output_dims", "capsconv_workspace_bytes", "capsconv_select_path",
                     "capsconv_set_path_override", "capsconv_fwd", "capsconv_bwd_data", "capsconv_bwd_kernel",
                     "capsconv_output_dims_pad", "capsconv_workspace_bytes_pad", "capsconv_select_path_pad",
                     "capsconv_fwd_pad", "capsconv_bwd_data_pad", "capsconv_bwd_kernel_pad"):
            getattr(lib, name).restype = ctypes.c_int
        lib.capsconv_status_string.argtypes = [ctypes.c_int]
        lib.capsconv_status_string.restype = ctypes.c_char_p
        lib.capsconv_last_error.argtypes = []
        lib.capsconv_last_error.restype = ctypes.c_char_p
        lib.capsconv_launch_count.argtypes = []
        lib.capsconv_launch_count.restype = ctypes.c_uint64
        lib.capsconv_version.argtypes = []
        lib.capsconv_version.restype = ctypes.c_char_p
        _lib = lib
        return lib


def _check(status: int, what: str):
    if status != 0:
        lib = load_library()
        raise CapsConvError("%s: %s (%s)" % (what, lib.capsconv_status_string(status).decode(),
                                             lib.capsconv_last_error().decode()))


def version() -> str:
    return load_library().capsconv_version().decode()


def launch_count() -> int:
    """Kernels enqueued by libcapsconv in this process so far."""
    return int(load_library().capsconv_launch_count())


_dims_cache = {}


def output_dims(H: int, W: int, KH: int, KW: int, stride: int, pad: int = 0) -> Tuple[int, int]:
    key = (H, W, KH, KW, stride, pad)
    v = _dims_cache.get(key)
    if v is None:
        lib = load_library()
        ho, wo = ctypes.c_int64(), ctypes.c_int64()
        _check(lib.capsconv_output_dims_pad(H, W, KH, KW, stride, pad, ctypes.byref(ho), ctypes.byref(wo)),
               "output_dims")
        v = _dims_cache[key] = (ho.value, wo.value)
    return v


def _dt(dtype) -> int:
    if dtype not in _DT:
        raise ValueError("libcapsconv supports float32 and bfloat16, got %s" % dtype)
    return _DT[dtype]


_ws_size_cache = {}


def _ext12(ext):
    """Extents (B,H,W,C,Cout,KH,KW,D1,D2,D3,stride[,pad]); pad defaults to 0."""
    ext = tuple(ext)
    return ext + (0,) if len(ext) == 11 else ext


def _layout(layout) -> int:
    if layout not in _LAYOUTS:
        raise ValueError("layout must be 'natural' or 'rows', got %r" % (layout,))
    return _LAYOUTS[layout]


def workspace_bytes(op: int, dtype, ext, layout="natural") -> int:
    ext = _ext12(ext)
    lay = _layout(layout)
    key = (op, dtype, ext, lay, _device_key())
    v = _ws_size_cache.get(key)
    if v is None:
        lib = load_library()
        out = ctypes.c_size_t()
        _check(lib.capsconv_workspace_bytes_ex(op, _dt(dtype), lay, *ext, ctypes.byref(out)), "workspace_bytes")
        v = _ws_size_cache[key] = out.value
    return v


def _device_key():
    return torch.cuda.current_device() if torch.cuda.is_available() else -1


def select_path(op: int, dtype, ext, layout="natural") -> int:
    lib = load_library()
    out = ctypes.c_int()
    _check(lib.capsconv_select_path_ex(op, _dt(dtype), _layout(layout), *_ext12(ext), ctypes.byref(out)),
           "select_path")
    return out.value


def set_path_override(path: int):
    _check(load_library().capsconv_set_path_override(path), "set_path_override")


# Workspace: one growable device buffer per (device, stream).
_ws_cache = {}


def _workspace(nbytes: int, device: torch.device, stream_handle: int):
    if nbytes == 0:
        return None
    key = (device.index, stream_handle)
    buf = _ws_cache.get(key)
    if buf is None or buf.numel() < nbytes:
        buf = torch.empty(nbytes, dtype=torch.uint8, device=device)
        _ws_cache[key] = buf
    return buf


def _need_cuda(*ts):
    for t in ts:
        if not isinstance(t, torch.Tensor) or not t.is_cuda:
            raise ValueError("libcapsconv takes CUDA tensors (no CPU path)")
        if not t.is_contiguous():
            raise ValueError("libcapsconv takes contiguous tensors")
    dev = ts[0].device
    for t in ts[1:]:
        if t.device != dev:
            raise ValueError("tensors are on different devices")
    return dev


def _call(name: str, op: int, dtype, ext, a, b, out, stream: Optional[torch.cuda.Stream], layout=LAYOUT_NATURAL):
    lib = load_library()
    s = stream if stream is not None else torch.cuda.current_stream(out.device)
    handle = s.cuda_stream
    ext = _ext12(ext)
    need = workspace_bytes(op, dtype, ext, layout)
    ws = _workspace(need, out.device, handle)
    fn = getattr(lib, name + "_ex")
    with torch.cuda.device(out.device):
        st = fn(_dt(dtype), _layout(layout), *ext, ctypes.c_void_p(a.data_ptr()), ctypes.c_void_p(b.data_ptr()),
                ctypes.c_void_p(out.data_ptr()), ctypes.c_void_p(ws.data_ptr() if ws is not None else 0),
                ctypes.c_size_t(need), ctypes.c_void_p(handle))
    _check(st, name)
    return out


def _split(t, layout):
    """(B, H, W, C, D1, D2) of a capsule tensor in either layout."""
    if _layout(layout) == LAYOUT_ROWS:
        B, H, W, D1, C, D2 = t.shape
    else:
        B, H, W, C, D1, D2 = t.shape
    return B, H, W, C, D1, D2


def _shape(B, H, W, C, D1, D2, layout):
    return (B, H, W, D1, C, D2) if _layout(layout) == LAYOUT_ROWS else (B, H, W, C, D1, D2)


def fwd(I: torch.Tensor, K: torch.Tensor, stride: int = 1, out: Optional[torch.Tensor] = None,
        stream: Optional[torch.cuda.Stream] = None, pad: int = 0, layout="natural") -> torch.Tensor:
    """O = capsule_conv(I, K, stride) (capsconv_fwd_ex); pad > 0: symmetric zero
    padding of H and W; layout: "natural" or "rows" (capsconv.h)."""
    dev = _need_cuda(I, K)
    if I.dim() != 6 or K.dim() != 6:
        raise ValueError("I must be (B,H,W,C,D1,D2) [natural] / (B,H,W,D1,C,D2) [rows] and K (KH,KW,C,Cout,D2,D3)")
    B, H, W, C, D1, D2 = _split(I, layout)
    KH, KW, C2, Cout, D2b, D3 = K.shape
    if C2 != C or D2b != D2 or I.dtype != K.dtype:
        raise ValueError("I %s and K %s disagree" % (tuple(I.shape), tuple(K.shape)))
    Ho, Wo = output_dims(H, W, KH, KW, stride, pad)
    shape = _shape(B, Ho, Wo, Cout, D1, D3, layout)
    if out is None:
        out = torch.empty(shape, dtype=I.dtype, device=dev)
    elif tuple(out.shape) != shape or out.dtype != I.dtype:
        raise ValueError("out has the wrong shape/dtype")
    ext = (B, H, W, C, Cout, KH, KW, D1, D2, D3, stride, pad)
    return _call("capsconv_fwd", OP_FWD, I.dtype, ext, I, K, out, stream, layout)


def bwd_data(dO: torch.Tensor, K: torch.Tensor, stride: int, H: int, W: int,
             out: Optional[torch.Tensor] = None, stream: Optional[torch.cuda.Stream] = None,
             pad: int = 0, layout="natural") -> torch.Tensor:
    """dI (capsconv_bwd_data_ex)."""
    dev = _need_cuda(dO, K)
    B, Ho, Wo, Cout, D1, D3 = _split(dO, layout)
    KH, KW, C, Cout2, D2, D3b = K.shape
    if Cout2 != Cout or D3b != D3 or dO.dtype != K.dtype:
        raise ValueError("dO %s and K %s disagree" % (tuple(dO.shape), tuple(K.shape)))
    if output_dims(H, W, KH, KW, stride, pad) != (Ho, Wo):
        raise ValueError("dO spatial extent does not match H, W, K, stride and pad")
    shape = _shape(B, H, W, C, D1, D2, layout)
    if out is None:
        out = torch.empty(shape, dtype=dO.dtype, device=dev)
    elif tuple(out.shape) != shape or out.dtype != dO.dtype:
        raise ValueError("out has the wrong shape/dtype")
    ext = (B, H, W, C, Cout, KH, KW, D1, D2, D3, stride, pad)
    return _call("capsconv_bwd_data", OP_BWD_DATA, dO.dtype, ext, dO, K, out, stream, layout)


def bwd_kernel(I: torch.Tensor, dO: torch.Tensor, stride: int, KH: int, KW: int,
               out: Optional[torch.Tensor] = None, stream: Optional[torch.cuda.Stream] = None,
               pad: int = 0, layout="natural") -> torch.Tensor:
    """dK in float32 (capsconv_bwd_kernel_ex)."""
    dev = _need_cuda(I, dO)
    B, H, W, C, D1, D2 = _split(I, layout)
    B2, Ho, Wo, Cout, D1b, D3 = _split(dO, layout)
    if B2 != B or D1b != D1 or I.dtype != dO.dtype:
        raise ValueError("I %s and dO %s disagree" % (tuple(I.shape), tuple(dO.shape)))
    if output_dims(H, W, KH, KW, stride, pad) != (Ho, Wo):
        raise ValueError("dO spatial extent does not match H, W, K, stride and pad")
    shape = (KH, KW, C, Cout, D2, D3)
    if out is None:
        out = torch.empty(shape, dtype=torch.float32, device=dev)
    elif tuple(out.shape) != shape or out.dtype != torch.float32:
        raise ValueError("out must be float32 of the kernel's shape")
    ext = (B, H, W, C, Cout, KH, KW, D1, D2, D3, stride, pad)
    return _call("capsconv_bwd_kernel", OP_BWD_KERNEL, I.dtype, ext, I, dO, out, stream, layout)


def sgd_update(w_master: torch.Tensor, grad: torch.Tensor, lr: float, w_out: Optional[torch.Tensor] = None,
               stream: Optional[torch.cuda.Stream] = None) -> torch.Tensor:
    """One SGD step (capsconv_sgd_update): w_master -= lr * grad in fp32, then
    w_out = w_master rounded to w_out's dtype (bf16 or fp32; default: w_master
    itself).  Returns w_out."""
    dev = _need_cuda(w_master, grad)
    if w_out is None:
        w_out = w_master
    _need_cuda(w_out)
    if w_master.dtype != torch.float32 or grad.dtype != torch.float32:
        raise ValueError("w_master and grad must be float32")
    n = w_master.numel()
    if grad.numel() != n or w_out.numel() != n:
        raise ValueError("w_master, grad and w_out must have the same number of elements")
    lib = load_library()
    s = stream if stream is not None else torch.cuda.current_stream(dev)
    with torch.cuda.device(dev):
        st = lib.capsconv_sgd_update(_dt(w_out.dtype), n, ctypes.c_float(lr), ctypes.c_void_p(w_master.data_ptr()),
                                     ctypes.c_void_p(grad.data_ptr()), ctypes.c_void_p(w_out.data_ptr()),
                                     ctypes.c_void_p(s.cuda_stream))
    _check(st, "sgd_update")
    return w_out


# ------------------------------------------------------------ S-slice capsules (R22)
def _slices_call(name: str, op: int, dtype, ext, a, b, out, stream):
    lib = load_library()
    s = stream if stream is not None else torch.cuda.current_stream(out.device)
    handle = s.cuda_stream
    need = ctypes.c_size_t()
    _check(lib.capsconv_workspace_bytes_slices(op, _dt(dtype), *ext, ctypes.byref(need)), "workspace_bytes_slices")
    ws = _workspace(need.value, out.device, handle)
    with torch.cuda.device(out.device):
        st = getattr(lib, name)(_dt(dtype), *ext, ctypes.c_void_p(a.data_ptr()), ctypes.c_void_p(b.data_ptr()),
                                ctypes.c_void_p(out.data_ptr()), ctypes.c_void_p(ws.data_ptr() if ws is not None else 0),
                                ctypes.c_size_t(need.value), ctypes.c_void_p(handle))
    _check(st, name)
    return out


def fwd_slices(I: torch.Tensor, K: torch.Tensor, stride: int = 1, out: Optional[torch.Tensor] = None,
               stream: Optional[torch.cuda.Stream] = None) -> torch.Tensor:
    """S-slice capsules: I (B,H,W,C,S,D1,D2), K (KH,KW,C,Cout,S,D2,D3) -> O (B,Ho,Wo,Cout,S,D1,D3)."""
    dev = _need_cuda(I, K)
    B, H, W, C, S, D1, D2 = I.shape
    KH, KW, C2, Cout, S2, D2b, D3 = K.shape
    if C2 != C or S2 != S or D2b != D2 or I.dtype != K.dtype:
        raise ValueError("I %s and K %s disagree" % (tuple(I.shape), tuple(K.shape)))
    Ho, Wo = output_dims(H, W, KH, KW, stride)
    shape = (B, Ho, Wo, Cout, S, D1, D3)
    out = torch.empty(shape, dtype=I.dtype, device=dev) if out is None else out
    if tuple(out.shape) != shape or out.dtype != I.dtype:
        raise ValueError("out has the wrong shape/dtype")
    ext = (B, H, W, C, Cout, KH, KW, S, D1, D2, D3, stride)
    return _slices_call("capsconv_fwd_slices", OP_FWD, I.dtype, ext, I, K, out, stream)


def bwd_data_slices(dO: torch.Tensor, K: torch.Tensor, stride: int, H: int, W: int,
                    out: Optional[torch.Tensor] = None, stream: Optional[torch.cuda.Stream] = None) -> torch.Tensor:
    dev = _need_cuda(dO, K)
    B, Ho, Wo, Cout, S, D1, D3 = dO.shape
    KH, KW, C, Cout2, S2, D2, D3b = K.shape
    if Cout2 != Cout or S2 != S or D3b != D3 or dO.dtype != K.dtype:
        raise ValueError("dO %s and K %s disagree" % (tuple(dO.shape), tuple(K.shape)))
    if output_dims(H, W, KH, KW, stride) != (Ho, Wo):
        raise ValueError("dO spatial extent does not match H, W, K and stride")
    shape = (B, H, W, C, S, D1, D2)
    out = torch.empty(shape, dtype=dO.dtype, device=dev) if out is None else out
    if tuple(out.shape) != shape or out.dtype != dO.dtype:
        raise ValueError("out has the wrong shape/dtype")
    ext = (B, H, W, C, Cout, KH, KW, S, D1, D2, D3, stride)
    return _slices_call("capsconv_bwd_data_slices", OP_BWD_DATA, dO.dtype, ext, dO, K, out, stream)


def bwd_kernel_slices(I: torch.Tensor, dO: torch.Tensor, stride: int, KH: int, KW: int,
                      out: Optional[torch.Tensor] = None, stream: Optional[torch.cuda.Stream] = None) -> torch.Tensor:
    dev = _need_cuda(I, dO)
    B, H, W, C, S, D1, D2 = I.shape
    B2, Ho, Wo, Cout, S2, D1b, D3 = dO.shape
    if B2 != B or S2 != S or D1b != D1 or I.dtype != dO.dtype:
        raise ValueError("I %s and dO %s disagree" % (tuple(I.shape), tuple(dO.shape)))
    if output_dims(H, W, KH, KW, stride) != (Ho, Wo):
        raise ValueError("dO spatial extent does not match H, W, K and stride")
    shape = (KH, KW, C, Cout, S, D2, D3)
    out = torch.empty(shape, dtype=torch.float32, device=dev) if out is None else out
    if tuple(out.shape) != shape or out.dtype != torch.float32:
        raise ValueError("out must be float32 of the kernel's shape")
    ext = (B, H, W, C, Cout, KH, KW, S, D1, D2, D3, stride)
    return _slices_call("capsconv_bwd_kernel_slices", OP_BWD_KERNEL, I.dtype, ext, I, dO, out, stream)


class CapsConvFunction(torch.autograd.Function):
    """autograd wrapper: forward = capsconv_fwd, backward = bwd_kernel + bwd_data."""

    @staticmethod
    def forward(ctx, I, K, stride, pad=0):
        ctx.save_for_backward(I, K)
        ctx.stride = stride
        ctx.pad = pad
        return fwd(I, K, stride, pad=pad)

    @staticmethod
    def backward(ctx, dO):
        I, K = ctx.saved_tensors
        dO = dO.contiguous()
        dI = dK = None
        if ctx.needs_input_grad[1]:
            dK = bwd_kernel(I, dO, ctx.stride, K.shape[0], K.shape[1], pad=ctx.pad).to(K.dtype)
        if ctx.needs_input_grad[0]:
            dI = bwd_data(dO, K, ctx.stride, I.shape[1], I.shape[2], pad=ctx.pad)
        return dI, dK, None, None


def caps_conv2d(I: torch.Tensor, K: torch.Tensor, stride: int = 1, pad: int = 0) -> torch.Tensor:
    """Differentiable capsule convolution; pad: symmetric
    zero padding."""
    return CapsConvFunction.apply(I, K, stride, pad)
