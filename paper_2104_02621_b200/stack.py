"""CapsNet stack driver: capsule conv layers composed with the identity in
between (reading R17), forward then backward, with the batch sharded across
GPUs and each layer's dK summed across ranks (the only collective).

Layout of one step:
  forward   : acts[l+1] = capsconv_fwd(acts[l], K[l])              l = 0..L-1
  backward  : for l = L-1 .. 0:
                dK[l] = capsconv_bwd_kernel(acts[l], g)            (fp32)
                -> record an event; the comm stream waits on it and
                   all-reduces dK[l] (SUM, fp32) while the compute stream
                   goes on with
                g     = capsconv_bwd_data(g, K[l])                 (dI)
  the step ends when the compute stream has waited for the comm stream.

``ops`` is the compute backend: by default the libcapsconv binding (CUDA
only).  Tests inject another backend to exercise the sharding and
all-reduce logic with the gloo backend on CPU.
"""
from __future__ import annotations

import contextlib
from dataclasses import dataclass
from typing import List, Optional, Sequence

import torch
import torch.distributed as dist


@dataclass(frozen=True)
class LayerSpec:
    C: int
    Cout: int
    KH: int
    KW: int
    stride: int
    pad: int = 0      # symmetric zero padding


def shard_range(global_batch: int, rank: int, world: int):
    """Contiguous batch shard [lo, hi) of ``rank``; sizes differ by at most 1."""
    lo = global_batch * rank // world
    hi = global_batch * (rank + 1) // world
    return lo, hi


class CapsStack:
    def __init__(self, specs: Sequence[LayerSpec], H: int, W: int, D: int, batch: int, weights: List[torch.Tensor],
                 device, ops=None, group=None, overlap: bool = True, layout: str = "natural",
                 dk_stream: bool = True, distributed: bool = True):
        if ops is None:
            from . import capsconv as ops
        self.ops = ops
        # capsule-tensor layout of the activations and gradients: "natural"
        # (B,H,W,C,D1,D2) or "rows" (B,H,W,D1,C,D2), see include/capsconv.h
        self.layout = layout
        self._lk = {} if layout == "natural" else {"layout": layout}
        self.specs = list(specs)
        self.device = torch.device(device)
        self.dtype = weights[0].dtype
        self.batch = batch
        self.D = D
        self.group = group
        # distributed=False: a rank-local stack (no collectives) even inside a
        # process group, e.g. a check one rank runs on its own
        self.world = (dist.get_world_size(group) if (distributed and dist.is_available() and dist.is_initialized())
                      else 1)
        self.overlap = overlap and self.device.type == "cuda"
        self.K = [w.to(self.device).contiguous() for w in weights]
        # spatial extents per layer
        self.hw = [(H, W)]
        for sp in self.specs:
            h, w = self.hw[-1]
            self.hw.append(ops.output_dims(h, w, sp.KH, sp.KW, sp.stride, sp.pad))
        # static buffers (stable pointers: the step can be captured in a CUDA graph).
        # acts[0] is the caller's input itself when it already has the layer-0
        # layout (no copy); the static buffer is only used otherwise.
        self.acts = [torch.empty(self.caps_shape(batch, h, w, sp.C), dtype=self.dtype, device=self.device)
                     for (h, w), sp in zip(self.hw[:-1], self.specs)]
        self._acts0 = self.acts[0]
        last = self.specs[-1]
        h, w = self.hw[-1]
        self.out = torch.empty(self.caps_shape(batch, h, w, last.Cout), dtype=self.dtype, device=self.device)
        self.grads = [torch.empty_like(a) for a in self.acts]           # dI of every layer
        # dK is fp32 for fp32/bf16 operands (libcapsconv's contract); wider
        # operand types (test backends) keep their own precision
        kdt = torch.float64 if self.dtype == torch.float64 else torch.float32
        self.dK = [torch.empty(k.shape, dtype=kdt, device=self.device) for k in self.K]
        self.comm_stream = torch.cuda.Stream(self.device) if self.overlap else None
        self.events = [torch.cuda.Event() for _ in self.K] if self.overlap else None
        # dK on a stream of its own: the dK chain and the dI chain of the
        # backward are independent once a layer's incoming gradient exists, so
        # their kernels fill each other's tails and share dO reads through L2
        self.dk_stream = torch.cuda.Stream(self.device) if (self.overlap and dk_stream) else None
        self.g_events = [torch.cuda.Event() for _ in self.K] if self.dk_stream is not None else None

    def caps_shape(self, b, h, w, c):
        """Shape of a capsule tensor of this stack's layout."""
        D = self.D
        return (b, h, w, D, c, D) if self.layout == "rows" else (b, h, w, c, D, D)

    # ------------------------------------------------------------ flops / bytes
    def layer_flops(self, li: int, batch: Optional[int] = None) -> int:
        """Algorithmic flops of one pass (fwd = dI = dK) of layer li: 2*M*N*K."""
        sp = self.specs[li]
        ho, wo = self.hw[li + 1]
        b = self.batch if batch is None else batch
        return 2 * b * ho * wo * self.D * sp.Cout * self.D * sp.KH * sp.KW * sp.C * self.D

    def step_flops(self, batch: Optional[int] = None) -> int:
        return 3 * sum(self.layer_flops(i, batch) for i in range(len(self.specs)))

    # ------------------------------------------------------------ one step
    def _bind_input(self, x: torch.Tensor):
        a0 = self._acts0
        if x.device == a0.device and x.dtype == a0.dtype and x.shape == a0.shape and x.is_contiguous():
            self.acts[0] = x            # read in place (forward input and layer-0 dK operand)
        else:
            a0.copy_(x)
            self.acts[0] = a0

    def forward(self, x: torch.Tensor) -> torch.Tensor:
        self._bind_input(x)
        for li, sp in enumerate(self.specs):
            dst = self.acts[li + 1] if li + 1 < len(self.specs) else self.out
            self.ops.fwd(self.acts[li], self.K[li], sp.stride, out=dst, pad=sp.pad, **self._lk)
        return self.out

    def backward(self, dy: torch.Tensor, timer=None) -> List[torch.Tensor]:
        g = dy
        cur = torch.cuda.current_stream(self.device) if self.overlap else None
        # per-pass timing (timer) runs the passes one after another so that each
        # event pair brackets one pass alone
        ks = self.dk_stream if timer is None else None
        if ks is not None:
            ks.wait_stream(cur)   # the previous step's readers of dK are behind us
        for li in range(len(self.specs) - 1, -1, -1):
            sp = self.specs[li]
            h, w = self.hw[li]
            if ks is not None:
                # dK(li) reads acts[li] and g on the dK stream once g exists
                self.g_events[li].record(cur)
                ks.wait_event(self.g_events[li])
            with torch.cuda.stream(ks) if ks is not None else contextlib.nullcontext():
                if timer: timer.begin(li, "dK")
                self.ops.bwd_kernel(self.acts[li], g, sp.stride, sp.KH, sp.KW, out=self.dK[li], pad=sp.pad,
                                    **self._lk)
                if timer: timer.end(li, "dK")
            if self.world > 1:
                if self.overlap:
                    self.events[li].record(ks if ks is not None else cur)
                    self.comm_stream.wait_event(self.events[li])
                    with torch.cuda.stream(self.comm_stream):
                        dist.all_reduce(self.dK[li], op=dist.ReduceOp.SUM, group=self.group)
                else:
                    dist.all_reduce(self.dK[li], op=dist.ReduceOp.SUM, group=self.group)
            if timer: timer.begin(li, "dI")
            self.ops.bwd_data(g, self.K[li], sp.stride, h, w, out=self.grads[li], pad=sp.pad, **self._lk)
            if timer: timer.end(li, "dI")
            g = self.grads[li]
        if ks is not None:
            cur.wait_stream(ks)
        if self.world > 1 and self.overlap:
            cur.wait_stream(self.comm_stream)
        return self.dK

    def step(self, x: torch.Tensor, dy: torch.Tensor, timer=None) -> List[torch.Tensor]:
        if timer is None:
            self.forward(x)
            return self.backward(dy)
        self._bind_input(x)
        for li, sp in enumerate(self.specs):
            dst = self.acts[li + 1] if li + 1 < len(self.specs) else self.out
            timer.begin(li, "fwd")
            self.ops.fwd(self.acts[li], self.K[li], sp.stride, out=dst, pad=sp.pad, **self._lk)
            timer.end(li, "fwd")
        return self.backward(dy, timer)
