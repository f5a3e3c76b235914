"""The routing-free P-CapsNet training step (
PAPER.md:278 "5-layer convolutional CapsNets", Fig 7): a primary layer from
the image to the first capsule map, the capsule stack (stack.py), and one SGD
step on every weight, all through libcapsconv.

Primary layer (reading R25): a plain KH x KW convolution from a
one-channel image to 128 channels, i.e. the capsule convolution with C = Cout
= 1, D1 = D2 = 1, D3 = 128 (the paper's own generalisation: a 1 x 1 input
capsule times a 1 x 128 kernel capsule, summed over the taps).  Its 128
output channels ARE the stack's first capsule map in the rows layout: channel
o = (d1 * C + c) * D2 + d2, so the primary output buffer is the stack input
and the stack's dX is the primary layer's dO, without a copy.  The image
gradient is not formed (nothing consumes it).

Optimizer: plain SGD on fp32 master copies of every weight, one
capsconv_sgd_update over flat buffers holding all weights, masters and dKs
(it also rewrites the working bf16 copies the convolution calls read).  The
whole step is capturable in one CUDA graph.
"""
from __future__ import annotations

from typing import List, Optional, Sequence

import torch
import torch.distributed as dist

from .stack import CapsStack, LayerSpec


class CapsTrainer:
    def __init__(self, specs: Sequence[LayerSpec], H: int, W: int, D: int, batch: int,
                 primary_kernel: torch.Tensor, weights: List[torch.Tensor], device, lr: float,
                 ops=None, group=None, overlap: bool = True, dk_stream: bool = True, distributed: bool = True):
        if ops is None:
            from . import capsconv as ops
        self.ops = ops
        self.device = torch.device(device)
        self.lr = float(lr)
        self.D = D
        self.batch = batch
        KP = primary_kernel
        if KP.dim() != 6 or KP.shape[2] != 1 or KP.shape[3] != 1 or KP.shape[4] != 1:
            raise ValueError("primary kernel must be (KH, KW, 1, 1, 1, C*D*D)")
        C0 = specs[0].C
        if KP.shape[5] != C0 * D * D:
            raise ValueError("primary kernel has %d channels, the stack's first map needs %d" % (KP.shape[5], C0 * D * D))
        self.KPH, self.KPW = int(KP.shape[0]), int(KP.shape[1])
        self.Himg, self.Wimg = H + self.KPH - 1, W + self.KPW - 1     # valid convolution onto H x W
        self.stack = CapsStack(specs, H, W, D, batch, weights, device, ops=ops, group=group, overlap=overlap,
                               layout="rows", dk_stream=dk_stream, distributed=distributed)
        self.dtype = self.stack.dtype
        # every weight, its fp32 master and its dK live in three flat buffers
        # (primary first, then the stack's layers), so the optimizer step is one
        # capsconv_sgd_update over all of them; every piece starts 16-byte aligned
        shapes = [tuple(KP.shape)] + [tuple(k.shape) for k in self.stack.K]
        sizes = [int(torch.Size(sh).numel()) for sh in shapes]
        if any(n % 8 for n in sizes):
            raise ValueError("weight sizes must be multiples of 8 elements (16-byte aligned pieces)")
        total = sum(sizes)
        self.kflat = torch.empty(total, dtype=self.dtype, device=self.device)
        self.mflat = torch.empty(total, dtype=torch.float32, device=self.device)
        self.gflat = torch.zeros(total, dtype=torch.float32, device=self.device)
        views = []
        off = 0
        for sh, n in zip(shapes, sizes):
            views.append((self.kflat[off:off + n].view(sh), self.mflat[off:off + n].view(sh),
                          self.gflat[off:off + n].view(sh)))
            off += n
        src = [KP.to(self.device, self.dtype)] + list(self.stack.K)
        for (kv, mv, gv), w in zip(views, src):
            kv.copy_(w)
            mv.copy_(kv.float())
        self.KP, self.masterP, self.dKP = views[0]
        self.stack.K = [v[0] for v in views[1:]]
        self.masters = [v[1] for v in views[1:]]
        self.stack.dK = [v[2] for v in views[1:]]
        # the primary output = the stack's first capsule map (rows layout)
        self.prim = torch.empty((batch, H, W, 1, 1, C0 * D * D), dtype=self.dtype, device=self.device)

    @property
    def specs(self):
        return self.stack.specs

    def rows_view(self, t: torch.Tensor) -> torch.Tensor:
        """(B, H, W, 1, 1, C*D*D) <-> the rows-layout capsule map (B, H, W, D, C, D)."""
        B, H, W = t.shape[0], t.shape[1], t.shape[2]
        return t.view(B, H, W, self.D, self.specs[0].C, self.D)

    def step_flops(self) -> int:
        """Algorithmic flops of one training step: the stack's 3 passes per
        layer plus the primary forward and its dK (no image gradient)."""
        b, h, w = self.batch, self.stack.hw[0][0], self.stack.hw[0][1]
        prim = 2 * b * h * w * self.KP.shape[5] * self.KPH * self.KPW
        return self.stack.step_flops() + 2 * prim

    def step(self, img: torch.Tensor, dy: torch.Tensor, timer=None) -> List[torch.Tensor]:
        """One training step on `img` (B, Himg, Wimg, 1, 1, 1) with the upstream
        gradient `dy` of the stack output (rows layout); returns the fp32
        master weights [primary, layer 0, ...] after the update.  `timer`
        (bench.py) brackets every pass; the primary layer's passes are layer -1."""
        ops = self.ops
        if timer: timer.begin(-1, "fwd")
        ops.fwd(img, self.KP, 1, out=self.prim)                       # primary layer
        if timer: timer.end(-1, "fwd")
        if timer is None:
            self.stack.forward(self.rows_view(self.prim))
            self.stack.backward(dy)                                   # dK of every layer, dX = stack.grads[0]
        else:
            self.stack.step(self.rows_view(self.prim), dy, timer)
        g0 = self.stack.grads[0]
        dprim = g0.view(g0.shape[0], g0.shape[1], g0.shape[2], 1, 1, -1)
        if timer: timer.begin(-1, "dK")
        ops.bwd_kernel(img, dprim, 1, self.KPH, self.KPW, out=self.dKP)
        if self.stack.world > 1:   # data parallel: the primary layer's dK is summed like the stack's
            dist.all_reduce(self.dKP, op=dist.ReduceOp.SUM, group=self.stack.group)
        if timer: timer.end(-1, "dK")
        if timer: timer.begin(-1, "opt")
        ops.sgd_update(self.mflat, self.gflat, self.lr, self.kflat)   # every weight in one pass
        if timer: timer.end(-1, "opt")
        return [self.masterP] + self.masters
