"""Seeded synthetic inputs and the workload registry.

This module is shared by the oracle side (tests, bench's CPU leg) and the
product side (bench, tests).  It holds shapes and random numbers only -- none
of the capsule convolution's arithmetic (no shape law, no contraction).
Output shapes are passed in by the caller.

Input recipe:
  * torch.Generator on the CPU; seed = base + 100 * layer, base 0 for I,
    1 for K, 2 for dO.
  * I ~ U[-1, 1);  K ~ U[-0.5, 0.5) * (KH*KW*C*D2)^-1/2 (keeps activations of a
    stack O(1)); dO ~ U[-1, 1).
  * kind="int": exact integers U{-2..2} (every product and partial sum stays
    exact in fp32; used for bitwise checks).  kind="ones": the paper's
    worked example.  kind="pos": U[0, 1).
  * Values are generated in fp32 and, for bf16 runs, rounded to bf16 once; the
    oracle receives exactly those (rounded) values.
"""
from __future__ import annotations

import dataclasses
from typing import List, Optional

import torch


@dataclasses.dataclass(frozen=True)
class Layer:
    """One capsule convolution: I (B,H,W,C,D1,D2) * K (KH,KW,C,Cout,D2,D3)."""
    B: int
    H: int
    W: int
    C: int
    Cout: int
    KH: int
    KW: int
    D1: int
    D2: int
    D3: int
    stride: int

    def i_shape(self):
        return (self.B, self.H, self.W, self.C, self.D1, self.D2)

    def k_shape(self):
        return (self.KH, self.KW, self.C, self.Cout, self.D2, self.D3)

    def o_shape(self, Ho: int, Wo: int):
        return (self.B, Ho, Wo, self.Cout, self.D1, self.D3)

    def with_batch(self, B: int) -> "Layer":
        return dataclasses.replace(self, B=B)


# BASELINE.json "configs" (BJ:7-11).  Config 5's layer sizes are the survey's
# proposal: the paper prints none (Fig 7 is stripped).
CONFIGS = {
    # 1. paper worked example, PAPER.md:43-54 (fp32, all ones)
    "fig2": Layer(B=1, H=5, W=5, C=1, Cout=1, KH=4, KW=4, D1=3, D2=3, D3=3, stride=1),
    # 2. single capsule conv layer
    "layer_s1": Layer(B=64, H=32, W=32, C=8, Cout=8, KH=3, KW=3, D1=4, D2=4, D3=4, stride=1),
    # 3. downsampling capsule conv
    "layer_s2": Layer(B=128, H=16, W=16, C=16, Cout=32, KH=3, KW=3, D1=4, D2=4, D3=4, stride=2),
    # 4. fully-connected capsule layer as a full-extent capsule conv
    "fc": Layer(B=256, H=8, W=8, C=32, Cout=10, KH=8, KW=8, D1=4, D2=4, D3=4, stride=1),
}

# 5. the CapsNet stack: 3 capsule conv layers + FC capsule layer, global batch 1024
STACK_BATCH = 1024
STACK_INPUT = dict(H=24, W=24, C=8, D=4)
STACK_LAYERS = [
    # (C, Cout, KH, KW, stride); spatial extent follows from the previous layer
    (8, 8, 3, 3, 1),
    (8, 16, 3, 3, 2),
    (16, 32, 3, 3, 1),
    (32, 10, 8, 8, 1),
]

# 6. the same stack with "same" zero padding on the 3x3 layers:
#    24x24 -> 24x24 -> 12x12 -> 12x12 -> FC over the 12x12 map
STACK_SAME_LAYERS = [
    # (C, Cout, KH, KW, stride, pad)
    (8, 8, 3, 3, 1, 1),
    (8, 16, 3, 3, 2, 1),
    (16, 32, 3, 3, 1, 1),
    (32, 10, 12, 12, 1, 0),
]


# 7. the routing-free P-CapsNet training step (PAPER.md:278 /
#    Fig 7): a primary layer from a one-channel 28x28 image (MNIST-shaped) to
#    the stack's 24x24 map of 8 capsules of 4x4 -- a plain 5x5 convolution to
#    128 channels, written as the capsule convolution with C = Cout = 1,
#    D1 = D2 = 1, D3 = 128 (reading R25) -- then the stack, then one SGD step
#    on every weight (fp32 master copies).
PRIMARY = dict(H=28, W=28, KH=5, KW=5, D3=128)
PRIMARY_SEED_LAYER = 9          # seeds of the image / primary kernel (layer_idx)
TRAIN_LR = 0.01


def primary_layer(batch: int) -> Layer:
    """The primary layer as a capsule-convolution Layer (reading R25)."""
    return Layer(B=batch, H=PRIMARY["H"], W=PRIMARY["W"], C=1, Cout=1, KH=PRIMARY["KH"], KW=PRIMARY["KW"],
                 D1=1, D2=1, D3=PRIMARY["D3"], stride=1)


def stack_layers(batch: int, out_hw) -> List[Layer]:
    """Materialise the stack for ``batch`` images.  ``out_hw(H, W, KH, KW, s)``
    is the caller's shape law (oracle or product), so this module stays free
    of the method's arithmetic."""
    H, W = STACK_INPUT["H"], STACK_INPUT["W"]
    D = STACK_INPUT["D"]
    layers = []
    for (C, Cout, KH, KW, s) in STACK_LAYERS:
        layers.append(Layer(B=batch, H=H, W=W, C=C, Cout=Cout, KH=KH, KW=KW,
                            D1=D, D2=D, D3=D, stride=s))
        H, W = out_hw(H, W, KH, KW, s)
    return layers


def _gen(seed: int) -> torch.Generator:
    g = torch.Generator(device="cpu")
    g.manual_seed(int(seed))
    return g


def _draw(shape, seed: int, kind: str, lo: float = -1.0, hi: float = 1.0) -> torch.Tensor:
    g = _gen(seed)
    if kind == "ones":
        return torch.ones(shape, dtype=torch.float32)
    if kind == "int":
        return torch.randint(-2, 3, shape, generator=g, dtype=torch.int32).to(torch.float32)
    if kind == "int1":
        return torch.randint(-1, 2, shape, generator=g, dtype=torch.int32).to(torch.float32)
    if kind == "pos":
        return torch.rand(shape, generator=g, dtype=torch.float32)
    if kind == "uniform":
        return torch.rand(shape, generator=g, dtype=torch.float32) * (hi - lo) + lo
    raise ValueError("unknown kind %r" % kind)


def _cast(t: torch.Tensor, dtype: torch.dtype) -> torch.Tensor:
    return t.to(dtype) if dtype != torch.float32 else t


def make_input(layer: Layer, kind: str = "uniform", dtype=torch.float32, layer_idx: int = 0,
               batch_offset: int = 0, batch: Optional[int] = None) -> torch.Tensor:
    """I of shape (B,H,W,C,D1,D2).  ``batch_offset``/``batch`` slice a shard of
    the full seeded batch (the full batch is generated, then sliced, so every
    rank of a sharded run sees the same global tensor)."""
    t = _draw(layer.i_shape(), 0 + 100 * layer_idx, kind)
    if batch is not None:
        t = t[batch_offset:batch_offset + batch].contiguous()
    return _cast(t, dtype)


def make_kernel(layer: Layer, kind: str = "uniform", dtype=torch.float32, layer_idx: int = 0) -> torch.Tensor:
    """K of shape (KH,KW,C,Cout,D2,D3)."""
    if kind == "uniform":
        fan_in = layer.KH * layer.KW * layer.C * layer.D2
        t = _draw(layer.k_shape(), 1 + 100 * layer_idx, "uniform", -0.5, 0.5) * (fan_in ** -0.5)
    else:
        t = _draw(layer.k_shape(), 1 + 100 * layer_idx, kind)
    return _cast(t, dtype)


def make_grad_output(o_shape, kind: str = "uniform", dtype=torch.float32, layer_idx: int = 0,
                     batch_offset: int = 0, batch: Optional[int] = None) -> torch.Tensor:
    """dO of the given output shape (B,Ho,Wo,Cout,D1,D3)."""
    t = _draw(tuple(o_shape), 2 + 100 * layer_idx, kind)
    if batch is not None:
        t = t[batch_offset:batch_offset + batch].contiguous()
    return _cast(t, dtype)
