#!/usr/bin/env python
"""Benchmark of the capsule convolution (arXiv 2104.02621) on B200.

Metric (BASELINE.json): capsule-conv TFLOP/s fwd+bwd, and % of the HBM /
tensor roofline.  Default workload (N = 1): BASELINE.json configs[4], the
CapsNet stack -- 3 capsule conv layers + the FC capsule layer -- forward and
backward on a global batch of 1024, bf16, synthetic seeded inputs and
random-init weights.  With N > 1 ranks (torchrun, or --gpus N self-launch)
every rank runs its own batch of 1024 images -- the batch is the unit the path
partitions (tier rule 5: shard the units, report "weak" scaling) -- and every
layer's dK is all-reduced over NCCL, the path's one exchange step.
`--scaling strong` instead shards the global batch of 1024 across the ranks.

A step = forward of every layer + (dK, dI) of every layer in reverse order
(+ the dK all-reduces).  Algorithmic flops per layer pass = 2*M*N*K with
M = B*Ho*Wo*D1, N = Cout*D3, K = KH*KW*C*D2; fwd+bwd = 3x forward.

Usage:  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                        [--config stack|layer_s1|layer_s2|fc] [--dtype bf16|fp32]
Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import capsinputs  # noqa: E402

METRIC = "capsule-conv TFLOP/s fwd+bwd at 1/2/4/8 B200; % of tensor/HBM roofline"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference", "paper-alg34"],
                    help="ours; reference = the CPU oracle; paper-alg34 = the paper's Algorithms 3/4 literally "
                         "(materialised im2col / extends + cuBLAS strided-batched matmuls via torch) on the GPU, "
                         "a context row (SURVEY NEXT-3 (ii))")
    ap.add_argument("--config", default="stack",
                    choices=["stack", "stack_same", "layer_s1", "layer_s2", "fc", "pcapsnet_train"])
    ap.add_argument("--dtype", default="bf16", choices=["bf16", "fp32"])
    ap.add_argument("--no-overlap", action="store_true", help="all-reduce on the compute stream")
    ap.add_argument("--no-dk-stream", action="store_true", help="dK passes on the compute stream (no second chain)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--eager", action="store_true", help="time eager launches instead of CUDA-graph replays")
    ap.add_argument("--layout", default=None, choices=["rows", "natural"],
                    help="capsule-tensor layout of the stack's activations (include/capsconv.h); default rows for "
                         "bf16 (its tensor-core kernels), natural for fp32 (the SIMT kernels' own layout) and for "
                         "the padded stack_same (the natural tensor-core kernels take padding)")
    ap.add_argument("--no-parity", action="store_true", help="skip the in-bench oracle parity check")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="N > 1: weak = 1024 images per rank (default), strong = 1024 images shared by the ranks")
    ap.add_argument("--batch", type=int, default=0,
                    help="override the global batch (e.g. 128/256/512: one rank's share of the batch-1024 stack "
                         "at 8/4/2 GPUs -- the compute side of strong scaling on one GPU)")
    args = ap.parse_args()
    if args.layout is None:   # the rows kernels take bf16 unpadded layers; the natural ones pad (NEXT-2) and fp32
        args.layout = "natural" if (args.dtype == "fp32" or args.config == "stack_same") else "rows"
    return args


def self_launch(args):
    """--gpus N > 1 without a torchrun environment: re-launch this script as N
    ranks of one node (torch.distributed.run, rendezvous on 127.0.0.1) and
    return its exit code; the launcher's rank 0 prints the JSON line."""
    import socket
    import subprocess
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(args.gpus),
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


# ---------------------------------------------------------------- workload
def workload(cfg: str, world: int):
    """(specs, H, W, D, global_batch, name) of the benchmarked workload."""
    from paper_2104_02621_b200.stack import LayerSpec
    if cfg == "stack":
        specs = [LayerSpec(*l) for l in capsinputs.STACK_LAYERS]
        si = capsinputs.STACK_INPUT
        return specs, si["H"], si["W"], si["D"], capsinputs.STACK_BATCH, "capsnet_stack_3conv_fc_b1024"
    if cfg == "pcapsnet_train":   # primary layer + the stack + SGD on every weight
        specs = [LayerSpec(*l) for l in capsinputs.STACK_LAYERS]
        si = capsinputs.STACK_INPUT
        return specs, si["H"], si["W"], si["D"], capsinputs.STACK_BATCH, "pcapsnet_train_step_b1024"
    if cfg == "stack_same":   # zero-padded ("same") 3x3 layers, SURVEY NEXT-2
        specs = [LayerSpec(*l) for l in capsinputs.STACK_SAME_LAYERS]
        si = capsinputs.STACK_INPUT
        return specs, si["H"], si["W"], si["D"], capsinputs.STACK_BATCH, "capsnet_stack_same_pad1_b1024"
    L = capsinputs.CONFIGS[cfg]
    return [LayerSpec(L.C, L.Cout, L.KH, L.KW, L.stride)], L.H, L.W, L.D1, L.B, "single_layer_" + cfg


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return {"hbm_gbs": float(d["hbm_gbs"]), "bf16_tflops": float(d["bf16_tflops"]),
                "bf16_tflops_sustained": float(d.get("bf16_tflops_sustained", d["bf16_tflops"])), "src": "measured"}
    except Exception:
        # fallback of /opt/skills/guides/B200_PROFILING.md
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "src": "fallback"}


# ---------------------------------------------------------------- clocks
REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
           0x80: "hw_power_brake_slowdown", 0x2: "applications_clocks_setting", 0x10: "sync_boost"}


class ClockSampler:
    def __init__(self, index: int):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        self._ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self._ok = True
        except Exception:
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                try:
                    r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                except AttributeError:
                    r = self.nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
                for bit, name in REASONS.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.002)

    def __enter__(self):
        if self._ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self._ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons)}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ---------------------------------------------------------------- per-call timer
class CallTimer:
    """CUDA events around every C-ABI call of a step, on the launching stream."""

    def __init__(self):
        self.pending = []
        self.open = {}

    def begin(self, li, kind):
        e = torch.cuda.Event(enable_timing=True)
        e.record()
        self.open[(li, kind)] = e

    def end(self, li, kind):
        e = torch.cuda.Event(enable_timing=True)
        e.record()
        self.pending.append(((li, kind), self.open.pop((li, kind)), e))

    def collect(self):
        out = {}
        for key, a, b in self.pending:
            out.setdefault(key, []).append(a.elapsed_time(b))
        self.pending = []
        return out


class GraphCallTimer:
    """The same per-call events, recorded while the step is captured into a
    CUDA graph (external events become event-record nodes, so every replay
    re-records them); collect() reads the last replay's durations."""

    def __init__(self):
        self.ev = {}
        self.order = []

    def _pair(self, key):
        if key not in self.ev:
            self.ev[key] = (torch.cuda.Event(enable_timing=True, external=True),
                            torch.cuda.Event(enable_timing=True, external=True))
            self.order.append(key)
        return self.ev[key]

    def begin(self, li, kind):
        self._pair((li, kind))[0].record()

    def end(self, li, kind):
        self._pair((li, kind))[1].record()

    def collect_into(self, out):
        for key in self.order:
            a, b = self.ev[key]
            out.setdefault(key, []).append(a.elapsed_time(b))


def pass_name(li, kind):
    return ("L%d_%s" % (li + 1, kind)) if li >= 0 else ("SGD" if kind == "opt" else "P_%s" % kind)


def pass_flops(st, li, kind):
    return st.layer_flops(li) if li >= 0 else st.aux_flops(kind)


def pass_bytes(st, li, kind, elem):
    """Algorithmic HBM bytes of one pass: every operand moved once
    (SURVEY §8(d)): fwd |I|+|K|+|O|; dI |dO|+|K|+|dI|; dK |I|+|dO|+4|dK|."""
    if li < 0:
        return st.aux_bytes(kind, elem)
    sp = st.specs[li]
    h, w = st.hw[li]
    ho, wo = st.hw[li + 1]
    D = st.D
    nI = st.batch * h * w * sp.C * D * D
    nO = st.batch * ho * wo * sp.Cout * D * D
    nK = sp.KH * sp.KW * sp.C * sp.Cout * D * D
    if kind == "fwd":
        return (nI + nK + nO) * elem
    if kind == "dI":
        return (nO + nK + nI) * elem
    return (nI + nO) * elem + 4 * nK


def pass_write_bytes(st, li, kind, elem):
    """The part of pass_bytes the pass writes: |O| (fwd), |dI| (dI), 4|dK| (dK)."""
    if li < 0:
        return st.aux_write_bytes(kind, elem)
    sp = st.specs[li]
    h, w = st.hw[li]
    ho, wo = st.hw[li + 1]
    D = st.D
    if kind == "fwd":
        return st.batch * ho * wo * sp.Cout * D * D * elem
    if kind == "dI":
        return st.batch * h * w * sp.C * D * D * elem
    return 4 * sp.KH * sp.KW * sp.C * sp.Cout * D * D


# ---------------------------------------------------------------- reference (oracle) arm
def run_reference(args, rank, world):
    if rank != 0:
        return
    import numpy as np
    import oracle
    oracle.build()
    specs, H, W, D, gbatch, name = workload(args.config, 1)
    dtype = torch.bfloat16 if args.dtype == "bf16" else torch.float32
    flops_per_image, Ks, strides, layers = stack_oracle_setup(specs, H, W, D, dtype)

    Xa, dYa = stack_oracle_inputs(layers, specs, H, W, D, gbatch, dtype, gbatch)
    train = args.config == "pcapsnet_train"
    if train:   # oracle.train_step (primary layer + stack + SGD)
        P = capsinputs.primary_layer(gbatch)
        Kp64 = capsinputs.make_kernel(P, dtype=dtype, layer_idx=capsinputs.PRIMARY_SEED_LAYER).to(torch.float64).numpy()
        imga = capsinputs.make_input(P, dtype=dtype, layer_idx=capsinputs.PRIMARY_SEED_LAYER).to(torch.float64).numpy()
        prim = 2 * 1 * H * W * specs[0].C * D * D * capsinputs.PRIMARY["KH"] * capsinputs.PRIMARY["KW"]
        flops_per_image += 2 * prim

    def one(b):
        t0 = time.perf_counter()
        if train:
            oracle.train_step(imga[:b], Kp64, Ks, strides[0], dYa[:b], capsinputs.TRAIN_LR, True)
        else:
            oracle.stack_fwd_bwd(Xa[:b], Ks, strides[0], dYa[:b], dtype == torch.bfloat16, pads=strides[1])
        return time.perf_counter() - t0

    t1 = one(1)
    budget = min(1.5, 120.0 / max(1, args.steps + args.warmup))
    b = int(max(1, min(gbatch, budget / max(t1, 1e-6))))
    for _ in range(args.warmup):
        one(b)
    ts = [one(b) for _ in range(args.steps)]
    t = sum(ts) / len(ts)
    tf = flops_per_image * b / t / 1e12
    cores = oracle.num_threads()
    line = {
        "impl": "reference", "metric": METRIC, "value": tf, "unit": "TFLOP/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
        "scaling": args.scaling if world > 1 else "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": name, "global_batch": gbatch, "sample_batch": b, "io_dtype": args.dtype},
        "cpu_baseline": {"value": tf, "unit": "TFLOP/s", "cores": cores, "kind": "oracle",
                         "sample": "oracle (C, fp64, OpenMP) %s fwd+bwd on %d of %d images per step" % (name, b, gbatch)},
        "e2e": {"value": tf, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def stack_oracle_setup(specs, H, W, D, dtype):
    import oracle
    layers, Ks, strides, pads = [], [], [], []
    h, w = H, W
    flops = 0
    for li, sp in enumerate(specs):
        L = capsinputs.Layer(B=1, H=h, W=w, C=sp.C, Cout=sp.Cout, KH=sp.KH, KW=sp.KW, D1=D, D2=D, D3=D,
                             stride=sp.stride)
        layers.append(L)
        Ks.append(capsinputs.make_kernel(L, dtype=dtype, layer_idx=li).to(torch.float64).numpy())
        strides.append(sp.stride)
        pads.append(sp.pad)
        ho, wo = oracle.output_dims(h, w, sp.KH, sp.KW, sp.stride, sp.pad)
        flops += 3 * 2 * ho * wo * D * sp.Cout * D * sp.KH * sp.KW * sp.C * D
        h, w = ho, wo
    return flops, Ks, (strides, pads), layers


def stack_oracle_inputs(layers, specs, H, W, D, b, dtype, gbatch):
    import oracle
    L0 = layers[0].with_batch(gbatch)
    X = capsinputs.make_input(L0, dtype=dtype, batch=b).to(torch.float64).numpy()
    h, w = H, W
    for sp in specs:
        h, w = oracle.output_dims(h, w, sp.KH, sp.KW, sp.stride, sp.pad)
    dY = capsinputs.make_grad_output((b, h, w, specs[-1].Cout, D, D), dtype=dtype, layer_idx=len(specs)).to(
        torch.float64).numpy()
    return X, dY


# The paper's own result, quoted as context: not comparable
# hardware, precision or workload, so vs_baseline stays null.
PAPER_CONTEXT = {
    "claim": "4x: capsule-conv CapsNet fwd+bwd 510 ms (ours, official APIs) vs 2220 ms ('GPU' baseline)",
    "gpu": "NVIDIA TITAN X (Pascal), CUDA 10.0",
    "source": "PAPER.md:29 (abstract), :278 (experiments), Table 1 :154-156",
    "comparable": False,
}


def host_cpu():
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"model": model, "logical_cpus": os.cpu_count()}


def parity_check(pkg, specs, H, W, D, PB, weights, X_nat, dY_nat, dtype, dev, layout):
    """Max normalised error max|gpu - oracle| / max|oracle| of every tensor of
    one stack step (forward outputs of every layer, dX, every dK) on PB images;
    bf16 outputs and dI are compared with the oracle rounded at the same bf16
    boundaries (reading R13).  Tolerance: north_star's 2e-2 (bf16) / 1e-5 (fp32)."""
    import numpy as np
    import oracle
    from paper_2104_02621_b200.stack import CapsStack
    st = CapsStack(specs, H, W, D, PB, weights, dev, overlap=False, layout=layout,
                   distributed=False)   # rank 0 alone runs the check: no collectives
    perm = (lambda t: t.permute(0, 1, 2, 4, 3, 5).contiguous()) if layout == "rows" else (lambda t: t)
    st.step(perm(X_nat.to(dev)), perm(dY_nat.to(dev)))
    torch.cuda.synchronize()
    f64 = lambda t: t.detach().to("cpu", torch.float64).numpy()
    strides = [sp.stride for sp in specs]
    pads = [sp.pad for sp in specs]
    acts, dX, dKs, _ = oracle.stack_fwd_bwd(f64(X_nat), [f64(k) for k in weights], strides, f64(dY_nat),
                                            dtype == torch.bfloat16, pads=pads)
    outs = [st.acts[i] for i in range(1, len(specs))] + [st.out]
    errs = {}

    def rel(a, b):
        m = float(np.abs(b).max())
        return float(np.abs(a - b).max()) / (m if m > 0 else 1.0)

    for li, o in enumerate(outs):
        errs["O%d" % (li + 1)] = rel(f64(perm(o)), acts[li + 1])
    errs["dX"] = rel(f64(perm(st.grads[0])), dX)
    for li, k in enumerate(st.dK):
        errs["dK%d" % (li + 1)] = rel(f64(k), dKs[li])
    tol = 2e-2 if dtype == torch.bfloat16 else 1e-5
    worst = max(errs.values())
    return {"images": PB, "max_norm_err": {k: float("%.3g" % v) for k, v in errs.items()}, "worst": float("%.3g" % worst),
            "tol": tol, "pass": worst <= tol}


# ---------------------------------------------------------------- the paper's scheme, literally
def alg34_layer(I, K, s, dO=None):
    """Algorithm 3 (forward) and 4 (backward) of the paper with its
    buffers materialised as the paper describes them: capsule_im2col,
    input_extend (x Cout), kernel_extend (x Ho*Wo), strided-batched 4x4 matmuls
    (torch.matmul -> cuBLAS batched GEMM), output_reduce; backward: output_extend
    (x KH*KW*C), the two batched products, the reduces and capsule_col2im.
    Natural layout, the dtype of I.  Returns O, or (dI, dK) when dO is given."""
    B, H, W, C, D1, D2 = I.shape
    KH, KW, _, Co, _, D3 = K.shape
    Ho, Wo = (H - KH) // s + 1, (W - KW) // s + 1
    sB, sH, sW, sC, s1, s2 = I.stride()
    If = I.as_strided((B, Ho, Wo, KH, KW, C, D1, D2), (sB, sH * s, sW * s, sH, sW, sC, s1, s2)).contiguous()
    Ip = If.unsqueeze(6).expand(B, Ho, Wo, KH, KW, C, Co, D1, D2).contiguous()              # input_extend
    del If
    Kp = K.unsqueeze(0).unsqueeze(0).expand(Ho, Wo, KH, KW, C, Co, D2, D3).contiguous()       # kernel_extend
    if dO is None:
        Op = torch.matmul(Ip, Kp.unsqueeze(0))                                                 # sbmm(K', I')
        return Op.sum(dim=(3, 4, 5))                                                           # output_reduce
    Odp = dO.view(B, Ho, Wo, 1, 1, 1, Co, D1, D3).expand(B, Ho, Wo, KH, KW, C, Co, D1, D3).contiguous()
    dK = torch.matmul(Ip.transpose(-1, -2), Odp).sum(dim=(0, 1, 2), dtype=torch.float32)      # K'_diff, reduce
    del Ip
    Id = torch.matmul(Odp, Kp.unsqueeze(0).transpose(-1, -2)).sum(dim=6)                       # I'_d, input_reduce
    del Odp
    dI = torch.zeros_like(I)
    for p in range(KH):                                                                        # capsule_col2im
        for q in range(KW):
            dI[:, p:p + s * (Ho - 1) + 1:s, q:q + s * (Wo - 1) + 1:s] += Id[:, :, :, p, q]
    return dI, dK


def run_paper_alg34(args, rank, world):
    if rank != 0:
        return
    specs, H, W, D, gbatch, name = workload(args.config, 1)
    dev = torch.device("cuda", 0)
    dtype = torch.bfloat16 if args.dtype == "bf16" else torch.float32
    ws, h, w = [], H, W
    hw = [(H, W)]
    for li, sp in enumerate(specs):
        L = capsinputs.Layer(B=gbatch, H=h, W=w, C=sp.C, Cout=sp.Cout, KH=sp.KH, KW=sp.KW, D1=D, D2=D, D3=D,
                             stride=sp.stride)
        ws.append(capsinputs.make_kernel(L, dtype=dtype, layer_idx=li).to(dev))
        h, w = (h - sp.KH) // sp.stride + 1, (w - sp.KW) // sp.stride + 1
        hw.append((h, w))
    L0 = capsinputs.Layer(B=gbatch, H=H, W=W, C=specs[0].C, Cout=specs[0].Cout, KH=specs[0].KH, KW=specs[0].KW,
                          D1=D, D2=D, D3=D, stride=specs[0].stride)
    X = capsinputs.make_input(L0, dtype=dtype).to(dev)
    dY = capsinputs.make_grad_output((gbatch, h, w, specs[-1].Cout, D, D), dtype=dtype, layer_idx=len(specs)).to(dev)
    flops = 0
    for li, sp in enumerate(specs):
        ho, wo = hw[li + 1]
        flops += 3 * 2 * gbatch * ho * wo * D * sp.Cout * D * sp.KH * sp.KW * sp.C * D

    def step():
        acts = [X]
        for sp, K in zip(specs, ws):
            acts.append(alg34_layer(acts[-1], K, sp.stride))
        g = dY
        for li in range(len(specs) - 1, -1, -1):
            g, _ = alg34_layer(acts[li], ws[li], specs[li].stride, g)
        return g

    for _ in range(max(1, args.warmup)):
        step()
    torch.cuda.synchronize()
    ts = []
    for _ in range(args.steps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        step()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ms = sum(ts) / len(ts)
    line = {"impl": "paper-alg34", "metric": METRIC, "value": round(flops / (ms * 1e-3) / 1e12, 3), "unit": "TFLOP/s",
            "n_gpus": 1, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 3),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": args.dtype,
            "data": "synthetic (seeded capsinputs)",
            "config": {"workload": name, "global_batch": gbatch,
                       "scheme": "PAPER.md Alg 3/4: materialised capsule_im2col, input/kernel/output extends, "
                                 "torch.matmul batched 4x4 products (cuBLAS), reduces, capsule_col2im",
                       "peak_mem_GB": round(torch.cuda.max_memory_allocated(dev) / 1e9, 1)}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- our arm
class TrainBench:
    """bench.py's view of a CapsTrainer (config pcapsnet_train):
    the stack's attributes, plus the primary layer (pass layer -1: fwd, dK) and
    the SGD step (layer -1, "opt") for the per-pass table."""

    def __init__(self, trainer):
        self.tr = trainer
        self.stack = trainer.stack

    def __getattr__(self, name):          # specs, hw, D, batch, acts, out, dk_stream, layer_flops ...
        return getattr(self.stack, name)

    @property
    def dK(self):                         # what a step returns (read back by the e2e leg)
        return [self.tr.masterP] + self.tr.masters

    def step(self, x, dy, timer=None):
        return self.tr.step(x, dy, timer)

    def step_flops(self, batch=None):
        return self.tr.step_flops()

    def _prim_elems(self):
        b, (h, w) = self.stack.batch, self.stack.hw[0]
        img = b * self.tr.Himg * self.tr.Wimg
        return img, b * h * w * self.tr.KP.shape[5], self.tr.KP.numel()

    def aux_flops(self, kind):
        nimg, nprim, nk = self._prim_elems()
        if kind == "opt":
            return 2 * sum(m.numel() for m in self.dK)
        return 2 * nprim * self.tr.KPH * self.tr.KPW

    def aux_bytes(self, kind, elem):
        nimg, nprim, nk = self._prim_elems()
        if kind == "fwd":
            return (nimg + nk + nprim) * elem
        if kind == "dK":
            return (nimg + nprim) * elem + 4 * nk
        n = sum(m.numel() for m in self.dK)       # master read+write, dK read, working copy write
        return n * (4 + 4 + 4 + elem)

    def aux_write_bytes(self, kind, elem):
        nimg, nprim, nk = self._prim_elems()
        if kind == "fwd":
            return nprim * elem
        if kind == "dK":
            return 4 * nk
        return sum(m.numel() for m in self.dK) * (4 + elem)


def train_parity(pkg, specs, H, W, D, PB, Kp, weights, img_nat, dY_nat, dev):
    """The training step on the first PB images (same trainer code, eager)
    against oracle.train_step: max normalised error of every dK and of every
    updated master weight (as lr * dK error)."""
    import oracle
    from paper_2104_02621_b200.train import CapsTrainer
    lr = capsinputs.TRAIN_LR
    tr = CapsTrainer(specs, H, W, D, PB, Kp, weights, dev, lr, distributed=False)   # rank 0 alone: no collectives
    tr.step(img_nat.to(dev), dY_nat.permute(0, 1, 2, 4, 3, 5).contiguous().to(dev))
    torch.cuda.synchronize()
    f64 = lambda t: t.detach().to("cpu", torch.float64).numpy()  # noqa: E731
    new, rdK, den = oracle.train_step(f64(img_nat), f64(Kp), [f64(k) for k in weights], [s.stride for s in specs],
                                      f64(dY_nat), lr, True)
    names = ["dKp"] + ["dK%d" % (i + 1) for i in range(len(specs))]
    errs = {}
    for name, got, ref, a in zip(names, [tr.dKP] + list(tr.stack.dK), rdK, den):
        errs[name] = float((abs(f64(got) - ref) / (a + 1e-30)).max())
    for i, (m, ref, a) in enumerate(zip([tr.masterP] + tr.masters, new, den)):
        errs["W%d" % i] = float((abs(f64(m) - ref) / (lr * a + 1e-6)).max())
    worst = max(errs.values())
    tol = 2e-2
    return {"images": PB, "max_norm_err": {k: float("%.3g" % v) for k, v in errs.items()},
            "worst": float("%.3g" % worst), "tol": tol, "pass": bool(worst <= tol),
            "note": "W_i: |w_gpu - w_oracle| / (lr * sum|dK terms| + 1e-6) after the SGD step"}


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(self_launch(args))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    if args.impl == "paper-alg34":
        run_paper_alg34(args, rank, world)
        if world > 1:
            dist.destroy_process_group()
        return
    if args.impl == "reference":
        run_reference(args, rank, world)
        if world > 1:
            dist.destroy_process_group()
        return

    import paper_2104_02621_b200 as pkg
    from paper_2104_02621_b200.stack import CapsStack, shard_range
    pkg.load_library()
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    dtype = torch.bfloat16 if args.dtype == "bf16" else torch.float32
    elem = 2 if dtype == torch.bfloat16 else 4
    specs, H, W, D, gbatch, name = workload(args.config, world)
    if args.scaling == "weak" and world > 1 and not args.batch:
        gbatch *= world      # every rank keeps the single-GPU batch
    if args.batch:
        gbatch = args.batch
        name = name.rsplit("_b", 1)[0] + "_b%d" % gbatch if "_b" in name else name + "_b%d" % gbatch
    lo, hi = shard_range(gbatch, rank, world)
    batch = hi - lo

    # seeded weights (identical on every rank) and this rank's shard of the global batch
    weights, h, w = [], H, W
    for li, sp in enumerate(specs):
        L = capsinputs.Layer(B=gbatch, H=h, W=w, C=sp.C, Cout=sp.Cout, KH=sp.KH, KW=sp.KW, D1=D, D2=D, D3=D,
                             stride=sp.stride)
        weights.append(capsinputs.make_kernel(L, dtype=dtype, layer_idx=li))
        h, w = pkg.output_dims(h, w, sp.KH, sp.KW, sp.stride, sp.pad)
    L0 = capsinputs.Layer(B=gbatch, H=H, W=W, C=specs[0].C, Cout=specs[0].Cout, KH=specs[0].KH, KW=specs[0].KW,
                          D1=D, D2=D, D3=D, stride=specs[0].stride)
    X_host = capsinputs.make_input(L0, dtype=dtype, batch_offset=lo, batch=batch)
    dY_host = capsinputs.make_grad_output((gbatch, h, w, specs[-1].Cout, D, D), dtype=dtype, layer_idx=len(specs),
                                          batch_offset=lo, batch=batch)
    PB = min(2, batch)            # images of the in-bench parity check (natural layout, for the oracle)
    X_nat, dY_nat = X_host[:PB].clone(), dY_host[:PB].clone()
    if args.layout == "rows":   # the same synthetic tensors stored D1-outer: (B, H, W, D1, C, D2)
        X_host = X_host.permute(0, 1, 2, 4, 3, 5).contiguous()
        dY_host = dY_host.permute(0, 1, 2, 4, 3, 5).contiguous()
    X_host, dY_host = X_host.pin_memory(), dY_host.pin_memory()
    X = X_host.to(dev)
    dY = dY_host.to(dev)

    train = args.config == "pcapsnet_train"
    if train:   # the input is the image; the stack's input is the primary layer's output
        if dtype != torch.bfloat16 or args.layout != "rows":
            raise SystemExit("bench: --config pcapsnet_train runs bf16 in the rows layout")
        from paper_2104_02621_b200.train import CapsTrainer
        P = capsinputs.primary_layer(gbatch)
        Kp = capsinputs.make_kernel(P, dtype=dtype, layer_idx=capsinputs.PRIMARY_SEED_LAYER)
        img_host = capsinputs.make_input(P, dtype=dtype, layer_idx=capsinputs.PRIMARY_SEED_LAYER,
                                         batch_offset=lo, batch=batch)
        img_nat = img_host[:PB].clone()
        X_host = img_host.pin_memory()
        X = X_host.to(dev)
        st = TrainBench(CapsTrainer(specs, H, W, D, batch, Kp, weights, dev, capsinputs.TRAIN_LR,
                                    overlap=not args.no_overlap, dk_stream=not args.no_dk_stream))
        gflops = st.step_flops() * world
    else:
        st = CapsStack(specs, H, W, D, batch, weights, dev, overlap=not args.no_overlap, layout=args.layout,
                       dk_stream=not args.no_dk_stream)
        gflops = st.step_flops(batch=gbatch)          # whole-job algorithmic flops per step
    peaks = load_peaks()

    # L2 flush buffer: 2x the L2 size, rewritten between timed steps
    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    flush = torch.empty(max(2 * l2, 64 << 20), dtype=torch.uint8, device=dev)

    def barrier():
        if world > 1:
            dist.barrier(device_ids=[local])

    for _ in range(args.warmup):
        st.step(X, dY)
    torch.cuda.synchronize()

    # The timed step is one CUDA-graph replay of the whole step (every kernel
    # of every pass, and for N > 1 the per-layer NCCL dK all-reduces on the
    # side stream; the graph removes host launch gaps between them).  The
    # per-call events are captured with it; launches are counted at capture.
    # If capture fails (e.g. an NCCL build without graph support) the step is
    # timed eagerly and the line says so.
    use_graph = not args.eager
    graph_note = None
    gtimer = GraphCallTimer() if use_graph else None
    launches_per_step = None
    if use_graph:
        try:
            cap_stream = torch.cuda.Stream(dev)
            cap_stream.wait_stream(torch.cuda.current_stream(dev))
            with torch.cuda.stream(cap_stream):
                st.step(X, dY)                      # warm the capture stream's workspace
            torch.cuda.synchronize()
            barrier()
            # the timed graph: the step alone (event nodes between kernels would
            # break the PDL overlap of consecutive kernels)
            graph = torch.cuda.CUDAGraph()
            c0 = pkg.launch_count()
            with torch.cuda.graph(graph, stream=cap_stream):
                st.step(X, dY)
            launches_per_step = pkg.launch_count() - c0
            # the per-pass graph: the same step with an event pair around every call
            tgraph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(tgraph, stream=cap_stream):
                st.step(X, dY, timer=gtimer)
            torch.cuda.synchronize()
            for _ in range(2):
                graph.replay()
                tgraph.replay()
            torch.cuda.synchronize()
        except Exception as exc:   # fall back to eager launches, reported in config.launch
            graph_note = "graph capture failed (%s): eager launches" % str(exc).splitlines()[0][:120]
            print("bench: " + graph_note, file=sys.stderr)
            torch.cuda.synchronize()
            use_graph, gtimer = False, None

    # HBM write bandwidth, live: the L2 flush is a plain write of 2x L2 (a
    # write-only stream reaches about half the copy figure on this part, so
    # the write-heavy passes get a second, write-aware floor in per_pass)
    wa, wb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    flush.zero_()
    wa.record()
    for _ in range(5):
        flush.zero_()
    wb.record()
    torch.cuda.synchronize()
    write_gbs = 5 * flush.numel() / (wa.elapsed_time(wb) * 1e-3) / 1e9

    timer = CallTimer()
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    barrier()
    torch.cuda.synchronize()
    n0 = pkg.launch_count()
    with ClockSampler(dev.index if dev.index is not None else 0) as clk:
        gcalls = {}
        for i in range(args.steps):
            flush.zero_()
            starts[i].record()
            if use_graph:
                graph.replay()
            else:
                st.step(X, dY, timer=timer)
            ends[i].record()
        torch.cuda.synchronize()
        barrier()
    if use_graph:   # per-pass durations: replays of the event-instrumented graph
        for i in range(max(3, min(args.steps, 20))):
            flush.zero_()
            tgraph.replay()
            torch.cuda.synchronize()
            gtimer.collect_into(gcalls)
    launches = launches_per_step * args.steps if use_graph else pkg.launch_count() - n0
    step_ms = [a.elapsed_time(b) for a, b in zip(starts, ends)]
    calls = gcalls if use_graph else timer.collect()
    ms = sum(step_ms) / len(step_ms)
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    value = gflops / (ms_max * 1e-3) / 1e12

    # ---- per-pass breakdown and the dominant kernel's roofline.  Compute
    # roof: bf16 -> the sustained tensor peak (MEASURED_PEAKS.json); fp32 runs
    # on CUDA-core FFMA (SIMT path) -> 148 SMs x 128 FP32 lanes x 2 flop x the
    # max SM clock (74.4 TF/s at 1965 MHz), bound "alu"
    if dtype == torch.bfloat16:
        cpeak, cbound = peaks["bf16_tflops_sustained"], "tensor"
    else:
        sm_mhz = clk.max_mhz or 1965
        cpeak = torch.cuda.get_device_properties(dev).multi_processor_count * 128 * 2 * sm_mhz * 1e6 / 1e12
        cbound = "alu"
        try:   # the FFMA microbenchmark's figure (tests/probe/ffma_peak.cu) when it has been run on this pool
            with open(os.path.join(ROOT, "profiles", "r2_ffma_peak.json")) as f:
                cpeak = float(json.load(f)["ffma_tflops"])
            peaks["src"] = "measured FFMA peak (profiles/r2_ffma_peak.json)"
        except Exception:
            pass
    per_pass, best = {}, None
    t_roof_sum = 0.0
    for (li, kind), v in sorted(calls.items()):
        avg = sum(v) / len(v)
        byts = pass_bytes(st, li, kind, elem)
        fl = pass_flops(st, li, kind)
        gbs = byts / (avg * 1e-3) / 1e9
        tr = max(byts / (peaks["hbm_gbs"] * 1e9), fl / (cpeak * 1e12)) * 1e3
        tw = max(tr, pass_write_bytes(st, li, kind, elem) / (write_gbs * 1e9) * 1e3)
        t_roof_sum += tr
        per_pass[pass_name(li, kind)] = {"ms": round(avg, 5), "GB_s": round(gbs, 1),
                                                "TFLOP_s": round(fl / (avg * 1e-3) / 1e12, 1),
                                                "roof_frac": round(tr / avg, 3),
                                                "wfloor_frac": round(tw / avg, 3)}
        if best is None or avg > best[1]:
            best = ((li, kind), avg, byts)
    (bli, bkind), bavg, bbytes = best
    traffic = None
    try:   # the committed captures are of the bf16 rows kernels of the stack
        if dtype == torch.bfloat16 and args.layout == "rows" and args.config in ("stack", "pcapsnet_train"):
            with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
                traffic = json.load(f).get(pass_name(bli, bkind))
    except Exception:
        pass
    # the binding roof of the dominant pass: HBM time of its algorithmic bytes
    # vs tensor time of its algorithmic flops, whichever is longer
    bflops = pass_flops(st, bli, bkind)
    t_hbm = bbytes / (peaks["hbm_gbs"] * 1e9)
    # kernels are timed inside a long step: the sustained tensor figure applies
    t_tc = bflops / (cpeak * 1e12)
    if t_tc > t_hbm:
        achieved = bflops / (bavg * 1e-3) / 1e12
        roofline = {"bound": cbound, "achieved": round(achieved, 2), "peak": cpeak,
                    "unit": "TFLOP/s", "frac": round(achieved / cpeak, 4)}
    else:
        achieved = bbytes / (bavg * 1e-3) / 1e9
        roofline = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peaks["hbm_gbs"], "unit": "GB/s",
                    "frac": round(achieved / peaks["hbm_gbs"], 4)}
    roofline.update({"traffic": traffic, "kernel": pass_name(bli, bkind), "bytes_per_launch": bbytes,
                     "flops_per_launch": bflops,
                     "peak_src": peaks["src"] if dtype == torch.bfloat16 or t_tc <= t_hbm or "FFMA" in peaks["src"]
                     else "derived: SMs x 128 FFMA lanes x 2 x max SM clock",
                     "step_frac": round(t_roof_sum / ms, 4),
                     "hbm_write_gbs_live": round(write_gbs, 1)})

    # ---- e2e: same steps through the public API with host buffers.  Every
    # step copies its input X and dY from pinned host memory and reads all dK
    # back; the copy of step i+1's inputs runs on a copy stream while step i
    # computes (double-buffered device inputs), as an input pipeline would.
    dk_host = torch.empty(sum(k.numel() for k in st.dK), dtype=torch.float32).pin_memory()
    copy_stream = torch.cuda.Stream(dev)
    xbuf = [torch.empty_like(X), torch.empty_like(X)]
    gbuf = [torch.empty_like(dY), torch.empty_like(dY)]
    ready = [torch.cuda.Event(), torch.cuda.Event()]
    consumed = [torch.cuda.Event(), torch.cuda.Event()]
    e2e_start, e2e_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    cur = torch.cuda.current_stream(dev)

    def h2d(slot):
        copy_stream.wait_event(consumed[slot])
        with torch.cuda.stream(copy_stream):
            xbuf[slot].copy_(X_host, non_blocking=True)
            gbuf[slot].copy_(dY_host, non_blocking=True)
            ready[slot].record(copy_stream)

    barrier()
    torch.cuda.synchronize()
    for ev in consumed:
        ev.record(cur)
    e2e_start.record(cur)
    h2d(0)
    for i in range(args.steps):
        slot = i & 1
        if i + 1 < args.steps:
            h2d(slot ^ 1)
        cur.wait_event(ready[slot])
        dks = st.step(xbuf[slot], gbuf[slot])
        consumed[slot].record(cur)
        off = 0
        for k in dks:
            dk_host[off:off + k.numel()].copy_(k.reshape(-1), non_blocking=True)
            off += k.numel()
    e2e_end.record(cur)
    torch.cuda.synchronize()
    e2e_ms = e2e_start.elapsed_time(e2e_end) / args.steps
    t = torch.tensor([e2e_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    e2e_ms = float(t.item())
    e2e = {"value": gflops / (e2e_ms * 1e-3) / 1e12, "unit": "TFLOP/s",
           "h2d_bytes_per_step": X_host.numel() * X_host.element_size() + dY_host.numel() * dY_host.element_size(),
           "d2h_bytes_per_step": dk_host.numel() * 4, "ms_per_step": e2e_ms,
           "note": "pinned host->device copy of step i+1 overlapped with step i on a copy stream"}

    # ---- CPU baseline: the oracle as it stands, on host cores, bounded
    # samples: all cores (OpenMP, ~10 s) and one thread (~5 s)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            import oracle
            oracle.build()
            fl1, Ks, strides, layers = stack_oracle_setup(specs, H, W, D, dtype)
            if train:
                fl1 = st.step_flops() / batch
                Kp64 = Kp.to(torch.float64).numpy()

            def timed(b):
                Xs, dYs = stack_oracle_inputs(layers, specs, H, W, D, b, dtype, gbatch)
                if train:
                    imgs = capsinputs.make_input(capsinputs.primary_layer(gbatch), dtype=dtype,
                                                 layer_idx=capsinputs.PRIMARY_SEED_LAYER, batch=b)
                    imgs = imgs.to(torch.float64).numpy()
                    t0 = time.perf_counter()
                    oracle.train_step(imgs, Kp64, Ks, strides[0], dYs, capsinputs.TRAIN_LR, True)
                    return time.perf_counter() - t0
                t0 = time.perf_counter()
                oracle.stack_fwd_bwd(Xs, Ks, strides[0], dYs, dtype == torch.bfloat16, pads=strides[1])
                return time.perf_counter() - t0

            ncores = oracle.num_threads()
            t1 = timed(1)
            # chunks of the same size the reference arm times per step (~1.5 s),
            # repeated for ~10 s: the oracle is memory-bound, so one big call over
            # hundreds of images would measure a different (slower) working set
            b = int(max(1, min(gbatch, 1.5 / max(t1, 1e-6))))
            timed(b)
            tb, nimg = 0.0, 0
            while tb < 10.0:
                tb += timed(b)
                nimg += b
            oracle.set_num_threads(1)
            try:
                s1 = timed(1)
                b1 = int(max(1, min(gbatch, 5.0 / max(s1, 1e-6))))
                sb1 = timed(b1) if b1 > 1 else s1
            finally:
                oracle.set_num_threads(ncores)
            cpu = {"value": fl1 * nimg / tb / 1e12, "unit": "TFLOP/s", "cores": ncores, "kind": "oracle",
                   "sample": "oracle (C, fp64, OpenMP) %s fwd+bwd, %d calls of %d of %d images, %.1f s" % (
                       name, nimg // b, b, gbatch, tb),
                   "single_thread": {"value": fl1 * b1 / sb1 / 1e12, "cores": 1,
                                     "sample": "%d images, %.1f s" % (b1, sb1)},
                   "host": host_cpu()}
        except Exception as e:  # the baseline is reported, never required
            cpu = {"value": None, "unit": "TFLOP/s", "cores": None, "kind": "oracle", "sample": "failed: %s" % e}

    # ---- parity: the benchmarked stack (same layout, weights, launch path) on
    # the first PB images of this rank's shard vs the oracle stack
    parity = None
    if rank == 0 and not args.no_parity:
        try:
            if train:
                parity = train_parity(pkg, specs, H, W, D, PB, Kp, weights, img_nat, dY_nat, dev)
            else:
                parity = parity_check(pkg, specs, H, W, D, PB, weights, X_nat, dY_nat, dtype, dev, args.layout)
        except Exception as e:
            parity = {"pass": False, "error": str(e)[:200]}

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 3), "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms_max, 5), "higher_is_better": True,
            "scaling": args.scaling if world > 1 else "weak",
            "vs_baseline": None, "dtype": args.dtype, "data": "synthetic (seeded capsinputs; random-init weights)",
            "config": {"workload": name, "global_batch": gbatch, "per_rank_batch": batch,
                       "layers": ["%dx%d s%d%s %d->%d" % (s.KH, s.KW, s.stride, " p%d" % s.pad if s.pad else "", s.C,
                                                          s.Cout) for s in specs],
                       "input": ("%dx%dx1 image -> %dx%d primary layer -> %dx%dx%d capsules %dx%d, SGD lr %g" % (
                           capsinputs.PRIMARY["H"], capsinputs.PRIMARY["W"], capsinputs.PRIMARY["KH"],
                           capsinputs.PRIMARY["KW"], H, W, specs[0].C, D, D, capsinputs.TRAIN_LR) if train
                           else "%dx%dx%d capsules %dx%d" % (H, W, specs[0].C, D, D)),
                       "layout": args.layout,
                       "parallelism": "dp%d" % world, "l2": "flushed between timed steps (%d MiB write)" % (flush.numel() >> 20),
                       "allreduce": "per-layer dK fp32 SUM on a side stream" if world > 1 else None,
                       "launch": ("one CUDA-graph replay of the captured step (%d libcapsconv kernels%s%s; "
                                  "per-pass times from a second graph running the passes one by one)" % (
                           launches_per_step, " + %d NCCL all-reduces" % len(specs) if world > 1 else "",
                           ", the dK chain on a second stream beside the dI chain" if st.dk_stream is not None else ""))
                       if use_graph else (graph_note or "eager launches")},
            "roofline": roofline,
            "cpu_baseline": cpu,
            "parity": parity,
            "paper_context": PAPER_CONTEXT,
            "e2e": e2e,
            "gpu_launches": launches,
            "clocks": clk.summary(),
            "per_pass": per_pass,
            "flops_per_step": gflops,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
