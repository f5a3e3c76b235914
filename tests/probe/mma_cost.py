"""Probe: SS tcgen05.mma cost (cycles per MMA, 148 CTAs issuing back to back)
vs N for swizzled K-major A with swizzled (mode 0) or no-swizzle (mode 2) B."""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from test_rows_probe_gpu import load_probe  # noqa: E402

lib = load_probe()
for mode in (0, 2):
    for swz in (64, 128):
        for nacc in (1, 2):
            row = []
            for N in (32, 64, 96, 128, 192, 256):
                row.append("%3d:%6.1f" % (N, lib.rows_bench(mode, swz, N, 4096, nacc, 148, 0, 0)))
            print("mode %d swz %3d nacc %d  " % (mode, swz, nacc) + "  ".join(row), flush=True)
