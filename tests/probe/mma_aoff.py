"""Probe: SS tcgen05.mma cost (cycles per MMA, 148 CTAs back to back) with the A
start shifted inside the swizzle atom (the walk's column taps start q pixels =
4q rows further), for B without swizzle (the packed weights)."""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from test_rows_probe_gpu import load_probe  # noqa: E402

lib = load_probe()
for swz in (64, 128):
    rowb = swz
    for aoff in (0, 4 * rowb, 8 * rowb, 12 * rowb):
        row = []
        for N in (32, 64, 96, 128, 192, 256):
            row.append("%3d:%6.1f" % (N, lib.rows_bench(2, swz, N, 4096, 1, 148, aoff, 0)))
        print("swz %3d aoff %4d  " % (swz, aoff) + "  ".join(row), flush=True)
    for walk in (4 * rowb, 8 * rowb):
        row = []
        for N in (32, 96, 192):
            row.append("%3d:%6.1f" % (N, lib.rows_bench(2, swz, N, 4096, 1, 148, 0, walk)))
        print("swz %3d walk %4d  " % (swz, walk) + "  ".join(row), flush=True)
