"""Measure tcgen05 MMA issue throughput (cycles per 128xNx16 bf16 MMA), SS vs TS."""
import ctypes, os
lib = ctypes.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "libumma_probe.so"))
lib.umma_bench.argtypes = [ctypes.c_int] * 6
lib.umma_bench.restype = ctypes.c_double
for ts in (0, 1):
    for lay in (0, 1, 2):
        row = []
        for N in (16, 32, 64, 128, 256):
            lib.umma_bench(N, 256, ts, 148, 1, lay)
            row.append("N=%d:%.1f" % (N, lib.umma_bench(N, 4096, ts, 148, 1, lay)))
        print("%s lay=%d " % ("TS" if ts else "SS", lay), "  ".join(row), flush=True)
