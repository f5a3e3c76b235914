"""TS MMA issue cost in wgrad's form: B MN-major vs K-major, A column walk."""
import ctypes, os
lib = ctypes.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "libumma_probe.so"))
lib.umma_bench2.argtypes = [ctypes.c_int] * 6
lib.umma_bench2.restype = ctypes.c_double
for astep in (0, 8, -1, -2, -3):
    row = []
    for N in (32, 64):
        lib.umma_bench2(N, 240, 1, astep, 148, 128)
        row.append("N=%d:%.1f" % (N, lib.umma_bench2(N, 4800, 1, astep, 148, 128)))
    print("a_step=%d " % astep, "  ".join(row), flush=True)
