import ctypes, os, subprocess
here = os.path.dirname(os.path.abspath(__file__))
csrc = os.path.join(here, "..", "..", "paper_2104_02621_b200", "csrc")
lib = os.path.join(here, "libtma_bench.so")
subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O2", "-std=c++17", "-Xcompiler", "-fPIC", "-shared",
                "-I", csrc, "-I", os.path.join(here, "..", "..", "include"), "-o", lib, os.path.join(here, "tma_bench.cu"),
                os.path.join(csrc, "tma.cpp"), "-lcuda"], check=True)
L = ctypes.CDLL(lib)
L.tma_bench.restype = ctypes.c_double
L.tma_bench.argtypes = [ctypes.c_int] * 6
for B in (2000, 8000):
    for W, rows, nbox in [(24, 1, 7), (24, 1, 28)]:
        for mode in (0, 1):
            print("B=%d mode=%s W=%d rows/box=%d nbox=%d box=%d B: %.0f GB/s" % (B, ["tensor", "bulk"][mode], W, rows, nbox,
                  W * 256 * rows, L.tma_bench(mode, nbox, 100, W, rows, B)), flush=True)
