import ctypes, os, subprocess
here = os.path.dirname(os.path.abspath(__file__))
csrc = os.path.join(here, "..", "..", "paper_2104_02621_b200", "csrc")
lib = os.path.join(here, "libtma_bench.so")
subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O2", "-std=c++17", "-Xcompiler", "-fPIC", "-shared",
                "-I", csrc, "-I", os.path.join(here, "..", "..", "include"), "-o", lib, os.path.join(here, "tma_bench.cu"),
                os.path.join(csrc, "tma.cpp"), "-lcuda"], check=True)
L = ctypes.CDLL(lib)
L.tma_bench.restype = ctypes.c_double
L.tma_bench.argtypes = [ctypes.c_int] * 8
for mode in (0, 2):
    for nbox in (8, 16):
        print("mode=%s nbox=%d: %.0f GB/s" % (["one map", "bulk", "two maps"][mode], nbox, L.tma_bench(mode, nbox, 100, 24, 1, 2000, 24, 32)), flush=True)
