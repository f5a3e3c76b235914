"""Build libcapsconv.so in-tree with nvcc for sm_100a (no JIT cache, no torch
extension machinery: the library is a plain C-ABI shared object)."""
from __future__ import annotations

import concurrent.futures
import glob
import os
import subprocess

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
BUILD = os.path.join(PKG, "build")
LIB = os.path.join(PKG, "libcapsconv.so")
# probe flavour (tests/probe/ only): same sources with -DCAPSCONV_PROBES, which
# compiles in the diagnostic knobs (skip switches, planner overrides, traces)
PROBE_LIB = os.path.join(PKG, "libcapsconv_probe.so")
PROBE_BUILD = os.path.join(PKG, "build_probe")

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
         "-I", INCLUDE, "-I", CSRC, "--expt-relaxed-constexpr"]


def _sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp")))


def _deps():
    return _sources() + sorted(glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh"))) + \
        [os.path.join(INCLUDE, "capsconv.h"), os.path.abspath(__file__)]


def needs_build(lib: str = LIB) -> bool:
    if not os.path.exists(lib):
        return True
    t = os.path.getmtime(lib)
    return any(os.path.getmtime(d) > t for d in _deps())


def _compile(src: str, verbose: bool, probes: bool = False) -> str:
    obj = os.path.join(PROBE_BUILD if probes else BUILD, os.path.basename(src) + ".o")
    extra = os.environ.get("CAPSCONV_EXTRA_FLAGS", "").split() if probes else []
    cmd = [NVCC] + ARCH + FLAGS + (["-DCAPSCONV_PROBES"] if probes else []) + extra + ["-c", src, "-o", obj]
    if src.endswith(".cu") and verbose:
        cmd += ["-Xptxas", "-v"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("nvcc failed for %s:\n%s\n%s" % (src, r.stdout, r.stderr))
    if verbose and r.stderr:
        print(r.stderr)
    return obj


def build(force: bool = False, verbose: bool = False, probes: bool = False) -> str:
    """Compile every CUDA / C++ source under csrc/ and link libcapsconv.so
    (probes=True: the diagnostic flavour libcapsconv_probe.so)."""
    lib = PROBE_LIB if probes else LIB
    if not force and not needs_build(lib):
        return lib
    os.makedirs(PROBE_BUILD if probes else BUILD, exist_ok=True)
    srcs = _sources()
    with concurrent.futures.ThreadPoolExecutor(max_workers=min(8, len(srcs))) as ex:
        objs = list(ex.map(lambda s: _compile(s, verbose, probes), srcs))
    tmp = lib + ".tmp.%d" % os.getpid()
    # -fvisibility=hidden + extern "C" with default visibility (see capsconv.h users):
    cmd = [NVCC] + ARCH + ["-shared", "-o", tmp] + objs + ["-lcudart", "-Xlinker", "-rpath=/usr/local/cuda/lib64"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("link failed:\n%s\n%s" % (r.stdout, r.stderr))
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    import sys
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, probes="--probes" in sys.argv))
