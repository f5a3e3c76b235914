"""Per-kernel SASS instruction summary of the built libcapsconv.so (run here,
no GPU): counts of the tcgen05 / TMA / TMEM / mbarrier instructions that prove
what each kernel issues, plus registers and local memory from -res-usage.
    python tests/probe/sass_summary.py > profiles/r2_sass_summary.txt"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
LIB = os.path.join(ROOT, "paper_2104_02621_b200", "libcapsconv.so")
OPS = ["UTCHMMA", "UTCQMMA", "UTCBAR", "UTMALDG", "UTMASTG", "UBLKCP", "LDTM", "STTM", "SYNCS", "HMMA", "FFMA",
       "LDS", "STS", "LDG", "STG", "LDL", "STL"]


def demangle(n):
    try:
        return subprocess.run(["c++filt", n], capture_output=True, text=True).stdout.strip()
    except OSError:
        return n


def main():
    sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
    res = subprocess.run(["cuobjdump", "-res-usage", LIB], capture_output=True, text=True).stdout
    regs = {}
    cur = None
    for line in res.splitlines():
        m = re.search(r"Function (\S+):", line)
        if m:
            cur = m.group(1)
        m = re.search(r"REG:(\d+) STACK:(\d+) SHARED:(\d+) LOCAL:(\d+)", line)
        if m and cur:
            regs[cur] = m.groups()
    kern = collections.OrderedDict()
    cur = None
    for line in sass.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            cur = m.group(1)
            kern[cur] = collections.Counter()
            continue
        m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", line)
        if m and cur:
            op = m.group(2)
            kern[cur]["total"] += 1
            for o in OPS:
                if op == o or op.startswith(o + "."):
                    kern[cur][o] += 1
    print("# SASS summary of %s (cuobjdump -sass / -res-usage, sm_100a)" % os.path.relpath(LIB, ROOT))
    print("# static instruction counts per kernel (not dynamic); REG/STACK from -res-usage")
    for k, c in kern.items():
        name = demangle(k)
        name = name.replace("(anonymous namespace)::", "").replace("capsconv::", "")
        name = re.sub(r"^void ", "", name)
        name = re.sub(r"\(.*", "", name)
        r = regs.get(k, ("?", "?", "?", "?"))
        ops = " ".join("%s=%d" % (o, c[o]) for o in OPS if c[o])
        print("%-60s REG=%s STACK=%s instr=%d  %s" % (name[:60], r[0], r[1], c["total"], ops))


if __name__ == "__main__":
    sys.exit(main())
