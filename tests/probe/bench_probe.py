"""Probe: run bench.py against the diagnostic library flavour (libcapsconv_probe.so,
-DCAPSCONV_PROBES) so its env knobs apply, e.g.
    CAPSCONV_SKIP_SMALL=1 python tests/probe/bench_probe.py --steps 20 --no-cpu-baseline --no-parity"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import paper_2104_02621_b200.capsconv as cc  # noqa: E402
from paper_2104_02621_b200 import _build  # noqa: E402

cc.load_library(_build.PROBE_LIB)   # the process-wide library handle: every later load returns it
sys.argv[0] = os.path.join(ROOT, "bench.py")
import bench  # noqa: E402
bench.main()
