"""GPU parity of the planner's alternative code paths.

The production plans of the stack layers are pinned bit-exactly by
test_parity_gpu.py; the planner also has alternatives that other shapes (or
the environment switches used for A/B measurements) select: row-box vs tall-box
staging, per-phase vs merged stride-2 dI items, descriptor-shift vs
materialised vs one-tap-per-slot dK, one or two materialised dO copies,
buffer/loader-group orderings, forced tile groups and channel chunks.  The
switches are read once per process, so each variant runs in a subprocess that
checks every pass of the stack layers (at a small batch, exact-integer inputs:
results must equal the oracle bit for bit in any summation order) against the
oracle.
"""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r'''
import json, sys
import numpy as np, torch
sys.path.insert(0, sys.argv[1])
import capsinputs, oracle
import paper_2104_02621_b200.capsconv as cc
cc.load_library()
res = {}
for name, (B, H, W, C, Co, KH, KW, s) in {
        "L1": (6, 24, 24, 8, 8, 3, 3, 1), "L2": (6, 22, 22, 8, 16, 3, 3, 2),
        "L3": (6, 10, 10, 16, 32, 3, 3, 1), "FC": (40, 8, 8, 32, 10, 8, 8, 1)}.items():
    L = capsinputs.Layer(B, H, W, C, Co, KH, KW, 4, 4, 4, s)
    I = capsinputs.make_input(L, "int1", torch.bfloat16)
    K = capsinputs.make_kernel(L, "int1", torch.bfloat16)
    Ho, Wo = oracle.output_dims(H, W, KH, KW, s)
    dO = capsinputs.make_grad_output(L.o_shape(Ho, Wo), "int1", torch.bfloat16)
    Id, Kd, dOd = I.cuda(), K.cuda(), dO.cuda()
    O = cc.fwd(Id, Kd, s).float().cpu().numpy()
    dI = cc.bwd_data(dOd, Kd, s, H, W).float().cpu().numpy()
    dK = cc.bwd_kernel(Id, dOd, s, KH, KW).cpu().numpy()
    f64 = lambda t: t.to(torch.float64).numpy()
    rO, _ = oracle.fwd(f64(I), f64(K), s)
    rdI, _ = oracle.bwd_data(f64(dO), f64(K), s, H, W)
    rdK, _ = oracle.bwd_kernel(f64(I), f64(dO), s, KH, KW)
    rb = lambda a: oracle.round_bf16(a)
    ext = (B, H, W, C, Co, KH, KW, 4, 4, 4, s)
    paths = [cc.select_path(op, torch.bfloat16, ext) for op in (0, 1, 2)]   # fwd, bwd_data, bwd_kernel
    res[name] = [float(np.abs(O - rb(rO)).max()), float(np.abs(dI - rb(rdI)).max()),
                 float(np.abs(dK - rdK).max()), paths]
print(json.dumps(res))
'''

VARIANTS = [
    ("default", {}),
    ("row_boxes", {"CAPSCONV_NO_TALL": "1"}),
    ("tall_h2", {"CAPSCONV_TALL_H": "2"}),
    ("dI_per_phase", {"CAPSCONV_NO_MERGE": "1"}),
    ("force_G1", {"CAPSCONV_FORCE_G": "1"}),
    ("force_CC4", {"CAPSCONV_FORCE_CC": "4"}),
    ("wg_materialised", {"CAPSCONV_WG_BDESC": "0"}),
    ("wg_two_copies", {"CAPSCONV_WG_BMAT": "2"}),
    ("wg_one_tap_per_slot", {"CAPSCONV_WG_NQ1": "1"}),
    ("wg_buffers_2_2", {"CAPSCONV_WG_CMODE": "1"}),
    ("wg_buffers_4_4", {"CAPSCONV_WG_CMODE": "2"}),
    ("wg_one_loader_group", {"CAPSCONV_WG_LG": "1"}),
    ("wg_kp16", {"CAPSCONV_WG_KP": "16"}),
]


@pytest.mark.parametrize("name,env", VARIANTS, ids=[v[0] for v in VARIANTS])
def test_variant_exact(name, env):
    e = dict(os.environ)
    e.update(env)
    r = subprocess.run([sys.executable, "-c", CHILD, ROOT], env=e, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    res = json.loads(r.stdout.strip().splitlines()[-1])
    for layer, (eO, edI, edK, paths) in res.items():
        assert eO == 0.0 and edI == 0.0 and edK == 0.0, (name, layer, eO, edI, edK)
        # the variant must still run on the tensor-core path (no silent SIMT fallback)
        assert paths == [2, 2, 2], (name, layer, paths)
