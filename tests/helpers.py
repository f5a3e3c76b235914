"""Test helpers: the error metric of reading R19 and oracle glue."""
import numpy as np
import torch

# Tolerances stated by BASELINE.json's north_star ("max relative error 1e-5 in
# fp32 and 2e-2 in bf16"), applied to the metric of reading R19:
#   err = max_i |g_i - r_i| / max(sum_k |a_k b_k|_i, tiny)
TOL = {torch.float32: 1e-5, torch.bfloat16: 2e-2}


def rel_err(got, ref, abs_sum):
    g = np.asarray(got, dtype=np.float64)
    r = np.asarray(ref, dtype=np.float64)
    a = np.asarray(abs_sum, dtype=np.float64)
    if g.shape != r.shape:
        raise AssertionError("shape %s != %s" % (g.shape, r.shape))
    if g.size == 0:
        return 0.0
    if not np.all(np.isfinite(g)):
        return float("inf")
    return float(np.max(np.abs(g - r) / np.maximum(a, 1e-30)))


def to_np(t: torch.Tensor) -> np.ndarray:
    return t.detach().to("cpu", torch.float64).numpy()


def assert_close(got, ref, abs_sum, dtype, what=""):
    e = rel_err(got, ref, abs_sum)
    assert e <= TOL[dtype], "%s: normalised error %.3e > %.1e" % (what, e, TOL[dtype])
    return e
