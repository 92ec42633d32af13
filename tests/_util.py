"""Shared test helpers: parity metrics and the north_star tolerance gates."""
import math

import numpy as np


def rel_fro(got, ref) -> float:
    """Whole-output relative Frobenius error in fp64 (reading R6)."""
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    nr = np.linalg.norm(ref)
    return float(np.linalg.norm(got - ref) / (nr if nr > 0 else 1.0))


def gate(dtype: str, h: int) -> float:
    """BASELINE.json north_star: max relative Frobenius error 1e-12 (fp64), 2e-5*sqrt(h) (fp32).
    h = 0 uses sqrt(1): the result is then a copy/scale, exact up to one rounding."""
    return 1e-12 if dtype == "f64" else 2e-5 * math.sqrt(max(h, 1))


def assert_parity(got, ref, dtype: str, h: int, what: str = ""):
    got = np.asarray(got)
    assert np.all(np.isfinite(got)), f"{what}: non-finite outputs"
    e = rel_fro(got, ref)
    assert e <= gate(dtype, h), f"{what}: rel_fro {e:.3e} > gate {gate(dtype, h):.3e}"
    return e
