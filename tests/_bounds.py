"""Shared tolerance helpers for the parity tests (no method arithmetic)."""
import numpy as np


def f64_within(got, exact, c):
    """SURVEY 8(c) a7 bound: |V - V_int/n| <= 1e-12 V_int/n when V_int/n >= 1e-9 R_nc, else
    <= 1e-12 R_nc (R_nc = T_N / n, the no-checkpoint expected recompute)."""
    c = np.asarray(c, np.float64)
    n = c.sum()
    rnc = (np.arange(c.size) * c).sum() / n if n > 0 else 0.0
    exact = np.asarray(exact, np.float64)
    tol = np.where(exact >= 1e-9 * rnc, 1e-12 * exact, 1e-12 * rnc)
    return np.abs(np.asarray(got) - exact) <= tol
