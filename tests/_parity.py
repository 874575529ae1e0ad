"""Shared parity metric for the GPU tests (BASELINE.json north_star): normalised marginals within
1e-10 RELATIVE per element in complex128 (1e-4 in complex64), applied to every marginal above a
floor (|dp| <= tol * p for p > 1e-12); below the floor an absolute bound."""

import numpy as np

REL_TOL_C128 = 1e-10
REL_TOL_C64 = 1e-4
P_FLOOR = 1e-12


def marginal_errors(p_gpu, p_cpu, floor=P_FLOOR):
    """(max |dp|, max |dp| / p over p_cpu > floor, number of marginals above the floor)."""
    d = np.abs(np.asarray(p_gpu) - np.asarray(p_cpu))
    big = p_cpu > floor
    rel = float((d[big] / p_cpu[big]).max()) if big.any() else 0.0
    return float(d.max()), rel, int(big.sum())
