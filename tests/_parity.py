"""Shared parity metric for the GPU tests (BASELINE.json north_star): normalised marginals within
1e-10 RELATIVE per element in complex128 (1e-4 in complex64), applied to every marginal above a
floor (|dp| <= tol * p for p > 1e-12); below the floor an absolute bound."""

import numpy as np

REL_TOL_C128 = 1e-10
REL_TOL_C64 = 1e-4
# complex128 K1 emulated on the INT8 tensor cores (gemm mode 8, 7 Ozaki digits, opt-in): its error is
# ~1e-13 of each row's scale, so the relative error of a marginal grows as that scale over p.  At
# D <= 10 it stays inside REL_TOL_C128; at D = 16 the smallest marginals reach 3.4e-10
# (tools/fuzz_large.py, profiles/r02_fuzz_large.txt), so the mode's stated bar is 1e-9 relative.
REL_TOL_OZAKI7 = 1e-9
P_FLOOR = 1e-12


def marginal_errors(p_gpu, p_cpu, floor=P_FLOOR):
    """(max |dp|, max |dp| / p over p_cpu > floor, number of marginals above the floor)."""
    d = np.abs(np.asarray(p_gpu) - np.asarray(p_cpu))
    big = p_cpu > floor
    rel = float((d[big] / p_cpu[big]).max()) if big.any() else 0.0
    return float(d.max()), rel, int(big.sum())
