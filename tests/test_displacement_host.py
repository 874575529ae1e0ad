"""Host check (no GPU) of the arithmetic the device's D(alpha) recurrence relies on
(csrc/displace_draw.cuh: cmul_rn, displacement_column0, displacement_entry).

The device forms complex products the way numpy's SIMD loops do: re = fma(ar, br, -(ai*bi)) and
im = fma(ar, bi, ai*br).  The recurrence below restates the device code with exact FMAs (rational
arithmetic) and must reproduce oracle.displacement_matrix bit for bit when given numpy's exp().
If this host's numpy forms complex products differently (no FMA3), the test skips: the oracle's
D(alpha) then differs from the device's by rounding (~1e-12 at D = 16, |alpha| ~ 2.4), which is
still inside the parity bar."""

import math
from fractions import Fraction

import numpy as np
import pytest

from oracle import mps_oracle as orc


def _fma(x, y, z):
    return float(Fraction(x) * Fraction(y) + Fraction(z))


def _cmul_rn(a, b):
    return complex(_fma(a.real, b.real, -(a.imag * b.imag)), _fma(a.real, b.imag, a.imag * b.real))


def _device_matrix(a, D):
    T = [[0j] * D for _ in range(D)]
    T[0][0] = complex(float(np.exp(np.array([-0.5 * (a.real * a.real + a.imag * a.imag)]))[0]), 0.0)
    for k in range(1, D):
        v, s = _cmul_rn(T[k - 1][0], a), 1.0 / math.sqrt(k)
        T[k][0] = complex(v.real * s, v.imag * s)
    for d in range(1, D):
        inv = 1.0 / math.sqrt(d)
        for k in range(D):
            t2 = _cmul_rn(complex(a.real, -a.imag), T[k][d - 1])
            if k == 0:
                T[k][d] = complex(-t2.real * inv, -t2.imag * inv)
                continue
            sk, t1 = math.sqrt(k), T[k - 1][d - 1]
            T[k][d] = complex((sk * t1.real - t2.real) * inv, (sk * t1.imag - t2.imag) * inv)
    return np.array(T)


def _numpy_uses_fma_form():
    rng = np.random.default_rng(0)
    a = rng.standard_normal(64) + 1j * rng.standard_normal(64)
    b = rng.standard_normal(64) + 1j * rng.standard_normal(64)
    p = a * b
    return all(_cmul_rn(x, y) == z for x, y, z in zip(a, b, p))


def test_device_displacement_recurrence_matches_oracle_bitwise():
    if not _numpy_uses_fma_form():
        pytest.skip("this host's numpy does not form complex products with FMA3 (see module docstring)")
    alphas = orc.alpha_stream(4, 0, 10, 2, 0.9).reshape(-1)
    for D in (4, 10, 16):
        ref = orc.displacement_matrix(alphas, D)
        dev = np.stack([_device_matrix(a, D) for a in alphas])
        assert np.array_equal(dev, ref), (D, int((dev != ref).sum()), float(np.abs(dev - ref).max()))
