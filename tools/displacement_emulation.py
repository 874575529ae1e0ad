"""CPU emulation of the device's D(alpha) recurrence (csrc/displace_draw.cuh: displacement_column0,
displacement_entry, cmul_rn) against the oracle's numpy construction (oracle.displacement_matrix).
Host only, no GPU.  Exact FMAs come from rational arithmetic.  With numpy's own exp() for T[0,0] the
emulation is bit-identical to the oracle at D = 4, 10 and 16.  With libm's exp() (a stand-in for
CUDA's) only exp's last bit differs, and that is a common factor of the matrix.
    python tools/displacement_emulation.py        (profiles/r02_conditioning.txt)"""
import math
import sys
from fractions import Fraction

import numpy as np

sys.path.insert(0, ".")
from oracle import mps_oracle as orc  # noqa: E402


def fma(x, y, z):
    return float(Fraction(x) * Fraction(y) + Fraction(z))


def cmul(a, b):  # cmul_rn: numpy's SIMD complex multiply
    return complex(fma(a.real, b.real, -(a.imag * b.imag)), fma(a.real, b.imag, a.imag * b.real))


def device_matrix(a, D, exp):
    T = [[0j] * D for _ in range(D)]
    T[0][0] = complex(exp(-0.5 * (a.real * a.real + a.imag * a.imag)), 0.0)
    for k in range(1, D):
        v, s = cmul(T[k - 1][0], a), 1.0 / math.sqrt(k)
        T[k][0] = complex(v.real * s, v.imag * s)
    for d in range(1, D):
        inv = 1.0 / math.sqrt(d)
        for k in range(D):
            t2 = cmul(complex(a.real, -a.imag), T[k][d - 1])
            if k == 0:
                T[k][d] = complex(-t2.real * inv, -t2.imag * inv)
                continue
            sk, t1 = math.sqrt(k), T[k - 1][d - 1]
            T[k][d] = complex((sk * t1.real - t2.real) * inv, (sk * t1.imag - t2.imag) * inv)
    return np.array(T)


def main():
    al = orc.alpha_stream(4, 0, 50, 3, 0.7).reshape(-1)
    exps = {"numpy exp": lambda x: float(np.exp(np.array([x]))[0]), "libm exp": math.exp}
    for D in (4, 10, 16):
        ref = orc.displacement_matrix(al, D)
        for name, ex in exps.items():
            dev = np.stack([device_matrix(a, D, ex) for a in al])
            print(f"D={D:2d} {name}: entries differing from the oracle {int((dev != ref).sum())} of {ref.size}, "
                  f"max |diff| {np.abs(dev - ref).max():.1e}", flush=True)


if __name__ == "__main__":
    main()
