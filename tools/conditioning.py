"""How accurately can ANY complex128 engine reproduce a small marginal?  Runs on the host (no GPU).

For one chain shape it samples a path with the oracle, then evaluates the normalised marginals along
that path three ways and compares each with an extended-precision reference (numpy clongdouble,
64-bit mantissa, the chain evaluated per row in the oracle's operation order):
  * the oracle itself (complex128 ZGEMM, 4M-style products),
  * a 3M (Gauss) complex128 product, the GPU's default K1 decomposition,
  * the oracle vs the 3M evaluation (what a GPU-vs-oracle parity test sees).
Reported: max |dp| / p over marginals p > floor, for several floors.  The relative error of a small
marginal is set by cancellation in the contraction (|C_jk| much smaller than sum_i |v_i||G_ijk|), not
by the engine, so this bounds what the 1e-10 relative bar can demand at a given floor.
    python tools/conditioning.py            (profiles/r02_conditioning.txt)
"""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from oracle import mps_oracle as orc  # noqa: E402
from paper_2511_14923_b200.mps import host_site  # noqa: E402


def displacement_ld(alpha, D):
    """orc.displacement_matrix's recurrence evaluated in clongdouble (the extended-precision D(alpha))."""
    a = np.asarray(alpha).astype(np.clongdouble)
    T = np.zeros(a.shape + (D, D), dtype=np.clongdouble)
    ac = np.conj(a)
    T[..., 0, 0] = np.exp(np.longdouble(-0.5) * (a.real * a.real + a.imag * a.imag))
    for k in range(1, D):
        T[..., k, 0] = T[..., k - 1, 0] * a / np.sqrt(np.longdouble(k))
    for d in range(1, D):
        inv = np.longdouble(1) / np.sqrt(np.longdouble(d))
        T[..., 0, d] = (-ac * T[..., 0, d - 1]) * inv
        for k in range(1, D):
            T[..., k, d] = (np.sqrt(np.longdouble(k)) * T[..., k - 1, d - 1] - ac * T[..., k, d - 1]) * inv
    return T


def chain_marginals(sites, counts, product, dtype, alpha=None):
    """Normalised marginals along the forced path `counts`, C = v @ G by `product`, then the
    displacement einsum with D(alpha) built in the evaluation's own precision."""
    n, M = counts.shape
    D = sites[0].shape[2]
    v = np.ones((n, 1), dtype=dtype)
    out = np.zeros((n, M, D))
    rows = np.arange(n)
    for m, G in enumerate(sites):
        chl, chr_, _ = G.shape
        C = product(v, G.reshape(chl, chr_ * D).astype(dtype)).reshape(n, chr_, D)
        if alpha is not None:
            Dm = displacement_ld(alpha[:, m], D) if dtype == np.clongdouble else orc.displacement_matrix(alpha[:, m], D)
            C = np.einsum("bjd,bkd->bjk", C, Dm)
        p = (C.real * C.real + C.imag * C.imag).sum(axis=1)
        out[:, m] = (p / p.sum(axis=1, keepdims=True)).astype(np.float64)
        k = counts[:, m]
        v = C[rows, :, k] / np.sqrt(p[rows, k])[:, None]
    return out


def prod_4m(v, G):
    return v @ G


def prod_3m(v, G):
    vr, vi, gr, gi = v.real, v.imag, G.real, G.imag
    t1, t2, t3 = vr @ gr, vi @ gi, (vr + vi) @ (gr + gi)
    return (t1 - t2) + 1j * (t3 - (t1 + t2))


def rel_err(p, ref, floor):
    big = ref > floor
    return float((np.abs(p - ref)[big] / ref[big]).max()) if big.any() else 0.0, int(big.sum())


def main():
    shapes = [([1, 16, 256, 513, 249, 16, 1], 16, 0.9), ([1, 16, 256, 513, 249, 16, 1], 16, 0.0),
              ([1, 10, 100, 1000, 100, 10, 1], 10, 0.9), ([1, 10, 100, 1000, 100, 10, 1], 10, 0.5 ** 0.5),
              ([1, 7, 49, 343, 777, 343, 49, 7, 1], 7, 0.9), ([1, 4, 16, 64, 256, 64, 16, 4, 1], 4, 0.9)]
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
    floors = (1e-12, 1e-10, 1e-8, 1e-6)
    print(f"n = {n} sampled paths per shape; max |dp|/p over marginals above each floor "
          f"(floors {floors}); reference = clongdouble evaluation of the same path")
    for dims, D, sigma in shapes:
        t0 = time.time()
        M = len(dims) - 1
        sites = [host_site(3, m, dims[m], dims[m + 1], D) for m in range(M)]
        u = orc.stream_uniforms(3, 0, n, M)
        al = orc.alpha_stream(3, 0, n, M, sigma) if sigma > 0 else None
        counts = orc.sample_chain(sites, u, alpha=al)["counts"]
        ref = chain_marginals(sites, counts, prod_4m, np.clongdouble, al)
        p4 = chain_marginals(sites, counts, prod_4m, np.complex128, al)
        p3 = chain_marginals(sites, counts, prod_3m, np.complex128, al)
        if al is not None:
            Dm = orc.displacement_matrix(al, D)
            dD = float(np.abs(Dm - displacement_ld(al, D)).max())
        else:
            dD = 0.0
        print(f"dims={dims} D={D} sigma={sigma:.3g}  max|D(alpha)_fp64 - D(alpha)_exact| {dD:.1e}, "
              f"max|alpha| {np.abs(al).max() if al is not None else 0:.2f}  ({time.time() - t0:.0f} s)")
        for name, a, b in (("oracle  vs exact", p4, ref), ("3M      vs exact", p3, ref), ("3M      vs oracle", p3, p4)):
            cols = []
            for f in floors:
                r, nb = rel_err(a, b, f)
                cols.append(f"p>{f:.0e}: {r:.1e} (n={nb})")
            print(f"  {name}: max|dp| {np.abs(a - b).max():.1e}; " + "; ".join(cols), flush=True)


if __name__ == "__main__":
    main()
