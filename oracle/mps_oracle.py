"""CPU oracle for the displaced-MPS sampler — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
``--impl reference`` legs may import this module, and only as the checker or
the timed CPU baseline.  The product path (``paper_2511_14923_b200``) never
imports it and fails loudly without its CUDA library.

What it restates
----------------
The reference (``/root/reference``, package ``gbsemu``) ships no MPS sampler;
the hot path exists only as prose about the third-party "Chicago" CPU sampler
``sampling_cpu.py`` (zenodo 10.5281/zenodo.7992735, no version pin, absent
here).  This module restates that prose plus the reference's own sampling
conventions:

* ``PAPER.md:9``   amplitude = ordered product of site matrices A^[m]_{d_m};
* ``PAPER.md:58``  shapes: temp_tensor 1 x chi, Gamma chi x chi x D,
                   displacements 1 x M x D x D (batched here: n x M x D x D);
* ``PAPER.md:62``  temp @ Gamma.reshape(chi, chi*D), reshaped to 1 x chi x D;
* ``PAPER.md:64``  einsum contracting d with the displacement's 2nd index,
                   i.e. E[j, k] = sum_d C[j, d] Disp[k, d]  (E = C @ Disp.T);
* ``PAPER.md:66``  loop order: samples x modes, modes sequential;
* ``sampler.py:109-125`` counter-based Philox uniforms (restated bit-exactly
                   in :func:`stream_uniforms`, pinned by tests/golden);
* ``sampler.py:692-697`` inverse-CDF rule: cdf = cumsum(p), cdf[-1] = 1,
                   k = searchsorted(cdf, u, side="right") clamped;
* ``gaussian.py:387-391`` QR with the diagonal phase fix (site generator);
* ``tests/test_gaussian.py:139-143`` coherent known answer |<0|D(a)|0>|^2 = exp(-|a|^2).

Decisions the prose leaves open, pinned here (DESIGN.md §3 repeats them):

1. bond profile chi_0 = chi_M = 1, chi_m = min(chi, D^m, D^(M-m));
2. sites are row-orthonormal: Gamma.reshape(chi_l, chi_r*D) has orthonormal
   rows (sum_d G_d G_d^+ = I), so the left-to-right chain rule is exact;
3. marginal p(k) = sum_j |E[j, k]|^2 (no Lambda weighting: the path has none);
4. cdf = cumsum(p) / sum(p) with cdf[-1] = 1.0, k = #{k' : cdf[k'] <= u},
   clamped to D-1; if that k has p(k) == 0 (only by rounding at the top) the
   draw steps down to the largest k' < k with p(k') > 0;
5. renormalise v' = E[:, k] / sqrt(p(k));
6. D(alpha) = exact truncated Fock matrix elements <k|D(alpha)|d> via the
   recurrence <k|D|d> = (sqrt(k) <k-1|D|d-1> - conj(alpha) <k|D|d-1>) / sqrt(d),
   <k|D|0> = exp(-|a|^2/2) a^k / sqrt(k!)  (not unitary after truncation; the
   per-step renormalisation absorbs the lost norm);
7. alpha_{i,m} ~ CN(0, sigma^2) from the counter stream keyed (seed, 2^62 + i//64),
   two uniforms per mode: alpha = sigma sqrt(-log1p(-u1)) exp(2 pi i u2);
8. a sample whose step norm sum_k p(k) is not finite and positive is failed;
   a sample is flagged when some draw had |cdf[k] - u| <= 1e-10 (k < D-1):
   only flagged samples may differ in counts between two correct engines.

Parity status: the restatement is PINNED against the reference's own
conventions (uniform stream bit-for-bit, inverse-CDF rule, coherent overlap;
tests/golden) and against builder-made known answers (brute-force Born
probabilities at tiny M, product states).  It is UNPINNED against the Chicago
implementation itself, which is not available anywhere in this environment.
"""

from __future__ import annotations

import math

import numpy as np

STREAM_BLOCK = 64          # sampler.py:106
ALPHA_BLOCK_OFFSET = 1 << 62
TIE_EPS = 1e-10


# ---------------------------------------------------------------------------
# counter-based randomness (sampler.py:106-130)
# ---------------------------------------------------------------------------


def _philox_rows(seed: int, blk: int, width: int) -> np.ndarray:
    gen = np.random.Generator(np.random.Philox(key=[seed & (2**64 - 1), blk]))
    return gen.random((STREAM_BLOCK, width))


def stream_uniforms(seed: int, start: int, count: int, M: int) -> np.ndarray:
    """Uniforms of samples start..start+count-1, shape (count, M).

    Restates ``gbsemu.sampler._stream_uniforms`` (sampler.py:109-125): sample i
    reads row i mod 64 of Philox(key=[seed, i // 64]).random((64, M)).
    """
    out = np.empty((count, M))
    if count == 0:
        return out
    for blk in range(start // STREAM_BLOCK, (start + count - 1) // STREAM_BLOCK + 1):
        rows = _philox_rows(seed, blk, M)
        lo = max(start, blk * STREAM_BLOCK)
        hi = min(start + count, (blk + 1) * STREAM_BLOCK)
        out[lo - start: hi - start] = rows[lo - blk * STREAM_BLOCK: hi - blk * STREAM_BLOCK]
    return out


def alpha_stream(seed: int, start: int, count: int, M: int, sigma: float) -> np.ndarray:
    """Per-sample per-mode displacements alpha ~ CN(0, sigma^2), shape (count, M).

    Same block structure as :func:`stream_uniforms` on the key
    (seed, 2^62 + i // 64) with 2M uniforms per sample: (u1, u2) = row[2m], row[2m+1];
    |alpha|^2 ~ Exp(sigma^2) and a uniform phase (decision 7).
    """
    out = np.empty((count, M), dtype=np.complex128)
    if count == 0:
        return out
    for blk in range(start // STREAM_BLOCK, (start + count - 1) // STREAM_BLOCK + 1):
        rows = _philox_rows(seed, ALPHA_BLOCK_OFFSET + blk, 2 * M)
        lo = max(start, blk * STREAM_BLOCK)
        hi = min(start + count, (blk + 1) * STREAM_BLOCK)
        r = rows[lo - blk * STREAM_BLOCK: hi - blk * STREAM_BLOCK]
        u1, u2 = r[:, 0::2], r[:, 1::2]
        rad = sigma * np.sqrt(-np.log1p(-u1))
        ph = 2.0 * np.pi * u2
        out[lo - start: hi - start] = rad * np.cos(ph) + 1j * (rad * np.sin(ph))
    return out


# ---------------------------------------------------------------------------
# MPS sites (decisions 1-2; QR + phase fix as gaussian.py:387-391)
# ---------------------------------------------------------------------------


def bond_dims(M: int, chi: int, D: int) -> list[int]:
    """chi_0 .. chi_M with chi_0 = chi_M = 1 and chi_m = min(chi, D^m, D^(M-m))."""
    dims = [1]
    for m in range(1, M):
        e = min(m, M - m)
        cap = chi
        p = 1
        for _ in range(e):
            p *= D
            if p >= cap:
                break
        dims.append(min(cap, p))
    dims.append(1)
    return dims


def random_site(seed: int, m: int, chi_l: int, chi_r: int, D: int) -> np.ndarray:
    """Row-orthonormal site tensor Gamma^[m] of shape (chi_l, chi_r, D), complex128.

    Z ~ CN(0, 1)^{(chi_r D) x chi_l} from default_rng([seed, m]); Q R = Z with the
    diagonal phase fix Q <- Q diag(R_ii / |R_ii|); Gamma[i, j, d] = conj(Q[j D + d, i]).
    """
    if chi_l > chi_r * D:
        raise ValueError(f"site {m}: chi_l={chi_l} > chi_r*D={chi_r * D}, no isometry")
    rng = np.random.default_rng([seed, m])
    Z = (rng.standard_normal((chi_r * D, chi_l)) + 1j * rng.standard_normal((chi_r * D, chi_l))) / np.sqrt(2.0)
    Q, R = np.linalg.qr(Z)
    d = np.diagonal(R)
    Q = Q * (d / np.abs(d))
    return np.ascontiguousarray(Q.conj().T.reshape(chi_l, chi_r, D))


def random_mps(M: int, chi: int, D: int, seed: int = 0) -> list[np.ndarray]:
    dims = bond_dims(M, chi, D)
    return [random_site(seed, m, dims[m], dims[m + 1], D) for m in range(M)]


# ---------------------------------------------------------------------------
# displacement (decision 6)
# ---------------------------------------------------------------------------


def displacement_matrix(alpha, D: int) -> np.ndarray:
    """Truncated Fock matrix <k|D(alpha)|d>, shape alpha.shape + (D, D), [out k, in d]."""
    a = np.asarray(alpha, dtype=np.complex128)
    T = np.zeros(a.shape + (D, D), dtype=np.complex128)
    ac = np.conj(a)
    T[..., 0, 0] = np.exp(-0.5 * (a.real * a.real + a.imag * a.imag))
    for k in range(1, D):
        T[..., k, 0] = T[..., k - 1, 0] * a / math.sqrt(k)
    for d in range(1, D):
        inv = 1.0 / math.sqrt(d)
        T[..., 0, d] = (-ac * T[..., 0, d - 1]) * inv
        for k in range(1, D):
            T[..., k, d] = (math.sqrt(k) * T[..., k - 1, d - 1] - ac * T[..., k, d - 1]) * inv
    return T


# ---------------------------------------------------------------------------
# the chain sampler (PAPER.md:58-66 + decisions 3-5, 8)
# ---------------------------------------------------------------------------


def draw(p: np.ndarray, u: np.ndarray):
    """Inverse-CDF draw per row of p (n x D) against u (n,).

    Returns (k, ok, tie): sampler.py:692-697 rule on the normalised cdf.
    """
    n, D = p.shape
    P = p.sum(axis=1)
    ok = np.isfinite(P) & (P > 0)
    Ps = np.where(ok, P, 1.0)
    cdf = np.cumsum(p, axis=1) / Ps[:, None]
    cdf[:, -1] = 1.0
    k = np.minimum((cdf <= u[:, None]).sum(axis=1), D - 1)
    rows = np.arange(n)
    # decision 4: never land on a zero-probability outcome
    for _ in range(D):
        zero = ok & (p[rows, k] <= 0) & (k > 0)
        if not zero.any():
            break
        k = np.where(zero, k - 1, k)
    tie = np.abs(cdf[:, :-1] - u[:, None]).min(axis=1) <= TIE_EPS if D > 1 else np.zeros(n, bool)
    return k.astype(np.int32), ok, tie


def sample_chain(sites, uniforms, disp=None, alpha=None, forced=None, return_marginals=False, state_in=None,
                 return_state=False):
    """Sample n paths through the MPS.

    sites: list of M arrays (chi_l, chi_r, D); uniforms: (n, M) in [0, 1);
    disp: (n, M, D, D) complex [out k, in d] or None; alpha: (n, M) complex or None
    (both None = no displacement); forced: (n, M) int outcomes to follow instead of
    drawing (teacher forcing, the pattern of sampler.py:394-416).  state_in: (n, chi_0)
    complex starting state for a chain that begins mid-MPS (a pipeline stage; default
    ones(n, 1)); return_state adds the final (n, chi_M) state as "state".

    Returns dict(counts (n, M) int32, failed (n,) bool, flagged (n,) bool,
    marginals (n, M, D) normalised p/P when requested, logp (n,) log joint
    probability of the realised path under the per-step-renormalised chain).
    """
    u = np.asarray(uniforms, dtype=np.float64)
    n, M = u.shape
    if len(sites) != M:
        raise ValueError("uniforms must have one column per site")
    D = sites[0].shape[2]
    v = np.ones((n, 1), dtype=np.complex128) if state_in is None else np.asarray(state_in, dtype=np.complex128)
    counts = np.zeros((n, M), dtype=np.int32)
    failed = np.zeros(n, dtype=bool)
    flagged = np.zeros(n, dtype=bool)
    logp = np.zeros(n)
    marg = np.zeros((n, M, D)) if return_marginals else None
    rows = np.arange(n)
    for m in range(M):
        G = sites[m]
        chl, chr_, _ = G.shape
        C = (v @ G.reshape(chl, chr_ * D)).reshape(n, chr_, D)
        if disp is not None:
            Dm = np.asarray(disp[:, m])
        elif alpha is not None:
            Dm = displacement_matrix(np.asarray(alpha)[:, m], D)
        else:
            Dm = None
        E = C if Dm is None else np.einsum("bjd,bkd->bjk", C, Dm)
        p = (E.real * E.real + E.imag * E.imag).sum(axis=1)             # decision 3
        k, ok, tie = draw(p, u[:, m])
        if forced is not None:
            k = np.asarray(forced)[:, m].astype(np.int32)
        failed |= ~ok
        flagged |= tie & ok
        P = np.where(ok, p.sum(axis=1), 1.0)
        pk = p[rows, k]
        if marg is not None:
            marg[:, m] = p / P[:, None]
        good = ok & (pk > 0)
        logp += np.where(good, np.log(np.where(good, pk / P, 1.0)), -np.inf)
        scale = np.where(good, 1.0 / np.sqrt(np.where(good, pk, 1.0)), 0.0)
        v = E[rows, :, k] * scale[:, None]                               # decision 5
        counts[:, m] = k
    counts[failed] = -1
    out = dict(counts=counts, failed=failed, flagged=flagged, logp=logp)
    if marg is not None:
        out["marginals"] = marg
    if return_state:
        out["state"] = v
    return out


def sample_serial(sites, uniforms, disp=None, alpha=None):
    """Chicago's serial form: one 1 x chi ZGEMV chain per sample.

    Same decisions as :func:`sample_chain`; kept for the memory-bound serial CPU
    baseline and as a cross-check that batching changes nothing.
    """
    u = np.asarray(uniforms)
    res = [sample_chain(sites, u[i: i + 1],
                        None if disp is None else disp[i: i + 1],
                        None if alpha is None else alpha[i: i + 1])["counts"][0]
           for i in range(u.shape[0])]
    return np.array(res, dtype=np.int32).reshape(u.shape[0], len(sites))


# ---------------------------------------------------------------------------
# brute force (tiny M): full contraction, the pattern of tests/oracles.py:12-82
# ---------------------------------------------------------------------------


def full_state(sites, local_ops=None) -> np.ndarray:
    """psi[d_0, ..., d_{M-1}] = prod_m Gamma^[m]_{d_m}, optionally with local D x D ops applied."""
    M = len(sites)
    D = sites[0].shape[2]
    psi = np.ones((1, 1), dtype=np.complex128)                  # (D^m, chi_m)
    for m, G in enumerate(sites):
        chl, chr_, _ = G.shape
        if local_ops is not None:
            G = np.einsum("ijd,kd->ijk", G, local_ops[m])
        t = psi @ G.reshape(chl, chr_ * D)                        # (D^m, chi_r*D)
        t = t.reshape(-1, chr_, D).transpose(0, 2, 1).reshape(-1, chr_)
        psi = t
    return psi.reshape((D,) * M)


def born_distribution(sites, local_ops=None) -> np.ndarray:
    psi = full_state(sites, local_ops)
    p = np.abs(psi) ** 2
    return p / p.sum()
