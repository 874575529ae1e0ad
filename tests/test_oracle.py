"""The CPU oracle against the reference's golden vectors and known answers (no GPU)."""

import itertools

import numpy as np
import pytest
import scipy.linalg as sl

from oracle import mps_oracle as orc


def test_uniforms_bit_exact_vs_reference(golden):
    j = 0
    while f"uniforms_{j}" in golden:
        seed, start, count, M = (int(x) for x in golden[f"uniforms_{j}_args"])
        assert np.array_equal(orc.stream_uniforms(seed, start, count, M), golden[f"uniforms_{j}"])
        j += 1
    assert j >= 4


def test_uniform_chunk_invariance():
    full = orc.stream_uniforms(9, 0, 300, 7)
    parts = np.concatenate([orc.stream_uniforms(9, s, 37, 7)[: min(37, 300 - s)] for s in range(0, 300, 37)])
    assert np.array_equal(full, parts)


def test_draw_rule_matches_reference_exact_sampler(golden):
    p, u, codes = golden["exact_p"], golden["exact_u"], golden["exact_codes"]
    k, ok, tie = orc.draw(np.broadcast_to(p, (len(u), len(p))).copy(), u)
    assert ok.all()
    cdf = np.cumsum(p)
    near = np.abs(cdf[:-1][None, :] - u[:, None]).min(axis=1) <= 1e-10
    assert np.array_equal(k[~near], codes[~near])


def test_draw_edges():
    p = np.array([[0.0, 0.5, 0.0, 0.5], [0.25, 0.25, 0.25, 0.25], [1.0, 0.0, 0.0, 0.0], [0, 0, 0, 0.0]])
    u = np.array([0.0, 0.999999, 0.7, 0.3])
    k, ok, tie = orc.draw(p, u)
    assert list(k[:3]) == [1, 3, 0]
    assert list(ok) == [True, True, True, False]
    # cdf boundary exactly at u is a tie and belongs to the next outcome (side="right")
    k, ok, tie = orc.draw(np.array([[0.5, 0.5]]), np.array([0.5]))
    assert k[0] == 1 and tie[0]


def test_displacement_coherent_column_vs_reference(golden):
    a = golden["coherent_alpha"]
    T = orc.displacement_matrix(a, 16)
    assert np.allclose(np.abs(T[:, 0, 0]) ** 2, golden["coherent_vacuum_prob"], rtol=0, atol=1e-14)
    k = np.arange(16)
    from math import factorial

    coh = np.exp(-np.abs(a)[:, None] ** 2 / 2) * a[:, None] ** k / np.sqrt([float(factorial(i)) for i in k])
    assert np.allclose(T[:, :, 0], coh, atol=1e-15)


def test_displacement_matches_expm_of_generator():
    Dbig = 80
    adag = np.diag(np.sqrt(np.arange(1, Dbig)), -1)
    for a in (0.3 + 0.4j, -0.7 + 0.1j, 1.1j):
        U = sl.expm(a * adag - np.conj(a) * adag.T)
        assert np.abs(U[:12, :12] - orc.displacement_matrix(a, 12)).max() < 1e-13


def test_displacement_unitary_limit():
    T = orc.displacement_matrix(0.5 - 0.2j, 60)
    assert np.abs(T[:, :20].conj().T @ T[:, :20] - np.eye(20)).max() < 1e-12


def test_sites_row_orthonormal_and_tapered():
    dims = orc.bond_dims(9, 50, 3)
    assert dims == [1, 3, 9, 27, 50, 50, 27, 9, 3, 1]
    sites = orc.random_mps(9, 50, 3, seed=2)
    for G in sites:
        A = G.reshape(G.shape[0], -1)
        assert np.abs(A @ A.conj().T - np.eye(A.shape[0])).max() < 1e-13


@pytest.mark.parametrize("M,chi,D", [(5, 4, 3), (4, 9, 3), (6, 3, 2)])
def test_chain_equals_born_with_unitary_local_ops(M, chi, D):
    """Brute-force full contraction (the pattern of tests/oracles.py): the
    per-step-renormalised chain reproduces Born probabilities exactly."""
    sites = orc.random_mps(M, chi, D, seed=M)
    rng = np.random.default_rng(1)
    ops = np.array([np.linalg.qr(rng.standard_normal((D, D)) + 1j * rng.standard_normal((D, D)))[0] for _ in range(M)])
    born = orc.born_distribution(sites, ops).reshape(-1)
    allk = np.array(list(itertools.product(range(D), repeat=M)))
    res = orc.sample_chain(sites, np.zeros((len(allk), M)), disp=np.broadcast_to(ops, (len(allk), M, D, D)),
                           forced=allk)
    assert np.abs(np.exp(res["logp"]) - born).max() < 1e-12


def test_chain_tvd_vs_born():
    M, chi, D = 4, 6, 3
    sites = orc.random_mps(M, chi, D, seed=4)
    born = orc.born_distribution(sites).reshape(-1)
    N = 40000
    res = orc.sample_chain(sites, orc.stream_uniforms(1, 0, N, M))
    codes = (res["counts"] * (D ** np.arange(M - 1, -1, -1))).sum(axis=1)
    emp = np.bincount(codes, minlength=D**M) / N
    assert 0.5 * np.abs(emp - born).sum() < 3 * np.sqrt(D**M / N) / 2


def test_product_state_vacuum_probability_vs_reference(golden):
    """chi = 1 vacuum sites + D(alpha): P(all zero) = prod exp(-|a|^2) = gbsemu.vacuum_overlap."""
    am = golden["coherent_multimode_alpha"]
    M, D = len(am), 16
    vac = np.zeros((1, 1, D), dtype=np.complex128)
    vac[0, 0, 0] = 1.0
    sites = [vac.copy() for _ in range(M)]
    res = orc.sample_chain(sites, np.zeros((1, M)), alpha=am[None, :], forced=np.zeros((1, M), int))
    assert abs(np.exp(res["logp"][0]) - float(golden["coherent_multimode_vacuum_prob"])) < 1e-14


def test_product_state_poisson_counts():
    M, D, N, sigma = 3, 16, 20000, 0.0
    a = np.array([0.6, 0.3 + 0.5j, -0.8j])
    vac = np.zeros((1, 1, D), dtype=np.complex128)
    vac[0, 0, 0] = 1.0
    res = orc.sample_chain([vac] * M, orc.stream_uniforms(2, 0, N, M), alpha=np.broadcast_to(a, (N, M)))
    for m in range(M):
        lam = abs(a[m]) ** 2
        mean = res["counts"][:, m].mean()
        assert abs(mean - lam) < 5 * np.sqrt(lam / N)


def test_batched_equals_serial(c1_sites):
    u = orc.stream_uniforms(0, 0, 50, 8)
    al = orc.alpha_stream(0, 0, 50, 8, 0.5)
    a = orc.sample_chain(c1_sites, u, alpha=al)["counts"]
    b = orc.sample_serial(c1_sites, u, alpha=al)
    assert np.array_equal(a, b)


def test_alpha_stream_law():
    al = orc.alpha_stream(3, 0, 20000, 4, 0.5)
    assert abs(np.mean(np.abs(al) ** 2) - 0.25) < 0.01
    assert abs(np.mean(al)) < 0.01
    assert np.array_equal(al[100:200], orc.alpha_stream(3, 100, 100, 4, 0.5))


def test_failed_sample_marked():
    sites = orc.random_mps(3, 2, 2, seed=0)
    sites = [s.copy() for s in sites]
    sites[1][:] = 0.0
    res = orc.sample_chain(sites, orc.stream_uniforms(0, 0, 4, 3))
    assert res["failed"].all() and (res["counts"] == -1).all()
