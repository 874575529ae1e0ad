"""Randomised parity sweep (needs a B200): seeded random chains through the C ABI against the oracle.

Every case draws its own shape (M, tapered chi, D), displacement law, micro-batch size, lane count,
micro-batching of the call, small-chain selection and complex128 K1 product, samples a seeded index
window, and is held to the parity bar of tests/_parity.py (the INT8 K1 at 7 digits included):
marginals within 1e-10 absolute and 1e-10 relative (p > 1e-12) along the GPU's path, counts identical
to the free-running oracle except on flagged near-ties.  The case list is fixed by the seed, so a
failure names a reproducible configuration.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

from oracle import mps_oracle as orc  # noqa: E402
from paper_2511_14923_b200 import MPS, MpsSampler, alpha_stream, stream_uniforms  # noqa: E402
from paper_2511_14923_b200 import _native  # noqa: E402

from _parity import REL_TOL_C128, marginal_errors  # noqa: E402


def _cases(n_cases=96, seed=2024):
    rng = np.random.default_rng(seed)
    out = []
    for i in range(n_cases):
        D = int(rng.choice([2, 3, 4, 5, 7, 10, 12, 16]))
        M = int(rng.integers(1, 9))
        chi = int(rng.choice([1, 2, 5, 16, 40, 100, 160]))
        N = int(rng.integers(1, 300))
        out.append(dict(
            M=M, chi=chi, D=D, N=N, first=int(rng.integers(0, 10**6)),
            batch=int(rng.choice([1, 7, 64, 128, N])), lanes=int(rng.integers(1, 4)),
            micro=int(rng.choice([0, 0, 16, 50])), small_chain=int(rng.integers(0, 3)),
            gemm=int(rng.choice([3, 3, 4, 8])), sigma=float(rng.choice([0.0, 0.3, 0.5, 0.9])),
            seed=int(rng.integers(0, 2**31)), site_seed=int(rng.integers(0, 1000))))
    return out


@pytest.mark.parametrize("case", _cases(), ids=lambda c: "M{M}-chi{chi}-D{D}-N{N}-g{gemm}-sc{small_chain}".format(**c))
def test_random_chain_vs_oracle(case):
    c = case
    sites = orc.random_mps(c["M"], c["chi"], c["D"], seed=c["site_seed"])
    sigma = c["sigma"] if c["sigma"] > 0 else None
    N, M, D, first = c["N"], c["M"], c["D"], c["first"]
    u = stream_uniforms(c["seed"], first, N, M)
    al = alpha_stream(c["seed"], first, N, M, sigma) if sigma else None
    with MpsSampler(MPS(sites)) as eng:
        eng.set_gemm_mode(c["gemm"])
        eng.set_lanes(c["lanes"])
        eng.set_small_chain(c["small_chain"])
        eng.set_micro_batch(c["micro"])
        eng.set_streams(c["seed"], sigma)
        counts = np.zeros((N, M), dtype=np.int32)
        status = np.zeros(N, dtype=np.uint8)
        marg = np.zeros((N, M, D))
        for s0 in range(0, N, c["batch"]):  # host arrays, device counter streams, index window `first`
            b = min(c["batch"], N - s0)
            eng.run(first + s0, b, counts[s0:s0 + b], marginals=marg[s0:s0 + b], status=status[s0:s0 + b])
    assert not (status & _native.MPS_STATUS_FAILED).any()
    ref = orc.sample_chain(sites, u, alpha=al, forced=counts, return_marginals=True)
    ab, rel, _ = marginal_errors(marg, ref["marginals"])
    assert ab <= 1e-10 and rel <= REL_TOL_C128, (ab, rel)
    free = orc.sample_chain(sites, u, alpha=al)
    flagged = (status & _native.MPS_STATUS_FLAGGED) != 0
    mism = (counts != free["counts"]).any(axis=1) & ~flagged & ~free["flagged"]
    assert not mism.any(), int(mism.sum())


def _split_cases(n_cases=24, seed=77):
    rng = np.random.default_rng(seed)
    out = []
    for i in range(n_cases):
        M = int(rng.integers(2, 9))
        out.append(dict(M=M, mid=int(rng.integers(1, M)), chi=int(rng.choice([3, 16, 40, 100])),
                        D=int(rng.choice([2, 4, 10])), N=int(rng.integers(1, 260)),
                        dtype=str(rng.choice(["complex128", "complex128", "complex64"])),
                        micro=int(rng.choice([0, 32])), small_chain=int(rng.integers(0, 3)),
                        lanes=int(rng.integers(1, 3)), seed=int(rng.integers(0, 2**31))))
    return out


@pytest.mark.parametrize("case", _split_cases(), ids=lambda c: "M{M}-mid{mid}-chi{chi}-D{D}-N{N}-{dtype}".format(**c))
def test_random_stage_split_equals_full_chain(case):
    """A chain run as two stages (modes [0, mid) then [mid, M), the n x chi state handed over on the
    device) gives the same bits as the one-stage run, for both dtypes, micro-batched host outputs,
    lanes and small-chain selection -- the mode-pipelined layout's invariant."""
    c = case
    sites = [s.astype(c["dtype"]) for s in orc.random_mps(c["M"], c["chi"], c["D"], seed=c["seed"] % 1000)]
    mps = MPS(sites)
    N, M, D, mid = c["N"], c["M"], c["D"], c["mid"]
    cdt = torch.complex64 if c["dtype"] == "complex64" else torch.complex128
    chi_mid = mps.bond_dims[mid]
    with MpsSampler(mps) as eng:
        eng.set_lanes(c["lanes"])
        eng.set_small_chain(c["small_chain"])
        eng.set_micro_batch(c["micro"])
        eng.set_streams(c["seed"], 0.5)
        full_c = np.zeros((N, M), dtype=np.int32)
        full_m = np.zeros((N, M, D))
        eng.run(0, N, full_c, marginals=full_m, status=np.zeros(N, dtype=np.uint8))
        st = np.zeros(N, dtype=np.uint8)
        c2, m2 = np.zeros((N, M), dtype=np.int32), np.zeros((N, M, D))
        mid_state = torch.zeros((N, chi_mid), dtype=cdt, device="cuda")
        eng.run(0, N, c2, m_begin=0, m_end=mid, state_out=mid_state, marginals=m2, status=st)
        eng.run(0, N, c2, m_begin=mid, m_end=M, state_in=mid_state, marginals=m2, status=st)
    dm = np.abs(full_m - m2).max(axis=(0, 2))
    assert np.array_equal(full_c, c2) and np.array_equal(full_m, m2), (
        c, "modes with marginal differences", np.nonzero(dm)[0].tolist(), float(dm.max()),
        "rows", np.nonzero(np.abs(full_m - m2).max(axis=(1, 2)))[0][:10].tolist())


def _knob_cases(n_cases=32, seed=5150):
    rng = np.random.default_rng(seed)
    out = []
    for i in range(n_cases):
        out.append(dict(M=int(rng.integers(1, 7)), chi=int(rng.choice([2, 16, 60, 130])), D=int(rng.choice([3, 4, 10])),
                        N=int(rng.integers(1, 400)), gemm=int(rng.choice([3, 8])), seed=int(rng.integers(0, 2**31)),
                        knobs=dict(lanes=int(rng.integers(1, 5)), micro=int(rng.choice([0, 40, 100])),
                                   small_chain=int(rng.integers(0, 3)), sum_planes=bool(rng.integers(0, 2)),
                                   stream_sites=bool(rng.integers(0, 2)), borrow=bool(rng.integers(0, 2)),
                                   oz_site_mode=int(rng.integers(0, 3)), batch=int(rng.choice([1, 33, 128, 1000])),
                                   forced=bool(rng.integers(0, 2)))))
    return out


def _run_knobs(sites, c, k):
    """One sampling (or, with k["forced"], teacher-forced evaluation) pass under the given knobs."""
    N, M, D = c["N"], c["M"], c["D"]
    stream = k.get("stream_sites", False) and c["gemm"] == 3
    if stream:
        mps = MPS(sites)
    elif k.get("borrow", False):
        mps = MPS([torch.from_numpy(G).cuda() for G in sites])
    else:
        mps = MPS(sites)
    with MpsSampler(mps, sum_planes=k.get("sum_planes", True), stream_sites=stream) as eng:
        eng.set_gemm_mode(c["gemm"])
        eng.set_lanes(k.get("lanes", 1))
        eng.set_micro_batch(k.get("micro", 0))
        eng.set_small_chain(k.get("small_chain", 2))
        eng.set_ozaki_site_mode(k.get("oz_site_mode", 0), 64)
        eng.set_streams(c["seed"], 0.5)
        counts = np.zeros((N, M), dtype=np.int32)
        if k.get("forced", False):
            counts[:] = np.random.default_rng(c["seed"]).integers(0, min(D, 3), size=(N, M))
            eng.set_forced(True)
        marg = np.zeros((N, M, D))
        status = np.zeros(N, dtype=np.uint8)
        B = k.get("batch", N)
        for s0 in range(0, N, B):
            b = min(B, N - s0)
            eng.run(s0, b, counts[s0:s0 + b], marginals=marg[s0:s0 + b], status=status[s0:s0 + b])
    return counts, marg, status


@pytest.mark.parametrize("case", _knob_cases(), ids=lambda c: "M{M}-chi{chi}-D{D}-N{N}-g{gemm}".format(**c))
def test_random_knobs_bit_identical(case):
    """Every engine knob that promises identical results (lanes, micro-batching, small-chain selection,
    sum planes, host-streamed / borrowed / copied sites, streamed INT8 digit planes, call batch size)
    gives the same bits as the plain configuration, sampling or teacher-forced."""
    c = case
    sites = orc.random_mps(c["M"], c["chi"], c["D"], seed=c["seed"] % 997)
    plain = _run_knobs(sites, c, dict(forced=c["knobs"]["forced"]))
    other = _run_knobs(sites, c, c["knobs"])
    for a, b, name in zip(plain, other, ("counts", "marginals", "status")):
        assert np.array_equal(a, b), (name, c)


# Large ragged chains (tools/fuzz_large.py runs the seeded sweep of these, profiles/r02_fuzz_large.txt):
# bond dimensions that are not multiples of any tile edge, up to chi = 1333, sample counts just past
# the 64-row K1 tiles and the 1024-row lane split, every complex128 K1 product.
_LARGE = [
    dict(dims=[1, 10, 100, 887, 1333, 1000, 100, 10, 1], D=10, N=1025, gemm=3, lanes=2, micro=0, sigma=0.5),
    dict(dims=[1, 7, 49, 343, 777, 343, 49, 7, 1], D=7, N=257, gemm=4, lanes=3, micro=200, sigma=0.9),
    dict(dims=[1, 16, 202, 1100, 256, 16, 1], D=16, N=65, gemm=8, lanes=1, micro=0, sigma=0.0),
]


@pytest.mark.parametrize("case", _LARGE, ids=lambda c: "chi{}-D{D}-N{N}-g{gemm}".format(max(c["dims"]), **c))
def test_large_ragged_chain_vs_oracle(case):
    from paper_2511_14923_b200.mps import device_site

    c = case
    dims, D, N = c["dims"], c["D"], c["N"]
    M = len(dims) - 1
    sites = [device_site(11, m, dims[m], dims[m + 1], D) for m in range(M)]
    sigma = c["sigma"] or None
    u = stream_uniforms(11, 5000, N, M)
    al = alpha_stream(11, 5000, N, M, sigma) if sigma else None
    counts = np.zeros((N, M), dtype=np.int32)
    status = np.zeros(N, dtype=np.uint8)
    marg = np.zeros((N, M, D))
    with MpsSampler(MPS(sites)) as eng:
        eng.set_gemm_mode(c["gemm"])
        eng.set_lanes(c["lanes"])
        eng.set_micro_batch(c["micro"])
        eng.set_streams(11, sigma)
        eng.run(5000, N, counts, marginals=marg, status=status)
    assert not (status & _native.MPS_STATUS_FAILED).any()
    host = [G.cpu().numpy() for G in sites]
    ref = orc.sample_chain(host, u, alpha=al, forced=counts, return_marginals=True)
    ab, rel, _ = marginal_errors(marg, ref["marginals"])
    assert ab <= 1e-10 and rel <= REL_TOL_C128, (ab, rel)
    free = orc.sample_chain(host, u, alpha=al)
    flagged = (status & _native.MPS_STATUS_FLAGGED) != 0
    mism = (counts != free["counts"]).any(axis=1) & ~flagged & ~free["flagged"]
    assert not mism.any(), int(mism.sum())


def test_large_ragged_chain_complex64_vs_oracle():
    """The complex64 engine (3xTF32 tcgen05 K1) on a ragged chi = 1000 chain against the complex128
    oracle on the same rounded sites: the north star's 1e-4 as an absolute bound on the normalised
    marginals, relative error for p > 1e-3 held to the 1e-2 asserted after the 64 C3 modes
    (DESIGN.md §4 and §8 item 6: the c64 K1's fp32 TMEM accumulation sets it)."""
    from paper_2511_14923_b200.mps import device_site

    dims, D, N = [1, 10, 100, 999, 1000, 100, 10, 1], 10, 257
    M = len(dims) - 1
    sites = [device_site(12, m, dims[m], dims[m + 1], D).to(torch.complex64) for m in range(M)]
    u = stream_uniforms(12, 0, N, M)
    al = alpha_stream(12, 0, N, M, 0.5)
    counts = np.zeros((N, M), dtype=np.int32)
    status = np.zeros(N, dtype=np.uint8)
    marg = np.zeros((N, M, D))
    with MpsSampler(MPS(sites)) as eng:
        assert eng.dtype == "complex64"
        eng.set_streams(12, 0.5)
        eng.run(0, N, counts, marginals=marg, status=status)
    assert not (status & _native.MPS_STATUS_FAILED).any()
    host = [G.to(torch.complex128).cpu().numpy() for G in sites]
    ref = orc.sample_chain(host, u, alpha=al, forced=counts, return_marginals=True)
    ab, _, _ = marginal_errors(marg, ref["marginals"])
    _, rel, _ = marginal_errors(marg, ref["marginals"], floor=1e-3)
    print(f"c64 chi=1000 chain: max |dp| {ab:.1e}, max |dp|/p (p > 1e-3) {rel:.1e}")
    assert ab <= 1e-4 and rel <= 1e-2, (ab, rel)
    free = orc.sample_chain(host, u, alpha=al)
    flagged = (status & _native.MPS_STATUS_FLAGGED) != 0
    assert not ((counts != free["counts"]).any(axis=1) & ~flagged).any()
