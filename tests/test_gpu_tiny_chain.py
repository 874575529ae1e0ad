"""The tiny-chain kernel (chain_tiny.cuh: one CTA per 8-row group, every site in shared memory) against
the 16-CTA cluster kernel (small-chain mode 3) and the per-mode kernels (mode 0).

All three run the same 3M DMMA k order, the same draw reduction (for chi_r <= 32 the per-mode
draw's 128-thread tree reduces to its warp 0 plus exact zeros) and the same draw rule, so every
output bit must agree; the tiny kernel is also held to the oracle directly.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

from oracle import mps_oracle as orc  # noqa: E402
from paper_2511_14923_b200 import MPS, MpsSampler, MpsSamplerConfig, alpha_stream, stream_uniforms  # noqa: E402
from paper_2511_14923_b200 import _native  # noqa: E402

from _parity import REL_TOL_C128, marginal_errors  # noqa: E402

MODES = (2, 3, 0)  # tiny, cluster, per-mode


def _three(mps, fn, n):
    outs = []
    for mode in MODES:
        with MpsSampler(mps) as eng:
            eng.set_small_chain(mode)
            kind = eng.small_chain_kind(n)
            outs.append(fn(eng))
        assert kind == {2: 2, 3: 1 if kind else 0, 0: 0}[mode], (mode, kind)
    return outs


def _same(outs):
    for o in outs[1:]:
        for k in outs[0]:
            assert np.array_equal(outs[0][k], o[k]), k


@pytest.mark.parametrize("M,chi,D,n", [(8, 16, 4, 100), (8, 16, 4, 1000), (8, 16, 4, 5003), (4, 10, 10, 77),
                                       (7, 7, 3, 37), (4, 32, 8, 64), (3, 1, 16, 9), (1, 1, 7, 5),
                                       (12, 4, 2, 130), (4, 9, 7, 999), (40, 3, 2, 17), (64, 2, 2, 11)])
def test_tiny_chain_bit_identical(M, chi, D, n):
    mps = MPS(orc.random_mps(M, chi, D, seed=M * 7 + chi))
    cfg = MpsSamplerConfig(N=n, seed=13, alpha_sigma=0.5, batch_size=n)
    outs = _three(mps, lambda e: e.sample(cfg, return_marginals=True), n)
    _same(outs)


@pytest.mark.parametrize("kind", ["alpha", "disp", "none", "uniforms", "device_alpha"])
def test_tiny_chain_inputs(kind):
    M, chi, D, n = 8, 16, 4, 203
    sites = orc.random_mps(M, chi, D, seed=3)
    u = stream_uniforms(4, 17, n, M)
    alpha = alpha_stream(4, 17, n, M, 0.5)
    disp = None
    if kind == "disp":
        rng = np.random.default_rng(2)
        z = rng.standard_normal((n, M, D, D)) + 1j * rng.standard_normal((n, M, D, D))
        disp = np.linalg.qr(z)[0]

    def run(eng):
        if kind in ("uniforms", "device_alpha"):
            eng.set_streams(4, 0.5)
        counts = np.zeros((n, M), np.int32)
        marg = np.zeros((n, M, D))
        status = np.zeros(n, np.uint8)
        eng.run(17, n, counts, uniforms=None if kind == "device_alpha" else u,
                alpha=alpha if kind == "alpha" else None, disp=disp, marginals=marg, status=status)
        return dict(counts=counts, marginals=marg, status=status)

    outs = _three(MPS(sites), run, n)
    _same(outs)
    if kind in ("alpha", "device_alpha", "disp", "none"):
        ref = orc.sample_chain(sites, u, alpha=alpha if kind in ("alpha", "device_alpha") else None,
                               disp=disp, forced=outs[0]["counts"], return_marginals=True)
        ab, rel, _ = marginal_errors(outs[0]["marginals"], ref["marginals"])
        assert ab <= 1e-10 and rel <= REL_TOL_C128, (ab, rel)


def test_tiny_chain_oracle_parity_c1(c1_sites):
    """BASELINE configs[0] through the tiny kernel: marginals vs the teacher-forced oracle (relative
    bar), counts vs the free-running oracle except flagged near-ties."""
    n, M = 1000, 8
    cfg = MpsSamplerConfig(N=n, seed=0, alpha_sigma=0.5, batch_size=100)
    with MpsSampler(MPS(c1_sites)) as eng:
        assert eng.small_chain_kind(100) == 2
        res = eng.sample(cfg, return_marginals=True)
    u, al = stream_uniforms(0, 0, n, M), alpha_stream(0, 0, n, M, 0.5)
    ref = orc.sample_chain(c1_sites, u, alpha=al, forced=res["counts"], return_marginals=True)
    ab, rel, _ = marginal_errors(res["marginals"], ref["marginals"])
    assert ab <= 1e-10 and rel <= REL_TOL_C128, (ab, rel)
    free = orc.sample_chain(c1_sites, u, alpha=al)
    flagged = (res["status"] & _native.MPS_STATUS_FLAGGED) != 0
    assert not (((res["counts"] != free["counts"]).any(1)) & ~flagged & ~free["flagged"]).any()


def test_tiny_chain_forced_and_failures():
    M, chi, D, n = 8, 16, 4, 120
    mps = MPS(orc.random_mps(M, chi, D, seed=5))
    rng = np.random.default_rng(0)
    counts = rng.integers(0, 3, size=(n, M)).astype(np.int32)
    counts[5, 3] = 10  # out of range: the sample fails
    counts[9, 0] = -2
    outs = _three(mps, lambda e: e.evaluate(MpsSamplerConfig(N=n, seed=2, alpha_sigma=0.5, batch_size=n), counts), n)
    _same(outs)
    assert outs[0]["status"][5] & _native.MPS_STATUS_FAILED and outs[0]["status"][9] & _native.MPS_STATUS_FAILED


@pytest.mark.parametrize("n", [1, 7, 8, 9, 100])
def test_tiny_chain_stage_split_state_bounds(n):
    """state_in / state_out through the tiny kernel == the other paths, and padding rows of the last
    8-row group write nothing past state_out's n rows."""
    M, chi, D, cut = 10, 20, 4, 4
    mps = MPS(orc.random_mps(M, chi, D, seed=n))
    chi_cut = mps.bond_dims[cut]
    res = []
    for mode in MODES:
        counts = torch.zeros((n, M), dtype=torch.int32, device="cuda")
        marg = torch.zeros((n, M, D), dtype=torch.float64, device="cuda")
        status = torch.zeros(n, dtype=torch.uint8, device="cuda")
        big = torch.full((n + 16, chi_cut), 7.0 + 3.0j, dtype=torch.complex128, device="cuda")
        out = torch.zeros((n, 1), dtype=torch.complex128, device="cuda")
        with MpsSampler(mps, sites_range=(0, cut), layout=1) as s0, \
                MpsSampler(mps, sites_range=(cut, M), layout=1) as s1:
            for e in (s0, s1):
                e.set_streams(9, 0.5)
                e.set_small_chain(mode)
            if mode == 2:
                assert s0.small_chain_kind(n) == 2 and s1.small_chain_kind(n) == 2
            s0.run(0, n, counts, state_out=big[:n], marginals=marg, status=status)
            s1.run(0, n, counts, state_in=big[:n], state_out=out, marginals=marg, status=status)
        torch.cuda.synchronize()
        assert bool((big[n:] == 7.0 + 3.0j).all())
        res.append([x.cpu().numpy() for x in (counts, marg, status, big[:n], out)])
    for other in res[1:]:
        for a, b in zip(res[0], other):
            assert np.array_equal(a, b)


def test_tiny_chain_not_taken_past_its_bounds():
    """chi = 33 or chi_r D > 256 falls back to the cluster kernel; c64 and 4M never take it."""
    with MpsSampler(MPS(orc.random_mps(14, 33, 2, seed=1))) as eng:  # bonds reach 33
        eng.set_small_chain(1)
        assert eng.small_chain_kind(100) == 1
    with MpsSampler(MPS(orc.random_mps(6, 30, 10, seed=1))) as eng:  # chi_r D = 300
        eng.set_small_chain(1)
        assert eng.small_chain_kind(100) == 1
    with MpsSampler(MPS(orc.random_mps(6, 16, 4, seed=1))) as eng:
        eng.set_gemm_mode(4)
        assert eng.small_chain_kind(100) == 0


def test_tiny_chain_micro_batched_chunks(c1_sites):
    """C1 through one micro-batched call (chunks of micro-batches run back to back under PDL):
    the same bits as one call per micro-batch."""
    N, M, D, nb = 2003, 8, 4, 100
    u, al = stream_uniforms(6, 0, N, M), alpha_stream(6, 0, N, M, 0.25)
    outs = []
    with MpsSampler(MPS(c1_sites)) as eng:
        for micro in (0, nb):
            eng.set_micro_batch(micro)
            c = np.zeros((N, M), dtype=np.int32)
            st = np.zeros(N, dtype=np.uint8)
            mg = np.zeros((N, M, D))
            if micro == 0:
                for s0 in range(0, N, nb):
                    b = min(nb, N - s0)
                    eng.run(s0, b, c[s0:s0 + b], uniforms=u[s0:s0 + b], alpha=al[s0:s0 + b], status=st[s0:s0 + b],
                            marginals=mg[s0:s0 + b])
            else:
                eng.run(0, N, c, uniforms=u, alpha=al, status=st, marginals=mg)
            outs.append((c, st, mg))
    assert all(np.array_equal(a, b) for a, b in zip(*outs))
