"""The small-chain persistent cluster kernel (chain_small.cuh) against the per-mode kernels.

Both paths run the same 3M DMMA k order, the same draw reduction tree and the same draw rule,
so every output bit must agree: counts, marginals, status and the handed-off state.  The
per-mode path is itself checked against the CPU oracle in test_gpu_parity.py; here the chain
kernel is also checked against the oracle directly.
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


def _both(mps, fn):
    outs = []
    for on in (False, True):
        with MpsSampler(mps) as eng:
            eng.set_small_chain(on)
            outs.append((fn(eng), eng.kernel_launches))
    return outs


def _same(a, b):
    for k in ("counts", "marginals", "status"):
        if k in a:
            assert np.array_equal(a[k], b[k]), k


@pytest.mark.parametrize("M,chi,D,n", [(8, 16, 4, 100), (16, 100, 10, 100), (16, 100, 10, 1000), (7, 7, 3, 37),
                                       (9, 40, 2, 257), (5, 128, 8, 61), (3, 1, 16, 9), (1, 1, 7, 5),
                                       (6, 64, 16, 130), (5, 128, 1, 33), (4, 9, 7, 1000)])
def test_small_chain_bit_identical_device_streams(M, chi, D, n):
    mps = MPS(orc.random_mps(M, chi, D, seed=M + chi))
    cfg = MpsSamplerConfig(N=n, seed=11, alpha_sigma=0.5, batch_size=n)
    (off, l0), (on, l1) = _both(mps, lambda e: e.sample(cfg, return_marginals=True))
    _same(off, on)
    assert l1 < l0  # one persistent launch instead of two per mode


@pytest.mark.parametrize("kind", ["alpha", "disp", "none", "uniforms"])
def test_small_chain_bit_identical_host_inputs(c2_sites, kind):
    M, D, n = 16, 10, 203
    u = stream_uniforms(4, 17, n, M)
    alpha = alpha_stream(4, 17, n, M, 0.5)
    disp = None
    if kind == "disp":
        rng = np.random.default_rng(2)
        z = rng.standard_normal((n, M, D, D)) + 1j * rng.standard_normal((n, M, D, D))
        disp = np.linalg.qr(z)[0]
    mps = MPS(c2_sites)

    def run(eng):
        if kind == "uniforms":  # host uniforms, device alpha stream
            eng.set_streams(4, 0.5)
        counts = np.zeros((n, M), np.int32)
        marg = np.zeros((n, M, D))
        status = np.zeros(n, np.uint8)
        eng.run(17, n, counts, uniforms=u, alpha=alpha if kind == "alpha" else None,
                disp=disp, marginals=marg, status=status)
        return dict(counts=counts, marginals=marg, status=status)

    (off, _), (on, _) = _both(mps, run)
    _same(off, on)
    if kind == "alpha":
        ref = orc.sample_chain(c2_sites, u, alpha=alpha, forced=on["counts"], return_marginals=True)
        assert np.abs(ref["marginals"] - on["marginals"]).max() <= 1e-10


def test_small_chain_oracle_parity_c2(c2_sites):
    n, M = 300, 16
    cfg = MpsSamplerConfig(N=n, seed=5, alpha_sigma=0.5, batch_size=n)
    with MpsSampler(MPS(c2_sites)) as eng:
        eng.set_small_chain(True)  # n = 300 is past the automatic crossover (two-plus waves of groups)
        res = eng.sample(cfg, return_marginals=True)
        assert eng.kernel_launches <= 3
    u = stream_uniforms(5, 0, n, M)
    alpha = alpha_stream(5, 0, n, M, 0.5)
    ref = orc.sample_chain(c2_sites, u, alpha=alpha, forced=res["counts"], return_marginals=True)
    assert np.abs(res["marginals"] - ref["marginals"]).max() <= 1e-10
    free = orc.sample_chain(c2_sites, u, alpha=alpha)
    flagged = (res["status"] & _native.MPS_STATUS_FLAGGED) != 0
    assert not (((res["counts"] != free["counts"]).any(1)) & ~flagged & ~free["flagged"]).any()


def test_small_chain_stage_split_and_state(c2_sites):
    """state_in / state_out through the chain kernel == the per-mode kernels, bit for bit."""
    N, M, cut = 150, 16, 6
    mps = MPS(c2_sites)
    chi_cut = mps.bond_dims[cut]
    res = []
    for on in (False, True):
        counts = torch.zeros((N, M), dtype=torch.int32, device="cuda")
        marg = torch.zeros((N, M, 10), dtype=torch.float64, device="cuda")
        status = torch.zeros(N, dtype=torch.uint8, device="cuda")
        state = torch.zeros((N, chi_cut), dtype=torch.complex128, device="cuda")
        out = torch.zeros((N, 1), dtype=torch.complex128, device="cuda")
        with MpsSampler(mps, sites_range=(0, cut), layout=1) as s0, \
                MpsSampler(mps, sites_range=(cut, M), layout=1) as s1:
            for e in (s0, s1):
                e.set_streams(9, 0.5)
                e.set_small_chain(on)
            s0.run(0, N, counts, state_out=state, marginals=marg, status=status)
            s1.run(0, N, counts, state_in=state, state_out=out, marginals=marg, status=status)
        torch.cuda.synchronize()
        res.append([x.cpu().numpy() for x in (counts, marg, status, state, out)])
    for a, b in zip(*res):
        assert np.array_equal(a, b)


def test_small_chain_forced(c2_sites):
    n, M = 120, 16
    mps = MPS(c2_sites)
    rng = np.random.default_rng(0)
    counts = rng.integers(0, 3, size=(n, M)).astype(np.int32)
    counts[5, 3] = 10  # out of range: the sample fails
    outs = []
    for on in (False, True):
        with MpsSampler(mps) as eng:
            eng.set_small_chain(on)
            outs.append(eng.evaluate(MpsSamplerConfig(N=n, seed=2, alpha_sigma=0.5, batch_size=n), counts))
    assert np.array_equal(outs[0]["marginals"], outs[1]["marginals"])
    assert np.array_equal(outs[0]["status"], outs[1]["status"])
    assert np.array_equal(outs[0]["logp"], outs[1]["logp"])
    assert outs[1]["status"][5] & _native.MPS_STATUS_FAILED


@pytest.mark.parametrize("n", [1, 37, 100])
def test_small_chain_state_out_stays_in_bounds(c2_sites, n):
    """Padding rows of the last 16-row group must not write past state_out's n rows (a view of a
    larger buffer whose tail holds a sentinel)."""
    M, cut = 16, 8
    mps = MPS(c2_sites)
    chi = mps.bond_dims[cut]
    big = torch.full((n + 32, chi), 7.0 + 3.0j, dtype=torch.complex128, device="cuda")
    counts = torch.zeros((n, M), dtype=torch.int32, device="cuda")
    status = torch.zeros(n, dtype=torch.uint8, device="cuda")
    with MpsSampler(mps, sites_range=(0, cut), layout=1) as s0:
        assert s0.small_chain_active(n)
        s0.set_streams(1, 0.5)
        s0.run(0, n, counts, state_out=big[:n], status=status)
    torch.cuda.synchronize()
    assert bool((big[n:] == 7.0 + 3.0j).all())
    assert bool((big[:n] != 7.0 + 3.0j).all())


def test_small_chain_auto_choice(c2_sites, c1_sites):
    """Automatic mode takes the cluster kernel for one wave of 16-row groups and the per-mode kernels
    once the batch is large enough for them to win, and the tiny-chain kernel for chi <= 32 at any n
    (all give the same bits)."""
    with MpsSampler(MPS(c2_sites)) as eng:
        assert eng.small_chain_active(100)
        assert not eng.small_chain_active(1024)
        eng.set_small_chain(True)
        assert eng.small_chain_active(1024)
        eng.set_small_chain(False)
        assert not eng.small_chain_active(100)
    with MpsSampler(MPS(c1_sites)) as eng:  # chi <= 32: the tiny-chain kernel, at any n
        assert eng.small_chain_kind(300) == 2 and eng.small_chain_kind(100_000) == 2
        eng.set_small_chain(3)  # without it: the cluster kernel whenever eligible
        assert eng.small_chain_kind(300) == 1 and eng.small_chain_kind(4096) == 1
        eng.set_small_chain(False)
        assert eng.small_chain_kind(300) == 0
