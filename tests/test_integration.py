"""The gbsemu plug-in (integration/gbsemu_mps.py) applied to the reference's own
``gbsemu.sampler``: method "mps" survives SamplerConfig validation (sampler.py:64-79), dispatches
through batch_sample (sampler.py:706-723) and returns the reference's SampleBatch.

gbsemu comes from the offline install in baseline/_ref (travels with the repo snapshot) or, in the
build container, from /root/reference/pkg/src; the tests skip when neither exists.  No reference
code is copied into this repository.
"""

import importlib
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
_CANDIDATES = [ROOT / "baseline" / "_ref", Path("/root/reference/pkg/src")]


@pytest.fixture(scope="module")
def gbs():
    for p in _CANDIDATES:
        if (p / "gbsemu" / "sampler.py").exists():
            sys.path.insert(0, str(p))
            try:
                sampler = importlib.import_module("gbsemu.sampler")
                errors = importlib.import_module("gbsemu.errors")
            finally:
                sys.path.remove(str(p))
            sys.path.insert(0, str(ROOT / "integration"))
            import gbsemu_mps

            gbsemu_mps.install(sampler)
            return sampler, errors, gbsemu_mps
    pytest.skip("gbsemu (the reference package) is not installed here")


def test_unpatched_reference_rejects_mps():
    """Why the plug-in exists: gbsemu itself has no method "mps" (sampler.py:45, :65)."""
    for p in _CANDIDATES:
        if (p / "gbsemu" / "sampler.py").exists():
            src = (p / "gbsemu" / "sampler.py").read_text()
            assert 'METHODS = ("single_elision", "double_elision", "exact_reference")' in src
            return
    pytest.skip("gbsemu not available")


def test_config_validation_after_install(gbs):
    sampler, errors, _ = gbs
    cfg = sampler.SamplerConfig(N=10, method="mps", seed=3, batch_size=4, workers=2)
    assert cfg.method == "mps" and "mps" in sampler.METHODS
    with pytest.raises(errors.ValidationError):
        sampler.SamplerConfig(N=-1, method="mps")
    with pytest.raises(errors.ValidationError):
        sampler.SamplerConfig(N=1, method="mps", batch_size=0)
    with pytest.raises(errors.ValidationError):
        sampler.SamplerConfig(N=1, method="mpss")
    # the reference's own methods still validate as before
    assert sampler.SamplerConfig(N=5, method="double_elision", K=4).aux_orders == (3, 3, 2)
    with pytest.raises(errors.ValidationError):
        sampler.SamplerConfig(N=5, method="single_elision", K=1)


def test_dispatch_and_errors_without_gpu(gbs):
    """batch_sample(method="mps") reaches the C ABI through ctypes; without a GPU the library
    refuses with status 3, surfaced as gbsemu's ResourceGuardError (errors.py:8-29)."""
    sampler, errors, plug = gbs
    cfg = sampler.SamplerConfig(N=4, method="mps")
    with pytest.raises(errors.ValidationError):
        sampler.batch_sample(cfg)                   # no MpsModel in the kappa slot
    from oracle import mps_oracle as orc

    model = plug.MpsModel(orc.random_mps(3, 4, 2, seed=0), alpha_sigma=0.5)
    empty = sampler.batch_sample(sampler.SamplerConfig(N=0, method="mps"), model)
    assert isinstance(empty, sampler.SampleBatch) and empty.N == 0 and empty.bitstrings.shape == (0, 3)
    try:
        import torch

        has_gpu = torch.cuda.is_available()
    except Exception:  # pragma: no cover
        has_gpu = False
    if not has_gpu:
        with pytest.raises(errors.ResourceGuardError):
            sampler.batch_sample(cfg, model)
    # the reference's own methods still dispatch to the reference's code
    gaussian = sys.modules["gbsemu.gaussian"]
    inst, _ = gaussian.random_instance(M=4, k=2, eta=0.7, r_max=1.0, seed=1)
    ref = sampler.batch_sample(sampler.SamplerConfig(N=20, method="exact_reference", seed=2), inst=inst)
    assert ref.method == "exact_reference" and ref.bitstrings.shape == (20, 4)


@pytest.mark.gpu
@pytest.mark.parametrize("workers,batch", [(1, None), (2, 37)])
def test_mps_through_gbsemu_matches_package(gbs, workers, batch):
    """gbsemu.batch_sample(SamplerConfig(method="mps")) == this package's batch_sample, clicks = counts > 0,
    for any worker count / batch size (the reference's invariance, tests/test_sampler.py:272-285)."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    sampler, errors, plug = gbs
    from oracle import mps_oracle as orc
    from paper_2511_14923_b200 import MPS, MpsSamplerConfig, batch_sample

    sites = orc.random_mps(8, 16, 4, seed=0)
    cfg = sampler.SamplerConfig(N=500, method="mps", seed=7, workers=workers, batch_size=batch)
    out = sampler.batch_sample(cfg, plug.MpsModel(sites, alpha_sigma=0.5))
    ours = batch_sample(MpsSamplerConfig(N=500, seed=7, alpha_sigma=0.5, batch_size=100), MPS(sites))
    assert isinstance(out, sampler.SampleBatch) and out.method == "mps" and out.M == 8
    assert out.N == ours.N and out.n_failed == ours.n_failed and out.n_flagged == ours.n_flagged
    assert np.array_equal(out.bitstrings, ours.bitstrings)
    # the reference's own text format round-trips the result (sampler.py:772-795)
    import tempfile

    with tempfile.TemporaryDirectory() as d:
        sampler.save_samples_text(Path(d) / "s.txt", out)
        back = sampler.load_samples_text(Path(d) / "s.txt")
    assert np.array_equal(back.bitstrings, out.bitstrings) and back.method == "mps"
