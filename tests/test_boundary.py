"""Host-side logic and the C-ABI boundary without a GPU: the library loads and exports
every symbol include/mps_sampler.h declares; configs validate like the reference's;
status codes map onto the reference's exception hierarchy (errors.py:8-29)."""

import ctypes
import re
from pathlib import Path

import numpy as np
import pytest

from oracle import mps_oracle as orc
from paper_2511_14923_b200 import (
    MPS,
    GbsError,
    MpsSamplerConfig,
    NumericalError,
    ResourceGuardError,
    ValidationError,
    alpha_stream,
    bond_dims,
    host_site,
    stream_uniforms,
)
from paper_2511_14923_b200 import _native
from paper_2511_14923_b200.errors import raise_for_status

ROOT = Path(__file__).resolve().parents[1]


def _header_symbols():
    text = (ROOT / "include" / "mps_sampler.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    text = re.sub(r"#ifdef [A-Z_]*TRACE.*?#endif", "", text, flags=re.S)  # debug-build-only entry points
    return sorted(set(re.findall(r"\b(mps_[a-z_0-9]+)\s*\(", text)))


def test_library_exports_every_header_symbol():
    L = _native.load_library()
    syms = _header_symbols()
    assert len(syms) >= 12
    for name in syms:
        assert hasattr(L, name), name
    assert sorted(_native.EXPORTS) == syms


def test_library_refuses_without_gpu_or_bad_args():
    L = _native.load_library()
    ctx = ctypes.c_void_p()
    assert L.mps_create(2, None, 0, ctypes.byref(ctx)) == 2      # one device per context
    assert L.mps_create(1, None, 7, ctypes.byref(ctx)) == 2      # unknown layout
    assert L.mps_configure(None, 4, 3) == 2
    assert L.mps_site_gemm(None, None, None, 1, 1, 1, 1, 0) == 2
    assert L.mps_stream_uniforms(0, 0, 4, 0, None, 0) == 2
    assert L.mps_last_error(None) == b"null context"
    L.mps_destroy(None)


def test_status_mapping_mirrors_reference_exit_codes():
    for code, cls in ((1, GbsError), (2, ValidationError), (3, ResourceGuardError), (4, NumericalError)):
        with pytest.raises(cls) as ei:
            raise_for_status(code, "x")
        assert ei.value.exit_code == code
    raise_for_status(0)


def test_config_validation():
    MpsSamplerConfig(N=0)
    for bad in (dict(N=-1), dict(N=1, method="exact_reference"), dict(N=1, alpha_sigma=-1.0),
                dict(N=1, alpha_sigma=float("nan")), dict(N=1, batch_size=0), dict(N=1, seed=-3), dict(N=1, device=-1)):
        with pytest.raises(ValidationError):
            MpsSamplerConfig(**bad)
    cfg = MpsSamplerConfig(N=5)
    with pytest.raises(Exception):
        cfg.N = 6  # frozen, like SamplerConfig


def test_host_streams_equal_oracle_and_reference(golden):
    assert np.array_equal(stream_uniforms(7, 100, 300, 16), golden["uniforms_1"])
    assert np.array_equal(alpha_stream(3, 10, 77, 5, 0.5), orc.alpha_stream(3, 10, 77, 5, 0.5))


def test_bond_dims_and_sites_match_oracle():
    assert bond_dims(64, 1000, 10) == orc.bond_dims(64, 1000, 10)
    assert bond_dims(144, 4000, 10)[:5] == [1, 10, 100, 1000, 4000]
    assert np.array_equal(host_site(0, 3, 4, 4, 3), orc.random_site(0, 3, 4, 4, 3))


def test_mps_container_validation():
    sites = orc.random_mps(4, 3, 2, seed=0)
    mps = MPS(sites)
    assert mps.M == 4 and mps.D == 2 and mps.bond_dims == orc.bond_dims(4, 3, 2)
    with pytest.raises(ValidationError):
        MPS([])
    with pytest.raises(ValidationError):
        MPS([sites[0], sites[2]])  # bond mismatch
    with pytest.raises(ValidationError):
        MPS([s.real.copy() for s in sites])  # real dtype
    with pytest.raises(ValidationError):
        MPS([sites[0].astype(np.complex64)] + sites[1:])  # mixed dtypes
    with pytest.raises(ValidationError):
        MPS(sites[1:])  # chi_0 != 1


def test_product_path_does_not_import_oracle():
    pkg = ROOT / "paper_2511_14923_b200"
    for f in pkg.rglob("*.py"):
        assert "oracle" not in re.sub(r'""".*?"""|#.*', "", f.read_text(), flags=re.S), f


def test_no_cpu_fallback_without_cuda():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2511_14923_b200 import MpsSampler

    with pytest.raises(ResourceGuardError):
        MpsSampler(MPS(orc.random_mps(3, 2, 2, 0)))
