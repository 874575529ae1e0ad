"""File formats and the CLI plumbing that need no GPU."""

import numpy as np
import pytest

from oracle import mps_oracle as orc
from paper_2511_14923_b200 import MPS, SiteShape, ValidationError
from paper_2511_14923_b200.cli import build_parser, main
from paper_2511_14923_b200.formats import (
    load_counts,
    load_mps,
    read_mps_header,
    save_clicks_text,
    save_counts,
    save_mps,
)


def test_mps_container_roundtrip(tmp_path):
    sites = orc.random_mps(6, 9, 3, seed=4)
    p = tmp_path / "a.gmps"
    save_mps(MPS(sites), p)
    M, D, dims, _ = read_mps_header(p)
    assert (M, D, dims) == (6, 3, orc.bond_dims(6, 9, 3))
    back = load_mps(p)
    for a, b in zip(sites, back.sites):
        assert np.array_equal(a, b)
    blk = load_mps(p, block=(2, 4))
    assert isinstance(blk.sites[0], SiteShape) and isinstance(blk.sites[5], SiteShape)
    assert np.array_equal(blk.sites[3], sites[3])


def test_mps_container_detects_corruption(tmp_path):
    p = tmp_path / "a.gmps"
    save_mps(MPS(orc.random_mps(4, 3, 2, seed=0)), p)
    raw = bytearray(p.read_bytes())
    raw[60] ^= 0x10
    p.write_bytes(bytes(raw))
    with pytest.raises(ValidationError):
        load_mps(p)
    p.write_bytes(bytes(raw[:-3]))
    with pytest.raises(ValidationError):
        load_mps(p)
    (tmp_path / "b.gmps").write_bytes(b"NOPE" + bytes(40))
    with pytest.raises(ValidationError):
        load_mps(tmp_path / "b.gmps")


def test_counts_roundtrip_and_checks(tmp_path):
    c = np.random.default_rng(0).integers(0, 10, size=(50, 7))
    p = tmp_path / "c.gmpc"
    save_counts(p, c, D=10, seed=3)
    back, D, seed = load_counts(p)
    assert np.array_equal(back, c) and D == 10 and seed == 3
    raw = bytearray(p.read_bytes())
    raw[40] ^= 1
    p.write_bytes(bytes(raw))
    with pytest.raises(ValidationError):
        load_counts(p)
    with pytest.raises(ValidationError):
        save_counts(p, np.full((2, 2), 10), D=10)


def test_counts_v2_provenance(tmp_path):
    """v2 counts files carry alpha_sigma and each row's sample index (failed samples dropped)."""
    from paper_2511_14923_b200.formats import load_counts_file

    c = np.random.default_rng(1).integers(0, 4, size=(5, 3))
    p = tmp_path / "c.gmpc"
    save_counts(p, c, D=4, seed=9, alpha_sigma=0.5, indices=[0, 1, 3, 4, 7])
    f = load_counts_file(p)
    assert f["version"] == 2 and f["alpha_sigma"] == 0.5 and list(f["indices"]) == [0, 1, 3, 4, 7]
    assert np.array_equal(f["counts"], c) and f["seed"] == 9
    save_counts(p, c, D=4, seed=9)
    f = load_counts_file(p)
    assert f["alpha_sigma"] is None and list(f["indices"]) == [0, 1, 2, 3, 4]
    with pytest.raises(ValidationError):
        save_counts(p, c, D=4, indices=[0, 1])


def _write_v1_counts(path, counts, D, seed):
    import struct

    payload = b"GMPC" + struct.pack("<IIQIQ", 1, counts.shape[1], counts.shape[0], D, seed) + \
        counts.astype(np.uint8).tobytes()
    path.write_bytes(payload + struct.pack("<Q", int(np.frombuffer(payload, np.uint8).sum(dtype=np.uint64))))


def test_evaluate_refuses_unknown_provenance(tmp_path, capsys):
    """A v1 counts file records neither alpha_sigma nor the row indices: `evaluate` refuses to guess
    (exit code 2) instead of scoring the rows under the wrong displacement streams."""
    from paper_2511_14923_b200.cli import main
    from paper_2511_14923_b200.formats import load_counts_file

    m = tmp_path / "m.gmps"
    save_mps(MPS.random(3, 4, 2, seed=0), m)
    p = tmp_path / "old.gmpc"
    _write_v1_counts(p, np.zeros((4, 3), dtype=np.int32), D=2, seed=1)
    assert load_counts_file(p)["alpha_sigma"] == "unknown" and load_counts(p)[2] == 1
    assert main(["evaluate", "--mps", str(m), "--counts", str(p), "--out", str(tmp_path / "l.npy")]) == 2
    assert main(["evaluate", "--mps", str(m), "--counts", str(p), "--alpha-sigma", "0.5",
                 "--out", str(tmp_path / "l.npy")]) == 2  # --start still missing
    save_counts(p, np.zeros((4, 3), dtype=np.int32), D=2, seed=1, alpha_sigma=0.5)
    assert main(["evaluate", "--mps", str(m), "--counts", str(p), "--alpha-sigma", "0.7",
                 "--out", str(tmp_path / "l.npy")]) == 2  # contradicts the file
    assert "contradicts" in capsys.readouterr().err


def test_clicks_text_matches_reference_format(tmp_path, golden):
    """counts > 0 written byte-for-byte like gbsemu's save_samples_text (sampler.py:772-778)."""
    bits = golden["text_bits"]
    counts = bits * np.random.default_rng(1).integers(1, 9, size=bits.shape)
    p = tmp_path / "s.txt"
    save_clicks_text(p, counts, seed=11)
    assert p.read_bytes() == golden["text_bytes"].tobytes()


def test_cli_gen_mps_and_argument_errors(tmp_path, capsys):
    out = tmp_path / "m.gmps"
    assert main(["gen-mps", "--modes", "5", "--chi", "4", "--dim", "3", "--seed", "2", "--out", str(out)]) == 0
    man = capsys.readouterr().out
    assert '"bond_dims"' in man
    mps = load_mps(out)
    assert mps.bond_dims == orc.bond_dims(5, 4, 3)
    assert main(["sample", "--mps", str(tmp_path / "missing.gmps"), "--samples", "3", "--out", str(tmp_path / "x")]) == 2
    with pytest.raises(SystemExit):
        build_parser().parse_args(["sample"])


def test_vidal_lambda_absorption():
    """Gamma-Lambda (Vidal) input: absorbing Lambda to the right of each Gamma gives the same
    amplitudes as the explicit contraction Gamma Lambda Gamma Lambda ... Gamma."""
    rng = np.random.default_rng(3)
    dims, D = [1, 3, 4, 3, 1], 3
    gam = [rng.standard_normal((dims[m], dims[m + 1], D)) + 1j * rng.standard_normal((dims[m], dims[m + 1], D))
           for m in range(4)]
    lam = [rng.random(dims[m + 1]) + 0.1 for m in range(3)]
    mps = MPS.from_vidal(gam, lam)
    psi = orc.full_state(mps.sites)
    for idx in [(0, 1, 2, 0), (2, 2, 1, 1), (1, 0, 0, 2)]:
        amp = np.ones((1, 1), complex)
        for m, d in enumerate(idx):
            amp = amp @ gam[m][:, :, d]
            if m < 3:
                amp = amp @ np.diag(lam[m])
        assert abs(psi[idx] - amp[0, 0]) < 1e-12
    with pytest.raises(ValidationError):
        MPS.from_vidal(gam, lam[:2])
    with pytest.raises(ValidationError):
        MPS.from_vidal(gam, [lam[0], lam[1][:2], lam[2]])
