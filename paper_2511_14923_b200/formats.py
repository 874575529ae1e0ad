"""File formats around the sampler.

* ``.gmps`` — MPS site-tensor container.  Chicago loads its MPS from disk
   in an unspecified format; this one follows the reference's
  own table container (cumulants.py:275-305): little-endian, magic + version
  header, payload, trailing uint64 byte-sum checksum.  Layout:
  ``b"GMPS" | <I version | <I M | <I D | <I reserved | (M+1) x <I bond dims |
  M sites, each chi_l*chi_r*D complex128 ('<c16', C order) | <Q checksum``.
  Sites are read one at a time (memory-mapped), so a stage can load just its
  block, straight to the device.
* ``.gmpc`` — photon-count samples with the provenance needed to re-evaluate them:
  v2 ``b"GMPC" | <I version=2 | <I M | <Q N | <I D | <Q seed | <d alpha_sigma (NaN = no
  displacement stream) | <Q flags (bit 0: alpha_sigma recorded) | N x <Q sample index |
  N x M uint8 counts | <Q checksum``.  Row i is sample ``index[i]`` of the counter streams
  (failed samples are dropped by ``batch_sample``, so indices need not be contiguous).
  v1 files (no alpha_sigma, no indices) still load; their provenance is reported unknown.
* click text — ``counts > 0`` in the reference's own sample text format
  (sampler.py:772-778), so gbsemu's ``load_samples`` and benchmark statistics
  (benchmark.py:332-371) consume MPS samples unchanged.
"""

from __future__ import annotations

import struct
from pathlib import Path

import numpy as np

from .errors import ValidationError
from .mps import MPS, SiteShape

_MPS_MAGIC = b"GMPS"
_COUNTS_MAGIC = b"GMPC"
_VERSION = 1
_TEXT_HEADER = "# gbs-samples v1"  # sampler.py:768


def _bytesum(buf) -> int:
    return int(np.frombuffer(buf, dtype=np.uint8).sum(dtype=np.uint64))


# --------------------------------------------------------------------------- MPS


def save_mps(mps: MPS, path) -> None:
    """Write every site (numpy or torch tensors; placeholders are refused)."""
    dims = mps.bond_dims
    header = _MPS_MAGIC + struct.pack("<IIII", _VERSION, mps.M, mps.D, 0) + struct.pack(f"<{len(dims)}I", *dims)
    checksum = _bytesum(header)
    with open(path, "wb") as fh:
        fh.write(header)
        for m, G in enumerate(mps.sites):
            if isinstance(G, SiteShape):
                raise ValidationError(f"site {m} is not materialised")
            arr = G.detach().cpu().numpy() if hasattr(G, "detach") else np.asarray(G)
            data = np.ascontiguousarray(arr, dtype="<c16").tobytes()
            checksum += _bytesum(data)
            fh.write(data)
        fh.write(struct.pack("<Q", checksum & (2**64 - 1)))


def read_mps_header(path) -> tuple[int, int, list[int], int]:
    """(M, D, bond dims, payload offset) of a .gmps file."""
    with open(path, "rb") as fh:
        head = fh.read(20)
        if len(head) < 20 or head[:4] != _MPS_MAGIC:
            raise ValidationError(f"{path} is not an MPS container")
        version, M, D, _ = struct.unpack("<IIII", head[4:20])
        if version != _VERSION:
            raise ValidationError(f"unsupported MPS container version {version}")
        dims = list(struct.unpack(f"<{M + 1}I", fh.read(4 * (M + 1))))
    return M, D, dims, 20 + 4 * (M + 1)


def load_mps(path, block=None, device=None, verify: bool = True) -> MPS:
    """Load a .gmps file.  ``block=(m_begin, m_end)`` materialises only those sites
    (the rest become :class:`SiteShape`); ``device`` moves them to a CUDA device;
    ``verify`` checks the trailing byte-sum over the whole file (streamed)."""
    M, D, dims, off = read_mps_header(path)
    sizes = [dims[m] * dims[m + 1] * D * 16 for m in range(M)]
    total = off + sum(sizes) + 8
    if Path(path).stat().st_size != total:
        raise ValidationError(f"{path} has wrong length")
    if verify:
        acc = 0
        with open(path, "rb") as fh:
            remaining = total - 8
            while remaining:
                chunk = fh.read(min(remaining, 1 << 26))
                acc += _bytesum(chunk)
                remaining -= len(chunk)
            (stored,) = struct.unpack("<Q", fh.read(8))
        if (acc & (2**64 - 1)) != stored:
            raise ValidationError(f"{path} checksum mismatch")
    lo, hi = block if block is not None else (0, M)
    mm = np.memmap(path, dtype=np.uint8, mode="r")
    sites = []
    pos = off
    for m in range(M):
        shape = (dims[m], dims[m + 1], D)
        if lo <= m < hi:
            arr = np.frombuffer(mm[pos: pos + sizes[m]], dtype="<c16").reshape(shape)
            if device is not None:
                import torch

                sites.append(torch.from_numpy(np.array(arr)).to(device))
            else:
                sites.append(np.array(arr, dtype=np.complex128))
        else:
            sites.append(SiteShape(shape))
        pos += sizes[m]
    del mm
    return MPS(sites)


# --------------------------------------------------------------------------- counts


def save_counts(path, counts: np.ndarray, D: int, seed: int = 0, alpha_sigma: float | None = None,
                indices=None) -> None:
    """Write a v2 counts file; ``indices`` (default 0..N-1) are the rows' sample indices."""
    counts = np.asarray(counts)
    if counts.ndim != 2:
        raise ValidationError("counts must be N x M")
    if counts.size and (counts.min() < 0 or counts.max() >= D or D > 256):
        raise ValidationError("counts must lie in [0, D) with D <= 256")
    N, M = counts.shape
    idx = np.arange(N, dtype="<u8") if indices is None else np.asarray(indices, dtype="<u8")
    if idx.shape != (N,):
        raise ValidationError(f"indices must have shape ({N},)")
    a = float("nan") if alpha_sigma is None else float(alpha_sigma)
    payload = (_COUNTS_MAGIC + struct.pack("<IIQIQdQ", 2, M, N, D, seed, a, 1) + idx.tobytes()
               + counts.astype(np.uint8).tobytes())
    Path(path).write_bytes(payload + struct.pack("<Q", _bytesum(payload) & (2**64 - 1)))


def load_counts_file(path) -> dict:
    """A counts file, checksum verified: dict(counts N x M int32, D, seed, alpha_sigma (float,
    None for "no displacement", or the string "unknown" for v1 files), indices (N,) int64 or
    None for v1 files, version)."""
    data = Path(path).read_bytes()
    if len(data) < 40 or data[:4] != _COUNTS_MAGIC:
        raise ValidationError(f"{path} is not a counts file")
    (version,) = struct.unpack("<I", data[4:8])
    if version == 1:
        _, M, N, D, seed = struct.unpack("<IIQIQ", data[4:32])
        off, alpha, idx = 32, "unknown", None
    elif version == 2:
        if len(data) < 56:
            raise ValidationError(f"{path} has wrong length")
        _, M, N, D, seed, a, flags = struct.unpack("<IIQIQdQ", data[4:48])
        alpha = "unknown" if not flags & 1 else (None if np.isnan(a) else float(a))
        off = 48 + 8 * N
        idx = None
    else:
        raise ValidationError(f"unsupported counts file version {version}")
    end = off + N * M
    if len(data) != end + 8:
        raise ValidationError(f"{path} has wrong length")
    (checksum,) = struct.unpack("<Q", data[end:])
    if (_bytesum(data[:end]) & (2**64 - 1)) != checksum:
        raise ValidationError(f"{path} checksum mismatch")
    if version == 2:
        idx = np.frombuffer(data[48:off], dtype="<u8").astype(np.int64)
    counts = np.frombuffer(data[off:end], dtype=np.uint8).reshape(N, M).astype(np.int32)
    return dict(counts=counts, D=int(D), seed=int(seed), alpha_sigma=alpha, indices=idx, version=int(version))


def load_counts(path) -> tuple[np.ndarray, int, int]:
    """(counts N x M int32, D, seed) of a counts file, checksum verified."""
    f = load_counts_file(path)
    return f["counts"], f["D"], f["seed"]


def save_clicks_text(path, counts: np.ndarray, seed: int = 0, method: str = "mps") -> None:
    """Threshold-detector view (counts > 0) in the reference's text format
    (sampler.py:772-778, K=0 as exact_reference writes it)."""
    counts = np.asarray(counts)
    N, M = counts.shape
    lines = [f"{_TEXT_HEADER} M={M} N={N} method={method} K=0 seed={seed}"]
    lines.extend("".join("1" if c > 0 else "0" for c in row) for row in counts)
    Path(path).write_text("\n".join(lines) + "\n")
