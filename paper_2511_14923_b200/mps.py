"""The MPS container: site tensors Gamma^[m] (chi_l x chi_r x D, complex128).

Convention: the amplitude of |d_0 .. d_{M-1}> is the ordered
product of Gamma^[m][:, :, d_m]; chi_0 = chi_M = 1.  Sites are row-orthonormal
(Gamma.reshape(chi_l, chi_r D) has orthonormal rows) so the left-to-right
chain rule samples the Born distribution exactly.

Random sites follow the reference's Haar recipe, QR of a complex Gaussian with
the diagonal phase fix (gaussian.py:387-391), on the host (numpy, seeded by
(seed, m)) or on the device (torch + cuSOLVER, for sites too large to build on
the host; BASELINE.json config 5 "generated on device from per-site seeds").
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import ValidationError


def bond_dims(M: int, chi: int, D: int) -> list[int]:
    """chi_0 .. chi_M: 1 at both ends, min(chi, D^m, D^(M-m)) inside."""
    if M < 1 or chi < 1 or D < 1:
        raise ValidationError("M, chi and D must be >= 1")
    dims = [1]
    for m in range(1, M):
        e = min(m, M - m)
        p = 1
        for _ in range(e):
            p *= D
            if p >= chi:
                break
        dims.append(min(chi, p))
    dims.append(1)
    return dims


def host_site(seed: int, m: int, chi_l: int, chi_r: int, D: int) -> np.ndarray:
    if chi_l > chi_r * D:
        raise ValidationError(f"site {m}: chi_l={chi_l} > chi_r*D={chi_r * D}: no row-orthonormal site")
    rng = np.random.default_rng([seed, m])
    Z = (rng.standard_normal((chi_r * D, chi_l)) + 1j * rng.standard_normal((chi_r * D, chi_l))) / np.sqrt(2.0)
    Q, R = np.linalg.qr(Z)
    d = np.diagonal(R)
    Q = Q * (d / np.abs(d))
    return np.ascontiguousarray(Q.conj().T.reshape(chi_l, chi_r, D))


def device_site(seed: int, m: int, chi_l: int, chi_r: int, D: int, device="cuda"):
    """Same recipe on the device; the Gaussian comes from torch's CUDA Philox keyed
    (seed, m), so values differ from :func:`host_site` but the law is identical."""
    import torch

    if chi_l > chi_r * D:
        raise ValidationError(f"site {m}: chi_l={chi_l} > chi_r*D={chi_r * D}: no row-orthonormal site")
    g = torch.Generator(device=device)
    g.manual_seed((int(seed) * 1_000_003 + int(m)) & (2**63 - 1))
    Z = torch.randn(chi_r * D, chi_l, dtype=torch.complex128, device=device, generator=g)
    Q, R = torch.linalg.qr(Z)
    del Z
    d = torch.diagonal(R)
    Q.mul_(d / d.abs())
    del R, d
    # resolve_conj: for chi_l = 1 the transpose-reshape is a view, so torch would hand back Q's memory
    # with only the lazy conjugate bit set -- the raw bytes the engine reads would be conj(Gamma)
    out = Q.conj().T.reshape(chi_l, chi_r, D).resolve_conj().contiguous()
    del Q
    if out.numel() * 16 > 2**31:  # multi-GB sites (config 5): return the QR transients to the device
        torch.cuda.empty_cache()
    return out


@dataclass(frozen=True)
class SiteShape:
    """Shape-only stand-in for a site held by another rank (mode-pipelined layout)."""

    shape: tuple
    dtype: str = "complex128"


@dataclass
class MPS:
    """Ordered site tensors (numpy arrays or CUDA torch tensors, complex128)."""

    sites: list

    def __post_init__(self):
        if not self.sites:
            raise ValidationError("an MPS needs at least one site")
        D = None
        prev = None
        for m, G in enumerate(self.sites):
            shape = tuple(G.shape)
            if len(shape) != 3:
                raise ValidationError(f"site {m}: expected (chi_l, chi_r, D), got shape {shape}")
            dt = str(G.dtype).replace("torch.", "")
            if dt not in ("complex128", "complex64"):
                raise ValidationError(f"site {m}: dtype {G.dtype} is neither complex128 nor complex64")
            if m > 0 and dt != self.dtype:
                raise ValidationError(f"site {m}: dtype {dt} differs from site 0's {self.dtype}")
            if D is None:
                D = shape[2]
            elif shape[2] != D:
                raise ValidationError(f"site {m}: D={shape[2]} differs from D={D}")
            if prev is not None and shape[0] != prev:
                raise ValidationError(f"site {m}: chi_l={shape[0]} != chi_r={prev} of site {m - 1}")
            prev = shape[1]
        if self.sites[0].shape[0] != 1:
            raise ValidationError("chi_0 must be 1")

    @property
    def dtype(self) -> str:
        """"complex128" or "complex64" (all sites share it)."""
        return str(self.sites[0].dtype).replace("torch.", "")

    def astype(self, dtype: str) -> "MPS":
        """Copy with every materialised site cast to complex64 / complex128."""
        out = []
        for G in self.sites:
            if isinstance(G, SiteShape):
                out.append(SiteShape(G.shape, dtype))
            elif hasattr(G, "detach"):
                import torch

                out.append(G.to(getattr(torch, dtype)))
            else:
                out.append(np.ascontiguousarray(G, dtype=dtype))
        return MPS(out)

    @property
    def M(self) -> int:
        return len(self.sites)

    @property
    def D(self) -> int:
        return int(self.sites[0].shape[2])

    @property
    def bond_dims(self) -> list[int]:
        return [int(G.shape[0]) for G in self.sites] + [int(self.sites[-1].shape[1])]

    @property
    def chi(self) -> int:
        return max(self.bond_dims)

    @property
    def nbytes(self) -> int:
        return sum(int(np.prod(G.shape)) * 16 for G in self.sites)

    @classmethod
    def from_vidal(cls, gammas, lambdas) -> "MPS":
        """Vidal form Gamma^[0] Lambda^[1] Gamma^[1] ... Lambda^[M-1] Gamma^[M-1] -> site tensors.

        lambdas[m] (length chi_{m+1}) is the bond between sites m and m+1; it is absorbed
        to the right of Gamma^[m] (B^[m] = Gamma^[m] diag(Lambda^[m+1]), the right-canonical
        sites of a Vidal-canonical state), which is exactly the Lambda^2-weighted marginal
        p(k) = sum_j Lambda_j^2 |E_jk|^2 of the unabsorbed chain."""
        gammas = list(gammas)
        if len(lambdas) != len(gammas) - 1:
            raise ValidationError(f"need {len(gammas) - 1} bond vectors, got {len(lambdas)}")
        sites = []
        for m, G in enumerate(gammas):
            if m < len(gammas) - 1:
                lam = lambdas[m]
                if tuple(lam.shape) != (G.shape[1],):
                    raise ValidationError(f"bond {m + 1}: Lambda has shape {tuple(lam.shape)}, site {m} has "
                                          f"chi_r={G.shape[1]}")
                if hasattr(G, "detach"):
                    G = G * lam.to(G.dtype)[None, :, None]
                else:
                    G = np.ascontiguousarray(np.asarray(G) * np.asarray(lam)[None, :, None], dtype=np.complex128)
            sites.append(G)
        return cls(sites)

    def holds(self, m: int) -> bool:
        return not isinstance(self.sites[m], SiteShape)

    @classmethod
    def random(cls, M: int, chi: int, D: int, seed: int = 0, device: str = "cpu", block=None) -> "MPS":
        """Random row-orthonormal MPS; ``block=(m_begin, m_end)`` materialises only those
        sites (the rest are :class:`SiteShape` placeholders), for a pipeline stage."""
        dims = bond_dims(M, chi, D)
        lo, hi = block if block is not None else (0, M)
        sites = []
        for m in range(M):
            if not lo <= m < hi:
                sites.append(SiteShape((dims[m], dims[m + 1], D)))
            elif device == "cpu":
                sites.append(host_site(seed, m, dims[m], dims[m + 1], D))
            else:
                sites.append(device_site(seed, m, dims[m], dims[m + 1], D, device))
        return cls(sites)
