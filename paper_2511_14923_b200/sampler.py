"""Sampling entry point for method "mps" — the reference's interface, B200 engine.

Mirrors ``gbsemu.sampler`` (pkg/src/gbsemu/sampler.py):

* :class:`MpsSamplerConfig` — frozen, validated on construction, raising
  :class:`ValidationError` (SamplerConfig, sampler.py:51-79);
* :class:`MpsSampleBatch` — samples plus provenance and timing, with
  ``n_failed`` / ``n_flagged`` accounting (SampleBatch, sampler.py:82-95);
* :func:`batch_sample` — N samples, chunked into micro-batches, failed samples
  dropped and counted (sampler.py:706-761);
* :func:`sample_one` — sample ``index`` of the configured stream
  (sampler.py:672-676);
* randomness is counter-based: the uniforms of sample i are
  ``_stream_uniforms(seed, i, M)`` (sampler.py:109-125), evaluated on the device
  bit-for-bit, so output is identical for any batch size and GPU count.

Everything heavy runs in libmps_b200.so (include/mps_sampler.h) through ctypes;
torch only allocates device memory.  There is no CPU fallback.
"""

from __future__ import annotations

import ctypes
import time
from dataclasses import dataclass, field

import numpy as np

from . import _native
from .errors import ValidationError
from .mps import MPS

METHODS = ("mps",)
DEFAULT_BATCH = 1024


@dataclass(frozen=True)
class MpsSamplerConfig:
    """Sampling parameters.

    N: samples; seed: counter-stream seed (uniforms and alpha); alpha_sigma:
    displacement alpha ~ CN(0, alpha_sigma^2) per sample and mode (None: no
    displacement unless explicit ``disp`` / ``alpha`` arrays are passed);
    batch_size: samples in flight per micro-batch (n); device: CUDA ordinal.
    """

    N: int
    seed: int = 0
    alpha_sigma: float | None = None
    batch_size: int | None = None
    device: int = 0
    method: str = "mps"

    def __post_init__(self):
        if self.method not in METHODS:
            raise ValidationError(f"unknown method {self.method!r}")
        if self.N < 0:
            raise ValidationError("N must be >= 0")
        if self.seed < 0 or self.seed >= 2**63:
            # numpy routes key lists holding ints >= 2^63 through float64, which would
            # collapse the alpha stream's block keys; the uniform stream alone keeps the quirk
            raise ValidationError("seed must lie in [0, 2^63)")
        if self.alpha_sigma is not None and not (self.alpha_sigma >= 0.0 and np.isfinite(self.alpha_sigma)):
            raise ValidationError("alpha_sigma must be a finite number >= 0")
        if self.batch_size is not None and self.batch_size < 1:
            raise ValidationError("batch_size must be >= 1")
        if self.device < 0:
            raise ValidationError("device must be >= 0")


@dataclass
class MpsSampleBatch:
    """Photon-count samples (N x M int32) plus provenance and per-sample timing."""

    M: int
    N: int
    counts: np.ndarray
    method: str
    seed: int
    D: int = 0
    chi: int = 0
    wall_time: float = 0.0
    per_sample_mean: float = 0.0
    n_failed: int = 0
    n_flagged: int = 0
    indices: np.ndarray = field(default=None, repr=False)

    @property
    def bitstrings(self) -> np.ndarray:
        """Threshold-detector view (clicks = counts > 0), the reference's sample format."""
        return (self.counts > 0).astype(np.uint8)


def _materialised(x):
    """torch tensors with a lazy conjugate / negative bit (x.conj(), views of them) store the
    UNconjugated values: the C ABI reads raw memory, so inputs are resolved to physical values."""
    if x is not None and hasattr(x, "is_conj") and (x.is_conj() or x.is_neg()):
        return x.resolve_conj().resolve_neg()
    return x


def _ptr(x) -> int | None:
    if x is None:
        return None
    if isinstance(x, int):  # a raw device pointer (e.g. a peer buffer mapped by distributed.P2PHandoff)
        return x
    if isinstance(x, np.ndarray):
        return x.ctypes.data
    if x.is_conj() or x.is_neg():  # an output view with a lazy conjugate bit would be written wrongly
        raise ValidationError("tensors with a lazy conjugate/negative bit must be resolved (resolve_conj())")
    return x.data_ptr()  # torch tensor


class MpsSampler:
    """A native context on one GPU holding (a block of) the sites of an MPS.

    ``sites_range`` = (m_begin, m_end) loads only that block (mode-pipelined stage).
    """

    def __init__(self, mps: MPS, device: int = 0, layout: int = 0, sites_range=None, borrow: bool = True,
                 sum_planes: bool = True, stream_sites: bool = False):
        """stream_sites: keep host (numpy) sites in pinned host memory and stream them into a
        2-slot HBM ring per call (MPS_SITE_HOST_STREAM), for MPS larger than the GPU."""
        _native.require_cuda()
        import torch

        self._torch = torch
        self.L = _native.lib()
        self.mps = mps
        self.M, self.D = mps.M, mps.D
        self.device = device
        self.dims = mps.bond_dims
        self.sites_range = tuple(sites_range) if sites_range else (0, mps.M)
        ctx = ctypes.c_void_p()
        dev = (ctypes.c_int * 1)(device)
        _native.check(self.L.mps_create(1, dev, layout, ctypes.byref(ctx)))
        self.ctx = ctx
        try:
            _native.check(self.L.mps_configure(self.ctx, self.M, self.D), self.ctx)
            _native.check(self.L.mps_set_sum_planes(self.ctx, int(sum_planes)), self.ctx)
            self._keep = []
            self.dtype = mps.dtype
            dcode = _native.MPS_C64 if self.dtype == "complex64" else _native.MPS_C128
            for m in range(*self.sites_range):
                if not mps.holds(m):
                    raise ValidationError(f"site {m} is in this context's range but not materialised")
                G = mps.sites[m]
                if isinstance(G, np.ndarray):
                    G = np.ascontiguousarray(G, dtype=self.dtype)
                    flags = _native.MPS_SITE_HOST_STREAM if stream_sites else _native.MPS_SITE_HOST
                    if stream_sites:
                        self._keep.append(G)  # the library streams from this buffer on every call
                else:
                    G = _materialised(G).contiguous()
                    flags = _native.MPS_SITE_DEVICE_BORROW if borrow else _native.MPS_SITE_DEVICE_COPY
                    if borrow:
                        self._keep.append(G)
                chl, chr_, D = (int(s) for s in G.shape)
                _native.check(self.L.mps_set_site(self.ctx, m, chl, chr_, D, _ptr(G), flags, dcode), self.ctx)
        except Exception:
            self.close()
            raise

    # -- low level -------------------------------------------------------------
    def set_streams(self, seed: int, alpha_sigma: float | None):
        _native.check(self.L.mps_set_streams(self.ctx, seed, -1.0 if alpha_sigma is None else float(alpha_sigma)),
                      self.ctx)

    def run(self, first_index: int, n: int, counts, *, m_begin=None, m_end=None, uniforms=None, disp=None,
            alpha=None, state_in=None, state_out=None, marginals=None, status=None, stream=None):
        """One mps_sample_range call.  Arrays are numpy (host) or torch (device);
        full-width (column = absolute mode)."""
        uniforms, disp, alpha, state_in = (_materialised(a) for a in (uniforms, disp, alpha, state_in))
        mb = self.sites_range[0] if m_begin is None else m_begin
        me = self.sites_range[1] if m_end is None else m_end
        ld_u = uniforms.shape[1] if uniforms is not None else self.M
        ld_c = counts.shape[1]
        if stream is None:  # run on torch's current stream so torch ops stay ordered with ours
            stream = self._torch.cuda.current_stream(self.device).cuda_stream
        rc = self.L.mps_sample_range(self.ctx, mb, me, first_index, n, _ptr(uniforms), ld_u, _ptr(disp), _ptr(alpha),
                                     _ptr(state_in), _ptr(state_out), _ptr(counts), ld_c, _ptr(marginals),
                                     _ptr(status), 0 if stream is None else int(stream))
        _native.check(rc, self.ctx)

    def set_forced(self, enable: bool):
        """Teacher forcing (mps_set_forced): follow the outcomes in `counts` instead of drawing."""
        _native.check(self.L.mps_set_forced(self.ctx, int(bool(enable))), self.ctx)

    def evaluate(self, config: MpsSamplerConfig, counts, start: int = 0, disp=None, alpha=None) -> dict:
        """Teacher-forced chain along given outcomes (the reference's forced path, sampler.py:394-416):
        counts (n, M) int for samples start..start+n-1 (their displacement streams).  Returns
        dict(marginals (n, M, D) normalised conditionals along the path, logp (n,) log joint
        probability, status (n,) uint8); a sample whose path leaves the support has logp = -inf."""
        torch = self._torch
        counts = np.ascontiguousarray(counts, dtype=np.int32)
        if counts.ndim != 2 or counts.shape[1] != self.M:
            raise ValidationError(f"counts must have shape (n, {self.M}), got {counts.shape}")
        n_all = counts.shape[0]
        dev = torch.device("cuda", self.device)
        c_dev = torch.from_numpy(counts).to(dev)
        status = torch.zeros(n_all, dtype=torch.uint8, device=dev)
        marg = torch.empty((n_all, self.M, self.D), dtype=torch.float64, device=dev)
        self.set_streams(config.seed, config.alpha_sigma)
        B = config.batch_size or DEFAULT_BATCH
        self.set_forced(True)
        try:
            for s0 in range(0, n_all, B):
                b = min(B, n_all - s0)
                sl = slice(s0, s0 + b)
                dsp = None if disp is None else np.ascontiguousarray(disp[sl], dtype=np.complex128)
                alp = None if alpha is None else np.ascontiguousarray(alpha[sl], dtype=np.complex128)
                self.run(start + s0, b, c_dev[sl], m_begin=0, m_end=self.M, disp=dsp, alpha=alp, marginals=marg[sl],
                         status=status[sl])
        finally:
            self.set_forced(False)
        torch.cuda.synchronize(dev)
        inside = (c_dev >= 0) & (c_dev < self.D)
        pk = torch.gather(marg, 2, c_dev.clamp(0, self.D - 1).long().unsqueeze(2)).squeeze(2)
        logp = torch.where(inside & (pk > 0), torch.log(pk.clamp_min(1e-300)), torch.full_like(pk, -np.inf)).sum(1)
        st = status.cpu().numpy()
        logp = logp.cpu().numpy()
        logp[(st & _native.MPS_STATUS_FAILED) != 0] = -np.inf
        return dict(marginals=marg.cpu().numpy(), logp=logp, status=st)

    def set_micro_batch(self, micro: int):
        """Micro-batch size for calls with host arrays (mps_set_micro_batch; 0 = off): a call over more
        samples runs as micro-batches whose host<->device copies overlap the neighbouring
        micro-batches' kernels, with one synchronisation per call.  Results do not depend on it."""
        _native.check(self.L.mps_set_micro_batch(self.ctx, int(micro)), self.ctx)

    def set_lanes(self, lanes: int):
        """Concurrent row-block chains per call (mps_set_lanes); results do not depend on it."""
        _native.check(self.L.mps_set_lanes(self.ctx, int(lanes)), self.ctx)

    def set_small_chain(self, mode):
        """Whole-chain kernels for small chains (mps_set_small_chain): False / 0 off, True / 1 whenever
        eligible, 2 automatic (default), 3 as 1 without the tiny-chain kernel.  Results are bit-identical."""
        _native.check(self.L.mps_set_small_chain(self.ctx, int(mode)), self.ctx)

    def small_chain_active(self, n: int) -> bool:
        """Whether a call of n samples over this context's sites runs a whole-chain kernel."""
        return self.small_chain_kind(n) != 0

    def small_chain_kind(self, n: int) -> int:
        """0 per-mode kernels, 1 the 16-CTA cluster kernel, 2 the tiny-chain kernel (mps_small_chain_eligible)."""
        return int(self.L.mps_small_chain_eligible(self.ctx, *self.sites_range, int(n)))

    def set_ozaki_digits(self, S: int):
        """Digits per operand of gemm mode 8 (mps_set_ozaki_digits): 7 (default), 6 or 5."""
        _native.check(self.L.mps_set_ozaki_digits(self.ctx, int(S)), self.ctx)

    def set_ozaki_site_mode(self, mode: int, block_cols: int = 0):
        """gemm mode 8 site digit planes (mps_set_ozaki_site_mode): 0 resident, 1 streamed per call in
        column blocks of `block_cols` complex columns (0: ~4 GB each) on a copy stream, 2 auto."""
        _native.check(self.L.mps_set_ozaki_site_mode(self.ctx, int(mode), int(block_cols)), self.ctx)

    def set_gemm_mode(self, mode: int):
        """K1 complex product: 3 (3M, default) or 4 (4M)."""
        _native.check(self.L.mps_set_gemm_mode(self.ctx, int(mode)), self.ctx)

    def profile(self, mask: int = 3):
        """Time kernel launches live with CUDA events (mask bit 0: K1, bit 1: K2+K3)."""
        _native.check(self.L.mps_profile(self.ctx, int(mask)), self.ctx)

    def profile_read(self) -> dict:
        buf = (ctypes.c_double * 6)()
        _native.check(self.L.mps_profile_read(self.ctx, buf), self.ctx)
        return dict(gemm_ms=buf[0], gemm_launches=int(buf[1]), gemm_flops=buf[2],
                    draw_ms=buf[3], draw_launches=int(buf[4]), draw_bytes=buf[5])

    @property
    def kernel_launches(self) -> int:
        return int(self.L.mps_kernel_launches(self.ctx)) if self.ctx else 0

    def close(self):
        if getattr(self, "ctx", None):
            self.L.mps_destroy(self.ctx)
            self.ctx = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- batch sampling ------------------------------------------------------------
    def sample(self, config: MpsSamplerConfig, start: int = 0, stop: int | None = None, disp=None, alpha=None,
               uniforms=None, return_marginals: bool = False):
        """Samples start..stop-1 of the configured stream (device-resident counts,
        one D2H at the end).  Explicit disp (N x M x D x D) / alpha (N x M) /
        uniforms (N x M) host arrays are indexed by global sample index - start."""
        torch = self._torch
        stop = config.N if stop is None else stop
        if start < 0 or stop < start:
            raise ValidationError(f"sample range [{start}, {stop}) invalid")
        n_all = stop - start
        M, D = self.M, self.D
        dev = torch.device("cuda", self.device)
        counts = torch.empty((n_all, M), dtype=torch.int32, device=dev)
        status = torch.zeros(n_all, dtype=torch.uint8, device=dev)
        marg = torch.empty((n_all, M, D), dtype=torch.float64, device=dev) if return_marginals else None
        self.set_streams(config.seed, config.alpha_sigma)
        B = config.batch_size or DEFAULT_BATCH
        for s0 in range(0, n_all, B):
            b = min(B, n_all - s0)
            sl = slice(s0, s0 + b)
            u = None if uniforms is None else np.ascontiguousarray(uniforms[sl], dtype=np.float64)
            dsp = None if disp is None else np.ascontiguousarray(disp[sl], dtype=np.complex128)
            alp = None if alpha is None else np.ascontiguousarray(alpha[sl], dtype=np.complex128)
            self.run(start + s0, b, counts[sl], m_begin=0, m_end=M, uniforms=u, disp=dsp, alpha=alp,
                     marginals=None if marg is None else marg[sl], status=status[sl])
        torch.cuda.synchronize(dev)
        out = dict(counts=counts.cpu().numpy(), status=status.cpu().numpy())
        if marg is not None:
            out["marginals"] = marg.cpu().numpy()
        return out


def batch_sample(config: MpsSamplerConfig, mps: MPS, disp=None, alpha=None, uniforms=None,
                 sampler: MpsSampler | None = None, start: int = 0) -> MpsSampleBatch:
    """Generate N samples with the B200 engine (gbsemu batch_sample, sampler.py:706-761): sample
    indices start..start+N-1 of the counter streams, so a long run resumes (or shards) by index
    range with identical output.

    Failed samples (non-finite or zero step norm) are dropped and counted;
    flagged samples (a draw within 1e-10 of a CDF boundary) are kept and counted.
    """
    if start < 0:
        raise ValidationError("start must be >= 0")
    if config.method not in METHODS:
        raise ValidationError(f"unknown method {config.method!r}")
    if not isinstance(mps, MPS):
        raise ValidationError("batch_sample needs an MPS")
    for name, arr, tail in (("disp", disp, (mps.M, mps.D, mps.D)), ("alpha", alpha, (mps.M,)),
                            ("uniforms", uniforms, (mps.M,))):
        if arr is not None and tuple(arr.shape) != (config.N,) + tail:
            raise ValidationError(f"{name} must have shape {(config.N,) + tail}, got {tuple(arr.shape)}")
    if disp is not None and alpha is not None:
        raise ValidationError("pass disp or alpha, not both")
    t0 = time.perf_counter()
    own = sampler is None
    eng = sampler or MpsSampler(mps, device=config.device)
    try:
        res = eng.sample(config, start=start, stop=start + config.N, disp=disp, alpha=alpha, uniforms=uniforms)
    finally:
        if own:
            eng.close()
    st = res["status"]
    failed = (st & _native.MPS_STATUS_FAILED) != 0
    keep = ~failed
    counts = res["counts"][keep]
    wall = time.perf_counter() - t0
    n_ok = int(keep.sum())
    return MpsSampleBatch(
        M=mps.M, N=n_ok, counts=counts, method="mps", seed=config.seed, D=mps.D, chi=mps.chi,
        wall_time=wall, per_sample_mean=wall / max(n_ok, 1), n_failed=int(config.N - n_ok),
        n_flagged=int(((st & _native.MPS_STATUS_FLAGGED) != 0)[keep].sum()),
        indices=start + np.nonzero(keep)[0],
    )


def sample_one(mps: MPS, config: MpsSamplerConfig, index: int = 0, sampler: MpsSampler | None = None) -> np.ndarray:
    """Counts of sample ``index`` of the configured stream (sampler.py:672-676)."""
    if index < 0:
        raise ValidationError("index must be >= 0")
    own = sampler is None
    eng = sampler or MpsSampler(mps, device=config.device)
    try:
        res = eng.sample(config, start=index, stop=index + 1)
    finally:
        if own:
            eng.close()
    if res["status"][0] & _native.MPS_STATUS_FAILED:
        raise ValidationError("sample failed: non-finite or zero step norm")
    return res["counts"][0]


def chain_log_probability(mps: MPS, counts, config: MpsSamplerConfig, start: int = 0, disp=None, alpha=None,
                          sampler: MpsSampler | None = None) -> np.ndarray:
    """log P(counts[b]) under the chain for samples start..start+n-1 (their displacement streams),
    evaluated on the GPU by teacher forcing (batched analogue of gbsemu's chain_joint_probability,
    sampler.py:590-601).  -inf where a path leaves the support."""
    own = sampler is None
    eng = sampler or MpsSampler(mps, device=config.device)
    try:
        return eng.evaluate(config, counts, start=start, disp=disp, alpha=alpha)["logp"]
    finally:
        if own:
            eng.close()


def chain_joint_probability(mps: MPS, counts, config: MpsSamplerConfig, index: int = 0,
                            sampler: MpsSampler | None = None) -> float:
    """Model joint probability of one fixed count string (length M) for sample `index` of the
    configured streams (gbsemu chain_joint_probability, sampler.py:590-601)."""
    counts = np.asarray(counts)
    if counts.shape != (mps.M,):
        raise ValidationError(f"counts must have length {mps.M}")
    return float(np.exp(chain_log_probability(mps, counts[None, :], config, start=index, sampler=sampler)[0]))
