"""gbsemu plug-in for the B200 MPS sampler: method "mps" behind gbsemu's own sampling interface.

This file is what a gbsemu maintainer adds.  It needs only numpy, ctypes and
``libmps_b200.so`` (the C ABI of include/mps_sampler.h) -- no torch, no paper_2511_14923_b200.

The reference's plug-in point is method dispatch (pkg/src/gbsemu/sampler.py):

* ``METHODS`` (sampler.py:45) gains ``"mps"``;
* ``SamplerConfig.__post_init__`` (sampler.py:64-79) validates method "mps" like
  ``exact_reference`` -- no truncation order / aux orders (``_DEFAULT_AUX``, sampler.py:48,
  has no entry for it, so the unpatched validation would raise KeyError);
* ``batch_sample(config, kappa=None, inst=None)`` (sampler.py:706-761) takes the MPS model in
  its ``kappa`` slot, the slot that carries the chain methods' precomputed table: an
  :class:`MpsModel` (sites + displacement law), and returns a ``SampleBatch``.

Conventions kept: sample i uses the counter streams (seed, i) -- ``_stream_uniforms``
(sampler.py:109-125) evaluated bit-for-bit on the GPU -- so output is identical for any
``workers`` / ``batch_size``; failed samples are dropped and counted (``n_failed``); draws within
1e-10 of a CDF boundary are counted in ``n_flagged``; ``bitstrings`` are clicks (counts > 0),
the format ``save_samples_text`` / ``benchmark`` consume.  ``workers`` > 1 runs that many engine
contexts (one per entry of ``MpsModel.devices``, round robin) on threads -- ctypes releases the
GIL -- over chunks of the index range, like the reference's process pool (sampler.py:731-751).

:func:`install` applies the three edits to an imported ``gbsemu.sampler`` module at run time
(used by tests/test_integration.py); the literal source edits are in INTEGRATION.md §2.
"""

from __future__ import annotations

import ctypes
import os
import threading
import time
from pathlib import Path

import numpy as np

_LIB = None
_LIB_LOCK = threading.Lock()
_DEFAULT_LIB = Path(__file__).resolve().parents[1] / "paper_2511_14923_b200" / "libmps_b200.so"


def mps_lib():
    """Load libmps_b200.so once ($GBS_MPS_LIB overrides the path) and declare the entry points."""
    global _LIB
    with _LIB_LOCK:
        if _LIB is None:
            L = ctypes.CDLL(os.environ.get("GBS_MPS_LIB", str(_DEFAULT_LIB)))
            vp, i32, i64, u64 = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_uint64
            L.mps_create.argtypes = [i32, ctypes.POINTER(i32), i32, ctypes.POINTER(vp)]
            L.mps_configure.argtypes = [vp, i32, i32]
            L.mps_set_site.argtypes = [vp, i32, i32, i32, i32, vp, i32, i32]
            L.mps_set_streams.argtypes = [vp, u64, ctypes.c_double]
            L.mps_sample.argtypes = [vp, i64, i32, vp, vp, vp, vp, vp, ctypes.POINTER(u64)]
            L.mps_last_error.argtypes = [vp]
            L.mps_last_error.restype = ctypes.c_char_p
            L.mps_destroy.argtypes = [vp]
            L.mps_destroy.restype = None
            _LIB = L
    return _LIB


class MpsModel:
    """What method "mps" samples: site tensors Gamma^[m] (chi_l, chi_r, D) complex128, row-orthonormal
    with chi_0 = chi_M = 1, and the per-sample per-mode displacement law
    alpha ~ CN(0, alpha_sigma^2) (None: no displacement).  Passed in batch_sample's ``kappa`` slot;
    like SubsetTable it exposes ``M``."""

    def __init__(self, sites, alpha_sigma: float | None = None, devices=(0,)):
        self.sites = [np.ascontiguousarray(G, dtype=np.complex128) for G in sites]
        if not self.sites or any(G.ndim != 3 for G in self.sites):
            raise ValueError("sites must be a non-empty list of (chi_l, chi_r, D) arrays")
        self.M = len(self.sites)
        self.D = int(self.sites[0].shape[2])
        self.alpha_sigma = alpha_sigma
        self.devices = tuple(int(d) for d in devices)


def _errors(sampler):
    from importlib import import_module

    err = import_module(sampler.__name__.rsplit(".", 1)[0] + ".errors")
    return err


def _check(rc, L, ctx, err):
    if rc:
        msg = L.mps_last_error(ctx).decode() if ctx else f"libmps_b200 status {rc}"
        cls = {2: err.ValidationError, 3: err.ResourceGuardError, 4: err.NumericalError}.get(rc, err.GbsError)
        raise cls(msg)


def mps_batch_sample(config, model: MpsModel, sampler):
    """Method "mps" of batch_sample: N samples through the B200 engine, as a gbsemu SampleBatch."""
    err = _errors(sampler)
    if not isinstance(model, MpsModel):
        raise err.ValidationError("method 'mps' needs an MpsModel in the kappa slot")
    if model.alpha_sigma is not None and not (model.alpha_sigma >= 0 and np.isfinite(model.alpha_sigma)):
        raise err.ValidationError("alpha_sigma must be a finite number >= 0")
    if not 0 <= config.seed < 2**63:
        raise err.ValidationError("seed must lie in [0, 2^63) for method 'mps'")
    L = mps_lib()
    M, N = model.M, config.N
    counts = np.empty((N, M), dtype=np.int32)
    t0 = time.perf_counter()
    nw = max(1, min(config.workers, max(N, 1)))
    chunk = max(32, -(-N // (nw * 2))) if N else 1          # two chunks per worker (sampler.py:734)
    tasks = [(s, min(s + chunk, N)) for s in range(0, N, chunk)]
    B = config.batch_size or 1024
    flagged = [0] * nw
    failures = []

    def worker(w):
        ctx = ctypes.c_void_p()
        try:
            dev = (ctypes.c_int * 1)(model.devices[w % len(model.devices)])
            _check(L.mps_create(1, dev, 0, ctypes.byref(ctx)), L, None, err)
            _check(L.mps_configure(ctx, M, model.D), L, ctx, err)
            for m, G in enumerate(model.sites):
                chl, chr_, D = G.shape
                _check(L.mps_set_site(ctx, m, chl, chr_, D, G.ctypes.data, 0, 0), L, ctx, err)
            _check(L.mps_set_streams(ctx, config.seed, -1.0 if model.alpha_sigma is None else model.alpha_sigma),
                   L, ctx, err)
            fl = ctypes.c_uint64()
            for s, e in tasks[w::nw]:
                for s0 in range(s, e, B):                   # micro-batches like _chunk_chain (sampler.py:639)
                    b = min(B, e - s0)
                    _check(L.mps_sample(ctx, s0, b, None, None, None, counts[s0:].ctypes.data, None,
                                        ctypes.byref(fl)), L, ctx, err)
                    flagged[w] += fl.value
        except BaseException as ex:  # noqa: BLE001 - re-raised in the caller
            failures.append(ex)
        finally:
            if ctx:
                L.mps_destroy(ctx)

    if N:
        threads = [threading.Thread(target=worker, args=(w,)) for w in range(nw)]
        for t in threads:
            t.start()
        for t in threads:
            t.join()
        if failures:
            raise failures[0]
    keep = (counts >= 0).all(axis=1)                       # failed sample: row of -1, dropped
    wall = time.perf_counter() - t0
    n_ok = int(keep.sum())
    return sampler.SampleBatch(
        M=M, N=n_ok, bitstrings=(counts[keep] > 0).astype(np.uint8), method="mps", K=0, seed=config.seed,
        wall_time=wall, per_sample_mean=wall / max(n_ok, 1), n_failed=int(N - n_ok), n_flagged=int(sum(flagged)),
    )


def install(sampler) -> None:
    """Apply INTEGRATION.md §2's three edits to an imported ``gbsemu.sampler`` module."""
    if "mps" in sampler.METHODS:
        return
    err = _errors(sampler)
    sampler.METHODS = tuple(sampler.METHODS) + ("mps",)
    orig_post_init = sampler.SamplerConfig.__post_init__

    def __post_init__(self):
        if self.method == "mps":  # like exact_reference: no truncation / aux orders
            if self.N < 0 or self.workers < 1:
                raise err.ValidationError("N must be >= 0 and workers >= 1")
            if self.batch_size is not None and self.batch_size < 1:
                raise err.ValidationError("batch_size must be >= 1")
            return
        orig_post_init(self)

    sampler.SamplerConfig.__post_init__ = __post_init__
    orig_batch_sample = sampler.batch_sample

    def batch_sample(config, kappa=None, inst=None):
        if config.method == "mps":
            return mps_batch_sample(config, kappa, sampler)
        return orig_batch_sample(config, kappa, inst)

    batch_sample.__doc__ = orig_batch_sample.__doc__
    sampler.batch_sample = batch_sample
    sampler.MpsModel = MpsModel
