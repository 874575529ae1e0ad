"""ctypes binding of libmps_b200.so (include/mps_sampler.h).

There is no fallback: if the library or a B200 is missing, :func:`lib` raises.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

from .errors import GbsError, ResourceGuardError, raise_for_status

LIB_NAME = "libmps_b200.so"
LIB_PATH = Path(__file__).resolve().parent / LIB_NAME

# every symbol include/mps_sampler.h declares (checked by tests/test_boundary.py)
EXPORTS = (
    "mps_create", "mps_configure", "mps_set_site", "mps_set_streams", "mps_sample", "mps_sample_range",
    "mps_kernel_launches", "mps_profile", "mps_profile_read", "mps_last_error", "mps_destroy",
    "mps_site_gemm", "mps_site_gemm_cfg", "mps_set_gemm_config", "mps_set_gemm_mode", "mps_set_lanes", "mps_set_micro_batch", "mps_set_small_chain", "mps_set_ozaki_digits", "mps_set_ozaki_site_mode", "mps_small_chain_eligible",
    "mps_set_sum_planes", "mps_displacement", "mps_stream_uniforms", "mps_site_gemm_c64",
    "mps_c64_state_planes", "mps_c64_site_planes", "mps_c64_gemm_planes", "mps_site_gemm_ozaki",
    "mps_ozaki_state_planes", "mps_ozaki_site_planes", "mps_ozaki_gemm_planes",
    "mps_ipc_alloc", "mps_ipc_free", "mps_ipc_open", "mps_ipc_close", "mps_ipc_event_create", "mps_ipc_event_open",
    "mps_event_record", "mps_stream_wait_event", "mps_event_destroy", "mps_set_forced",
)

MPS_SITE_HOST, MPS_SITE_DEVICE_COPY, MPS_SITE_DEVICE_BORROW, MPS_SITE_HOST_STREAM = 0, 1, 2, 3
MPS_C128, MPS_C64 = 0, 1
MPS_STATUS_FAILED, MPS_STATUS_FLAGGED = 1, 2

_lib = None

c_int, c_int64, c_uint64, c_void_p, c_double = (ctypes.c_int, ctypes.c_int64, ctypes.c_uint64,
                                                ctypes.c_void_p, ctypes.c_double)


def _declare(L):
    L.mps_create.argtypes = [c_int, ctypes.POINTER(c_int), c_int, ctypes.POINTER(c_void_p)]
    L.mps_configure.argtypes = [c_void_p, c_int, c_int]
    L.mps_set_site.argtypes = [c_void_p, c_int, c_int, c_int, c_int, c_void_p, c_int, c_int]
    L.mps_set_streams.argtypes = [c_void_p, c_uint64, c_double]
    L.mps_sample.argtypes = [c_void_p, c_int64, c_int, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                             ctypes.POINTER(c_uint64)]
    L.mps_sample_range.argtypes = [c_void_p, c_int, c_int, c_int64, c_int, c_void_p, c_int64, c_void_p, c_void_p,
                                   c_void_p, c_void_p, c_void_p, c_int64, c_void_p, c_void_p, c_uint64]
    L.mps_kernel_launches.argtypes = [c_void_p]
    L.mps_kernel_launches.restype = c_uint64
    L.mps_profile.argtypes = [c_void_p, c_int]
    L.mps_profile_read.argtypes = [c_void_p, ctypes.POINTER(c_double)]
    L.mps_last_error.argtypes = [c_void_p]
    L.mps_last_error.restype = ctypes.c_char_p
    L.mps_destroy.argtypes = [c_void_p]
    L.mps_destroy.restype = None
    L.mps_site_gemm.argtypes = [c_void_p, c_void_p, c_void_p, c_int, c_int, c_int, c_int64, c_uint64]
    L.mps_site_gemm_cfg.argtypes = [c_void_p, c_void_p, c_void_p, c_int, c_int, c_int, c_int64, c_uint64, c_int, c_int]
    L.mps_set_gemm_mode.argtypes = [c_void_p, c_int]
    L.mps_set_lanes.argtypes = [c_void_p, c_int]
    L.mps_set_micro_batch.argtypes = [c_void_p, c_int]
    L.mps_set_small_chain.argtypes = [c_void_p, c_int]
    L.mps_set_ozaki_digits.argtypes = [c_void_p, c_int]
    L.mps_set_ozaki_site_mode.argtypes = [c_void_p, c_int, c_int]
    L.mps_small_chain_eligible.argtypes = [c_void_p, c_int, c_int, c_int]
    L.mps_set_sum_planes.argtypes = [c_void_p, c_int]
    L.mps_set_forced.argtypes = [c_void_p, c_int]
    L.mps_site_gemm_c64.argtypes = [c_void_p, c_void_p, c_void_p, c_int, c_int, c_int, c_uint64]
    L.mps_site_gemm_ozaki.argtypes = [c_void_p, c_void_p, c_void_p, c_int, c_int, c_int, c_int, c_uint64]
    L.mps_ozaki_state_planes.argtypes = [c_void_p, c_int, c_int, c_int, c_void_p, c_void_p, c_int, c_int, c_uint64]
    L.mps_ozaki_site_planes.argtypes = [c_void_p, c_int, c_int, c_int, c_void_p, c_void_p, c_int, c_int, c_uint64]
    L.mps_ozaki_gemm_planes.argtypes = [c_void_p, c_int, c_void_p, c_void_p, c_int, c_void_p, c_int, c_void_p, c_int,
                                        c_int, c_int, c_int, c_uint64]
    L.mps_c64_state_planes.argtypes = [c_void_p, c_int, c_int, c_void_p, c_void_p, c_int, c_uint64]
    L.mps_c64_site_planes.argtypes = [c_void_p, c_int, c_int, c_void_p, c_void_p, c_int, c_uint64]
    L.mps_c64_gemm_planes.argtypes = [c_void_p, c_void_p, c_void_p, c_void_p, c_int, c_void_p, c_int, c_int, c_int,
                                      c_uint64]
    L.mps_set_gemm_config.argtypes = [c_void_p, c_int]
    L.mps_displacement.argtypes = [c_void_p, c_int, c_int, c_void_p, c_uint64]
    L.mps_stream_uniforms.argtypes = [c_uint64, c_int64, c_int, c_int, c_void_p, c_uint64]
    L.mps_ipc_alloc.argtypes = [c_uint64, ctypes.POINTER(c_void_p), c_void_p]
    L.mps_ipc_free.argtypes = [c_void_p]
    L.mps_ipc_open.argtypes = [c_void_p, ctypes.POINTER(c_void_p)]
    L.mps_ipc_close.argtypes = [c_void_p]
    L.mps_ipc_event_create.argtypes = [ctypes.POINTER(c_void_p), c_void_p]
    L.mps_ipc_event_open.argtypes = [c_void_p, ctypes.POINTER(c_void_p)]
    L.mps_event_record.argtypes = [c_void_p, c_uint64]
    L.mps_stream_wait_event.argtypes = [c_uint64, c_void_p]
    L.mps_event_destroy.argtypes = [c_void_p]
    for name in EXPORTS:  # everything else returns an int status (include/mps_sampler.h)
        if name not in ("mps_kernel_launches", "mps_last_error", "mps_destroy"):
            getattr(L, name).restype = c_int


def load_library(path: str | os.PathLike | None = None):
    """Load (once) and return the CDLL.  Loading needs no GPU; calls do."""
    global _lib
    if _lib is None:
        p = Path(path) if path else Path(os.environ.get("MPS_LIB", LIB_PATH))
        if not p.exists():
            raise GbsError(f"{p} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`")
        L = ctypes.CDLL(str(p))
        _declare(L)
        _lib = L
    return _lib


def lib():
    return load_library()


def check(status: int, ctx=None) -> None:
    if status:
        msg = ""
        if ctx:
            msg = (lib().mps_last_error(ctx) or b"").decode(errors="replace")
        raise_for_status(status, msg)


def require_cuda():
    import torch

    if not torch.cuda.is_available():
        raise ResourceGuardError("the MPS sampler needs a CUDA device (B200, sm_100a); none is visible")
    major, _ = torch.cuda.get_device_capability()
    if major != 10:
        raise ResourceGuardError(f"the MPS sampler is built for sm_100a (B200); device capability major={major}")
