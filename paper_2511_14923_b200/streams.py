"""Counter-based host streams (the product's host-side copy of the convention).

``stream_uniforms`` is the reference's ``_stream_uniforms`` (sampler.py:109-125):
sample i reads row i mod 64 of Philox(key=[seed, i // 64]).random((64, M)), so
any sample range is regenerable and output never depends on chunking.  The
CUDA library evaluates the same streams on the device (``mps_stream_uniforms``,
``mps_set_streams``); tests/test_gpu_parity.py checks the two agree bit-for-bit.

``alpha_stream`` draws the per-sample per-mode displacement alpha ~ CN(0, sigma^2)
from the key (seed, 2^62 + i // 64), two uniforms per mode.
"""

from __future__ import annotations

import numpy as np

STREAM_BLOCK = 64
ALPHA_BLOCK_OFFSET = 1 << 62


def _blocks(seed: int, start: int, count: int, width: int, offset: int = 0):
    for blk in range(start // STREAM_BLOCK, (start + count - 1) // STREAM_BLOCK + 1):
        gen = np.random.Generator(np.random.Philox(key=[seed & (2**64 - 1), offset + blk]))
        rows = gen.random((STREAM_BLOCK, width))
        lo = max(start, blk * STREAM_BLOCK)
        hi = min(start + count, (blk + 1) * STREAM_BLOCK)
        yield lo - start, hi - start, rows[lo - blk * STREAM_BLOCK: hi - blk * STREAM_BLOCK]


def stream_uniforms(seed: int, start: int, count: int, M: int) -> np.ndarray:
    out = np.empty((count, M))
    if count > 0:
        for a, b, rows in _blocks(seed, start, count, M):
            out[a:b] = rows
    return out


def alpha_stream(seed: int, start: int, count: int, M: int, sigma: float) -> np.ndarray:
    out = np.empty((count, M), dtype=np.complex128)
    if count > 0:
        for a, b, rows in _blocks(seed, start, count, 2 * M, ALPHA_BLOCK_OFFSET):
            rad = sigma * np.sqrt(-np.log1p(-rows[:, 0::2]))
            ph = 2.0 * np.pi * rows[:, 1::2]
            out[a:b] = rad * np.cos(ph) + 1j * (rad * np.sin(ph))
    return out
