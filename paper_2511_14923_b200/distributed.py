"""Multi-GPU layouts: one process per GPU, torch.distributed (NCCL) for the plumbing.

Two layouts (the Chicago pipeline of PAPER.md:2499-2506):

* **sample-sharded** — every rank holds the whole MPS and samples a contiguous
  index range [rank N / G, (rank+1) N / G).  Uniforms and alpha are pure
  functions of (seed, index), so the output is identical for any G.  No
  collective on the data path; counts are gathered once at the end.
* **mode-pipelined** — rank g holds a contiguous block of sites and runs them for
  micro-batch t while rank g+1 runs micro-batch t-1; the n x chi complex128
  state is the only thing handed on (NCCL send/recv over NVLink).  With T
  micro-batches and G stages there are T + G - 1 pipeline steps.

The schedule (:func:`run_pipeline`) is independent of the compute: the product
passes a stage function that calls mps_sample_range on its device; the CPU
tests pass an oracle stage function over gloo.
"""

from __future__ import annotations

import numpy as np

from .errors import ValidationError


def shard_range(N: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous balanced sample-index range of `rank` (sizes differ by at most 1)."""
    if world < 1 or not 0 <= rank < world or N < 0:
        raise ValidationError("need 0 <= rank < world and N >= 0")
    return (N * rank) // world, (N * (rank + 1)) // world


def stage_blocks(bond_dims, D: int, world: int) -> list[tuple[int, int]]:
    """Split sites 0..M-1 into `world` contiguous blocks of roughly equal GEMM flops
    (sum chi_l chi_r D), each with at least one site.  Tapered edge sites are cheap,
    so equal-count blocks would leave the first and last stages idle."""
    M = len(bond_dims) - 1
    if world < 1 or world > M:
        raise ValidationError(f"cannot split {M} sites over {world} stages")
    w = np.array([bond_dims[m] * bond_dims[m + 1] * D for m in range(M)], dtype=np.float64)
    cum = np.concatenate([[0.0], np.cumsum(w)])
    bounds = [0]
    for g in range(1, world):
        target = cum[-1] * g / world
        b = int(np.searchsorted(cum, target))
        b = min(max(b, bounds[-1] + 1), M - (world - g))
        bounds.append(b)
    bounds.append(M)
    return [(bounds[g], bounds[g + 1]) for g in range(world)]


def run_pipeline(stage_fn, n_micro: int, recv_like, send_like, rank: int, world: int, group=None):
    """Drive one pipeline stage over `n_micro` micro-batches.

    stage_fn(t, state_in) -> state_out: runs this stage's sites for micro-batch t;
    state_in is None on stage 0, state_out is ignored on the last stage.
    recv_like / send_like: callables returning an empty buffer for the incoming /
    outgoing state (double-buffered).  Receives for t+1 are posted before stage t
    computes, sends are asynchronous, so communication overlaps compute.
    """
    import torch.distributed as dist

    prev, nxt = rank - 1, rank + 1
    rbuf = [recv_like(), recv_like()] if rank > 0 else None
    sbuf = [send_like(), send_like()] if rank < world - 1 else None
    sreq = [None, None]
    rreq = None
    if rank > 0 and n_micro > 0:
        rreq = dist.irecv(_as_real(rbuf[0]), src=prev, group=group)
    for t in range(n_micro):
        x = None
        if rank > 0:
            rreq.wait()
            x = rbuf[t % 2]
            if t + 1 < n_micro:
                rreq = dist.irecv(_as_real(rbuf[(t + 1) % 2]), src=prev, group=group)
        y = stage_fn(t, x)
        if rank < world - 1:
            if sreq[t % 2] is not None:
                sreq[t % 2].wait()
            sbuf[t % 2].copy_(y)
            sreq[t % 2] = dist.isend(_as_real(sbuf[t % 2]), dst=nxt, group=group)
    for r in sreq:
        if r is not None:
            r.wait()


def _as_real(t):
    import torch

    return torch.view_as_real(t) if t.is_complex() else t


def gather_rows(local, rank: int, world: int, dst: int = 0, group=None):
    """Gather variable-length row blocks (first axis) to `dst`, in rank order."""
    import torch
    import torch.distributed as dist

    rows = torch.tensor([local.shape[0]], dtype=torch.int64, device=local.device)
    all_rows = [torch.zeros_like(rows) for _ in range(world)]
    dist.all_gather(all_rows, rows, group=group)
    mx = int(max(int(r.item()) for r in all_rows))
    pad = torch.zeros((mx,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    pad[: local.shape[0]] = local
    bufs = [torch.empty_like(pad) for _ in range(world)] if rank == dst else None
    dist.gather(pad, bufs, dst=dst, group=group)
    if rank != dst:
        return None
    return torch.cat([b[: int(r.item())] for b, r in zip(bufs, all_rows)])


def gather_columns(local, m_begin: int, M: int, rank: int, world: int, dst: int = 0, group=None):
    """Assemble per-stage column blocks (counts of the stage's modes) into N x M on `dst`."""
    import torch
    import torch.distributed as dist

    meta = torch.tensor([m_begin, local.shape[1]], dtype=torch.int64, device=local.device)
    metas = [torch.zeros_like(meta) for _ in range(world)]
    dist.all_gather(metas, meta, group=group)
    width = int(max(int(m[1].item()) for m in metas))
    pad = torch.zeros((local.shape[0], width) + tuple(local.shape[2:]), dtype=local.dtype, device=local.device)
    pad[:, : local.shape[1]] = local
    bufs = [torch.empty_like(pad) for _ in range(world)] if rank == dst else None
    dist.gather(pad, bufs, dst=dst, group=group)
    if rank != dst:
        return None
    out = torch.empty((local.shape[0], M) + tuple(local.shape[2:]), dtype=local.dtype, device=local.device)
    for b, m in zip(bufs, metas):
        mb, w = int(m[0].item()), int(m[1].item())
        out[:, mb: mb + w] = b[:, :w]
    return out
