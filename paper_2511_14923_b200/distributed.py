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
    """Drive one pipeline stage over `n_micro` micro-batches (NCCL / gloo send-recv hand-off).

    stage_fn(t, state_in, out) runs this stage's sites for micro-batch t and writes its output state
    into `out`, the send buffer of micro-batch t (state_in is None on stage 0, out is None on the
    last stage): the producing kernel fills the buffer that is sent, so there is no staging copy.
    recv_like / send_like: callables returning an empty buffer for the incoming / outgoing state
    (double-buffered).  Receives for t+1 are posted before stage t computes and sends are
    asynchronous, so communication overlaps compute; a send buffer is reused only after its send
    of micro-batch t-2 completed (for NCCL, ``wait`` orders the current stream after the send).
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
        out = None
        if rank < world - 1:
            if sreq[t % 2] is not None:
                sreq[t % 2].wait()
            out = sbuf[t % 2]
        stage_fn(t, x, out)
        if rank < world - 1:
            sreq[t % 2] = dist.isend(_as_real(out), dst=nxt, group=group)
    for r in sreq:
        if r is not None:
            r.wait()


class P2PHandoff:
    """Fused stage hand-off over peer memory (the B200-native alternative to the NCCL send/recv of
    run_pipeline).  Rank g > 0 owns two receive buffers for its input state and two "consumed"
    interprocess events; rank g < G-1 maps rank g+1's receive buffers (CUDA IPC, NVLink peer
    memory) and owns two "filled" events.  A stage's last draw kernel writes the next stage's input
    directly into the mapped buffer (state_out = the peer pointer): no collective and no staging
    copy on the data path.  GPU-side ordering uses the events; the only host traffic is one tiny
    message per micro-batch and direction on a gloo group (which event record to wait on)."""

    @classmethod
    def create(cls, rank: int, world: int, recv_bytes: int, host_group=None):
        """A P2PHandoff if EVERY rank could export and map its peer's buffers and events (CUDA IPC
        over NVLink needs peer access between the two GPUs), else None on every rank, so the caller
        falls back to the NCCL send/recv hand-off together."""
        import torch.distributed as dist

        hp = cls(rank, world, recv_bytes, host_group=host_group)  # runs the same collectives on every rank
        oks = [None] * world
        dist.all_gather_object(oks, hp.opened, group=host_group)
        if all(oks):
            return hp
        hp.close()
        return None

    def __init__(self, rank: int, world: int, recv_bytes: int, host_group=None):
        import ctypes

        import torch.distributed as dist

        from . import _native

        self.L = _native.lib()
        self.rank, self.world, self.group = rank, world, host_group
        self.recv, self.consumed, self.filled = [None, None], [None, None], [None, None]
        self.peer_recv, self.peer_consumed, self.peer_filled = [None, None], [None, None], [None, None]
        mine = {}
        H = ctypes.c_char * 64

        def new_event():
            ev, h = ctypes.c_void_p(), H()
            _native.check(self.L.mps_ipc_event_create(ctypes.byref(ev), h))
            return ev.value, bytes(h)

        self.opened = False
        try:  # export this rank's buffers / events; a failure still joins the all_gather below
            if rank > 0:
                mine["recv"], mine["consumed"] = [], []
                for b in range(2):
                    p, h = ctypes.c_void_p(), H()
                    _native.check(self.L.mps_ipc_alloc(recv_bytes, ctypes.byref(p), h))
                    self.recv[b] = p.value
                    mine["recv"].append(bytes(h))
                    self.consumed[b], hb = new_event()
                    mine["consumed"].append(hb)
            if rank < world - 1:
                mine["filled"] = []
                for b in range(2):
                    self.filled[b], hb = new_event()
                    mine["filled"].append(hb)
        except Exception as e:  # noqa: BLE001 - reported through `opened` / create()
            mine = {"error": str(e)}
        everyone = [None] * world
        dist.all_gather_object(everyone, mine, group=host_group)
        if any("error" in e for e in everyone):
            return

        def open_mem(hb):
            p = ctypes.c_void_p()
            _native.check(self.L.mps_ipc_open(H.from_buffer_copy(hb), ctypes.byref(p)))
            return p.value

        def open_event(hb):
            ev = ctypes.c_void_p()
            _native.check(self.L.mps_ipc_event_open(H.from_buffer_copy(hb), ctypes.byref(ev)))
            return ev.value

        try:
            if rank < world - 1:
                nxt = everyone[rank + 1]
                self.peer_recv = [open_mem(h) for h in nxt["recv"]]
                self.peer_consumed = [open_event(h) for h in nxt["consumed"]]
            if rank > 0:
                self.peer_filled = [open_event(h) for h in everyone[rank - 1]["filled"]]
            self.opened = True
        except Exception:
            # keep the collective schedule intact (create() agrees on the outcome with every rank)
            self.opened = False

    def close(self):
        for p in self.peer_recv:
            if p:
                self.L.mps_ipc_close(p)
        for ev in self.peer_consumed + self.peer_filled + self.consumed + self.filled:
            if ev:
                self.L.mps_event_destroy(ev)
        for p in self.recv:
            if p:
                self.L.mps_ipc_free(p)
        self.recv = self.peer_recv = [None, None]
        self.consumed = self.filled = self.peer_consumed = self.peer_filled = [None, None]


def run_pipeline_p2p(stage_fn, n_micro: int, handoff: P2PHandoff, stream: int, rank: int, world: int,
                     group=None):
    """Drive one pipeline stage with the fused peer-memory hand-off.

    stage_fn(t, state_in_ptr, state_out_ptr) enqueues this stage's sites for micro-batch t on
    `stream` (raw cudaStream_t); state_in_ptr is None on stage 0 and state_out_ptr None on the last
    stage.  Buffer b = t % 2 on both sides; the producer waits for the consumer's "consumed"
    record of micro-batch t - 2 before overwriting buffer b, the consumer for the producer's
    "filled" record of t.  Host messages (gloo, asynchronous sends) say which record to wait on;
    nothing blocks the GPU or spins in a kernel."""
    import torch
    import torch.distributed as dist

    L = handoff.L
    pending = []

    def send(dst, t):
        msg = torch.tensor([t], dtype=torch.int64)
        pending.append((dist.isend(msg, dst=dst, group=group), msg))

    def recv(src, expect):
        msg = torch.zeros(1, dtype=torch.int64)
        dist.recv(msg, src=src, group=group)
        if int(msg.item()) != expect:
            raise ValidationError(f"pipeline hand-off out of order: got {int(msg.item())}, expected {expect}")

    consumed_seen = 0
    for t in range(n_micro):
        b = t % 2
        x = out = None
        if rank > 0:
            recv(rank - 1, t)  # stage rank-1 has enqueued micro-batch t into my buffer b
            L.mps_stream_wait_event(stream, handoff.peer_filled[b])
            x = handoff.recv[b]
        if rank < world - 1:
            if t >= 2:
                recv(rank + 1, t - 2)  # the next stage has enqueued its read of buffer b (t - 2)
                consumed_seen += 1
                L.mps_stream_wait_event(stream, handoff.peer_consumed[b])
            out = handoff.peer_recv[b]
        stage_fn(t, x, out)
        if rank > 0:
            L.mps_event_record(handoff.consumed[b], stream)
            send(rank - 1, t)
        if rank < world - 1:
            L.mps_event_record(handoff.filled[b], stream)
            send(rank + 1, t)
    if rank < world - 1:  # drain the consumer's last acknowledgements
        for t in range(consumed_seen, n_micro):
            recv(rank + 1, t)
    for req, _ in pending:
        req.wait()


def _as_real(t):
    import torch

    return torch.view_as_real(t) if t.is_complex() else t


def _for_backend(t, group):
    """gloo collectives take host tensors, NCCL device tensors."""
    import torch.distributed as dist

    return t.cpu() if dist.get_backend(group) == "gloo" else t


def gather_rows(local, rank: int, world: int, dst: int = 0, group=None):
    """Gather variable-length row blocks (first axis) to `dst`, in rank order."""
    import torch
    import torch.distributed as dist

    local = _for_backend(local, group)

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

    local = _for_backend(local, group)

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


# ---------------------------------------------------------------------------------------------
# user-facing multi-GPU sampling (one process per GPU, torch.distributed initialised)
# ---------------------------------------------------------------------------------------------


def _dist_info():
    import torch.distributed as dist

    if dist.is_available() and dist.is_initialized():
        return dist.get_rank(), dist.get_world_size()
    return 0, 1


def sample_sharded(config, mps, device: int | None = None, group=None):
    """Sample-sharded batch_sample: every rank holds the whole MPS and samples the contiguous
    index block shard_range(N, rank, world); counts are gathered to rank 0 (the only
    collective, after sampling).  Returns an MpsSampleBatch on rank 0, None elsewhere.
    Output is identical to single-GPU batch_sample for any world size (counter streams)."""
    import time

    import torch

    from .sampler import MpsSampleBatch, MpsSampler
    from . import _native

    rank, world = _dist_info()
    dev = torch.cuda.current_device() if device is None else device
    a, b = shard_range(config.N, rank, world)
    t0 = time.perf_counter()
    with MpsSampler(mps, device=dev) as eng:
        res = eng.sample(config, start=a, stop=b)
    counts = torch.from_numpy(res["counts"]).to(dev)
    status = torch.from_numpy(res["status"]).to(dev)
    if world > 1:
        counts = gather_rows(counts, rank, world, group=group)
        status = gather_rows(status, rank, world, group=group)
    if rank != 0:
        return None
    counts, status = counts.cpu().numpy(), status.cpu().numpy()
    failed = (status & _native.MPS_STATUS_FAILED) != 0
    keep = ~failed
    wall = time.perf_counter() - t0
    return MpsSampleBatch(M=mps.M, N=int(keep.sum()), counts=counts[keep], method="mps", seed=config.seed, D=mps.D,
                          chi=mps.chi, wall_time=wall, per_sample_mean=wall / max(int(keep.sum()), 1),
                          n_failed=int(failed.sum()),
                          n_flagged=int(((status & _native.MPS_STATUS_FLAGGED) != 0)[keep].sum()),
                          indices=np.nonzero(keep)[0])


def sample_pipelined(config, mps_block, device: int | None = None, group=None, handoff: str = "nccl",
                     host_group=None):
    """Mode-pipelined batch_sample: rank g holds the sites of stage_blocks(...)[g] (the other
    sites may be SiteShape placeholders), micro-batches of config.batch_size samples flow
    through the ranks with the n x chi state handed on by NCCL send/recv (handoff="nccl") or
    written by the stage's last draw kernel straight into the next rank's buffer over peer memory
    (handoff="p2p", P2PHandoff; host_group: a gloo group for its per-micro-batch messages, default
    `group`); each rank's count columns are gathered to rank 0.  Returns an MpsSampleBatch on
    rank 0, None elsewhere; the counts do not depend on the hand-off."""
    import time

    import torch

    from .sampler import MpsSampleBatch, MpsSampler
    from . import _native

    rank, world = _dist_info()
    dev = torch.cuda.current_device() if device is None else device
    dims = mps_block.bond_dims
    mb, me = stage_blocks(dims, mps_block.D, world)[rank]
    n = config.batch_size or 1024
    N = config.N
    T = (N + n - 1) // n
    cdt = torch.complex64 if mps_block.dtype == "complex64" else torch.complex128
    counts = torch.zeros((T * n, mps_block.M), dtype=torch.int32, device=dev)
    status = torch.zeros(T * n, dtype=torch.uint8, device=dev)
    t0 = time.perf_counter()
    with MpsSampler(mps_block, device=dev, sites_range=(mb, me), layout=1) as eng:
        eng.set_streams(config.seed, config.alpha_sigma)

        def stage(t, x, out=None):
            # the last micro-batch may be short: pad to n rows (the padding samples are dropped);
            # the stage's last draw kernel writes the hand-off state straight into the send buffer
            eng.run(t * n, n, counts[t * n:(t + 1) * n], m_begin=mb, m_end=me, state_in=x, state_out=out,
                    status=status[t * n:(t + 1) * n])

        hp = None
        if world > 1 and handoff == "p2p":
            hp = P2PHandoff.create(rank, world, n * dims[mb] * (8 if cdt == torch.complex64 else 16),
                                   host_group=host_group if host_group is not None else group)
            if hp is None:
                import warnings

                warnings.warn("peer-memory hand-off unavailable between these GPUs: using NCCL send/recv")
        if hp is not None:
            stream = torch.cuda.current_stream(dev).cuda_stream

            def stage_p2p(t, x, out):
                eng.run(t * n, n, counts[t * n:(t + 1) * n], m_begin=mb, m_end=me, state_in=x, state_out=out,
                        status=status[t * n:(t + 1) * n], stream=stream)

            try:
                run_pipeline_p2p(stage_p2p, T, hp, stream, rank, world,
                                 group=host_group if host_group is not None else group)
                torch.cuda.synchronize(dev)
            finally:
                import torch.distributed as dist

                dist.barrier(group=host_group if host_group is not None else group)  # peers are done with my buffers
                hp.close()
        elif world > 1:
            run_pipeline(stage, T, recv_like=lambda: torch.empty((n, dims[mb]), dtype=cdt, device=dev),
                         send_like=lambda: torch.empty((n, dims[me]), dtype=cdt, device=dev), rank=rank, world=world,
                         group=group)
        else:
            for t in range(T):
                stage(t, None, None)
        torch.cuda.synchronize(dev)
    local = counts[:, mb:me].contiguous()
    if world > 1:
        allc = gather_columns(local, mb, mps_block.M, rank, world, group=group)
        import torch.distributed as dist

        # status bits OR-ed over the stages (NCCL has no bitwise reduce: MAX per bit)
        bits = _for_backend(torch.stack([status & 1, (status >> 1) & 1]).to(torch.int32), group)
        dist.all_reduce(bits, op=dist.ReduceOp.MAX, group=group)
        status = (bits[0] | (bits[1] << 1)).to(torch.uint8)
    else:
        allc = counts
    if rank != 0:
        return None
    counts_np = allc[:N].cpu().numpy()
    st = status[:N].cpu().numpy()
    failed = (st & _native.MPS_STATUS_FAILED) != 0
    keep = ~failed
    wall = time.perf_counter() - t0
    return MpsSampleBatch(M=mps_block.M, N=int(keep.sum()), counts=counts_np[keep], method="mps", seed=config.seed,
                          D=mps_block.D, chi=max(dims), wall_time=wall,
                          per_sample_mean=wall / max(int(keep.sum()), 1), n_failed=int(failed.sum()),
                          n_flagged=int(((st & _native.MPS_STATUS_FLAGGED) != 0)[keep].sum()),
                          indices=np.nonzero(keep)[0])
