"""bench.py — displaced-MPS sampling throughput on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c3] [--impl ours|reference]

Workload (default c3 = BASELINE.json configs[2], the single-GPU-resident config the
metric's "at 1/2/4/8 B200" is quoted on): M=64, chi=1000, D=10, complex128 sites
(~10 GB, random row-orthonormal, generated on the device from per-site seeds),
alpha ~ CN(0, 0.5), micro-batch n=1024.  A *step* is one micro-batch of n samples
through all M modes.  Multi-GPU is sample-sharded (scaling "weak"): every rank holds
a replica of the MPS and takes its own contiguous sample-index blocks; there is no
collective on the data path.  Timing: W warm-up steps, then K steps bracketed by
barrier + synchronize, CUDA events on the launch stream, max over ranks.  The 10 GB
of sites streamed per step exceed the 126 MB L2, so no explicit flush is needed.

value    — samples/s with inputs (uniforms, alpha) already resident in HBM;
e2e      — samples/s through the reference-facing call with HOST buffers: pinned
           uniforms + alpha copied in and counts copied out inside the timed region;
roofline — the dominant kernel (site_gemm, K1) against the measured FP64 DMMA peak
           (profiles/fp64_peak.json), timed live with CUDA events on its stream;
cpu_baseline — the NumPy oracle (all host cores via BLAS) on a bounded sample,
           extrapolated by per-site flops (rank 0, N=1 only).
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

CONFIGS = {
    # name: (M, chi, D, n, alpha_sigma, N_total, description)
    "c1": (8, 16, 4, 100, 0.5, 1000, "BASELINE configs[0]: M=8 chi=16 D=4 n=100 alpha~CN(0,0.25)"),
    "c2": (16, 100, 10, 100, 0.5, 10000, "BASELINE configs[1]: M=16 chi=100 D=10 n=100 alpha~CN(0,0.25)"),
    "c3": (64, 1000, 10, 1024, 0.5 ** 0.5, 100000, "BASELINE configs[2]: M=64 chi=1000 D=10 n=1024 alpha~CN(0,0.5)"),
    "c4": (144, 4000, 10, 2048, 0.5 ** 0.5, 1000000,
           "BASELINE configs[3]: M=144 chi=4000 D=10 n=2048 alpha~CN(0,0.5), mode-pipelined"),
    "c5": (64, 10000, 10, 4096, 0.5 ** 0.5, 100000,
           "BASELINE configs[4]: M=64 chi=10000 D=10 n=4096 alpha~CN(0,0.5), mode-pipelined"),
}
HBM_USABLE = 170e9  # bytes per B200 we plan to fill with sites + workspaces
LANES = {"3m": 2, "4m": 2, "ozaki": 1}  # concurrent row-block chains per micro-batch (mps_set_lanes), per K1
METRIC = "MPS samples/sec (chi,D,M stated) at 1/2/4/8 B200; % of FP64 tensor-core peak"
# Multi-rank plumbing: NCCL, one GPU per rank.  MPS_BENCH_BACKEND=gloo + MPS_BENCH_ONE_GPU=1 run the
# same N>1 code path with every rank on cuda:0 (a plumbing check on a one-GPU box: ranks never wait
# on each other inside kernels in the sample-sharded layout; its timings mean nothing).
BACKEND = os.environ.get("MPS_BENCH_BACKEND", "nccl")
ONE_GPU = os.environ.get("MPS_BENCH_ONE_GPU") == "1"
# MPS_BENCH_PROFILE_RANGE=1: bracket the timed steps with cudaProfilerStart/Stop, so
# `ncu --profile-from-start off --metrics gpu__time_duration.sum` lists exactly their launches
PROFILE_RANGE = os.environ.get("MPS_BENCH_PROFILE_RANGE") == "1"
RANK_INFO: dict = {}  # every rank's device (N > 1), printed next to `config`


def dist_barrier(local):
    import torch.distributed as dist

    if dist.is_initialized() and dist.get_world_size() > 1:
        if BACKEND == "nccl":
            dist.barrier(device_ids=[local])
        else:
            dist.barrier()


def dist_max(x, dev):
    """Max over ranks of a host float (device tensor for NCCL, host tensor for gloo)."""
    import torch
    import torch.distributed as dist

    if not (dist.is_initialized() and dist.get_world_size() > 1):
        return x
    t = torch.tensor([x], device=dev if BACKEND == "nccl" else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def fp64_peak():
    p = ROOT / "profiles" / "fp64_peak.json"
    try:
        return float(json.loads(p.read_text())["fp64_dmma_tflops"]), ("builder-measured (profiles/fp64_peak.json, register-resident DMMA loop, tools/fp64_peak.cu; MEASURED_PEAKS.json has no FP64 entry; nominal 37.2)")
    except Exception:
        return 37.2, "nominal (148 SMs x 64 FP64 FMA/clk x 2 x 1.965 GHz)"


def measured_bf16():
    for p in (ROOT / "MEASURED_PEAKS.json",):
        try:
            return float(json.loads(p.read_text())["bf16_tflops"]), "measured (MEASURED_PEAKS.json)"
        except Exception:
            pass
    return 1590.0, "fallback (B200_PROFILING.md)"


def ncu_traffic(cfg_name, n):
    """DRAM bytes per K1 launch from the committed ncu --set full capture of the CURRENT default K1
    (site_gemm3m_kernel with sum planes) at a full-chi mode (profiles/), with the algorithmic bytes
    of that same launch, or (None, None)."""
    if cfg_name != "c3" or n != 1024:
        return None, None
    p = ROOT / "profiles" / "r02_ncu_k1_site_gemm3m_c3_mode30_n1024.json"
    try:
        rep = json.loads(p.read_text())[0]
    except Exception:
        return None, None
    chi, D = 1000, 10
    # Gamma (16 chi^2 D) + its 3M sum plane Gr+Gi (8 chi^2 D) + V (16 n chi) + its sum plane (8 n chi)
    # + C written (16 n chi D)
    algo = 24.0 * chi * chi * D + 24.0 * n * chi + 16.0 * n * chi * D
    return rep["dram_bytes_total"], {"source": str(p.relative_to(ROOT)), "launch": "mode 30 (chi_l = chi_r = 1000), "
                                     "one lane, the default 3M kernel with sum planes", "kernel": rep["Kernel Name"],
                                     "algorithmic_bytes": algo, "traffic_over_algorithmic": rep["dram_bytes_total"] / algo}


def site_flops(dims, D, n):
    return [8.0 * n * dims[m] * dims[m + 1] * D + 8.0 * n * dims[m + 1] * D * D for m in range(len(dims) - 1)]


def parity_tol(args):
    """The stated parity bar of the configured K1."""
    if args.dtype == "c64":
        return 1e-4
    if args.gemm == "ozaki":
        return {7: 1e-10, 6: 1e-8}.get(args.oz_digits, 1e-6)
    return 1e-10


def parity_rel_tol(args):
    """Relative bar on the marginals above parity_rel_floor: the absolute bar, except complex64, whose
    fp32 state drifts to ~1e-3 relative over the 64 C3 modes (1e-2 relative above p = 1e-3,
    tests/test_gpu_headline.py)."""
    return 1e-2 if args.dtype == "c64" else parity_tol(args)


def parity_rel_floor(args):
    """Marginals above this floor are held to the relative bar (tests/_parity.py P_FLOOR; complex64:
    tests/test_gpu_parity.py C64_REL_FLOOR -- fp32 state rounding gives ~1e-7 / p where the einsum
    cancels); smaller ones to the absolute bar."""
    return 1e-3 if args.dtype == "c64" else 1e-12


def parity_spot_check(eng, mps, m_begin, m_end, first, n_chk, stream, sigma, uniforms=None, alpha=None,
                      state_in=None, ref_counts=None, gemm_mode=None, tol=1e-10, rel_floor=1e-12,
                      rel_tol=None):
    """Parity of the bench's own run against the oracle (the checker, never the thing timed):
    n_chk samples starting at global index `first` through sites [m_begin, m_end) of the bench's
    device-resident sites, with marginals; the oracle follows the GPU's realised path
    (teacher-forced) and also runs free on the same uniforms / alpha / input state.  Returns the
    JSON "parity" object (north_star bar: marginals within 1e-10 relative, counts identical except
    flagged near-ties).  ref_counts: the timed run's counts of those rows, which must equal these."""
    import torch

    from oracle import mps_oracle as orc
    from paper_2511_14923_b200 import alpha_stream as a_stream, stream_uniforms as u_stream

    dev = torch.device("cuda", eng.device)
    M, D = eng.M, eng.D
    t0 = time.perf_counter()
    cnt = torch.zeros((n_chk, M), dtype=torch.int32, device=dev)
    st = torch.zeros(n_chk, dtype=torch.uint8, device=dev)
    marg = torch.zeros((n_chk, M, D), dtype=torch.float64, device=dev)
    u_all = u_stream(0, first, n_chk, M) if uniforms is None else uniforms.cpu().numpy()
    a_all = a_stream(0, first, n_chk, M, sigma) if alpha is None else alpha.cpu().numpy()
    eng.run(first, n_chk, cnt, m_begin=m_begin, m_end=m_end,
            uniforms=None if uniforms is None else uniforms, alpha=None if alpha is None else alpha,
            state_in=state_in, marginals=marg, status=st, stream=stream)
    torch.cuda.synchronize(dev)
    cnt_h, st_h, marg_h = cnt.cpu().numpy(), st.cpu().numpy(), marg.cpu().numpy()
    sites = [np.asarray(mps.sites[m].resolve_conj().cpu().numpy() if isinstance(mps.sites[m], torch.Tensor)
                        else mps.sites[m], dtype=np.complex128) for m in range(m_begin, m_end)]
    cols = slice(m_begin, m_end)
    v0 = None if state_in is None else state_in.cpu().numpy().astype(np.complex128)
    forced = orc.sample_chain(sites, u_all[:, cols], alpha=a_all[:, cols], forced=cnt_h[:, cols],
                              return_marginals=True, state_in=v0)
    free = orc.sample_chain(sites, u_all[:, cols], alpha=a_all[:, cols], state_in=v0)
    pg, pc = marg_h[:, cols], forced["marginals"]
    d = np.abs(pg - pc)
    big = pc > rel_floor
    rel = float((d[big] / pc[big]).max()) if big.any() else 0.0
    flagged = (st_h & 2) != 0
    mism = (cnt_h[:, cols] != free["counts"]).any(axis=1) & ~flagged & ~free["flagged"]
    ortho = 0.0
    for m in sorted({m_begin, m_begin + 1, (m_begin + m_end) // 2, m_end - 1} & set(range(m_begin, m_end))):
        G = mps.sites[m] if isinstance(mps.sites[m], torch.Tensor) else torch.from_numpy(np.asarray(mps.sites[m])).to(dev)
        A = G.reshape(G.shape[0], -1)[:256]  # a row subset keeps the check small at chi = 10^4 (16 GB sites)
        eye = torch.eye(A.shape[0], dtype=A.dtype, device=A.device)
        ortho = max(ortho, float((A @ A.conj().T - eye).abs().max().item()))
    same = None if ref_counts is None else bool(np.array_equal(ref_counts[:, cols], cnt_h[:, cols]))
    site_tol = 1e-12 if tol <= 1e-9 else 1e-4  # complex64 sites are orthonormal to fp32 rounding (~sqrt(N) eps)
    rel_tol = tol if rel_tol is None else rel_tol
    ok = bool(d.max() <= tol and rel <= rel_tol and not mism.any() and not (st_h & 1).any() and ortho < site_tol
              and same is not False)
    return {"ok": ok, "n_checked": int(n_chk), "modes": [int(m_begin), int(m_end)], "max_abs_dp": float(d.max()),
            "max_rel_dp": rel, "tolerance": tol, "rel_tolerance": rel_tol, "rel_floor": rel_floor, "n_marginals_above_floor": int(big.sum()),
            "counts_mismatch_unflagged": int(mism.sum()), "n_flagged": int(flagged.sum()),
            "same_as_timed_run": same, "site_orthonormality_max": ortho,
            "gemm_mode": gemm_mode, "oracle": "oracle.sample_chain teacher-forced along the GPU path + free run",
            "seconds": time.perf_counter() - t0}


# ---------------------------------------------------------------------------------------------
# CPU leg (oracle; only here and in tests)
# ---------------------------------------------------------------------------------------------


def host_site_fast(rng, chi_l, chi_r, D):
    """Row-orthonormal complex128 site for the CPU leg at large chi: Cholesky-QR of a complex
    Gaussian (Gamma.reshape(chi_l, chi_r D) = L^-1 Z^H with L L^H = Z^H Z), orthonormal to ~1e-14.
    The oracle's exact QR recipe (oracle.random_site) takes ~9 s per chi = 1000 site on the host;
    the CPU leg's time does not depend on the site values, only on their shapes."""
    import scipy.linalg as sl

    Z = rng.standard_normal((chi_r * D, chi_l)) + 1j * rng.standard_normal((chi_r * D, chi_l))
    Lc = np.linalg.cholesky(Z.conj().T @ Z)
    return np.ascontiguousarray(sl.solve_triangular(Lc, Z.conj().T, lower=True).reshape(chi_l, chi_r, D))


class CpuBaseline:
    """The NumPy oracle (oracle.sample_chain: batched BLAS ZGEMM chain on all host cores) timed on
    REAL steps: each step is a micro-batch of samples through ALL M sites (no extrapolation) for the
    sample-sharded configs c1-c3.  c1/c2 use the oracle's own sites; c3's 64 sites (10 GB) are
    generated row-orthonormal by Cholesky-QR (host_site_fast).  The pipelined configs c4/c5 do not
    fit host memory: there a block of full-chi sites is timed and extrapolated by flops."""

    def __init__(self, cfg_name):
        from oracle import mps_oracle as orc

        self.orc = orc
        M, chi, D, n, sigma, _, _ = CONFIGS[cfg_name]
        self.M, self.chi, self.D, self.n, self.sigma = M, chi, D, n, sigma
        self.dims = orc.bond_dims(M, chi, D)
        try:
            from threadpoolctl import threadpool_info

            self.cores = max([i.get("num_threads", 1) for i in threadpool_info()] or [os.cpu_count() or 1])
        except Exception:
            self.cores = os.cpu_count() or 1
        t0 = time.perf_counter()
        self.full = M * chi * chi * D * 16 <= 16e9
        if self.full:
            if chi <= 128:
                self.sites, self.site_note = orc.random_mps(M, chi, D, seed=0), "the oracle's sites (seed 0)"
            else:
                rng = np.random.default_rng(0)
                self.sites = [host_site_fast(rng, self.dims[m], self.dims[m + 1], D) for m in range(M)]
                self.site_note = "row-orthonormal sites by Cholesky-QR (seed 0)"
            self.setup_s = time.perf_counter() - t0
            return
        mid = M // 2
        site_bytes = 16.0 * chi * chi * D
        self.S = 2 if site_bytes <= 2e8 else 1
        self.block = list(range(mid, mid + self.S))
        self.slice_cols = chi if site_bytes <= 1e9 else max(1, int(1e9 / (16.0 * chi * D)))
        rng = np.random.default_rng(0)
        self.sites = [(rng.standard_normal((chi, self.slice_cols, D)) + 1j * rng.standard_normal(
            (chi, self.slice_cols, D))) / np.sqrt(2.0 * chi * D) for _ in self.block]
        self.n_cpu = 256
        self.u = orc.stream_uniforms(0, 0, self.n_cpu, self.S)
        self.al = orc.alpha_stream(0, 0, self.n_cpu, self.S, sigma)
        v0 = rng.standard_normal((self.n_cpu, chi)) + 1j * rng.standard_normal((self.n_cpu, chi))
        self.v0 = v0 / np.linalg.norm(v0, axis=1, keepdims=True)
        self.setup_s = time.perf_counter() - t0

    def step(self, first, n):
        """One real step: samples first..first+n-1 through all M sites; returns seconds."""
        orc = self.orc
        u = orc.stream_uniforms(0, first, n, self.M)
        al = orc.alpha_stream(0, first, n, self.M, self.sigma)
        t0 = time.perf_counter()
        orc.sample_chain(self.sites, u, alpha=al)
        return time.perf_counter() - t0

    def size_step(self, budget_s):
        """Samples per step so one full-chain step takes about budget_s (a multiple of 16, at most
        the config's n), from a timed 16-sample step."""
        if not self.full:
            return self.n_cpu
        t16 = self.step(0, 16)
        return int(max(16, min(self.n, (budget_s / max(t16, 1e-9)) * 16 // 16 * 16)))

    def describe(self, n_step, reps):
        if n_step >= self.n:
            what = f"{reps} full steps of n = {n_step} samples through all {self.M} sites"
        else:
            what = (f"{reps} steps of {n_step} samples (of the config's n = {self.n}) through all {self.M} sites "
                    f"(real steps, no extrapolation)")
        return what + f"; {self.site_note}; oracle.sample_chain (numpy BLAS, {self.cores} threads)"

    def run(self, target_s=15.0):
        """Returns (samples/s, cores, sample description) over about target_s of CPU time."""
        orc, D = self.orc, self.D
        if self.full:
            n_step = self.size_step(target_s / 2)
            reps, t, done = 0, 0.0, 0
            while reps < 2 or (t < target_s and reps < 100):
                t += self.step(done, n_step)
                done += n_step
                reps += 1
            return done / t, self.cores, self.describe(n_step, reps)
        n_cpu = self.n_cpu
        rows = np.arange(n_cpu)
        reps, t = 0, 0.0
        while t < target_s and reps < 50:
            t0 = time.perf_counter()
            v = self.v0
            for j, G in enumerate(self.sites):  # the oracle's per-mode step (sample_chain body)
                chl, chr_, _ = G.shape
                C = (v @ G.reshape(chl, chr_ * D)).reshape(n_cpu, chr_, D)
                E = np.einsum("bjd,bkd->bjk", C, orc.displacement_matrix(self.al[:, j], D))
                p = (E.real * E.real + E.imag * E.imag).sum(axis=1)
                k, ok, _ = orc.draw(p, self.u[:, j])
                v = E[rows, :, k] / np.sqrt(p[rows, k])[:, None]
                if chr_ != self.chi:  # column slice: keep the next state at full width for the next site
                    v = np.resize(v, (n_cpu, self.chi))
            t += time.perf_counter() - t0
            reps += 1
        fl = site_flops(self.dims, D, n_cpu)
        timed = sum(8.0 * n_cpu * G.shape[0] * G.shape[1] * D + 8.0 * n_cpu * G.shape[1] * D * D for G in self.sites)
        t_all = (t / reps) * sum(fl) / timed
        what = "full sites" if self.slice_cols == self.chi else f"a {self.slice_cols}-column slice of a site"
        return (n_cpu / t_all, self.cores,
                f"{reps} reps of {n_cpu} samples through {len(self.sites)} x {what} (chi={self.chi}); per-sample "
                f"time extrapolated to all {self.M} sites by algorithmic flops")


# ---------------------------------------------------------------------------------------------
# clocks during the timed region
# ---------------------------------------------------------------------------------------------


class Clocks:
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.path = Path(f"/tmp/mps_bench_clocks_{os.getpid()}.csv")

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        self.proc.wait()
        rows = [r.split(",") for r in self.path.read_text().strip().splitlines() if r.strip()]
        sm = [float(r[1]) for r in rows if len(r) >= 9 and r[1].strip().replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if len(r) >= 9 and r[2].strip().replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows if len(r) >= 9 for i in range(4) if "Active" in r[5 + i]
                          and "Not" not in r[5 + i]})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


# ---------------------------------------------------------------------------------------------


def run_pipelined(args, rank, world, local, W, K, config, dims):
    """Mode-pipelined layout: rank g holds a contiguous,
    flops-balanced block of sites; micro-batches of n samples flow rank 0 -> G-1, the
    n x chi complex128 state handed on by NCCL send/recv (the only exchange).  A step is one
    micro-batch entering the pipeline; the timed K steps include fill and drain (K + G - 1
    pipeline ticks).  Uniforms and alpha come from the device counter streams on every
    stage (column = absolute mode), so no inputs travel between ranks."""
    import torch
    import torch.distributed as dist

    from paper_2511_14923_b200 import MPS, MpsSampler
    from paper_2511_14923_b200.distributed import P2PHandoff, run_pipeline, run_pipeline_p2p, stage_blocks

    M, chi, D, n, sigma, _, desc = CONFIGS[args.config]
    dev = torch.device("cuda", local)
    blocks = stage_blocks(dims, D, world)
    mb, me = blocks[rank]
    t_setup = time.perf_counter()
    mps = MPS.random(M, chi, D, seed=0, device=dev, block=(mb, me))
    if args.dtype == "c64":
        mps = mps.astype("complex64")
    block_bytes = sum(dims[m] * dims[m + 1] for m in range(mb, me)) * D * 16.0
    eng = MpsSampler(mps, device=local, sites_range=(mb, me), layout=1, sum_planes=block_bytes * 1.5 < HBM_USABLE)
    eng.set_lanes(args.lanes)
    eng.set_streams(0, sigma)
    torch.cuda.synchronize()
    setup_s = time.perf_counter() - t_setup
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    nsteps = W + K
    counts = torch.empty((nsteps, n, M), dtype=torch.int32, device=dev)
    status = torch.zeros((nsteps, n), dtype=torch.uint8, device=dev)
    cdt = torch.complex64 if args.dtype == "c64" else torch.complex128
    c_host = torch.empty((n, me - mb), dtype=torch.int32).pin_memory()

    def stage_for(offset, copy_out=False):
        def stage(t, x, out):
            # the stage's last draw kernel writes the hand-off state straight into the send buffer
            s_ = offset + t
            eng.run(s_ * n, n, counts[s_], m_begin=mb, m_end=me, state_in=x, state_out=out, status=status[s_],
                    stream=stream.cuda_stream)
            if copy_out:
                c_host.copy_(counts[s_, :, mb:me], non_blocking=True)
        return stage

    hp = None
    if args.handoff == "p2p" and world > 1:  # fused hand-off: the draw kernel writes into the next GPU
        host_group = dist.new_group(backend="gloo") if BACKEND == "nccl" else None
        hp = P2PHandoff.create(rank, world, n * dims[mb] * (8 if args.dtype == "c64" else 16), host_group=host_group)
        if hp is None and rank == 0:
            print("[bench] peer-memory hand-off unavailable: NCCL send/recv instead", file=sys.stderr, flush=True)

    def pipe(offset, count, copy_out=False):
        if hp is not None:
            def stage_p2p(t, x, out):
                s_ = offset + t
                eng.run(s_ * n, n, counts[s_], m_begin=mb, m_end=me, state_in=x, state_out=out, status=status[s_],
                        stream=stream.cuda_stream)
                if copy_out:
                    c_host.copy_(counts[s_, :, mb:me], non_blocking=True)

            run_pipeline_p2p(stage_p2p, count, hp, stream.cuda_stream, rank, world, group=hp.group)
            return
        run_pipeline(stage_for(offset, copy_out), count,
                     recv_like=lambda: torch.empty((n, dims[mb]), dtype=cdt, device=dev),
                     send_like=lambda: torch.empty((n, dims[me]), dtype=cdt, device=dev),
                     rank=rank, world=world)

    def barrier():
        dist_barrier(local)
        torch.cuda.synchronize()

    def max_ms(ms):
        return dist_max(ms, dev)

    pipe(0, W)
    barrier()
    clocks = Clocks(local)
    clocks.start()
    l0 = eng.kernel_launches
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    pipe(W, K)
    e1.record(stream)
    barrier()
    launches = eng.kernel_launches - l0
    ck = clocks.stop()
    ms = max_ms(e0.elapsed_time(e1))
    value = K * n / (ms / 1e3)
    # e2e: each stage also copies its count columns to pinned host memory per micro-batch
    e2, e3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e2.record(stream)
    pipe(W, K, copy_out=True)
    e3.record(stream)
    barrier()
    ms_e2e = max_ms(e2.elapsed_time(e3))
    # roofline: K1 per launch on this rank, one lane, events around each launch
    eng.set_lanes(1)
    pipe(0, min(W, 2))
    barrier()
    eng.profile(1)
    pipe(W, min(K, 3))
    barrier()
    prof = eng.profile_read()
    eng.profile(0)
    peak, peak_src = fp64_peak()
    gemm_ms_avg = prof["gemm_ms"] / max(prof["gemm_launches"], 1)
    gemm_flops_avg = prof["gemm_flops"] / max(prof["gemm_launches"], 1)
    achieved = gemm_flops_avg / (gemm_ms_avg / 1e3) / 1e12 if gemm_ms_avg > 0 else 0.0
    kernel_name = {"3m": "site_gemm3m_kernel (K1, FP64 DMMA, 3M)", "4m": "site_gemm_kernel (K1, FP64 DMMA, 4M)",
                   "ozaki": f"ozaki2_gemm_kernel (K1, fp64 emulated on INT8 tcgen05, {args.oz_digits} digits)"}[args.gemm]
    bound_note = None
    if args.gemm == "3m":
        bound_note = ("achieved counts algorithmic flops (8 per complex MAC, SURVEY.md §8d); the 3M product executes "
                      "6 on the DMMA pipe, so the executed rate is 0.75 x achieved and frac can exceed 1")
    if args.dtype == "c64":
        # tcgen05 kind::tf32 executes 3 passes (hi.hi, hi.lo, lo.hi) of the real-doubled
        # product = 24 tensor flops per complex MAC; the roofline is the dense TF32 rate,
        # half the measured dense bf16 rate (MEASURED_PEAKS.json)
        bf16, src = measured_bf16()
        achieved, peak = 3.0 * achieved, bf16 / 2.0
        peak_src = f"dense TF32 = 1/2 of {src} bf16 {bf16:.0f} TFLOP/s"
        kernel_name = "c64_gemm_kernel (K1, tcgen05 kind::tf32, 3xTF32)"
        bound_note = "achieved counts executed tensor flops (3 passes x 8 per complex MAC)"
    elif args.gemm == "ozaki":
        # S(S+1)/2 int8 digit products (diagonals i + j < S; 28 at S = 7) of the real-doubled product per complex MAC;
        # the roofline is the measured kind::i8 issue rate
        achieved, peak = args.oz_digits * (args.oz_digits + 1) / 2.0 * achieved, 4510.5
        peak_src = "profiles/r01_umma_probe.jsonl (kind::i8 M=128 N=128 issue-rate probe), TOP/s"
        kernel_name = f"ozaki2_gemm_kernel (K1, complex128 emulated on INT8 tcgen05, {args.oz_digits} digits, CTA pairs)"
        bound_note = (f"achieved counts executed int8 tensor ops ({args.oz_digits * (args.oz_digits + 1) // 2} digit "
                      "products x 8 per complex MAC)")
    step_flops = sum(site_flops(dims, D, n))
    whole_tf = K * step_flops / (ms / 1e3) / 1e12
    ok = not bool((status[W:] & 1).any().item())
    cfg = dict(config, layout="mode-pipelined", stage_blocks=blocks,
               handoff=("fused peer-memory hand-off: the stage's last draw kernel writes the n x chi state into "
                        "the next GPU's CUDA-IPC buffer, interprocess events order the stages")
               if hp is not None else "NCCL send/recv of the n x chi state",
               pipeline=f"{K} micro-batches over {world} stages = {K + world - 1} ticks (fill+drain timed)")
    line = {
        "metric": METRIC, "value": value, "unit": "samples/s", "n_gpus": world, "steps": K, "warmup": W,
        "ms_per_step": ms / K, "higher_is_better": True, "scaling": "weak" if world == 1 else "strong",
        "vs_baseline": None, "dtype": args.dtype,
        "data": "synthetic (random row-orthonormal sites from per-site seeds on each stage's device, "
                "device counter-stream uniforms and alpha)",
        "config": cfg,
        "e2e": {"value": K * n / (ms_e2e / 1e3), "unit": "samples/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": n * M * 4},
        "gpu_launches": int(launches),
        "value_l2_warm": None if ms_warm is None else world * K * n / (ms_warm / 1e3),
        "roofline": {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                     "frac": achieved / peak if peak else None, "traffic": None,
                     "kernel": "site_gemm3m_kernel (K1, FP64 DMMA, 3M), rank 0's stage", "peak_source": peak_src,
                     "per_launch": {"ms": gemm_ms_avg, "algorithmic_flops": gemm_flops_avg},
                     "whole_chain_tflops": whole_tf, "whole_chain_frac": whole_tf / (world * peak)},
        "clocks": ck, "valid_outputs": ok, "setup_s": setup_s,
    }
    if hp is not None:
        dist_barrier(local)
        hp.close()
    eng.close()
    return line


def run_stage(args, local, W, K, config, dims):
    """One stage of a G-stage mode pipeline on this GPU (configs c4/c5 exceed one B200):
    the flops-balanced site block of stage g (distributed.stage_blocks), fed a random
    normalised n x chi state per micro-batch as the upstream stage's hand-off would be.
    Stages are flops-balanced and the hand-off (n x chi complex per micro-batch) is < 0.1%
    of a stage's time, so the pipeline's steady-state throughput is
    the slowest stage's samples/s, and with T micro-batches it is that x T / (T + G - 1)."""
    import torch

    from paper_2511_14923_b200 import MPS, MpsSampler
    from paper_2511_14923_b200.distributed import stage_blocks

    M, chi, D, n, sigma, N_total, desc = CONFIGS[args.config]
    n = args.n or n
    G, g = args.stage_of, args.stage
    dev = torch.device("cuda", local)
    blocks = stage_blocks(dims, D, G)
    mb, me = blocks[g]
    t_setup = time.perf_counter()
    mps = MPS.random(M, chi, D, seed=0, device=dev, block=(mb, me))
    if args.dtype == "c64":
        mps = mps.astype("complex64")
    torch.cuda.empty_cache()
    block_bytes = sum(dims[m] * dims[m + 1] for m in range(mb, me)) * D * (8.0 if args.dtype == "c64" else 16.0)
    eng = MpsSampler(mps, device=local, sites_range=(mb, me), layout=1)
    eng.set_lanes(args.lanes)
    eng.set_gemm_mode({"3m": 3, "4m": 4, "ozaki": 8}[args.gemm])
    eng.set_ozaki_digits(args.oz_digits)
    eng.set_streams(0, sigma)
    cdt = torch.complex64 if args.dtype == "c64" else torch.complex128
    gen = torch.Generator(device=dev)
    gen.manual_seed(1234 + g)
    nst = W + K
    x = torch.randn((nst, n, dims[mb]), dtype=cdt, device=dev, generator=gen)
    x /= torch.linalg.vector_norm(x, dim=2, keepdim=True)
    counts = torch.empty((nst, n, M), dtype=torch.int32, device=dev)
    status = torch.zeros((nst, n), dtype=torch.uint8, device=dev)
    y = torch.empty((n, dims[me]), dtype=cdt, device=dev) if me < M else None
    torch.cuda.synchronize()
    setup_s = time.perf_counter() - t_setup
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)

    def step(s, copy_out=None):
        eng.run(s * n, n, counts[s], m_begin=mb, m_end=me, state_in=x[s] if mb > 0 else None, state_out=y,
                status=status[s], stream=stream.cuda_stream)
        if copy_out is not None:
            copy_out.copy_(counts[s, :, mb:me], non_blocking=True)

    for s in range(W):
        step(s)
    torch.cuda.synchronize()
    clocks = Clocks(local)
    clocks.start()
    l0 = eng.kernel_launches
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for s in range(W, W + K):
        step(s)
    e1.record(stream)
    torch.cuda.synchronize()
    launches = eng.kernel_launches - l0
    ck = clocks.stop()
    ms = e0.elapsed_time(e1)
    c_host = torch.empty((n, me - mb), dtype=torch.int32).pin_memory()
    e2, e3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e2.record(stream)
    for s in range(W, W + K):
        step(s, copy_out=c_host)
    e3.record(stream)
    torch.cuda.synchronize()
    ms_e2e = e2.elapsed_time(e3)
    eng.set_lanes(1)
    step(0)
    torch.cuda.synchronize()
    eng.profile(1)
    for s in range(W, W + min(K, 2)):
        step(s)
    torch.cuda.synchronize()
    prof = eng.profile_read()
    eng.profile(0)
    peak, peak_src = fp64_peak()
    gemm_ms_avg = prof["gemm_ms"] / max(prof["gemm_launches"], 1)
    gemm_flops_avg = prof["gemm_flops"] / max(prof["gemm_launches"], 1)
    achieved = gemm_flops_avg / (gemm_ms_avg / 1e3) / 1e12 if gemm_ms_avg > 0 else 0.0
    kernel_name = {"3m": "site_gemm3m_kernel (K1, FP64 DMMA, 3M)", "4m": "site_gemm_kernel (K1, FP64 DMMA, 4M)",
                   "ozaki": f"ozaki2_gemm_kernel (K1, fp64 emulated on INT8 tcgen05, {args.oz_digits} digits)"}[args.gemm]
    if args.dtype == "c64":
        bf16, src = measured_bf16()
        achieved, peak = 3.0 * achieved, bf16 / 2.0
        peak_src = f"dense TF32 = 1/2 of {src} bf16 {bf16:.0f} TFLOP/s"
        kernel_name = "c64_gemm_kernel (K1, tcgen05 kind::tf32, 3xTF32; achieved = executed tensor flops)"
    elif args.gemm == "ozaki":
        achieved, peak = args.oz_digits * (args.oz_digits + 1) / 2.0 * achieved, 4510.5
        peak_src = "profiles/r01_umma_probe.jsonl (kind::i8 M=128 N=128 issue-rate probe), TOP/s"
        kernel_name = (f"ozaki2_gemm_kernel (K1, INT8 tcgen05; achieved = executed int8 ops, "
                       f"{args.oz_digits * (args.oz_digits + 1) // 2} per algorithmic flop)")
    stage_flops = sum(site_flops(dims, D, n)[mb:me])
    value = K * n / (ms / 1e3)
    T = (N_total + n - 1) // n
    ok = not bool((status[W:] & 1).any().item())
    # parity of this stage's kernels at full chi: its first two sites, 16 samples of step W fed the same
    # input state, against the oracle (sites copied to the host: ~2 x 2.6 GB at C4, 2 x 16 GB at C5)
    eng.set_lanes(args.lanes)
    n_chk = min(16, n)
    parity = parity_spot_check(eng, mps, mb, min(mb + 2, me), W * n, n_chk, stream.cuda_stream, sigma,
                               state_in=x[W][:n_chk].contiguous() if mb > 0 else None,
                               ref_counts=counts[W][:n_chk].cpu().numpy(), gemm_mode=args.gemm,
                               tol=parity_tol(args), rel_floor=parity_rel_floor(args),
                               rel_tol=parity_rel_tol(args))
    ok = ok and parity["ok"]
    cfg = dict(config, layout=f"one stage of a {G}-stage mode pipeline, measured alone on one B200",
               l2="inputs larger than L2 (stage sites %.1f GB streamed per step)" % (block_bytes / 1e9),
               stage=g, stage_blocks=blocks, stage_sites=[mb, me], stage_site_bytes=block_bytes,
               state_in="random normalised n x chi_l state per micro-batch (the upstream hand-off)")
    line = {
        "metric": METRIC, "value": value, "unit": "samples/s", "n_gpus": 1, "steps": K, "warmup": W,
        "ms_per_step": ms / K, "higher_is_better": True, "scaling": "stage", "vs_baseline": None,
        "dtype": args.dtype, "data": "synthetic (random row-orthonormal sites of this stage's block, generated "
                                     "on the device from per-site seeds; device counter-stream uniforms and alpha)",
        "config": cfg,
        "e2e": {"value": K * n / (ms_e2e / 1e3), "unit": "samples/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": n * (me - mb) * 4},
        "gpu_launches": int(launches),
        "pipeline_estimate": {
            "samples_per_s": value * T / (T + G - 1), "micro_batches": T, "stages": G,
            "note": f"{G}-GPU pipeline steady state = this stage's rate (stages flops-balanced, hand-off < 0.1%), "
                    f"x T/(T+G-1) fill/drain for N={N_total}"},
        "roofline": {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                     "frac": achieved / peak if peak else None, "traffic": None, "kernel": kernel_name,
                     "peak_source": peak_src, "per_launch": {"ms": gemm_ms_avg, "algorithmic_flops": gemm_flops_avg},
                     "stage_chain_tflops": K * stage_flops / (ms / 1e3) / 1e12},
        "clocks": ck, "valid_outputs": ok, "parity": parity, "setup_s": setup_s,
    }
    eng.close()
    return line


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None,
                    help="timed steps (default: 10; c1/c2, whose steps take 0.03-0.13 ms, 20000/10000 so the "
                         "timed region spans the clock sampler's interval)")
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c3", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--lanes", type=int, default=0,
                    help="concurrent row-block chains per micro-batch (default: 2 for the DMMA K1, 1 for INT8)")
    ap.add_argument("--l2", default="auto", choices=["auto", "replicas", "flush", "warm"],
                    help="keeping the timed steps honest about L2 (126 MB): 'auto' = the sites already exceed "
                         "L2 (C3-C5), else R replicas of the sites cycled per step when R <= 16 suffice (C2), "
                         "else an L2 flush between steps timed out with per-step events (C1); 'warm' = "
                         "back-to-back steps with the sites L2-resident (reported as value_l2_warm anyway)")
    ap.add_argument("--stream-sites", action="store_true",
                    help="keep the sites in pinned host memory and stream them into HBM every step")
    ap.add_argument("--gemm", default="3m", choices=["3m", "4m", "ozaki"],
                    help="complex128 K1: 3M / 4M on the FP64 DMMA pipe, or fp64 emulated on INT8 tcgen05")
    ap.add_argument("--oz-digits", type=int, default=7, choices=[5, 6, 7],
                    help="--gemm ozaki: digits of 7 bits per operand (7: ~1e-13 of the row scales, 6: ~1e-11)")
    ap.add_argument("--dtype", default="c128", choices=["c128", "c64"],
                    help="c64: complex64 chain, K1 on tcgen05 (3xTF32), parity 1e-4")
    ap.add_argument("--layout", default="auto", choices=["auto", "sharded", "pipelined"],
                    help="auto: sample-sharded when the MPS fits one GPU, else mode-pipelined")
    ap.add_argument("--handoff", default="p2p", choices=["p2p", "nccl"],
                    help="mode-pipelined stage hand-off: fused peer-memory writes (p2p) or NCCL send/recv")
    ap.add_argument("--stage-of", type=int, default=0,
                    help="measure one stage (--stage g) of a G-stage mode pipeline alone on one GPU (c4/c5)")
    ap.add_argument("--stage", type=int, default=0)
    ap.add_argument("--n", type=int, default=0,
                    help="micro-batch size (default: the config's batch n); with --lanes L it runs as L "
                         "concurrent chains of n / L rows; per-sample results do not depend on either")
    args = ap.parse_args()
    if args.gpus < 1:
        raise SystemExit("--gpus must be >= 1")
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: a bare `bench.py --gpus N` re-executes itself under torchrun (the
        # driver's own launch for N > 1), so --gpus can never silently measure one GPU
        import socket

        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr=127.0.0.1", f"--master-port={port}", str(Path(__file__).resolve()), *sys.argv[1:]]
        print("[bench] re-executing under torchrun: " + " ".join(cmd), file=sys.stderr, flush=True)
        os.execv(sys.executable, cmd)
    args.lanes = args.lanes or LANES[args.gemm]
    W = max(args.warmup, 3)
    K = args.steps if args.steps is not None else {"c1": 20000, "c2": 10000}.get(args.config, 10)
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = 0 if ONE_GPU else int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}: launch one process per GPU")
    M, chi, D, n, sigma, N_total, desc = CONFIGS[args.config]
    if args.n and args.stage_of == 0:  # micro-batch override for the sample-sharded / pipelined runs
        n = args.n
    from paper_2511_14923_b200.mps import bond_dims

    dims = bond_dims(M, chi, D)
    config = {"workload": f"{args.config}: {desc}", "M": M, "chi": chi, "D": D, "n": n, "lanes": args.lanes,
              "gemm": args.gemm if args.gemm != "ozaki" else f"ozaki (S={args.oz_digits})",
              "sites_in": "host, streamed per step" if args.stream_sites else "HBM",
              "alpha": "CN(0,%.3g)" % (sigma * sigma), "sites": "random row-orthonormal, seed 0",
              "layout": "sample-sharded" if world > 1 else "single GPU",
              "l2": "inputs larger than L2 (sites %.2f GB streamed per step)" % (
                  sum(a * b for a, b in zip(dims[:-1], dims[1:])) * D * 16 / 1e9)}
    L2_BYTES = 126e6
    site_bytes = sum(a * b for a, b in zip(dims[:-1], dims[1:])) * D * (8 if args.dtype == "c64" else 16)
    l2_mode, n_rep = args.l2, 1
    if ONE_GPU and l2_mode == "auto":  # plumbing check with every rank on cuda:0: its timing means nothing
        l2_mode = "warm"
    if l2_mode == "auto":
        if site_bytes >= L2_BYTES or args.stream_sites:
            l2_mode = "large"
        else:
            n_rep = int(np.ceil(1.25 * L2_BYTES / site_bytes))
            l2_mode = "replicas" if n_rep <= 16 else "flush"
    if l2_mode == "replicas":
        n_rep = max(2, int(np.ceil(1.25 * L2_BYTES / site_bytes)))
    if l2_mode == "replicas":
        config["l2"] = ("inputs larger than L2: %d device copies of the sites (%.1f MB each, %.0f MB in all) used in "
                        "turn, one per step" % (n_rep, site_bytes / 1e6, n_rep * site_bytes / 1e6))
    elif l2_mode == "flush":
        config["l2"] = ("L2 flushed between timed steps (a 512 MB write on the stream); each step timed by its own "
                        "CUDA events, the flushes excluded (sites %.2f MB)" % (site_bytes / 1e6))
    elif l2_mode == "warm":
        config["l2"] = "sites L2-resident across back-to-back steps (%.2f MB; --l2 warm)" % (site_bytes / 1e6)

    if args.impl == "reference":
        # The reference ships no MPS sampler; its arm is the CPU oracle restating
        # PAPER.md:58-66, timed on the host cores (all BLAS threads), rank 0 only.  Every step is a
        # REAL micro-batch through all M sites, sized so the W + K steps take a few minutes; the
        # line's ms_per_step is the measured median step time.
        if rank != 0:
            return
        cpu = CpuBaseline(args.config)
        budget = float(os.environ.get("MPS_REF_BUDGET_S", "240"))
        n_step = cpu.size_step(budget / (W + K)) if cpu.full else cpu.n_cpu
        times, rates = [], []
        first = 0
        for i in range(W + K):
            if cpu.full:
                dt = cpu.step(first, n_step)
                first += n_step
                v = n_step / dt
            else:
                v, _, _ = cpu.run(target_s=max(1.0, budget / (W + K)))
                dt = n_step / v
            if i >= W:
                times.append(dt)
                rates.append(v)
        v = float(np.median(rates))
        sample = cpu.describe(n_step, K) if cpu.full else cpu.run(target_s=0.0)[2]
        line = {"metric": METRIC, "value": v, "unit": "samples/s", "impl": "reference", "n_gpus": world, "steps": K,
                "warmup": W, "ms_per_step": 1000.0 * float(np.median(times)), "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "c128", "data": "synthetic", "config": config,
                "step_samples": n_step, "setup_s": cpu.setup_s,
                "cpu_baseline": {"value": v, "unit": "samples/s", "cores": cpu.cores, "kind": "port", "sample": sample},
                "e2e": {"value": v, "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return

    import torch
    import torch.distributed as dist

    from paper_2511_14923_b200 import MPS, MpsSampler, alpha_stream, stream_uniforms

    site_bytes = sum(a * b for a, b in zip(dims[:-1], dims[1:])) * D * 16.0
    layout = args.layout
    if layout == "auto":
        layout = "sharded" if site_bytes * 1.5 < HBM_USABLE else "pipelined"
    if not ONE_GPU and torch.cuda.device_count() < world:
        raise SystemExit(f"{world} ranks but only {torch.cuda.device_count()} visible GPU(s)")
    torch.cuda.set_device(local)
    if args.stage_of > 0:
        if world > 1 or not 0 <= args.stage < args.stage_of:
            raise SystemExit("--stage-of runs one stage on one GPU: need world 1 and 0 <= --stage < --stage-of")
        print(json.dumps(run_stage(args, local, W, K, config, dims)), flush=True)
        return
    if world > 1:
        if BACKEND == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(BACKEND)
        # communicator evidence for the driver: every rank's device, gathered on rank 0
        me = {"rank": rank, "local_rank": local, "device": torch.cuda.get_device_name(local),
              "pci_bus_id": torch.cuda.get_device_properties(local).pci_bus_id
              if hasattr(torch.cuda.get_device_properties(local), "pci_bus_id") else None}
        ranks = [None] * world
        dist.all_gather_object(ranks, me)
        RANK_INFO.update(ranks=ranks, backend=BACKEND)  # top-level keys: `config` stays the reference arm's
        if rank == 0:
            print(f"[bench] {BACKEND} process group up: world={world}, devices "
                  + ", ".join(f"r{r['rank']}:cuda:{r['local_rank']}" for r in ranks), file=sys.stderr, flush=True)
    if layout == "pipelined":
        if site_bytes / world > HBM_USABLE:
            if rank == 0:
                print(json.dumps({"metric": METRIC, "value": None, "unit": "samples/s", "n_gpus": world,
                                  "config": config, "infeasible": "the MPS (%.0f GB) does not fit %d B200(s)"
                                  % (site_bytes / 1e9, world)}), flush=True)
            return
        line = run_pipelined(args, rank, world, local, W, K, config, dims)
        if rank == 0:
            print(json.dumps(dict(line, **RANK_INFO)), flush=True)
        if world > 1:
            dist.destroy_process_group()
        return
    dev = torch.device("cuda", local)
    t_setup = time.perf_counter()
    mps = MPS.random(M, chi, D, seed=0, device=dev) if M * chi * chi * D * 16 > 2e8 else MPS.random(M, chi, D, 0)
    if args.dtype == "c64":
        mps = mps.astype("complex64")
    if args.stream_sites:  # host-resident sites, streamed per step (PCIe) instead of resident in HBM
        mps = MPS([G.cpu().numpy() if hasattr(G, "cpu") else G for G in mps.sites])
        torch.cuda.empty_cache()
    eng = MpsSampler(mps, device=local, stream_sites=args.stream_sites)
    eng.set_lanes(args.lanes)
    eng.set_gemm_mode({"3m": 3, "4m": 4, "ozaki": 8}[args.gemm])
    eng.set_ozaki_digits(args.oz_digits)
    sc_kind = eng.small_chain_kind(n)  # whole chain in one launch: 1 cluster kernel (chi <= 128), 2 tiny (chi <= 32)
    small_chain = sc_kind != 0
    path = {0: "per-mode K1 + K2/K3 kernels", 1: "small_chain_kernel (one launch per step)",
            2: "tiny_chain_kernel (one launch per step)"}[sc_kind]
    torch.cuda.synchronize()
    setup_s = time.perf_counter() - t_setup
    stream = torch.cuda.Stream(dev)  # explicit stream: events and kernels share it
    torch.cuda.set_stream(stream)

    def block_index(step):  # global first sample index of this rank's micro-batch
        return (step * world + rank) * n

    # resident inputs: uniforms + alpha for every step, in HBM before timing
    nsteps = W + K
    u_dev = [torch.from_numpy(stream_uniforms(0, block_index(s), n, M)).to(dev) for s in range(nsteps)]
    a_dev = [torch.from_numpy(alpha_stream(0, block_index(s), n, M, sigma)).to(dev) for s in range(nsteps)]
    counts = torch.empty((nsteps, n, M), dtype=torch.int32, device=dev)
    status = torch.zeros((nsteps, n), dtype=torch.uint8, device=dev)

    def step(s, e=None):
        (e or eng).run(block_index(s), n, counts[s], uniforms=u_dev[s], alpha=a_dev[s], status=status[s],
                       stream=stream.cuda_stream)

    def barrier():
        dist_barrier(local)
        torch.cuda.synchronize()

    # L2 policy of the timed region (--l2): replicas = extra contexts, each with its own device copy
    # of the sites (and of their chain / sum-plane layouts), used in turn, one per step
    engs = [eng]
    if l2_mode == "replicas":
        for _ in range(n_rep - 1):
            e = MpsSampler(mps, device=local, borrow=False)
            e.set_lanes(args.lanes)
            e.set_gemm_mode({"3m": 3, "4m": 4, "ozaki": 8}[args.gemm])
            e.set_ozaki_digits(args.oz_digits)
            engs.append(e)
    flush_buf = torch.empty(512 << 20, dtype=torch.uint8, device=dev) if l2_mode == "flush" else None

    for s in range(W):
        for e in engs:
            step(s, e)
    barrier()
    clocks = Clocks(local)
    clocks.start()
    l0 = sum(e.kernel_launches for e in engs)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    if PROFILE_RANGE:  # ncu --profile-from-start off sees exactly the timed steps
        torch.cuda.profiler.start()
    if l2_mode == "flush":
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
        for i, s in enumerate(range(W, W + K)):
            flush_buf.fill_(i & 0xFF)
            evs[i][0].record(stream)
            step(s)
            evs[i][1].record(stream)
    else:
        e0.record(stream)
        for s in range(W, W + K):
            step(s, engs[s % len(engs)])
        e1.record(stream)
    barrier()
    if PROFILE_RANGE:
        torch.cuda.profiler.stop()
    launches = sum(e.kernel_launches for e in engs) - l0
    ck = clocks.stop()
    ms_main = sum(a.elapsed_time(b) for a, b in evs) if l2_mode == "flush" else e0.elapsed_time(e1)
    ms_warm = None
    if l2_mode in ("replicas", "flush"):  # the same K steps back to back on one context, sites L2-resident
        w0, w1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        barrier()
        w0.record(stream)
        for s in range(W, W + K):
            step(s)
        w1.record(stream)
        barrier()
        ms_warm = dist_max(w0.elapsed_time(w1), dev)
    for e in engs[1:]:
        e.close()
    del flush_buf
    # Instrumented repeat of the same K steps: CUDA events around every K1 launch on its
    # stream (the roofline kernel), then around every K2+K3 launch.  Kept out of the
    # clean timed region because events between launches defeat programmatic
    # dependent launch (the next kernel's prologue overlapping this one's tail).
    eng.set_lanes(1)  # per-launch K1 duration of the kernel alone (no concurrent lane)
    for s in range(W):  # warm the one-lane shapes (autotune) outside the instrumented steps
        step(s)
    barrier()
    eng.profile(1)
    ei0, ei1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ei0.record(stream)
    for s in range(W, W + K):
        step(s)
    ei1.record(stream)
    barrier()
    prof = eng.profile_read()
    ms_instr = ei0.elapsed_time(ei1)
    eng.profile(2)
    for s in range(W, W + K):
        step(s)
    barrier()
    prof_draw = eng.profile_read()
    prof.update({k: v for k, v in prof_draw.items() if k.startswith("draw")})
    eng.profile(0)
    eng.set_lanes(args.lanes)
    ms = dist_max(ms_main, dev)
    value = world * K * n / (ms / 1e3)

    # e2e: host (pinned) uniforms + alpha in, counts + status out, through the same C ABI call, every
    # step's H2D and D2H inside the timed region.  The K steps are ONE call over K n samples with
    # micro-batch n (mps_set_micro_batch): each micro-batch's inputs go up and its counts come down on
    # the copy engines while the neighbouring micro-batches compute, one host synchronisation per call.
    e2e_first = (rank * (W + K)) * n  # this rank's contiguous index block for the e2e run

    def host_block(first, count):
        u = torch.from_numpy(stream_uniforms(0, first, count, M)).pin_memory()
        a = torch.from_numpy(alpha_stream(0, first, count, M, sigma)).pin_memory()
        return u, a, torch.empty((count, M), dtype=torch.int32).pin_memory(), torch.zeros(count, dtype=torch.uint8).pin_memory()

    eng.set_micro_batch(n)
    uw, aw, cw, sw = host_block(e2e_first, W * n)
    ue, ae, ce, se = host_block(e2e_first + W * n, K * n)
    eng.run(e2e_first, W * n, cw.numpy(), uniforms=uw.numpy(), alpha=aw.numpy(), status=sw.numpy(),
            stream=stream.cuda_stream)
    barrier()
    e2 = torch.cuda.Event(enable_timing=True)
    e3 = torch.cuda.Event(enable_timing=True)
    e2.record(stream)
    eng.run(e2e_first + W * n, K * n, ce.numpy(), uniforms=ue.numpy(), alpha=ae.numpy(), status=se.numpy(),
            stream=stream.cuda_stream)
    e3.record(stream)
    barrier()
    eng.set_micro_batch(0)
    ms_e2e = dist_max(e2.elapsed_time(e3), dev)
    e2e = world * K * n / (ms_e2e / 1e3)
    e2e_ok = bool((ce >= 0).all().item()) and not bool((se & 1).any().item())

    ok = bool((counts[W:] >= 0).all().item()) and not bool((status[W:] & 1).any().item()) and e2e_ok
    # parity of this run's own outputs: the first samples of timed step W against the oracle
    # (rank 0 only: every rank runs the same kernels; the host oracle would contend for the CPU)
    n_chk = min(32, n)
    parity = None
    if rank == 0:
        parity = parity_spot_check(eng, mps, 0, M, block_index(W), n_chk, stream.cuda_stream, sigma,
                                   uniforms=u_dev[W][:n_chk], alpha=a_dev[W][:n_chk],
                                   ref_counts=counts[W][:n_chk].cpu().numpy(), gemm_mode=args.gemm,
                                   tol=parity_tol(args), rel_floor=parity_rel_floor(args),
                                   rel_tol=parity_rel_tol(args))
        ok = ok and parity["ok"]

    # Same run, same inputs, K1 emulated on the INT8 tensor cores (gemm mode 8, Ozaki, ~1e-13):
    # reported next to the FP64-DMMA headline (the path the north star names) as "alt_gemm".
    alt = None
    if args.dtype == "c128" and args.gemm != "ozaki" and not args.stream_sites:
        eng.set_gemm_mode(8)
        eng.set_lanes(LANES["ozaki"])
        for s in range(W):
            step(s)
        barrier()
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a0.record(stream)
        for s in range(W, W + K):
            step(s)
        a1.record(stream)
        barrier()
        ms_alt = dist_max(a0.elapsed_time(a1), dev)
        ok_alt = not bool((status[W:] & 1).any().item())
        eng.set_lanes(1)
        step(0)
        barrier()
        eng.profile(1)
        for s in range(W, W + min(K, 3)):
            step(s)
        barrier()
        pa = eng.profile_read()
        eng.profile(0)
        eng.set_lanes(args.lanes)
        eng.set_gemm_mode({"3m": 3, "4m": 4}[args.gemm])
        k1_ms = pa["gemm_ms"] / max(pa["gemm_launches"], 1)
        k1_tf = (pa["gemm_flops"] / max(pa["gemm_launches"], 1)) / (k1_ms / 1e3) / 1e12 if k1_ms > 0 else 0.0
        i8_peak = 4510.5  # TOP/s: profiles/r01_umma_probe.jsonl, kind::i8 M=128 N=128 issue-rate probe
        S = args.oz_digits
        npr = S * (S + 1) // 2
        alt = {"gemm": f"ozaki_gemm (complex128 K1 emulated on INT8 tcgen05: {S} digits of 7 bits, "
                       f"{'~1e-13' if S == 7 else '~1e-11' if S == 6 else '~1e-9'} of the row scales; mps_set_gemm_mode 8)",
               "value": world * K * n / (ms_alt / 1e3), "unit": "samples/s", "ms_per_step": ms_alt / K,
               "lanes": LANES["ozaki"],
               "valid_outputs": ok_alt,
               "k1": {"ms_per_launch": k1_ms, "algorithmic_tflops": k1_tf, "vs_fp64_dmma_peak": k1_tf / fp64_peak()[0],
                      "executed_int8_tops": npr * k1_tf, "int8_frac": npr * k1_tf / i8_peak,
                      "int8_peak_source": "profiles/r01_umma_probe.jsonl (kind::i8 N=128, 4510 TOP/s)"}}
        if S == 7:
            # the 6-digit variant (21 INT8 products instead of 28; marginals ~7e-12 from the oracle at
            # chi = 1000 and 4000, tests/test_gpu_parity.py), same inputs, timed the same way
            eng.set_gemm_mode(8)
            eng.set_ozaki_digits(6)
            eng.set_lanes(LANES["ozaki"])
            for s in range(W):
                step(s)
            barrier()
            a0.record(stream)
            for s in range(W, W + K):
                step(s)
            a1.record(stream)
            barrier()
            ms6 = dist_max(a0.elapsed_time(a1), dev)
            alt["value_6_digits"] = world * K * n / (ms6 / 1e3)
            alt["valid_outputs_6_digits"] = not bool((status[W:] & 1).any().item())
            eng.set_ozaki_digits(7)
            eng.set_lanes(args.lanes)
            eng.set_gemm_mode({"3m": 3, "4m": 4}[args.gemm])
    peak, peak_src = fp64_peak()
    traffic, traffic_note = ncu_traffic(args.config, n)
    if args.dtype == "c64":
        traffic, traffic_note = None, None
    gemm_ms_avg = prof["gemm_ms"] / max(prof["gemm_launches"], 1)
    gemm_flops_avg = prof["gemm_flops"] / max(prof["gemm_launches"], 1)
    achieved = gemm_flops_avg / (gemm_ms_avg / 1e3) / 1e12 if gemm_ms_avg > 0 else 0.0
    kernel_name = {"3m": "site_gemm3m_kernel (K1, FP64 DMMA, 3M)", "4m": "site_gemm_kernel (K1, FP64 DMMA, 4M)",
                   "ozaki": f"ozaki2_gemm_kernel (K1, fp64 emulated on INT8 tcgen05, {args.oz_digits} digits)"}[args.gemm]
    bound_note = None
    if args.gemm == "3m":
        bound_note = ("achieved counts algorithmic flops (8 per complex MAC, SURVEY.md §8d); the 3M product executes "
                      "6 on the DMMA pipe, so the executed rate is 0.75 x achieved and frac can exceed 1")
    if small_chain:
        kernel_name = ("small_chain_kernel (whole mode chain in one persistent launch: K1 3M FP64 DMMA + K2/K3 "
                       "draw, 16-CTA clusters, st.async exchange)") if sc_kind == 1 else (
                       "tiny_chain_kernel (whole mode chain in one launch: one CTA per 8-row group, every site in "
                       "shared memory, K1 3M FP64 DMMA + K2/K3 draw)")
        bound_note = ("achieved = K1 algorithmic flops over the fused kernel's whole duration (the draw and the "
                      "exchanges included); " + bound_note)
    if args.dtype == "c64":
        # tcgen05 kind::tf32 executes 3 passes (hi.hi, hi.lo, lo.hi) of the real-doubled
        # product = 24 tensor flops per complex MAC; the roofline is the dense TF32 rate,
        # half the measured dense bf16 rate (MEASURED_PEAKS.json)
        bf16, src = measured_bf16()
        achieved, peak = 3.0 * achieved, bf16 / 2.0
        peak_src = f"dense TF32 = 1/2 of {src} bf16 {bf16:.0f} TFLOP/s"
        kernel_name = "c64_gemm_kernel (K1, tcgen05 kind::tf32, 3xTF32)"
        bound_note = "achieved counts executed tensor flops (3 passes x 8 per complex MAC)"
    elif args.gemm == "ozaki":
        # S(S+1)/2 int8 digit products (diagonals i + j < S; 28 at S = 7) of the real-doubled product per complex MAC;
        # the roofline is the measured kind::i8 issue rate
        achieved, peak = args.oz_digits * (args.oz_digits + 1) / 2.0 * achieved, 4510.5
        peak_src = "profiles/r01_umma_probe.jsonl (kind::i8 M=128 N=128 issue-rate probe), TOP/s"
        kernel_name = f"ozaki2_gemm_kernel (K1, complex128 emulated on INT8 tcgen05, {args.oz_digits} digits, CTA pairs)"
        bound_note = (f"achieved counts executed int8 tensor ops ({args.oz_digits * (args.oz_digits + 1) // 2} digit "
                      "products x 8 per complex MAC)")
    step_flops = sum(site_flops(dims, D, n))
    whole_tf = world * K * step_flops / (ms / 1e3) / 1e12

    line = {
        "metric": METRIC, "value": value, "unit": "samples/s", "n_gpus": world, "steps": K, "warmup": W,
        "ms_per_step": ms / K, "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": args.dtype,
        "data": "synthetic (random row-orthonormal sites from seeds, counter-stream uniforms and alpha)",
        "config": config, "path": path,
        "e2e": {"value": e2e, "unit": "samples/s", "h2d_bytes_per_step": n * M * (8 + 16) + n,
                "d2h_bytes_per_step": n * M * 4 + n,
                "how": "one C-ABI call over the K steps' K n samples from pinned host arrays, micro-batch n: "
                       "per step an H2D of its uniforms + alpha + status and a D2H of its counts + status, "
                       "overlapping the neighbouring steps' kernels; one host synchronisation"
                       + ("" if l2_mode == "large" else "; one context, so the sites stay L2-resident across "
                          "the call's micro-batches as in any production call")},
        "gpu_launches": int(launches),
        "value_l2_warm": None if ms_warm is None else world * K * n / (ms_warm / 1e3),
        "roofline": {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                     "frac": achieved / peak, "traffic": traffic, "traffic_note": traffic_note,
                     "kernel": kernel_name, "note": bound_note,
                     "executed_frac": (0.75 * achieved / peak) if (args.gemm == "3m" and args.dtype == "c128") else None,
                     "peak_source": peak_src,
                     "per_launch": {"ms": gemm_ms_avg, "algorithmic_flops": gemm_flops_avg},
                     "share_of_step": prof["gemm_ms"] / ms_instr if ms_instr > 0 else None,
                     "timing": "K1 launches bracketed by CUDA events on their stream in an instrumented "
                               "repeat of the K timed steps with one lane (events would defeat PDL and "
                               "lane overlap in the clean run)",
                     "whole_chain_tflops": whole_tf,
                     "whole_chain_frac": (3.0 if args.dtype == "c64" else 1.0) * whole_tf / (world * peak),
                     "displace_draw": None if small_chain else
                     {"ms_per_launch": prof["draw_ms"] / max(prof["draw_launches"], 1),
                      "achieved_gbs": (prof["draw_bytes"] / (prof["draw_ms"] / 1e3) / 1e9)
                      if prof["draw_ms"] > 0 else None}},
        "clocks": ck,
        "valid_outputs": ok,
        "parity": parity,
        "setup_s": setup_s,
    }
    if alt is not None:
        line["alt_gemm"] = alt
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        v, cores, sample = CpuBaseline(args.config).run()
        line["cpu_baseline"] = {"value": v, "unit": "samples/s", "cores": cores, "kind": "port", "sample": sample}
    if rank == 0:
        print(json.dumps(dict(line, **RANK_INFO)), flush=True)
    eng.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
