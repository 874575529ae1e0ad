"""Large-shape parity sweep (B200): seeded random chains with RAGGED bond dimensions up to chi ~ 2000
and odd sample counts up to 1500, against the oracle.  tests/test_gpu_fuzz.py keeps chi <= 160 so the
suite stays fast; this covers the per-mode kernels at the sizes the bench runs (K1 row tiles, lane
splits and column tiles with ragged edges, full-chi draw kernels), for every complex128 K1 product.
    python tools/fuzz_large.py SEED N_CASES [BUDGET_S [c64]]       (profiles/r02_fuzz_large.txt)
With c64 the sites are rounded to complex64 and the chain runs the complex64 engine (3xTF32 tcgen05 K1),
checked against the complex128 oracle on the same rounded sites under the complex64 bar (DESIGN.md §4:
1e-4 absolute on the normalised marginals; the relative error for p > 1e-3 is reported and held to the
1e-2 that tests/test_gpu_headline.py asserts after the 64 C3 modes).

Bar: tests/_parity.py's (normalised marginals within 1e-10 absolute and 1e-10 relative for p > 1e-12
along the GPU's path, 1e-9 relative for the opt-in INT8 K1 (REL_TOL_OZAKI7); free-running counts
identical except on flagged near-ties).  The per-case line prints the measured errors, so either bar
can be read off."""
import sys
import time
from collections.abc import Sequence

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import torch  # noqa: E402

from _parity import REL_TOL_C64, REL_TOL_C128, REL_TOL_OZAKI7, marginal_errors  # noqa: E402  # noqa: E402
from oracle import mps_oracle as orc  # noqa: E402
from paper_2511_14923_b200 import MPS, MpsSampler, alpha_stream, stream_uniforms  # noqa: E402
from paper_2511_14923_b200 import _native  # noqa: E402
from paper_2511_14923_b200.mps import device_site  # noqa: E402


class HostView(Sequence):
    def __init__(self, sites):
        self.sites = sites

    def __len__(self):
        return len(self.sites)

    def __getitem__(self, m):
        return self.sites[m].cpu().numpy()


def ragged_dims(rng, M, D, cap):
    """chi_0 = chi_M = 1, each bond a random size admitting row-orthonormal sites (chi_l <= chi_r D)
    and reachable from the right end (chi_m <= D^(M-m)), at least one bond near `cap`."""
    dims = [1]
    for m in range(1, M):
        hi = min(dims[-1] * D, D ** (M - m), cap)
        lo = max(1, -(-dims[-1] // D))
        dims.append(hi if (m == M // 2 or rng.random() < 0.6) else int(rng.integers(max(lo, hi // 3), hi + 1)))
    dims.append(1)
    for m in range(M - 1, 0, -1):  # chi_{m} <= chi_{m+1} D (site m row-orthonormal)
        dims[m] = min(dims[m], dims[m + 1] * D)
    return dims


def cases(n, seed):
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(n):
        D = int(rng.choice([4, 7, 10, 16]))
        M = int(rng.integers(6, 9))
        out.append(dict(D=D, M=M, cap=int(rng.choice([300, 513, 777, 1000, 1333, 2048])),
                        N=int(rng.choice([1, 63, 65, 257, 511, 1023, 1025, 1499])),
                        gemm=int(rng.choice([3, 3, 4, 8])), lanes=int(rng.integers(1, 4)),
                        micro=int(rng.choice([0, 0, 200])), sigma=float(rng.choice([0.0, 0.5, 0.9])),
                        seed=int(rng.integers(0, 2**31)), first=int(rng.integers(0, 10**6))))
        out[-1]["dims"] = ragged_dims(rng, M, D, out[-1]["cap"])
    return out


def run_case(c, c64=False):
    dims, D, N, M = c["dims"], c["D"], c["N"], c["M"]
    sites = [device_site(c["seed"], m, dims[m], dims[m + 1], D) for m in range(M)]
    if c64:
        sites = [G.to(torch.complex64) for G in sites]
    sigma = c["sigma"] if c["sigma"] > 0 else None
    u = stream_uniforms(c["seed"], c["first"], N, M)
    al = alpha_stream(c["seed"], c["first"], N, M, sigma) if sigma else None
    counts = np.zeros((N, M), dtype=np.int32)
    status = np.zeros(N, dtype=np.uint8)
    marg = np.zeros((N, M, D))
    with MpsSampler(MPS(sites)) as eng:
        if not c64:
            eng.set_gemm_mode(c["gemm"])
        eng.set_lanes(c["lanes"])
        eng.set_micro_batch(c["micro"])
        eng.set_streams(c["seed"], sigma)
        eng.run(c["first"], N, counts, marginals=marg, status=status)
    assert not (status & _native.MPS_STATUS_FAILED).any(), "failed samples"
    host = HostView([G.to(torch.complex128) for G in sites])
    ref = orc.sample_chain(host, u, alpha=al, forced=counts, return_marginals=True)
    if c64:
        ab, _, _ = marginal_errors(marg, ref["marginals"])
        _, rel, nbig = marginal_errors(marg, ref["marginals"], floor=1e-3)
    else:
        ab, rel, nbig = marginal_errors(marg, ref["marginals"])
    free = orc.sample_chain(host, u, alpha=al)
    flagged = (status & _native.MPS_STATUS_FLAGGED) != 0
    mism = int(((counts != free["counts"]).any(axis=1) & ~flagged & ~free["flagged"]).sum())
    if c64:
        ok = ab <= REL_TOL_C64 and rel <= 1e-2 and mism == 0
    else:
        ok = ab <= 1e-10 and rel <= (REL_TOL_OZAKI7 if c["gemm"] == 8 else REL_TOL_C128) and mism == 0
    return ok, ab, rel, nbig, mism, int(flagged.sum())


def main():
    seed, n = int(sys.argv[1]), int(sys.argv[2])
    budget = float(sys.argv[3]) if len(sys.argv) > 3 else 1e9
    c64 = len(sys.argv) > 4 and sys.argv[4] == "c64"
    t0 = time.time()
    worst_ab = worst_rel = 0.0
    fails = done = 0
    for i, c in enumerate(cases(n, seed)):
        if time.time() - t0 > budget:
            break
        t1 = time.time()
        try:
            ok, ab, rel, nbig, mism, nflag = run_case(c, c64)
        except Exception as e:  # a crash is a failure too
            ok, ab, rel, nbig, mism, nflag = False, float("nan"), float("nan"), 0, -1, 0
            print("  exception:", repr(e)[:300])
        done += 1
        fails += not ok
        worst_ab, worst_rel = max(worst_ab, ab if ab == ab else 0), max(worst_rel, rel if rel == rel else 0)
        print(f"{i:3d} {'ok  ' if ok else 'FAIL'} dims={c['dims']} D={c['D']} N={c['N']} "
              f"{'c64' if c64 else 'gemm=%d' % c['gemm']} "
              f"lanes={c['lanes']} micro={c['micro']} sigma={c['sigma']}  |dp|={ab:.1e} |dp|/p={rel:.1e} "
              f"(n_p={nbig}) mism={mism} flagged={nflag}  {time.time() - t1:.1f}s", flush=True)
        torch.cuda.empty_cache()
    print(f"cases {done}, fails {fails}, worst |dp| {worst_ab:.2e}, worst |dp|/p {worst_rel:.2e}, "
          f"{time.time() - t0:.0f} s", flush=True)


if __name__ == "__main__":
    main()
