"""Stress probe (not product code): repeat tests/test_gpu_parity.py::test_batch_size_invariance and
report where results differ (which batch size, samples, modes, magnitude)."""
import sys, numpy as np
sys.path.insert(0, '.')
from paper_2511_14923_b200 import MPS, MpsSampler, MpsSamplerConfig
from oracle import mps_oracle as orc
sites = orc.random_mps(16, 100, 10, seed=0)
N = 700
R = int(sys.argv[1]) if len(sys.argv) > 1 else 20
LANES = int(sys.argv[2]) if len(sys.argv) > 2 else 2
PIN = int(sys.argv[3]) if len(sys.argv) > 3 else -1
fails = 0
for it in range(R):
    outs = []
    with MpsSampler(MPS(sites)) as eng:
        eng.set_lanes(LANES)
        if PIN >= 0:
            eng.L.mps_set_gemm_config(eng.ctx, PIN)
        for B in (7, 64, 700):
            outs.append(eng.sample(MpsSamplerConfig(N=N, seed=9, alpha_sigma=0.5, batch_size=B), return_marginals=True))
    for bi, o in zip((64, 700), outs[1:]):
        dm = np.abs(o["marginals"] - outs[0]["marginals"])
        dc = o["counts"] != outs[0]["counts"]
        if dm.max() > 0 or dc.any():
            fails += 1
            rows = np.nonzero(dm.max(axis=(1, 2)))[0]
            modes = np.nonzero(dm.max(axis=(0, 2)))[0]
            print(f"iter {it} B={bi}: max|dm|={dm.max():.3e} rows={rows[:12]} (n={len(rows)}) modes={modes} "
                  f"count diffs={int(dc.sum())}", flush=True)
print("fails", fails, "of", R)
