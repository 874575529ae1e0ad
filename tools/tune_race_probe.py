"""Debug probe (not product code): every iteration uses a new micro-batch size, so the first call
autotunes its GEMM shapes (two lanes) and the second call reuses the cached configs; the two must
be bit-identical."""
import os, sys, numpy as np
sys.path.insert(0, '.')
from paper_2511_14923_b200 import MPS, MpsSampler, MpsSamplerConfig
from oracle import mps_oracle as orc
sites = (orc.random_mps(16, 100, 10, seed=0) if os.environ.get("PROBE_CHI", "100") == "100"
         else orc.random_mps(6, int(os.environ["PROBE_CHI"]), 10, seed=0))
R = int(sys.argv[1]) if len(sys.argv) > 1 else 30
bad = 0
mps = MPS(sites)
if os.environ.get("PROBE_C64") == "1":
    mps = mps.astype("complex64")
with MpsSampler(mps, sum_planes=os.environ.get("PROBE_SUMS", "1") == "1") as eng:
    if "PROBE_MODE" in os.environ:
        eng.set_gemm_mode(int(os.environ["PROBE_MODE"]))
    eng.set_lanes(int(os.environ.get("PROBE_LANES", "2")))
    if "PROBE_PIN" in os.environ:
        eng.L.mps_set_gemm_config(eng.ctx, int(os.environ["PROBE_PIN"]))
    for i in range(R):
        n = int(os.environ.get("PROBE_N0", "700")) - 2 * i
        cfg = MpsSamplerConfig(N=n, seed=9, alpha_sigma=0.5, batch_size=n)
        a = eng.sample(cfg, return_marginals=True)
        b = eng.sample(cfg, return_marginals=True)
        d = np.abs(a["marginals"] - b["marginals"])
        if d.max() > 0:
            bad += 1
            rows = np.nonzero(d.max(axis=(1, 2)))[0]
            print(f"n={n}: first-call differs, rows {rows.min()}..{rows.max()} (n={len(rows)}), first mode "
                  f"{int(np.nonzero(d.max(axis=(0, 2)))[0][0])}, max {d.max():.2e}", flush=True)
print("bad", bad, "of", R)
