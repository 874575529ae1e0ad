import sys, torch, numpy as np
sys.path.insert(0, '.')
from paper_2511_14923_b200 import MPS, MpsSampler, MpsSamplerConfig, _native
from oracle import mps_oracle as orc
sites = orc.random_mps(16, 100, 10, seed=1)
N = 700
ref = None
for cfg in [-1] + list(range(11)):
    for B in (7, 64, 700):
        with MpsSampler(MPS(sites)) as eng:
            _native.check(eng.L.mps_set_gemm_config(eng.ctx, cfg), eng.ctx)
            o = eng.sample(MpsSamplerConfig(N=N, seed=9, alpha_sigma=0.5, batch_size=B), return_marginals=True)
        if ref is None:
            ref = o; continue
        dc = int((o["counts"] != ref["counts"]).sum())
        dm = np.abs(o["marginals"] - ref["marginals"]).max()
        if dc or dm:
            rows = np.nonzero(np.abs(o["marginals"] - ref["marginals"]).max(axis=(1, 2)))[0]
            modes = np.nonzero(np.abs(o["marginals"] - ref["marginals"]).max(axis=(0, 2)))[0]
            print("cfg", cfg, "B", B, "count diffs", dc, "max marg diff", dm, "rows", rows[:10], "modes", modes[:10])
print("done")
