"""One fresh-process repetition of the batch-size invariance sequence (B = 7, 64, 700 on one
context) that also checks the B = 700 marginals against the teacher-forced oracle and reports
the first mode where any sample deviates (debug probe, not product code)."""
import sys, numpy as np
sys.path.insert(0, '.')
from paper_2511_14923_b200 import MPS, MpsSampler, MpsSamplerConfig, stream_uniforms, alpha_stream
from oracle import mps_oracle as orc
sites = orc.random_mps(16, 100, 10, seed=0)
N, M = 700, 16
outs = []
with MpsSampler(MPS(sites)) as eng:
    for B in (7, 64, 700):
        outs.append(eng.sample(MpsSamplerConfig(N=N, seed=9, alpha_sigma=0.5, batch_size=B), return_marginals=True))
d = np.abs(outs[2]["marginals"] - outs[0]["marginals"])
if d.max() > 0:
    u, al = stream_uniforms(9, 0, N, M), alpha_stream(9, 0, N, M, 0.5)
    ref = orc.sample_chain(sites, u, alpha=al, forced=outs[2]["counts"], return_marginals=True)
    e700 = np.abs(outs[2]["marginals"] - ref["marginals"]).max(axis=2)
    e7 = np.abs(outs[0]["marginals"] - ref["marginals"]).max(axis=2)
    rows = np.nonzero(d.max(axis=(1, 2)))[0]
    first_mode = int(np.nonzero(d.max(axis=(0, 2)))[0][0])
    print(f"MISMATCH rows {rows.min()}..{rows.max()} (n={len(rows)}), first mode {first_mode}, "
          f"B700 vs oracle max {e700[rows].max():.2e}, B7 vs oracle max {e7[rows].max():.2e}, "
          f"per-mode max diff {np.round(d.max(axis=(0, 2)), 4).tolist()}", flush=True)
else:
    print("ok")
