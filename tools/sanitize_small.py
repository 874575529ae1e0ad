"""Small end-to-end run for compute-sanitizer (one tool per gpurun call):
C1 and C2-sized chains in complex128 (3M with sum planes, 4M, lanes 1 and 2) and complex64,
a pipeline-stage split, the small-chain kernel forced on a ragged stage split (state_in / state_out
views of larger buffers), and every K1 tile config on a ragged shape."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from oracle import mps_oracle as orc  # noqa: E402
from paper_2511_14923_b200 import MPS, MpsSampler, MpsSamplerConfig, _native  # noqa: E402

L = _native.lib()
for M, chi, D, N, n in ((8, 16, 4, 130, 100), (6, 100, 10, 70, 70)):
    sites = orc.random_mps(M, chi, D, seed=1)
    for dtype in ("complex128", "complex64"):
        mps = MPS([s.astype(dtype) for s in sites])
        for lanes in (1, 2):
            with MpsSampler(mps) as eng:
                eng.set_lanes(lanes)
                r = eng.sample(MpsSamplerConfig(N=N, seed=3, alpha_sigma=0.5, batch_size=n), return_marginals=True)
                assert (r["counts"] >= 0).all()
    with MpsSampler(MPS(sites)) as eng:
        eng.set_gemm_mode(4)
        eng.sample(MpsSamplerConfig(N=N, seed=3, alpha_sigma=0.5, batch_size=n))
sites = orc.random_mps(9, 100, 10, seed=2)
for n in (37, 100):
    big_in = torch.zeros((n + 16, 100), dtype=torch.complex128, device="cuda")
    big_out = torch.zeros((n + 16, 100), dtype=torch.complex128, device="cuda")
    counts = torch.zeros((n, 9), dtype=torch.int32, device="cuda")
    status = torch.zeros(n, dtype=torch.uint8, device="cuda")
    with MpsSampler(MPS(sites), sites_range=(0, 4), layout=1) as s0, \
            MpsSampler(MPS(sites), sites_range=(4, 9), layout=1) as s1:
        for e in (s0, s1):
            e.set_small_chain(1)
            e.set_streams(5, 0.5)
        s0.run(0, n, counts, state_out=big_in[:n], status=status)
        s1.run(0, n, counts, state_in=big_in[:n], status=status)
    torch.cuda.synchronize()
    assert bool((big_in[n:] == 0).all())
g = torch.Generator(device="cuda").manual_seed(0)
V = torch.randn(37, 21, dtype=torch.complex128, device="cuda", generator=g)
G = torch.randn(21, 45, dtype=torch.complex128, device="cuda", generator=g)
C = torch.empty(37, 45, dtype=torch.complex128, device="cuda")
for mode, ncfg in ((3, 9), (4, 6)):
    for cfg in range(ncfg):
        assert L.mps_site_gemm_cfg(V.data_ptr(), G.data_ptr(), C.data_ptr(), 37, 21, 45, 45, 0, cfg, mode) == 0
V32, G32 = V.to(torch.complex64), G.to(torch.complex64)
C32 = torch.empty(37, 45, dtype=torch.complex64, device="cuda")
assert L.mps_site_gemm_c64(V32.data_ptr(), G32.data_ptr(), C32.data_ptr(), 37, 21, 45, 0) == 0
torch.cuda.synchronize()
print("sanitize_small ok")
