"""One bench step under the CUDA profiler API (for ncu --profile-from-start off).

python tools/profile_step.py [--config c3] [--steps 1] [--gemm 3m|4m|ozaki] [--lanes 2]: builds the config's MPS on the
device, runs 3 warm-up steps (autotune included), then brackets --steps steps with
cudaProfilerStart/Stop so ncu sees exactly the kernels of those steps."""
import argparse
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from bench import CONFIGS  # noqa: E402
from paper_2511_14923_b200 import MPS, MpsSampler, alpha_stream, stream_uniforms  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c3")
ap.add_argument("--steps", type=int, default=1)
ap.add_argument("--gemm", default="3m", choices=["3m", "4m", "ozaki"])
ap.add_argument("--lanes", type=int, default=2)
args = ap.parse_args()
M, chi, D, n, sigma, _, _ = CONFIGS[args.config]
mps = MPS.random(M, chi, D, seed=0, device="cuda") if chi >= 500 else MPS.random(M, chi, D, seed=0)
eng = MpsSampler(mps)
eng.set_gemm_mode({"3m": 3, "4m": 4, "ozaki": 8}[args.gemm])
eng.set_lanes(args.lanes)
counts = torch.empty((n, M), dtype=torch.int32, device="cuda")
status = torch.zeros(n, dtype=torch.uint8, device="cuda")
u = torch.from_numpy(stream_uniforms(0, 0, n, M)).cuda()
a = torch.from_numpy(alpha_stream(0, 0, n, M, sigma)).cuda()
for _ in range(3):
    status.zero_()
    eng.run(0, n, counts, uniforms=u, alpha=a, status=status)
torch.cuda.synchronize()
torch.cuda.profiler.start()
for _ in range(args.steps):
    eng.run(0, n, counts, uniforms=u, alpha=a, status=status)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("ok", eng.kernel_launches)
