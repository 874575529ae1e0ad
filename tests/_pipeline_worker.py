"""torchrun worker for tests/test_gpu_parity.py::test_pipelined_handoffs_on_one_gpu: two ranks
sharing cuda:0 over gloo run sample_pipelined with the given hand-off and rank 0 saves the counts."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import mps_oracle as orc  # noqa: E402
from paper_2511_14923_b200 import MPS, MpsSamplerConfig  # noqa: E402
from paper_2511_14923_b200.distributed import sample_pipelined, sample_sharded  # noqa: E402

handoff, out = sys.argv[1], sys.argv[2]
dist.init_process_group("gloo")
torch.cuda.set_device(0)
sites = orc.random_mps(16, 100, 10, seed=0)
cfg = MpsSamplerConfig(N=350, seed=4, alpha_sigma=0.5, batch_size=100)
if handoff == "sharded":  # sample-sharded layout: contiguous index blocks per rank, counts gathered
    res = sample_sharded(cfg, MPS(sites), device=0)
else:
    res = sample_pipelined(cfg, MPS(sites), device=0, handoff=handoff)
if dist.get_rank() == 0:
    np.save(out, res.counts)
dist.destroy_process_group()
