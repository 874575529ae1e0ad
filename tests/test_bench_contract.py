"""bench.py's driver contract: the reference arm's JSON line on the CPU, the GPU arm's line and
its N>1 sample-sharded code path on a B200 (pytest -m gpu)."""

import json
import sys
from pathlib import Path

import pytest
from _proc import run_group

ROOT = Path(__file__).resolve().parents[1]


def test_reference_arm_json_line():
    out = run_group([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--config", "c1",
                          "--steps", "1", "--warmup", "3"], timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "impl", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["higher_is_better"] is True
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert d["config"]["workload"].startswith("c1")


def test_gpus_flag_must_match_world_size():
    """--gpus N under a launcher with another WORLD_SIZE refuses instead of measuring the wrong N."""
    import os

    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    out = run_group([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--config", "c1", "--steps", "1"],
                         timeout=600, cwd=ROOT, env=env)
    assert out.returncode != 0 and "WORLD_SIZE=1" in out.stderr


def test_gpu_arm_fails_loudly_without_gpu():
    import torch

    if torch.cuda.is_available():
        return
    out = run_group([sys.executable, str(ROOT / "bench.py"), "--config", "c1", "--steps", "1"],
                         timeout=600, cwd=ROOT)
    assert out.returncode != 0  # no CPU fallback for the product path


@pytest.mark.gpu
@pytest.mark.timeout(1500)  # above the sum of the subprocess timeouts, so a stuck child is killed by them
def test_gpu_arm_json_line_and_two_rank_path():
    """One GPU arm line at N=1 (c2), then the N>1 sample-sharded code path under torchrun with
    two ranks sharing cuda:0 over gloo (MPS_BENCH_ONE_GPU plumbing mode: keys, max-over-ranks,
    whole-job value; the timing of that run means nothing)."""
    import os

    out = run_group([sys.executable, str(ROOT / "bench.py"), "--config", "c2", "--steps", "2", "--warmup", "3",
                          "--no-cpu-baseline"], timeout=420, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    d = json.loads([l for l in out.stdout.splitlines() if l.startswith("{")][-1])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "e2e", "gpu_launches", "roofline", "clocks", "alt_gemm"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["value"] > 0 and d["gpu_launches"] > 0 and d["valid_outputs"]
    assert d["roofline"]["bound"] == "tensor" and d["roofline"]["frac"] > 0
    env = dict(os.environ, MPS_BENCH_BACKEND="gloo", MPS_BENCH_ONE_GPU="1")
    # the bare driver command: `bench.py --gpus 2` re-executes itself under torchrun (2 ranks)
    out = run_group([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--config", "c2", "--steps", "2",
                          "--warmup", "3", "--no-cpu-baseline"],
                         timeout=600, cwd=ROOT, env=env)
    assert out.returncode == 0, out.stderr[-3000:]
    assert "re-executing under torchrun" in out.stderr and "process group up: world=2" in out.stderr
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1  # rank 0 only
    d2 = json.loads(lines[0])
    assert d2["n_gpus"] == 2 and d2["scaling"] == "weak" and d2["value"] > 0 and d2["valid_outputs"]
    assert [r["rank"] for r in d2["ranks"]] == [0, 1] and "ranks" not in d2["config"]
    # torchrun with a world size that contradicts --gpus fails loudly
    out = run_group([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                          "--master-addr", "127.0.0.1", "--master-port", "29547", str(ROOT / "bench.py"), "--gpus", "3",
                          "--config", "c2", "--steps", "2", "--no-cpu-baseline"],
                         timeout=300, cwd=ROOT, env=env)
    assert out.returncode != 0
