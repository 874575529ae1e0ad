"""Phase timeline of the small-chain kernel (CTA 0), from a -DSC_TRACE debug build.

    python tools/chain_trace.py [--config c2]

Builds /tmp/libmps_trace.so, runs one C2 micro-batch through it and prints, per mode, the
clock64 deltas of the compute warps (GEMM mainloop, epilogue + exchange barrier, draw, state
barrier) and of the helper warp (Gamma issue, next-mode head, D(alpha) build).
"""
import argparse
import ctypes
import subprocess
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--M", type=int, default=16)
    ap.add_argument("--chi", type=int, default=100)
    ap.add_argument("--D", type=int, default=10)
    ap.add_argument("--n", type=int, default=100)
    ap.add_argument("--sigma", type=float, default=0.5, help="alpha sigma (negative: no displacement)")
    ap.add_argument("-D", dest="defs", action="append", default=[], help="extra -D for the trace build")
    a = ap.parse_args()
    lib = Path("/tmp/libmps_trace.so")
    subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17", "-DSC_TRACE", *[f"-D{d}" for d in a.defs],
                    "-shared", "-Xcompiler", "-fPIC", "-I", str(ROOT / "include"), "-o", str(lib),
                    str(ROOT / "paper_2511_14923_b200/csrc/mps_capi.cu")], check=True)
    from paper_2511_14923_b200 import _native

    _native.LIB_PATH = lib
    import torch

    from paper_2511_14923_b200 import MPS, MpsSampler, MpsSamplerConfig

    mps = MPS.random(a.M, a.chi, a.D, seed=0)
    with MpsSampler(mps) as eng:
        cfg = MpsSamplerConfig(N=a.n, seed=0, alpha_sigma=a.sigma if a.sigma >= 0 else None, batch_size=a.n)
        for _ in range(3):
            eng.sample(cfg)
        torch.cuda.synchronize()
        buf = np.zeros((2, 256, 8), np.int64)
        L = _native.lib()
        L.mps_debug_chain_trace.argtypes = [ctypes.c_void_p]
        assert L.mps_debug_chain_trace(buf.ctypes.data) == 0
    c = buf[0, :a.M]
    print("mode   gemm  xchg  draw  tail   (cycles; xchg = C row + D(alpha) waits, tail = to next GEMM)")
    for q in range(a.M):
        nxt = c[q + 1, 0] if q + 1 < a.M else c[q, 3]
        print(f"{q:4d} {c[q,1]-c[q,0]:6d} {c[q,2]-c[q,1]:5d} {c[q,3]-c[q,2]:5d} {nxt-c[q,3]:5d}")
    print("total cycles", c[a.M - 1, 3] - c[0, 0])
    print("of which waiting for the previous mode's states (V) before the K1 loop:",
          [int(c[q, 7] - c[q, 0]) for q in range(a.M)])
    print("GEMM cycles thread 0 spent waiting for ring data, per mode:", list(buf[1, :a.M, 0] // 3))
    q = min(5, a.M - 2)
    print(f"draw of mode {q}: pass1 {c[q,4]-c[q,2]}  reduce {c[q,5]-c[q,4]}  draw {c[q,6]-c[q,5]}  "
          f"pass2+emit {c[q,3]-c[q,6]}")


if __name__ == "__main__":
    main()
