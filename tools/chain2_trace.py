"""clock64 phase timeline of the pipelined-halves small-chain kernel (chain_small2.cuh) at C2 -- debug only.

Build:  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -shared -Xcompiler -fPIC -I include \
            -DSC_TRACE -o /tmp/lib_sctrace.so paper_2511_14923_b200/csrc/mps_capi.cu
Run:    MPS_LIB=/tmp/lib_sctrace.so python tools/chain2_trace.py      (profiles/r02_small_chain2_trace.txt)"""
import ctypes, sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_2511_14923_b200 import MPS, MpsSampler, MpsSamplerConfig
from oracle import mps_oracle as orc
sites = orc.random_mps(16, 100, 10, seed=0)
with MpsSampler(MPS(sites)) as eng:
    eng.set_small_chain(1)
    import os
    cfg = MpsSamplerConfig(N=100, seed=0, alpha_sigma=None if os.environ.get('TRACE_IDENT') else 0.5, batch_size=100)
    for _ in range(3):
        eng.sample(cfg)
    L = eng.L
    buf = np.zeros((4, 256, 8), dtype=np.int64)
    L.mps_debug_chain2_trace.argtypes = [ctypes.c_void_p]
    assert L.mps_debug_chain2_trace(buf.ctypes.data) == 0
t0 = buf[0, 0, 1]
for q in range(16):
    k1a, k1b, d_a, d_b = buf[0, q], buf[1, q], buf[2, q], buf[3, q]
    f = lambda x: x - t0
    print(f"mode {q:2d}: K1(cta0) A wait {f(k1a[0]):7d} start {f(k1a[1]):7d} end {f(k1a[2]):7d} | B wait {f(k1a[4]):7d} start {f(k1a[5]):7d} end {f(k1a[6]):7d}"
          f" || drawA(cta0) cwait {f(d_a[0]):7d} cdone {f(d_a[1]):7d} T {f(d_a[5]):7d} p1 {f(d_a[2]):7d} draw {f(d_a[3]):7d} end {f(d_a[4]):7d}"
          f" || drawB(cta8) cdone {f(d_b[1]):7d} end {f(d_b[4]):7d}")
