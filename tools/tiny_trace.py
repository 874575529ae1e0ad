"""clock64 phase timeline of the tiny-chain kernel (chain_tiny.cuh) at C1 -- debug build only.

Build:  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -shared -Xcompiler -fPIC -I include \
            -DTC_TRACE -o /tmp/lib_tctrace.so paper_2511_14923_b200/csrc/mps_capi.cu
Run:    MPS_LIB=/tmp/lib_tctrace.so python tools/tiny_trace.py      (profiles/r02_tiny_chain_trace.txt)
Phases per mode of CTA 0, warp 0: chunk prep (uniforms + D(alpha)), barrier + site wait, K1, barrier,
pass 1 + xor tree, draw, pass 2, to the next mode."""
import ctypes, sys, numpy as np, torch
sys.path.insert(0, '.')
from oracle import mps_oracle as orc
from paper_2511_14923_b200 import MPS, MpsSampler, _native
sites = orc.random_mps(8, 16, 4, seed=0)
n, M = 100, 8
for mode in ("alpha", "ident"):
    with MpsSampler(MPS(sites)) as eng:
        eng.set_streams(0, 0.5 if mode == "alpha" else None)
        counts = torch.zeros((n, M), dtype=torch.int32, device="cuda")
        st = torch.zeros(n, dtype=torch.uint8, device="cuda")
        for i in range(5):
            eng.run(i * n, n, counts, status=st)
        torch.cuda.synchronize()
        buf = (ctypes.c_longlong * (64 * 8))()
        _native.lib().mps_debug_tiny_trace(buf)
        a = np.array(buf).reshape(64, 8)[:M]
        t0 = a[0, 0]
        print(mode, "phases per mode (cycles): [prep, bar1+sitewait, K1, bar2, pass1+tree, draw, pass2, ->next]")
        for q in range(M):
            d = np.diff(a[q]).tolist() + ([a[q + 1, 0] - a[q, 7]] if q + 1 < M else [0])
            print(q, a[q, 0] - t0, d)
