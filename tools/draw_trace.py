"""Per-CTA timeline of the K2+K3 draw kernel at C3 mode 30 (debug build only).

Build:  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -shared -Xcompiler -fPIC -I include \
            -DDRAW_TRACE -o /tmp/lib_drtrace.so paper_2511_14923_b200/csrc/mps_capi.cu -lcuda
Run:    MPS_LIB=/tmp/lib_drtrace.so python tools/draw_trace.py [mode] [c64]
Stamps (globaltimer, ns) per CTA: 0 entry, 1 D(alpha) built, 2 after griddepcontrol.wait, 3 pass 1 done
(partials reduced), 4 draw published, 5 exit; plus the SM id.  One lane (so the launch is not overlapped
by another lane's GEMM), n = 1024."""
import ctypes, sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_2511_14923_b200 import MPS, MpsSampler
from bench import CONFIGS
M, chi, D, n, sigma, _, _ = CONFIGS["c3"]
mode = int(sys.argv[1]) if len(sys.argv) > 1 else 30
c64 = len(sys.argv) > 2 and sys.argv[2] == "c64"
mps = MPS.random(M, chi, D, seed=0, device="cuda")
if c64:
    mps = mps.astype("complex64")
with MpsSampler(mps) as eng:
    eng.set_lanes(1)
    eng.set_streams(0, sigma)
    counts = torch.zeros((n, M), dtype=torch.int32, device="cuda")
    st = torch.zeros(n, dtype=torch.uint8, device="cuda")
    L = eng.L
    L.mps_debug_draw_trace.argtypes = [ctypes.c_int, ctypes.c_void_p]
    for i in range(2):
        eng.run(i * n, n, counts, status=st)
    torch.cuda.synchronize()
    assert L.mps_debug_draw_trace(mode, None) == 0
    eng.run(2 * n, n, counts, status=st)
    torch.cuda.synchronize()
    buf = np.zeros((8192, 8), dtype=np.int64)
    assert L.mps_debug_draw_trace(-1, buf.ctypes.data) == 0
a = buf[:n].astype(np.float64)
t0 = a[:, 0].min()
rel = (a[:, :6] - t0) / 1e3  # us
dur = np.diff(a[:, :6], axis=1) / 1e3
print(f"draw kernel ({'complex64' if c64 else 'complex128'}), C3 mode {mode}, n={n}: launch span {rel[:, 5].max():.1f} us (first entry -> last exit)")
print("phase means (us): D(alpha) %.2f | PDL wait %.2f | pass 1 %.2f | draw %.2f | pass 2 %.2f" % tuple(dur.mean(0)))
print("phase max   (us): D(alpha) %.2f | PDL wait %.2f | pass 1 %.2f | draw %.2f | pass 2 %.2f" % tuple(dur.max(0)))
print("CTA lifetime mean %.2f us, max %.2f" % ((a[:, 5] - a[:, 0]).mean() / 1e3, (a[:, 5] - a[:, 0]).max() / 1e3))
sm = a[:, 7].astype(int)
per_sm = np.bincount(sm, minlength=148)
print("CTAs per SM: min %d max %d" % (per_sm.min(), per_sm.max()))
# concurrency over time: CTAs resident, sampled every 1 us
ts = np.arange(0, rel[:, 5].max(), 1.0)
res = [((rel[:, 0] <= x) & (rel[:, 5] > x)).sum() for x in ts]
p1 = [((rel[:, 2] <= x) & (rel[:, 3] > x)).sum() for x in ts]
print("resident CTAs / in pass 1, per us:")
print(" ".join(f"{r}/{p}" for r, p in zip(res, p1)))
# entry order
order = np.argsort(rel[:, 0])
print("entries (us) of CTA ranks 0, 592, 800, 1000:", [round(rel[order[i], 0], 1) for i in (0, 592, 800, 1000) if i < n])
