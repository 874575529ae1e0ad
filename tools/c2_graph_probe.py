"""Probe (not product code): GPU-side time of one C2 micro-batch chain when the host launch cost
is taken out, by capturing mps_sample_range into a CUDA graph with torch.cuda.graph and replaying
it, vs eager calls.  Tells whether a graph / device-argument path would pay at small chi."""
import sys, time, torch
sys.path.insert(0, '.')
from paper_2511_14923_b200 import MPS, MpsSampler
from oracle import mps_oracle as orc
M, chi, D, n = 16, 100, 10, 100
mps = MPS(orc.random_mps(M, chi, D, seed=0))
eng = MpsSampler(mps)
eng.set_streams(0, 0.5)
dev = torch.device("cuda", 0)
counts = torch.empty((n, M), dtype=torch.int32, device=dev)
status = torch.zeros(n, dtype=torch.uint8, device=dev)
st = torch.cuda.Stream(dev)
with torch.cuda.stream(st):
    for _ in range(20): eng.run(0, n, counts, status=status, stream=st.cuda_stream)
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=st):
    eng.run(0, n, counts, status=status, stream=torch.cuda.current_stream().cuda_stream)
torch.cuda.synchronize()
R = 500
for label, fn in (("eager", lambda: eng.run(0, n, counts, status=status, stream=st.cuda_stream)), ("graph", g.replay)):
    with torch.cuda.stream(st):
        for _ in range(10): fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st); t0 = time.perf_counter()
        for _ in range(R): fn()
        t1 = time.perf_counter(); e1.record(st); torch.cuda.synchronize()
    print(label, "host us/call %.1f" % ((t1 - t0) / R * 1e6), "gpu us/call %.1f" % (e0.elapsed_time(e1) / R * 1e3),
          "samples/s %.0f" % (n * R / (e0.elapsed_time(e1) / 1e3)))
