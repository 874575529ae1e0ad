import sys, time, torch
sys.path.insert(0, '.')
from paper_2511_14923_b200 import MPS, MpsSampler
from oracle import mps_oracle as orc
M, chi, D, n = 16, 100, 10, 100
mps = MPS(orc.random_mps(M, chi, D, seed=0))
eng = MpsSampler(mps)
dev = torch.device("cuda", 0)
counts = torch.empty((n, M), dtype=torch.int32, device=dev)
status = torch.zeros(n, dtype=torch.uint8, device=dev)
st = torch.cuda.Stream(dev)
for sig in (0.5, None):
    eng.set_streams(0, sig)
    with torch.cuda.stream(st):
        for _ in range(20): eng.run(0, n, counts, status=status, stream=st.cuda_stream)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for i in range(300): eng.run(i * n, n, counts, status=status, stream=st.cuda_stream)
        e1.record(st); torch.cuda.synchronize()
    print("sigma", sig, "us/call", e0.elapsed_time(e1) / 300 * 1e3)
