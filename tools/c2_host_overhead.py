import sys, time, torch
sys.path.insert(0, '.')
from paper_2511_14923_b200 import MPS, MpsSampler, alpha_stream, stream_uniforms
from oracle import mps_oracle as orc
M, chi, D, n = 16, 100, 10, 100
mps = MPS(orc.random_mps(M, chi, D, seed=0))
eng = MpsSampler(mps)
eng.set_streams(0, 0.5)
dev = torch.device("cuda", 0)
st = torch.cuda.Stream(dev); torch.cuda.set_stream(st)
counts = torch.empty((n, M), dtype=torch.int32, device=dev)
status = torch.zeros(n, dtype=torch.uint8, device=dev)
for lanes in (1,):
    eng.set_lanes(lanes)
    for _ in range(20): eng.run(0, n, counts, status=status, stream=st.cuda_stream)
    torch.cuda.synchronize()
    R = 200
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st); t0 = time.perf_counter()
    for i in range(R): eng.run(i * n, n, counts, status=status, stream=st.cuda_stream)
    t1 = time.perf_counter(); e1.record(st); torch.cuda.synchronize()
    print("lanes", lanes, "host us/call", (t1 - t0) / R * 1e6, "gpu us/call", e0.elapsed_time(e1) / R * 1e3, "launches", eng.kernel_launches)
