"""Per-call host cost of the C ABI at C1 size (8 modes, chi 16, n 100): device-resident vs pinned host
arrays (profiles/r01_e2e_overhead.txt).  python tools/e2e_overhead.py"""
import sys, time; sys.path.insert(0, str(__import__("pathlib").Path(__file__).resolve().parents[1]))
import numpy as np, torch
from oracle import mps_oracle as orc
from paper_2511_14923_b200 import MPS, MpsSampler, alpha_stream, stream_uniforms
M, chi, D, n = 8, 16, 4, 100
mps = MPS(orc.random_mps(M, chi, D, seed=0))
eng = MpsSampler(mps); eng.set_streams(0, 0.5)
u = torch.from_numpy(stream_uniforms(0, 0, n, M)).pin_memory(); a = torch.from_numpy(alpha_stream(0, 0, n, M, 0.5)).pin_memory()
c = torch.zeros((n, M), dtype=torch.int32).pin_memory(); st = torch.zeros(n, dtype=torch.uint8).pin_memory()
ud, ad, cd, sd = u.cuda(), a.cuda(), c.cuda(), st.cuda()
s = torch.cuda.current_stream().cuda_stream
def bench(f, k=2000):
    for _ in range(50): f()
    torch.cuda.synchronize(); t = time.perf_counter()
    for _ in range(k): f()
    torch.cuda.synchronize(); return (time.perf_counter() - t) / k * 1e6
print("device in/out, no sync      %.1f us" % bench(lambda: eng.run(0, n, cd, uniforms=ud, alpha=ad, status=sd, stream=s)))
print("device + sync each          %.1f us" % bench(lambda: (eng.run(0, n, cd, uniforms=ud, alpha=ad, status=sd, stream=s), torch.cuda.synchronize())))
print("host pinned in/out (e2e)    %.1f us" % bench(lambda: eng.run(0, n, c.numpy(), uniforms=u.numpy(), alpha=a.numpy(), status=st.numpy(), stream=s)))
print("host, device streams only   %.1f us" % bench(lambda: eng.run(0, n, c.numpy(), status=st.numpy(), stream=s)))
