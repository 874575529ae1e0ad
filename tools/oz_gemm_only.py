import sys, torch
sys.path.insert(0, '.')
from paper_2511_14923_b200 import _native
L = _native.lib()
n, K, N = 1024, 1000, 10000
S = 7
g = torch.Generator(device="cuda").manual_seed(0)
V = torch.randn(n, K, dtype=torch.complex128, device="cuda", generator=g)
G = torch.randn(K, N, dtype=torch.complex128, device="cuda", generator=g)
C = torch.empty(n, N, dtype=torch.complex128, device="cuda")
ld, n_pad, b_pad = (2 * K + 31) // 32 * 32, (n + 255) // 256 * 256, (2 * N + 255) // 256 * 256
ap = torch.empty(S * n_pad * ld, dtype=torch.int8, device="cuda")
bp = torch.empty(S * b_pad * ld, dtype=torch.int8, device="cuda")
ea = torch.empty(n, dtype=torch.int32, device="cuda")
eb = torch.empty(2 * N, dtype=torch.int32, device="cuda")
assert L.mps_ozaki_site_planes(G.data_ptr(), K, N, S, bp.data_ptr(), eb.data_ptr(), ld, b_pad, 0) == 0
assert L.mps_ozaki_state_planes(V.data_ptr(), n, K, S, ap.data_ptr(), ea.data_ptr(), ld, n_pad, 0) == 0
for _ in range(3):
    L.mps_ozaki_gemm_planes(ap.data_ptr(), n_pad, ea.data_ptr(), bp.data_ptr(), b_pad, eb.data_ptr(), ld, C.data_ptr(), n, K, N, S, 0)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    L.mps_ozaki_gemm_planes(ap.data_ptr(), n_pad, ea.data_ptr(), bp.data_ptr(), b_pad, eb.data_ptr(), ld, C.data_ptr(), n, K, N, S, 0)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 5
print("gemm only ms", ms, "TF", 8.0 * n * K * N / ms / 1e9, "err", ((C - V @ G).abs().max() / (V @ G).abs().max()).item())
