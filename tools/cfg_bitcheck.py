import sys, torch, itertools
sys.path.insert(0, '.')
from paper_2511_14923_b200 import _native
L = _native.lib()
bad = []
for n, (K, N) in itertools.product([7, 64, 700, 1], [(1, 100), (10, 1000), (100, 1000), (100, 100), (10, 10)]):
    g = torch.Generator(device="cuda").manual_seed(n * 31 + K)
    V = torch.randn(n, K, dtype=torch.complex128, device="cuda", generator=g)
    G = torch.randn(K, N, dtype=torch.complex128, device="cuda", generator=g)
    ref = None
    for cfg in range(11):
        C = torch.full((n, N), complex(float('nan'), 0), dtype=torch.complex128, device="cuda")
        rc = L.mps_site_gemm_cfg(V.data_ptr(), G.data_ptr(), C.data_ptr(), n, K, N, N, 0, cfg, 3)
        torch.cuda.synchronize()
        if rc != 0:
            bad.append((n, K, N, cfg, "rc", rc)); continue
        if ref is None:
            ref = C.clone(); continue
        if not torch.equal(torch.view_as_real(C), torch.view_as_real(ref)):
            d = (C - ref).abs().max().item()
            bad.append((n, K, N, cfg, d, bool(torch.isnan(torch.view_as_real(C)).any())))
print("mismatches:", bad)
