"""cuBLAS DGEMM / ZGEMM throughput probe (library baseline for the FP64 roofline)."""
import json, torch
def bench(dtype, n, flops_per_mac, reps=10):
    a = torch.randn(n, n, dtype=dtype, device="cuda"); b = torch.randn(n, n, dtype=dtype, device="cuda")
    for _ in range(3): c = a @ b
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); c = a @ b; e1.record(); e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return flops_per_mac * n**3 / best / 1e9
print(json.dumps({"probe": "cublas_dgemm_8192", "tflops": bench(torch.float64, 8192, 2)}))
print(json.dumps({"probe": "cublas_zgemm_4096", "tflops": bench(torch.complex128, 4096, 8)}))
# the C3 site-GEMM shape: (1024 x 1000) @ (1000 x 10000) complex128
a = torch.randn(1024, 1000, dtype=torch.complex128, device="cuda"); b = torch.randn(1000, 10000, dtype=torch.complex128, device="cuda")
for _ in range(3): c = a @ b
torch.cuda.synchronize()
best = 1e30
for _ in range(10):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); c = a @ b; e1.record(); e1.synchronize(); best = min(best, e0.elapsed_time(e1))
print(json.dumps({"probe": "cublas_zgemm_c3_site", "ms": best, "tflops": 8 * 1024 * 1000 * 10000 / best / 1e9}))
