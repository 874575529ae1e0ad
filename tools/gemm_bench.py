"""K1 (site GEMM) sweep on the BASELINE site shapes: every FP64 DMMA tile config of both
products (4M, 3M), the INT8 Ozaki emulation, the complex64 tcgen05 kernel, vs cuBLAS.

python tools/gemm_bench.py [c2 c3 c4 c3_n512]  ->  one JSON line per (shape, kernel)."""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2511_14923_b200 import _native  # noqa: E402

L = _native.lib()
SHAPES = {"c2": (100, 100, 1000), "c3": (1024, 1000, 10000), "c4": (2048, 4000, 40000), "c3_n512": (512, 1000, 10000)}


def timeit(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best


def emit(**kw):
    print(json.dumps(kw), flush=True)


for name in sys.argv[1:] or list(SHAPES):
    n, K, N = SHAPES[name]
    g = torch.Generator(device="cuda").manual_seed(0)
    V = torch.randn(n, K, dtype=torch.complex128, device="cuda", generator=g)
    G = torch.randn(K, N, dtype=torch.complex128, device="cuda", generator=g)
    C = torch.empty(n, N, dtype=torch.complex128, device="cuda")
    flops = 8.0 * n * K * N
    ref = V @ G
    ms = timeit(lambda: torch.matmul(V, G, out=C))
    emit(shape=name, cfg="cublas", ms=ms, tflops=flops / ms / 1e9)
    for mode in (4, 3):
        for cfg in [-1] + list(range(6 if mode == 4 else 11)):
            ms = timeit(lambda: L.mps_site_gemm_cfg(V.data_ptr(), G.data_ptr(), C.data_ptr(), n, K, N, N, 0, cfg, mode))
            err = ((C - ref).abs().max() / ref.abs().max()).item()
            emit(shape=name, mode=mode, cfg=cfg, ms=ms, tflops=flops / ms / 1e9, rel_err=err)

    # complex128 emulated on INT8 tcgen05 (Ozaki): site digits prepared once (as in the chain),
    # state digits + GEMM timed
    for S in (7, 6):
        ld, n_pad, b_pad = (2 * K + 31) // 32 * 32, (n + 255) // 256 * 256, (2 * N + 255) // 256 * 256
        ap = torch.empty(S * n_pad * ld, dtype=torch.int8, device="cuda")
        bp = torch.empty(S * b_pad * ld, dtype=torch.int8, device="cuda")
        ea = torch.empty(n, dtype=torch.int32, device="cuda")
        eb = torch.empty(2 * N, dtype=torch.int32, device="cuda")
        assert L.mps_ozaki_site_planes(G.data_ptr(), K, N, S, bp.data_ptr(), eb.data_ptr(), ld, b_pad, 0) == 0

        def run():
            L.mps_ozaki_state_planes(V.data_ptr(), n, K, S, ap.data_ptr(), ea.data_ptr(), ld, n_pad, 0)
            L.mps_ozaki_gemm_planes(ap.data_ptr(), n_pad, ea.data_ptr(), bp.data_ptr(), b_pad, eb.data_ptr(), ld,
                                    C.data_ptr(), n, K, N, S, 0)
        ms = timeit(run)
        err = ((C - ref).abs().max() / ref.abs().max()).item()
        emit(shape=name, mode=f"ozaki_int8_S{S}", ms=ms, tflops=flops / ms / 1e9, rel_err=err)
        del ap, bp

    # complex64 on tcgen05 (3xTF32), planes prepared once, GEMM timed alone
    ld = (2 * K + 3) & ~3
    V32, G32 = V.to(torch.complex64), G.to(torch.complex64)
    ahi = torch.empty(n, ld, device="cuda")
    alo = torch.empty_like(ahi)
    bhi = torch.empty(2 * N, ld, device="cuda")
    blo = torch.empty_like(bhi)
    C32 = torch.empty(n, N, dtype=torch.complex64, device="cuda")
    assert L.mps_c64_state_planes(V32.data_ptr(), n, K, ahi.data_ptr(), alo.data_ptr(), ld, 0) == 0
    assert L.mps_c64_site_planes(G32.data_ptr(), K, N, bhi.data_ptr(), blo.data_ptr(), ld, 0) == 0
    ms = timeit(lambda: L.mps_c64_gemm_planes(ahi.data_ptr(), alo.data_ptr(), bhi.data_ptr(), blo.data_ptr(), ld,
                                              C32.data_ptr(), n, K, N, 0))
    err = ((C32.to(torch.complex128) - ref).abs().max() / ref.abs().max()).item()
    emit(shape=name, mode="c64_tcgen05_3xtf32", ms=ms, tflops=flops / ms / 1e9, rel_err=err)
    ms = timeit(lambda: torch.matmul(V32, G32, out=C32))
    emit(shape=name, cfg="cublas_c64", ms=ms, tflops=flops / ms / 1e9)
    del V, G, C, ref, ahi, alo, bhi, blo, V32, G32, C32
    torch.cuda.empty_cache()
