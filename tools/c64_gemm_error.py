"""Where the complex64 chain loses accuracy (B200): the 3xTF32 tcgen05 K1 against (a) the exact
product of its complex64 inputs and (b) a host emulation of 3xTF32 with exact accumulation, and a
plain fp32 cuBLAS product for scale.  Errors are max |dC| / (max|V| max|G| sqrt(K)).
    python tools/c64_gemm_error.py        (profiles/r02_c64_gemm_error.txt)"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2511_14923_b200 import _native  # noqa: E402


def tf32(x):
    b = np.asarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    return ((b + 0x1000) & 0xFFFFE000).astype(np.uint32).view(np.float32)


def split(z):
    out = []
    for part in (z.real, z.imag):
        hi = tf32(part)
        lo = (np.asarray(part, np.float32) - hi).view(np.uint32) & np.uint32(0xFFFFE000)  # tensor core truncates lo
        out.append((hi.astype(np.float64), lo.view(np.float32).astype(np.float64)))
    (rh, rl), (ih, il) = out
    return rh + 1j * ih, rl + 1j * il


def main():
    L = _native.lib()
    for n, K, N in ((256, 100, 1000), (256, 1000, 4000), (256, 2048, 2048)):
        g = torch.Generator(device="cuda").manual_seed(n + K)
        V = torch.randn(n, K, dtype=torch.complex64, device="cuda", generator=g)
        G = torch.randn(K, N, dtype=torch.complex64, device="cuda", generator=g)
        C = torch.empty(n, N, dtype=torch.complex64, device="cuda")
        assert L.mps_site_gemm_c64(V.data_ptr(), G.data_ptr(), C.data_ptr(), n, K, N, 0) == 0
        C32 = V @ G  # cuBLAS complex64 (fp32 accumulate)
        torch.cuda.synchronize()
        v, w = V.cpu().numpy(), G.cpu().numpy()
        exact = v.astype(np.complex128) @ w.astype(np.complex128)
        vh, vl = split(v)
        wh, wl = split(w)
        emu = vh @ wh + vh @ wl + vl @ wh
        scale = float(np.abs(v).max() * np.abs(w).max() * np.sqrt(K))
        e_gpu = np.abs(C.cpu().numpy().astype(np.complex128) - exact).max() / scale
        e_emu = np.abs(emu - exact).max() / scale
        e_emu32 = np.abs(emu.astype(np.complex64).astype(np.complex128) - exact).max() / scale
        e_blas = np.abs(C32.cpu().numpy().astype(np.complex128) - exact).max() / scale
        print(f"n={n} K={K} N={N}: tcgen05 3xTF32 {e_gpu:.1e} | host 3xTF32 emulation, exact accumulation {e_emu:.1e} "
              f"(rounded to c64 {e_emu32:.1e}) | cuBLAS c64 {e_blas:.1e}", flush=True)


if __name__ == "__main__":
    main()
