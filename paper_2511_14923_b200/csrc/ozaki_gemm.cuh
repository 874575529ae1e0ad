// ozaki_gemm.cuh — complex128 K1 emulated on the INT8 5th-gen tensor cores (Ozaki scheme I),
// an opt-in product mode (mps_set_gemm_mode(ctx, 8)) next to the FP64 DMMA 3M / 4M kernels.
//
// B200 has no FP64 tcgen05 kind, but it has kind::i8 at ~60x the DMMA rate.  Every fp64 row x
// of an operand is written as  x = 2^e * sum_{i<S} x_i 2^{-7(i+1)}  with signed 7-bit digits
// x_i (int8, |x_i| <= 127; e = frexp exponent of the row's max |x|, so the digit expansion is
// exact up to 2^{-7S} of the row scale).  A product of two rows is then
//   a.b = 2^{e_a + e_b} sum_d 2^{-7(d+2)} sum_{i+j=d} a_i . b_j
// where every a_i . b_j is an exact int32 dot product (|.| <= K 127^2 < 2^31 for K < 2^17).
// Diagonals d = i + j >= S are dropped (their weight is <= 2^{-7(S+2)}: S = 7 leaves ~1e-13
// of the row scales, far inside the 1e-10 parity bar; tests/test_gpu_parity.py checks it).
//
// Complex product: real-doubled 4M (like the complex64 kernel), so A = the interleaved state
// (n x 2K, one exponent per sample) and B = B_r^T (2N x 2K, one exponent per output real
// column), both K-major int8 digit planes.  One CTA owns a 128 x 64 (real) output tile and
// keeps S int32 accumulators (one per diagonal) in TMEM (S x 64 columns); per 32-byte K step
// it issues the S(S+1)/2 digit products (tcgen05.mma kind::i8, M=128 N=64 K=32), operands
// staged by TMA with the 32-byte swizzle.  The epilogue folds the diagonals smallest-first in
// fp64 and applies the exponents.  Digit planes of a site are built once (mps_set_site); the
// state's by ozaki_slice_kernel after each draw.
#pragma once
#include "c64_gemm.cuh"
#include "ptx.cuh"

namespace mps {

constexpr int OZ_MAX_S = 7;

// K-major, 32-byte swizzle (rows of 32 B = one K step): SBO = 8 rows x 32 B
__device__ __forceinline__ uint64_t umma_desc_k_sw32(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(256 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)6 << 61;  // SWIZZLE_32B
  return d;
}

// kind::i8 instruction descriptor: D s32, A/B signed int8, K-major, M x N
__host__ __device__ constexpr uint32_t idesc_i8(int M, int N) {
  return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void umma_i8(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void tmem_ld_32x32b_x16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}

// digits of x * 2^-e (|x| < 2^e): d_i = trunc(128 t), t <- 128 t - d_i (all exact in fp64)
__device__ __forceinline__ void ozaki_digits(double x, int e, int S, int8_t* out, long long plane_stride) {
  double t = ldexp(x, -e);
  for (int i = 0; i < S; ++i) {
    t *= 128.0;
    const double d = trunc(t);
    out[i * plane_stride] = (int8_t)(int)d;
    t -= d;
  }
}

template <int S_>
struct OzCfg {
  static constexpr int S = S_;
  static constexpr int BM = 128, BN = 64, BK = 32, STAGES = 4;
  static constexpr int A_BYTES = BM * BK;  // one digit plane tile (4 KiB)
  static constexpr int B_BYTES = BN * BK;  // 2 KiB
  static constexpr int STAGE_BYTES = S * (A_BYTES + B_BYTES);
  static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 + 2 * STAGES * 8 + 8 + 16;
  static constexpr int TMEM_COLS = (S * BN <= 256) ? 256 : 512;
  static constexpr int THREADS = 192;
  static_assert(S * BN <= 512, "diagonal accumulators exceed TMEM");
};

// C (n x N complex128 = n x 2N real, interleaved) from the digit planes:
//   tm_a : S planes stacked as rows (S*n_pad) x ld bytes, plane i at rows [i*n_pad, (i+1)*n_pad)
//   tm_b : S planes stacked the same way over 2N rows (pad b_pad)
//   ea[n], eb[2N]: exponents
template <class Cfg>
__global__ void __launch_bounds__(Cfg::THREADS, 1)
    ozaki_gemm_kernel(const __grid_constant__ CUtensorMap tm_a, const __grid_constant__ CUtensorMap tm_b,
                      const int* __restrict__ ea, const int* __restrict__ eb, double* __restrict__ C, int n, int N2,
                      int n_pad, int b_pad, int KB, long long ldc) {
  constexpr int S = Cfg::S;
  extern __shared__ __align__(16) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + Cfg::STAGES * Cfg::STAGE_BYTES);
  uint64_t* empty = full + Cfg::STAGES;
  uint64_t* tmem_full = empty + Cfg::STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_full + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m0 = blockIdx.x * Cfg::BM, n0 = blockIdx.y * Cfg::BN;

  griddep_launch_dependents();
  if (threadIdx.x == 0) {
    for (int s = 0; s < Cfg::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tmem_full, 1);
    fence_barrier_init();
    prefetch_tmap(&tm_a);
    prefetch_tmap(&tm_b);
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"((uint32_t)Cfg::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {  // ---- TMA producer: S digit tiles of A and of B per 32-byte K step ----
      griddep_wait();
      for (int kb = 0; kb < KB; ++kb) {
        const int s = kb % Cfg::STAGES;
        mbar_wait(&empty[s], ((kb / Cfg::STAGES) & 1) ^ 1);
        uint8_t* st = smem + s * Cfg::STAGE_BYTES;
        mbar_arrive_expect_tx(&full[s], Cfg::STAGE_BYTES);
        // one 3-D box per operand: {32 B of K} x {tile rows} x {S digit planes}
        tma_load_3d(st, &tm_a, kb * Cfg::BK, m0, 0, &full[s]);
        tma_load_3d(st + S * Cfg::A_BYTES, &tm_b, kb * Cfg::BK, n0, 0, &full[s]);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---- MMA issuer: diagonal d accumulates sum_{i+j=d} A_i . B_j ----
      constexpr uint32_t idesc = idesc_i8(Cfg::BM, Cfg::BN);
      for (int kb = 0; kb < KB; ++kb) {
        const int s = kb % Cfg::STAGES;
        mbar_wait(&full[s], (kb / Cfg::STAGES) & 1);
        tc_fence_after();
        const uint32_t st = smem_u32(smem + s * Cfg::STAGE_BYTES);
#pragma unroll
        for (int d = 0; d < S; ++d) {
#pragma unroll
          for (int i = 0; i <= d; ++i) {
            const int j = d - i;
            const uint64_t da = umma_desc_k_sw32(st + i * Cfg::A_BYTES);
            const uint64_t db = umma_desc_k_sw32(st + S * Cfg::A_BYTES + j * Cfg::B_BYTES);
            umma_i8(tmem + d * Cfg::BN, da, db, idesc, (kb != 0 || i != 0) ? 1u : 0u);
          }
        }
        umma_commit(&empty[s]);
      }
      umma_commit(tmem_full);
    }
  } else {
    // ---- epilogue: fold diagonals smallest-first in fp64, apply 2^(ea + eb) ----
    mbar_wait(tmem_full, 0);
    tc_fence_after();
    const int q = warp & 3;
    const int row = m0 + 32 * q + lane;
    const int era = (row < n) ? ea[row] : 0;
    double* crow = C + (long long)row * ldc;
    const uint32_t tbase = tmem + ((uint32_t)(32 * q) << 16);
#pragma unroll 1
    for (int c0 = 0; c0 < Cfg::BN; c0 += 16) {
      double acc[16];
#pragma unroll
      for (int c = 0; c < 16; ++c) acc[c] = 0.0;
#pragma unroll
      for (int d = S - 1; d >= 0; --d) {
        uint32_t r[16];
        tmem_ld_32x32b_x16(tbase + d * Cfg::BN + c0, r);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        const double w = ldexp(1.0, -7 * (d + 2));
#pragma unroll
        for (int c = 0; c < 16; ++c) acc[c] = fma((double)(int)r[c], w, acc[c]);
      }
      if (row < n) {
#pragma unroll
        for (int c = 0; c < 16; c += 2) {
          const int col = n0 + c0 + c;  // real column = 2 * complex column + (0 re, 1 im)
          if (col < N2)
            *reinterpret_cast<double2*>(crow + col) =
                make_double2(ldexp(acc[c], era + eb[col]), ldexp(acc[c + 1], era + eb[col + 1]));
        }
      }
    }
    tc_fence_before();
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"((uint32_t)Cfg::TMEM_COLS));
  }
}

// Digit planes of the real-doubled state: one CTA per sample row of V (K complex = 2K reals).
// e = frexp exponent of max |x| (0 for an all-zero row); planes: S x (n_pad x ld) int8.
__global__ void ozaki_slice_rows_kernel(const double2* __restrict__ V, int K, int S, int8_t* __restrict__ planes,
                                        long long plane_stride, int ld, int* __restrict__ e_out) {
  __shared__ double red[32];
  const int b = blockIdx.x;
  const double2* v = V + (long long)b * K;
  double m = 0.0;
  for (int k = threadIdx.x; k < K; k += blockDim.x) m = fmax(m, fmax(fabs(v[k].x), fabs(v[k].y)));
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x < 32) {
    m = (threadIdx.x < (blockDim.x + 31) / 32) ? red[threadIdx.x] : 0.0;
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (threadIdx.x == 0) red[0] = m;
  }
  __syncthreads();
  int e = 0;
  if (red[0] > 0.0) frexp(red[0], &e);  // max < 2^e
  if (threadIdx.x == 0) e_out[b] = e;
  int8_t* row = planes + (long long)b * ld;
  for (int kk = threadIdx.x; kk < ld; kk += blockDim.x) {
    const double x = (kk < 2 * K) ? ((kk & 1) ? v[kk >> 1].y : v[kk >> 1].x) : 0.0;
    ozaki_digits(x, e, S, row + kk, plane_stride);
  }
}

// Digit planes of a site's B_r^T (2N rows x 2K): row 2c = (Gr, -Gi, ...), row 2c+1 = (Gi, Gr, ...)
// over the site's rows i; one CTA per B_r^T row r.
__global__ void ozaki_slice_site_kernel(const double2* __restrict__ G, int K, int N, int S, int8_t* __restrict__ planes,
                                        long long plane_stride, int ld, int* __restrict__ e_out) {
  __shared__ double red[32];
  const int r = blockIdx.x;
  const int c = r >> 1, q = r & 1;
  double m = 0.0;
  for (int i = threadIdx.x; i < K; i += blockDim.x) {
    const double2 g = G[(long long)i * N + c];
    m = fmax(m, fmax(fabs(g.x), fabs(g.y)));
  }
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x < 32) {
    m = (threadIdx.x < (blockDim.x + 31) / 32) ? red[threadIdx.x] : 0.0;
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (threadIdx.x == 0) red[0] = m;
  }
  __syncthreads();
  int e = 0;
  if (red[0] > 0.0) frexp(red[0], &e);
  if (threadIdx.x == 0) e_out[r] = e;
  int8_t* row = planes + (long long)r * ld;
  for (int kk = threadIdx.x; kk < ld; kk += blockDim.x) {
    double x = 0.0;
    if (kk < 2 * K) {
      const double2 g = G[(long long)(kk >> 1) * N + c];
      const int p = kk & 1;
      x = (p == 0) ? (q == 0 ? g.x : g.y) : (q == 0 ? -g.y : g.x);
    }
    ozaki_digits(x, e, S, row + kk, plane_stride);
  }
}

}  // namespace mps
