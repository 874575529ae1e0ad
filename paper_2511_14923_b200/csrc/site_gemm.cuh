// site_gemm.cuh — K1: the per-mode site contraction C = V . Gamma.
//
//   V     : n x K complex128 (the n in-flight temp_tensors)
//   Gamma : K x N complex128, N = chi_r * D (Gamma^[m] reshaped chi_l x chi_r D)
//   C     : n x N complex128
//
// B200 has no FP64 tcgen05 kind, so the FP64 tensor pipe is reached through
// mma.sync .f64 (SASS DMMA.8x8x4: 256 FMA per warp instruction, measured peak
// 37.0 TFLOP/s, profiles/fp64_peak.json).  The complex product is a "real-doubled"
// 4M GEMM done without any repacking:
//   A_r[b][2i+p]  = V[b][i].(re, im)[p]          (V's own interleaved layout)
//   B_r[2i][2c+q] = Gamma[i][c].(re, im)[q]       (Gamma's own interleaved layout)
//   B_r[2i+1][2c] = -Gamma[i][c].im,  B_r[2i+1][2c+1] = Gamma[i][c].re
// so C_r = A_r B_r holds C interleaved, and the odd rows of B_r are produced while
// loading fragments (component swap + sign flip) from the same smem tile.
//
// Pipeline: thread 0 issues TMA loads of the V tile (BM x 16 doubles) and BN_R/16
// Gamma boxes (8 rows x 16 doubles each), 128-byte swizzled, into a STAGES-deep ring
// guarded by full/empty mbarriers, refilling each slot one iteration after it was
// consumed.  No dedicated producer warp: 8 warps = 2 per SM sub-partition keeps the
// 255-register budget (a 9th warp caps every warp at 168 and spills).  Each warp owns
// a (8 MF) x (8 NF) real sub-tile of DMMA fragments.  The k order inside a 16-double
// stage row is permuted (x = 2s + 8(t&1) + (t>>1) for lane-in-group t, step s) so both
// fragment loads are bank-conflict free against the TMA 128B swizzle.
//
// Summation order per output element is fixed by (K, stage, step) only — the same for
// every tile configuration, n, tile position and grid — so results are bit-identical
// across batch sizes and GPU counts (sampler.py:272-285 invariance tests).
#pragma once
#include "ptx.cuh"

namespace mps {

template <int BM_, int BN_R_, int WARPS_M_, int WARPS_N_, int STAGES_, int MIN_BLOCKS_>
struct GemmCfgT {
  static constexpr int BM = BM_;          // rows (samples) per CTA tile
  static constexpr int BN_R = BN_R_;      // real columns per CTA tile
  static constexpr int BK_C = 8;          // complex K rows per stage (16 real) — fixed: sets the sum order
  static constexpr int STAGES = STAGES_;
  static constexpr int WARPS_M = WARPS_M_, WARPS_N = WARPS_N_;
  static constexpr int WARPS = WARPS_M * WARPS_N;
  static constexpr int THREADS = WARPS * 32;
  static constexpr int MIN_BLOCKS = MIN_BLOCKS_;
  static constexpr int WM = BM / WARPS_M, WN = BN_R / WARPS_N;  // warp tile (real)
  static constexpr int MF = WM / 8, NF = WN / 8;                // DMMA 8x8 fragments per warp (4M)
  static constexpr int NF3 = WN / 16;                           // 8-complex-column fragments (3M)
  static constexpr int A_BYTES = BM * 16 * 8;
  static constexpr int B_GROUPS = BN_R / 16;
  static constexpr int B_BYTES = B_GROUPS * BK_C * 128;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 /*align*/ + 2 * STAGES * 8;
  static_assert(BM % (8 * WARPS_M) == 0 && BN_R % (16 * WARPS_N) == 0 && WN % 16 == 0, "tile shape");
  static_assert(A_BYTES % 1024 == 0 && B_BYTES % 1024 == 0, "128B-swizzle atoms need 1 KiB alignment");
};

template <class Cfg>
__global__ void __launch_bounds__(Cfg::THREADS, Cfg::MIN_BLOCKS)
    site_gemm_kernel(const __grid_constant__ CUtensorMap tmap_v, const __grid_constant__ CUtensorMap tmap_g,
                     double2* __restrict__ C, int n, int N, int KT, long long ldc) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  // align to 1 KiB by pointer arithmetic on the __shared__ array (keeps LDS addressing)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + Cfg::STAGES * Cfg::STAGE_BYTES);
  uint64_t* empty = full + Cfg::STAGES;

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int m0 = blockIdx.x * Cfg::BM;
  const int n0r = blockIdx.y * Cfg::BN_R;

  auto issue_g = [&](int kt) {  // one k-stage: expect the whole stage, load the B_GROUPS Gamma boxes
    const int s = kt % Cfg::STAGES;
    uint8_t* Bs = smem + s * Cfg::STAGE_BYTES + Cfg::A_BYTES;
    mbar_arrive_expect_tx(&full[s], Cfg::STAGE_BYTES);
#pragma unroll
    for (int gi = 0; gi < Cfg::B_GROUPS; ++gi)
      tma_load_2d(Bs + gi * (Cfg::BK_C * 128), &tmap_g, n0r + gi * 16, kt * Cfg::BK_C, &full[s]);
  };
  auto issue_v = [&](int kt) {  // the V tile of the stage (written by the previous kernel)
    const int s = kt % Cfg::STAGES;
    tma_load_2d(smem + s * Cfg::STAGE_BYTES, &tmap_v, kt * 16, m0, &full[s]);
  };
  auto issue = [&](int kt) {
    issue_g(kt);
    issue_v(kt);
  };

  // PDL: let the next kernel's CTAs launch into SMs this grid's tail leaves idle
  griddep_launch_dependents();
  if (threadIdx.x == 0) {
    for (int s = 0; s < Cfg::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], Cfg::WARPS);
    }
    fence_barrier_init();
    prefetch_tmap(&tmap_v);
    prefetch_tmap(&tmap_g);
    // Gamma is resident input: prefetch the first stages while the predecessor drains
    for (int kt = 0; kt < Cfg::STAGES && kt < KT; ++kt) issue_g(kt);
    griddep_wait();  // predecessor (draw of the previous mode) complete: V valid, C free to overwrite
    for (int kt = 0; kt < Cfg::STAGES && kt < KT; ++kt) issue_v(kt);
  }
  __syncthreads();

  const int g = lane >> 2;  // group id: fragment row (A) / column (B)
  const int t = lane & 3;   // thread in group: fragment k index
  const int warp_m = warp % Cfg::WARPS_M;
  const int warp_n = warp / Cfg::WARPS_M;
  const int p = t >> 1;  // 0: real row of B_r, 1: rotated row
  const uint64_t sign = ((p == 1) && ((g & 1) == 0)) ? 0x8000000000000000ull : 0ull;

  double acc[Cfg::MF][Cfg::NF][2];
#pragma unroll
  for (int i = 0; i < Cfg::MF; ++i)
#pragma unroll
    for (int j = 0; j < Cfg::NF; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  for (int kt = 0; kt < KT; ++kt) {
    const int s = kt % Cfg::STAGES;
    mbar_wait(&full[s], (kt / Cfg::STAGES) & 1);
    const uint8_t* As = smem + s * Cfg::STAGE_BYTES + (warp_m * Cfg::WM + g) * 128 + (p << 3);
    const uint8_t* Bs = smem + s * Cfg::STAGE_BYTES + Cfg::A_BYTES + warp_n * (Cfg::WN / 16) * (Cfg::BK_C * 128);
#pragma unroll
    for (int step = 0; step < 4; ++step) {
      const int i = step + 4 * (t & 1);  // complex row of the stage == 16B chunk of the A row
      double a[Cfg::MF], b[Cfg::NF];
#pragma unroll
      for (int mf = 0; mf < Cfg::MF; ++mf)
        a[mf] = *reinterpret_cast<const double*>(As + mf * 8 * 128 + ((i ^ g) << 4));
#pragma unroll
      for (int nf = 0; nf < Cfg::NF; ++nf) {
        const int xb = (((nf & 1) * 8) + g) ^ p;
        const uint64_t bits = *reinterpret_cast<const uint64_t*>(
            Bs + (nf >> 1) * (Cfg::BK_C * 128) + i * 128 + (((xb >> 1) ^ i) << 4) + ((xb & 1) << 3));
        b[nf] = __longlong_as_double(static_cast<long long>(bits ^ sign));
      }
#pragma unroll
      for (int mf = 0; mf < Cfg::MF; ++mf)
#pragma unroll
        for (int nf = 0; nf < Cfg::NF; ++nf) dmma_8x8x4(acc[mf][nf][0], acc[mf][nf][1], a[mf], b[nf]);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
    // Producer (thread 0): refill the slot of k-stage kt-1 — every warp has long left it
    // by the time warp 0 finishes kt, so this wait rarely blocks.
    if (threadIdx.x == 0 && kt >= 1 && kt - 1 + Cfg::STAGES < KT) {
      mbar_wait(&empty[(kt - 1) % Cfg::STAGES], ((kt - 1) / Cfg::STAGES) & 1);
      fence_proxy_async();  // the slot's generic-proxy reads before the TMA (async-proxy) refill
      issue(kt - 1 + Cfg::STAGES);
    }
  }

  // ---------------- epilogue: (c0, c1) of a fragment is one complex entry ----------------
#pragma unroll
  for (int mf = 0; mf < Cfg::MF; ++mf) {
    const int row = m0 + warp_m * Cfg::WM + mf * 8 + g;
    if (row >= n) continue;
    double2* crow = C + (long long)row * ldc;
#pragma unroll
    for (int nf = 0; nf < Cfg::NF; ++nf) {
      const int col = (n0r >> 1) + warp_n * (Cfg::WN / 2) + nf * 4 + t;
      if (col < N) crow[col] = make_double2(acc[mf][nf][0], acc[mf][nf][1]);
    }
  }
}

// ---------------------------------------------------------------------------------------
// 3M variant: three real GEMMs instead of four (Gauss / Karatsuba):
//   T1 = Vr.Gr,  T2 = Vi.Gi,  T3 = (Vr+Vi).(Gr+Gi);   Re C = T1 - T2,  Im C = T3 - (T1 + T2)
// 25% fewer DMMAs for the same algorithmic (8 flops per complex MAC) work.  Same TMA
// tiles as 4M; the MMA k index is the complex index, each lane reads (re, im) pairs
// with one LDS.128 (k of lane t at step s is i = 2t + s: conflict-free against the
// 128B swizzle for both operands).
//
// SUMS: the operand sums Vr+Vi and Gr+Gi come precomputed from "sum planes" (the draw
// kernel writes the state's, mps_set_site the site's) through two more TMA boxes per
// stage, instead of DADDs that queue behind DMMAs on the FP64 pipe (+7.5% measured).
// The planes hold exactly the IEEE sums the in-kernel DADD would form, so SUMS and
// non-SUMS launches give bit-identical C.  All 3M configs share the k order, so 3M
// results are bit-identical across configs, batch sizes and GPU counts.
// ---------------------------------------------------------------------------------------
template <class Cfg, bool SUMS>
struct Sums3M {
  // state sums: BM rows x 8 doubles (64 B rows, 64B swizzle); site sums: 8 rows x 16-double boxes
  static constexpr int AS_BYTES = SUMS ? Cfg::BM * 64 : 0;
  static constexpr int BS_BOXES = SUMS ? Cfg::BN_R / 32 : 0;
  static constexpr int BS_BYTES = BS_BOXES * 1024;
  static constexpr int STAGE_BYTES = Cfg::STAGE_BYTES + BS_BYTES + AS_BYTES;
  static constexpr int SMEM_BYTES = Cfg::STAGES * STAGE_BYTES + 1024 + 2 * Cfg::STAGES * 8;
  static_assert(!SUMS || (Cfg::BN_R % 32 == 0 && AS_BYTES % 512 == 0), "sum-plane tiles");
};

template <class Cfg, bool SUMS>
__global__ void __launch_bounds__(Cfg::THREADS, Cfg::MIN_BLOCKS)
    site_gemm3m_kernel(const __grid_constant__ CUtensorMap tmap_v, const __grid_constant__ CUtensorMap tmap_g,
                       const __grid_constant__ CUtensorMap tmap_vs, const __grid_constant__ CUtensorMap tmap_gs,
                       double2* __restrict__ C, int n, int N, int KT, long long ldc) {
  static_assert(Cfg::NF3 >= 1 && Cfg::WN % 16 == 0, "3M warp tile needs whole 8-complex fragments");
  using S = Sums3M<Cfg, SUMS>;
  extern __shared__ __align__(16) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + Cfg::STAGES * S::STAGE_BYTES);
  uint64_t* empty = full + Cfg::STAGES;
  // stage layout: [V tile | Gamma boxes | Gamma-sum boxes | V-sum tile]
  constexpr int OFF_A = 0, OFF_B = Cfg::A_BYTES, OFF_BS = Cfg::STAGE_BYTES, OFF_AS = Cfg::STAGE_BYTES + S::BS_BYTES;

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int m0 = blockIdx.x * Cfg::BM;
  const int n0r = blockIdx.y * Cfg::BN_R;

  auto issue_g = [&](int kt) {  // resident operands: Gamma (+ its sum plane)
    const int s = kt % Cfg::STAGES;
    uint8_t* st = smem + s * S::STAGE_BYTES;
    mbar_arrive_expect_tx(&full[s], S::STAGE_BYTES);
#pragma unroll
    for (int gi = 0; gi < Cfg::B_GROUPS; ++gi)
      tma_load_2d(st + OFF_B + gi * (Cfg::BK_C * 128), &tmap_g, n0r + gi * 16, kt * Cfg::BK_C, &full[s]);
    if constexpr (SUMS) {
#pragma unroll
      for (int gi = 0; gi < S::BS_BOXES; ++gi)
        tma_load_2d(st + OFF_BS + gi * 1024, &tmap_gs, (n0r >> 1) + gi * 16, kt * Cfg::BK_C, &full[s]);
    }
  };
  auto issue_v = [&](int kt) {  // the state (written by the previous kernel) (+ its sum plane)
    const int s = kt % Cfg::STAGES;
    uint8_t* st = smem + s * S::STAGE_BYTES;
    tma_load_2d(st + OFF_A, &tmap_v, kt * 16, m0, &full[s]);
    if constexpr (SUMS) tma_load_2d(st + OFF_AS, &tmap_vs, kt * 8, m0, &full[s]);
  };

  griddep_launch_dependents();
  if (threadIdx.x == 0) {
    for (int s = 0; s < Cfg::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], Cfg::WARPS);
    }
    fence_barrier_init();
    prefetch_tmap(&tmap_v);
    prefetch_tmap(&tmap_g);
    if constexpr (SUMS) {
      prefetch_tmap(&tmap_vs);
      prefetch_tmap(&tmap_gs);
    }
    for (int kt = 0; kt < Cfg::STAGES && kt < KT; ++kt) issue_g(kt);
    griddep_wait();
    for (int kt = 0; kt < Cfg::STAGES && kt < KT; ++kt) issue_v(kt);
  }
  __syncthreads();

  const int g = lane >> 2;
  const int t = lane & 3;
  const int warp_m = warp % Cfg::WARPS_M;
  const int warp_n = warp / Cfg::WARPS_M;
  constexpr int MF = Cfg::MF, NF = Cfg::NF3;

  double t1[MF][NF][2], t2[MF][NF][2], t3[MF][NF][2];
#pragma unroll
  for (int i = 0; i < MF; ++i)
#pragma unroll
    for (int j = 0; j < NF; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) t1[i][j][e] = t2[i][j][e] = t3[i][j][e] = 0.0;

  for (int kt = 0; kt < KT; ++kt) {
    const int s = kt % Cfg::STAGES;
    mbar_wait(&full[s], (kt / Cfg::STAGES) & 1);
    const uint8_t* st = smem + s * S::STAGE_BYTES;
    const uint8_t* As = st + OFF_A + (warp_m * Cfg::WM + g) * 128;
    const uint8_t* Bs = st + OFF_B + warp_n * NF * (Cfg::BK_C * 128);
    const uint8_t* Ass = st + OFF_AS + (warp_m * Cfg::WM + g) * 64;
    const uint8_t* Bss = st + OFF_BS;
#pragma unroll
    for (int step = 0; step < 2; ++step) {
      const int i = 2 * t + step;  // complex k of this lane: row of the Gamma box, chunk of the V row
      double ar[MF], ai[MF], as[MF], br[NF], bi[NF], bs[NF];
#pragma unroll
      for (int mf = 0; mf < MF; ++mf) {
        const double2 v = *reinterpret_cast<const double2*>(As + mf * 8 * 128 + ((i ^ g) << 4));
        ar[mf] = v.x;
        ai[mf] = v.y;
        if constexpr (SUMS) {
          // 64B swizzle: 16B chunk t of a 64B row XOR (row >> 1) & 3, row & 7 == g
          as[mf] = *reinterpret_cast<const double*>(Ass + mf * 8 * 64 + ((t ^ ((g >> 1) & 3)) << 4) + (step << 3));
        } else {
          as[mf] = __dadd_rn(v.x, v.y);
        }
      }
#pragma unroll
      for (int nf = 0; nf < NF; ++nf) {
        const double2 w = *reinterpret_cast<const double2*>(Bs + nf * (Cfg::BK_C * 128) + i * 128 + ((g ^ i) << 4));
        br[nf] = w.x;
        bi[nf] = w.y;
        if constexpr (SUMS) {
          // sum boxes: 8 rows x 16 doubles (complex cols); fragment fi covers cols 8 fi .. 8 fi + 7:
          // box fi/2, col (fi&1)*8 + g -> 16B chunk ((fi&1)*4 + g/2) ^ i (128B swizzle, row i)
          const int fi = warp_n * NF + nf;
          const int c = ((fi & 1) * 4 + (g >> 1)) ^ i;
          bs[nf] = *reinterpret_cast<const double*>(Bss + (fi >> 1) * 1024 + i * 128 + (c << 4) + ((g & 1) << 3));
        } else {
          bs[nf] = __dadd_rn(w.x, w.y);
        }
      }
#pragma unroll
      for (int mf = 0; mf < MF; ++mf)
#pragma unroll
        for (int nf = 0; nf < NF; ++nf) {
          dmma_8x8x4(t1[mf][nf][0], t1[mf][nf][1], ar[mf], br[nf]);
          dmma_8x8x4(t2[mf][nf][0], t2[mf][nf][1], ai[mf], bi[nf]);
          dmma_8x8x4(t3[mf][nf][0], t3[mf][nf][1], as[mf], bs[nf]);
        }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
    if (threadIdx.x == 0 && kt >= 1 && kt - 1 + Cfg::STAGES < KT) {
      mbar_wait(&empty[(kt - 1) % Cfg::STAGES], ((kt - 1) / Cfg::STAGES) & 1);
      // cross-proxy WAR: the warps' generic-proxy reads of this slot (ordered before us by the
      // empty barrier) must be ordered before the async-proxy (TMA) writes that refill it
      fence_proxy_async();
      issue_g(kt - 1 + Cfg::STAGES);
      issue_v(kt - 1 + Cfg::STAGES);
    }
  }

  // epilogue: lane holds complex columns 2t, 2t+1 of row g in each fragment
#pragma unroll
  for (int mf = 0; mf < MF; ++mf) {
    const int row = m0 + warp_m * Cfg::WM + mf * 8 + g;
    if (row >= n) continue;
    double2* crow = C + (long long)row * ldc;
#pragma unroll
    for (int nf = 0; nf < NF; ++nf) {
      const int col = (n0r >> 1) + warp_n * (Cfg::WN / 2) + nf * 8 + 2 * t;
#pragma unroll
      for (int e = 0; e < 2; ++e)
        if (col + e < N)
          crow[col + e] = make_double2(t1[mf][nf][e] - t2[mf][nf][e], t3[mf][nf][e] - (t1[mf][nf][e] + t2[mf][nf][e]));
    }
  }
}

// Sum plane of complex data: out[r * ld_out + c] = re + im (the exact DADD the 3M kernel forms)
__global__ void sum_plane_kernel(const double2* __restrict__ in, long long rows, int cols, double* __restrict__ out,
                                 int ld_out) {
  long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= rows * cols) return;
  const long long r = idx / cols;
  const int c = (int)(idx % cols);
  const double2 v = in[idx];
  out[r * ld_out + c] = __dadd_rn(v.x, v.y);
}

}  // namespace mps
