// ozaki_gemm.cuh — complex128 K1 emulated on the INT8 5th-gen tensor cores (Ozaki scheme I),
// product mode 8 (mps_set_gemm_mode(ctx, 8)) next to the FP64 DMMA 3M / 4M kernels.
//
// B200 has no FP64 tcgen05 kind, but it has kind::i8 at ~120x the DMMA rate.  Every fp64 row x
// of an operand is written as  x = 2^e * sum_{i<S} x_i 2^{-7(i+1)}  with signed 7-bit digits
// x_i (int8, |x_i| <= 127; e = frexp exponent of the row's max |x|, so the digit expansion is
// exact up to 2^{-7S} of the row scale).  A product of two rows is then
//   a.b = 2^{e_a + e_b} sum_d 2^{-7(d+2)} sum_{i+j=d} a_i . b_j
// where every a_i . b_j is an exact int32 dot product, and a diagonal's int32 accumulator holds
// at most S products: |sum| <= S K 127^2 < 2^31 needs K (real) <= 18862 for S = 7, so a longer K
// runs as several launches of <= 588 K steps, each adding its fp64 partial into C.  Diagonals d = i + j >= S are dropped (their weight is
// <= 2^{-7(S+2)}: S = 7 leaves ~1e-13 of the row scales, far inside the 1e-10 parity bar;
// tests/test_gpu_parity.py checks it).
//
// Complex product: real-doubled 4M (like the complex64 kernel), so A = the interleaved state
// (n x 2K, one exponent per sample) and B = B_r^T (2N x 2K, one exponent per output real
// column), both K-major int8 digit planes in a tiled global layout that equals the shared-memory
// stage layout (one bulk copy per operand slice and K step).  The default kernel
// (ozaki2_gemm_kernel) gives every 128 x 128 output tile to a CTA pair that splits the diagonals;
// ozaki_gemm_kernel (MPS_OZ_KERNEL=v1) keeps all S diagonals in one CTA at N = 64.  Digit planes
// of a site are built once (mps_set_site / first use); the state's by ozaki_slice_rows_kernel
// after each draw.
#pragma once
#include <type_traits>
#include "c64_gemm.cuh"
#include "ptx.cuh"

namespace mps {

constexpr int OZ_MAX_S = 7;
constexpr int OZ_MAX_K = 9400;  // complex K per launch of the single-CTA kernel: 7 x (2 K) x 127^2 < 2^31
constexpr int OZ_SEG_KB = 588;  // 32-byte K steps per launch of the pair kernel (18816 reals, same bound)

// K-major, 32-byte swizzle (rows of 32 B = one K step); sbo = byte stride between 8-row atoms
__device__ __forceinline__ uint64_t umma_desc_k_sw32(uint32_t saddr, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
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

// digits of x * 2^-e (|x| < 2^e): d_i = trunc(128 t), t <- 128 t - d_i (all exact in fp64);
// digit i goes to out[i * 256] (the next plane's atom, see the tiled layout below)
__device__ __forceinline__ void ozaki_digits(double x, int e, int S, int8_t* out) {
  double t = ldexp(x, -e);
  for (int i = 0; i < S; ++i) {
    t *= 128.0;
    const double d = trunc(t);
    out[i * 256] = (int8_t)(int)d;
    t -= d;
  }
}

// Tiled global layout of the int8 digit planes = the kernels' shared-memory stage layout, so a
// CTA fetches its slice of a stage with ONE linear bulk copy (TMA tensor boxes of 32-byte rows
// move ~1 row per clock and starved the tensor pipe).  Rows are cut into tiles of TR rows and K
// into 32-byte steps; for (tile t, k step k) the bytes of all S planes are contiguous as
//   [8-row group g][plane i][8 rows][32 B, 32B-swizzled]   (S * TR * 32 bytes)
// i.e. byte (row, kk, plane i) lives at
//   ((t * KS + kk / 32) * TR / 8 + (row % TR) / 8) * S * 256 + i * 256 + swz32((row % 8) * 32 + kk % 32)
// where swz32 swaps the two 16-byte halves of rows 4..7 of an 8 x 32 B atom (the SWIZZLE_32B
// pattern: byte-offset bit 4 ^= bit 7), exactly what a 32B-swizzled TMA box would have written.
constexpr int OZ_TR_A = 128;  // state tiles (M)
constexpr int OZ_TR_B = 64;   // site tiles (N): both kernels' B slices lie inside one 64-row tile
__host__ __device__ __forceinline__ long long oz_tiled(int row, int kk, int TR, int KS, int S) {
  const int o = (row & 7) * 32 + (kk & 31);
  const int sw = o ^ (((o >> 7) & 1) << 4);
  return ((((long long)(row / TR) * KS + kk / 32) * (TR / 8) + (row % TR) / 8) * S) * 256 + sw;
}
// start of the slice of rows [r0, r0 + 8 G) (inside one tile) at k step k; size G * S * 256 bytes
__host__ __device__ __forceinline__ long long oz_slice(int r0, int k, int TR, int KS, int S) {
  return ((((long long)(r0 / TR) * KS + k) * (TR / 8) + (r0 % TR) / 8) * S) * 256;
}

__device__ __forceinline__ void bulk_load_mc(void* smem_dst, const void* src, uint32_t bytes, uint64_t* bar,
                                             uint16_t mask) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1], %2, [%3], %4;" ::
          "r"(smem_u32(smem_dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "h"(mask)
      : "memory");
}

// Shared-memory tile layout: [row group of 8][digit plane][8 rows][32 B], i.e. the 8-row x 32-B
// swizzle atoms of all S planes of a row group are adjacent.  One 4-D TMA box
// {32 B, 8 rows, S planes, groups} (global: rows at pitch ld, planes at plane_stride, groups at
// 8 ld) lands in exactly this order, so a CTA fetches a slice of rows for every digit plane with
// ONE copy, and plane i of the tile is the UMMA operand at base + 256 i with atom stride S * 256.
template <int S_, int CM_, int CN_>
struct OzCfg {
  static constexpr int S = S_;
  static constexpr int CM = CM_, CN = CN_;  // cluster: CM CTAs along M share B, CN along N share A
  static constexpr int BM = 128, BN = 64, BK = 32, STAGES = 5;
  static constexpr int A_BYTES = S * BM * BK;  // all digit planes of the A tile (S x 4 KiB)
  static constexpr int B_BYTES = S * BN * BK;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int A_SLICE_ROWS = BM / CN, B_SLICE_ROWS = BN / CM;
  static constexpr int ATOM_STRIDE = S * 256;  // bytes between 8-row atoms of one plane
  static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 + 2 * STAGES * 8 + 8 + 16;
  static constexpr int TMEM_COLS = (S * BN <= 256) ? 256 : 512;
  static constexpr int THREADS = 192;
  static_assert(S * BN <= 512, "diagonal accumulators exceed TMEM");
  static_assert(A_SLICE_ROWS % 8 == 0 && B_SLICE_ROWS % 8 == 0, "slices are whole 8-row atoms");
};

// C (n x N complex128 = n x 2N real, interleaved) from the digit planes:
//   tm_a : 4-D view {K bytes, 8, S, n_pad / 8} of the state's S planes (n_pad x ld bytes each)
//   tm_b : the same over the site's 2N (padded b_pad) B_r^T rows
//   ea[n], eb[2N]: exponents
// Clusters of CM x CN CTAs: CTA (x, y) fetches A slice y (BM / CN rows, all planes) and
// multicasts it to the CN CTAs of its M tile, and B slice x to the CM CTAs of its N tile, so the
// L2 -> SM traffic per CTA and K step is (BM / CN + BN / CM) S 32 B instead of (BM + BN) S 32 B
// (the CN = CM = 1 kernel is L2-bandwidth bound at 36% tensor-pipe activity).  A stage slot of
// CTA (x, y) is written by the CTAs of row x and column y of the cluster, so every CTA's MMA
// commit releases the slot to exactly those (empty barrier count CM + CN - 1).
template <class Cfg>
__global__ void __launch_bounds__(Cfg::THREADS, 1)
    ozaki_gemm_kernel(const int8_t* __restrict__ a_planes, const int8_t* __restrict__ b_planes,
                      const int* __restrict__ ea, const int* __restrict__ eb, double* __restrict__ C, int n, int N2,
                      int KB, long long ldc) {
  constexpr int S = Cfg::S, CM = Cfg::CM, CN = Cfg::CN;
  constexpr bool MC = CM * CN > 1;
  extern __shared__ __align__(16) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + Cfg::STAGES * Cfg::STAGE_BYTES);
  uint64_t* empty = full + Cfg::STAGES;
  uint64_t* tmem_full = empty + Cfg::STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_full + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m0 = blockIdx.x * Cfg::BM, n0 = blockIdx.y * Cfg::BN;
  // cluster coordinates (rank = x + CM y, the %cluster_ctarank order)
  const int cx = MC ? (int)(blockIdx.x % CM) : 0, cy = MC ? (int)(blockIdx.y % CN) : 0;
  uint16_t mask_a = 0, mask_b = 0;  // receivers of my A slice (my M tile) / my B slice (my N tile)
#pragma unroll
  for (int y = 0; y < CN; ++y) mask_a |= (uint16_t)(1u << (cx + CM * y));
#pragma unroll
  for (int x = 0; x < CM; ++x) mask_b |= (uint16_t)(1u << (x + CM * cy));

  griddep_launch_dependents();
  if (threadIdx.x == 0) {
    for (int s = 0; s < Cfg::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], CM + CN - 1);
    }
    mbar_init(tmem_full, 1);
    fence_barrier_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"((uint32_t)Cfg::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  if constexpr (MC) cluster_sync_all();  // peers' barriers initialised before any multicast lands
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {  // ---- bulk-copy producer: my A slice and my B slice of every digit plane ----
      griddep_wait();
      const uint32_t a_off = cy * (Cfg::A_SLICE_ROWS / 8) * Cfg::ATOM_STRIDE;
      const uint32_t b_off = cx * (Cfg::B_SLICE_ROWS / 8) * Cfg::ATOM_STRIDE;
      const int ar = m0 + cy * Cfg::A_SLICE_ROWS, br = n0 + cx * Cfg::B_SLICE_ROWS;
      constexpr uint32_t a_bytes = Cfg::A_SLICE_ROWS / 8 * Cfg::ATOM_STRIDE, b_bytes = Cfg::B_SLICE_ROWS / 8 * Cfg::ATOM_STRIDE;
      for (int kb = 0; kb < KB; ++kb) {
        const int s = kb % Cfg::STAGES;
        mbar_wait(&empty[s], ((kb / Cfg::STAGES) & 1) ^ 1);
        uint8_t* st = smem + s * Cfg::STAGE_BYTES;
        mbar_arrive_expect_tx(&full[s], Cfg::STAGE_BYTES);
        const int8_t* asrc = a_planes + oz_slice(ar, kb, OZ_TR_A, KB, S);
        const int8_t* bsrc = b_planes + oz_slice(br, kb, OZ_TR_B, KB, S);
        if constexpr (CN > 1)
          bulk_load_mc(st + a_off, asrc, a_bytes, &full[s], mask_a);
        else
          bulk_load_1d(st + a_off, asrc, a_bytes, &full[s]);
        if constexpr (CM > 1)
          bulk_load_mc(st + Cfg::A_BYTES + b_off, bsrc, b_bytes, &full[s], mask_b);
        else
          bulk_load_1d(st + Cfg::A_BYTES + b_off, bsrc, b_bytes, &full[s]);
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
            const uint64_t da = umma_desc_k_sw32(st + i * 256, Cfg::ATOM_STRIDE);
            const uint64_t db = umma_desc_k_sw32(st + Cfg::A_BYTES + j * 256, Cfg::ATOM_STRIDE);
            umma_i8(tmem + d * Cfg::BN, da, db, idesc, (kb != 0 || i != 0) ? 1u : 0u);
          }
        }
        if constexpr (MC)
          umma_commit_mc(&empty[s], (uint16_t)(mask_a | mask_b));  // free the slot for every writer into it
        else
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
  if constexpr (MC) cluster_sync_all();  // no CTA leaves while a peer may still multicast into it
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"((uint32_t)Cfg::TMEM_COLS));
  }
}

// ---------------------------------------------------------------------------------------------
// Diagonal-split kernel (the default Ozaki K1).  tools/umma_probe.cu measured kind::i8 M=128 MMAs
// at 48 clk for N=64 (operand reads: 4 KiB A + 2 KiB B at 128 B/clk) and 64 clk for N=128 (the
// full 8192 MAC/clk rate), so a 128 x 64 tile caps the tensor pipe at 2/3.  N=128 needs
// 128 TMEM columns per diagonal accumulator, and 7 diagonals do not fit 512 columns, so a CTA
// PAIR computes each 128 x 128 output tile: CTA z accumulates only its group of diagonals
// (S=7: {6,3,1,0} and {5,4,2}, 14 products each), both CTAs fetch half of the A rows and
// multicast them to the pair, and B is shared by the whole cluster (MP pairs along M).  The
// epilogue folds each group smallest-first in fp64, the pair swaps the halves it does not own
// through distributed shared memory, and the owner writes 2^(ea + eb) (fold_0 + fold_1).
// ---------------------------------------------------------------------------------------------
// diagonal groups of the two CTAs of a pair, descending (fold smallest weight first); -1 = none.
// S=7: {6,3,1,0} / {5,4,2} (14 products each); S=6: {5,2,1} / {4,3,0}; S=5: {4,1,0} / {3,2}.
__host__ __device__ constexpr int oz2_diag(int S, int z, int t) {
  return S == 7 ? (z == 0 ? (t == 0 ? 6 : t == 1 ? 3 : t == 2 ? 1 : 0) : (t == 0 ? 5 : t == 1 ? 4 : t == 2 ? 2 : -1))
       : S == 6 ? (z == 0 ? (t == 0 ? 5 : t == 1 ? 2 : t == 2 ? 1 : -1) : (t == 0 ? 4 : t == 1 ? 3 : t == 2 ? 0 : -1))
                : (z == 0 ? (t == 0 ? 4 : t == 1 ? 1 : t == 2 ? 0 : -1) : (t == 0 ? 3 : t == 1 ? 2 : -1));
}

template <int S_, int MP_, bool MC_ = true>
struct Oz2Cfg {
  static constexpr int S = S_, MP = MP_;  // MP pairs (M tiles) per cluster share B
  static constexpr bool MC = MC_;         // false: every CTA fetches whole tiles itself (no multicast)
  static constexpr int CL = 2 * MP;       // cluster size
  static constexpr int BM = 128, BN = 128, BK = 32, STAGES = S >= 7 ? 4 : 4;
  static constexpr int A_BYTES = S * BM * BK, B_BYTES = S * BN * BK;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int A_SLICE_ROWS = BM / 2, B_SLICE_ROWS = BN / CL;
  static constexpr int ATOM_STRIDE = S * 256;
  static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 + 2 * STAGES * 8 + 8 + 16;
  static constexpr int TMEM_COLS = 512;
  static constexpr int THREADS = 192;
  static_assert(STAGES * STAGE_BYTES >= BM * (BN / 2) * 8 + BM * 66 * 8 + BN * 8, "the epilogue reuses the stage buffers");
};

// int32 -> double without I2F.F64 (a slow conversion pipe): the bits 0x43300000:(x ^ 2^31) are
// 2^52 + x + 2^31 exactly, so one DADD removes the offset (exact; same value as (double)x)
__device__ __forceinline__ double oz_i2d(uint32_t x) {
  return __hiloint2double(0x43300000, (int)(x ^ 0x80000000u)) - 4503601774854144.0;  // 2^52 + 2^31
}

// x * 2^e, bit-identical to ldexp(x, e) (one correctly rounded multiply by an exact power of two)
__device__ __forceinline__ double oz_scale(double x, int e) {
  if (e >= -1022 && e <= 1023) return x * __longlong_as_double((long long)(e + 1023) << 52);
  return ldexp(x, e);
}

__device__ __forceinline__ uint32_t mapa_shared(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
__device__ __forceinline__ void st_dsmem_f64(uint32_t addr, double v) {
  asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(addr), "d"(v) : "memory");
}

template <class Cfg>
__global__ void __launch_bounds__(Cfg::THREADS, 1)
    ozaki2_gemm_kernel(const int8_t* __restrict__ a_planes, const int8_t* __restrict__ b_planes,
                       const int* __restrict__ ea, const int* __restrict__ eb, double* __restrict__ C, int n, int N2,
                       int KB, long long ldc, int KS, int kb0, int accumulate) {
  // K steps [kb0, kb0 + KB) of the KS of the tiled planes; accumulate: C += this segment's product
  // (K longer than the int32-exact OZ_SEG_KB steps runs as several launches, see launch_ozaki2)
  constexpr int S = Cfg::S, CL = Cfg::CL;
  extern __shared__ __align__(16) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + Cfg::STAGES * Cfg::STAGE_BYTES);
  uint64_t* empty = full + Cfg::STAGES;
  uint64_t* tmem_full = empty + Cfg::STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_full + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int rank = (int)(blockIdx.x % CL);  // cluster rank (1-D cluster along x)
  const int z = rank & 1, mp = rank >> 1;   // diagonal group, pair within the cluster
  const int m0 = (int)(blockIdx.x >> 1) * Cfg::BM, n0 = blockIdx.y * Cfg::BN;
  const uint16_t mask_a = (uint16_t)(3u << (2 * mp)), mask_all = (uint16_t)((1u << CL) - 1);

  griddep_launch_dependents();
  if (threadIdx.x == 0) {
    for (int s = 0; s < Cfg::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], Cfg::MC ? CL : 1);  // my slot is written by my pair (A) and the whole cluster (B)
    }
    mbar_init(tmem_full, 1);
    fence_barrier_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"((uint32_t)Cfg::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  int era = 0, eb0 = 0, eb1 = 0;
  if (warp == 0) {
    if (lane == 0) {  // ---- bulk-copy producer: A rows [z*64, +64) to my pair, B slice `rank` to all ----
      griddep_wait();
      const uint32_t a_off = z * (Cfg::A_SLICE_ROWS / 8) * Cfg::ATOM_STRIDE;
      const uint32_t b_off = rank * (Cfg::B_SLICE_ROWS / 8) * Cfg::ATOM_STRIDE;
      const int ar = m0 + z * Cfg::A_SLICE_ROWS, br = n0 + rank * Cfg::B_SLICE_ROWS;
      constexpr uint32_t a_bytes = Cfg::A_SLICE_ROWS / 8 * Cfg::ATOM_STRIDE, b_bytes = Cfg::B_SLICE_ROWS / 8 * Cfg::ATOM_STRIDE;
      for (int kb = 0; kb < KB; ++kb) {
        const int s = kb % Cfg::STAGES;
        mbar_wait(&empty[s], ((kb / Cfg::STAGES) & 1) ^ 1);
        uint8_t* st = smem + s * Cfg::STAGE_BYTES;
        mbar_arrive_expect_tx(&full[s], Cfg::STAGE_BYTES);
        if constexpr (Cfg::MC) {
          bulk_load_mc(st + a_off, a_planes + oz_slice(ar, kb0 + kb, OZ_TR_A, KS, S), a_bytes, &full[s], mask_a);
          bulk_load_mc(st + Cfg::A_BYTES + b_off, b_planes + oz_slice(br, kb0 + kb, OZ_TR_B, KS, S), b_bytes, &full[s],
                       mask_all);
        } else {
          bulk_load_1d(st, a_planes + oz_slice(m0, kb0 + kb, OZ_TR_A, KS, S), Cfg::A_BYTES, &full[s]);
          bulk_load_1d(st + Cfg::A_BYTES, b_planes + oz_slice(n0, kb0 + kb, OZ_TR_B, KS, S), Cfg::B_BYTES / 2,
                       &full[s]);
          bulk_load_1d(st + Cfg::A_BYTES + Cfg::B_BYTES / 2, b_planes + oz_slice(n0 + 64, kb0 + kb, OZ_TR_B, KS, S),
                       Cfg::B_BYTES / 2, &full[s]);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---- MMA issuer: my diagonals, accumulator slot t <- sum_{i+j=d_t} A_i . B_j ----
      constexpr uint32_t idesc = idesc_i8(Cfg::BM, Cfg::BN);
      auto kstep = [&](uint32_t st, int kb, auto zc) {
        constexpr int ZZ = decltype(zc)::value;
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          constexpr int dd[4] = {oz2_diag(S, ZZ, 0), oz2_diag(S, ZZ, 1), oz2_diag(S, ZZ, 2), oz2_diag(S, ZZ, 3)};
          const int d = dd[t];
#pragma unroll
          for (int i = 0; i <= d; ++i) {
            const uint64_t da = umma_desc_k_sw32(st + i * 256, Cfg::ATOM_STRIDE);
            const uint64_t db = umma_desc_k_sw32(st + Cfg::A_BYTES + (d - i) * 256, Cfg::ATOM_STRIDE);
            umma_i8(tmem + t * Cfg::BN, da, db, idesc, (kb != 0 || i != 0) ? 1u : 0u);
          }
        }
      };
      for (int kb = 0; kb < KB; ++kb) {
        const int s = kb % Cfg::STAGES;
        mbar_wait(&full[s], (kb / Cfg::STAGES) & 1);
        tc_fence_after();
        const uint32_t st = smem_u32(smem + s * Cfg::STAGE_BYTES);
        if (z == 0)
          kstep(st, kb, std::integral_constant<int, 0>{});
        else
          kstep(st, kb, std::integral_constant<int, 1>{});
        if constexpr (Cfg::MC)
          umma_commit_mc(&empty[s], mask_all);  // free the slot for every writer into it
        else
          umma_commit(&empty[s]);
      }
      umma_commit(tmem_full);
    }
  } else {
    // exponents of my rows / my half's columns: fetched while the mainloop runs
    const int rw = m0 + 32 * (warp & 3) + lane, cl = n0 + z * (Cfg::BN / 2) + 2 * lane;
    era = (rw < n) ? ea[rw] : 0;
    eb0 = (cl < N2) ? eb[cl] : 0;
    eb1 = (cl < N2) ? eb[cl + 1] : 0;
    mbar_wait(tmem_full, 0);
    tc_fence_after();
  }
  // every CTA of the cluster is past its mainloop: all stage buffers are free
  __syncthreads();
  cluster_sync_all();
  const int q = warp & 3;
  const int rl = 32 * q + lane;  // row within the tile = TMEM lane
  const int row = m0 + rl;
  const uint32_t tbase = tmem + ((uint32_t)(32 * q) << 16);
  double* part = reinterpret_cast<double*>(smem);  // [64 cols][128 rows] partial from the partner
  // fold my group's diagonals (smallest weight first) over 64 columns [cb, cb + 64) in 16-column
  // chunks; the TMEM loads of chunk k + 1 are in flight while chunk k is folded
  auto fold_half = [&](int cb, auto&& emit) {
    uint32_t r[2][4][16];
    auto tld = [&](int c0, uint32_t (&rr)[4][16]) {
#pragma unroll
      for (int t = 0; t < 4; ++t)
        if ((z ? oz2_diag(S, 1, t) : oz2_diag(S, 0, t)) >= 0) tmem_ld_32x32b_x16(tbase + t * Cfg::BN + c0, rr[t]);
    };
    tld(cb, r[0]);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      if (k + 1 < 4) tld(cb + 16 * (k + 1), r[(k + 1) & 1]);
      double acc[16];
#pragma unroll
      for (int c = 0; c < 16; ++c) acc[c] = 0.0;
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const int d = z ? oz2_diag(S, 1, t) : oz2_diag(S, 0, t);
        if (d >= 0) {
          const double w = __longlong_as_double((long long)(1023 - 7 * (d + 2)) << 52);  // 2^-7(d+2)
#pragma unroll
          for (int c = 0; c < 16; ++c) acc[c] = fma(oz_i2d(r[k & 1][t][c]), w, acc[c]);
        }
      }
      emit(16 * k, acc);
    }
  };
  if (warp >= 2) {  // ---- phase 1: fold the partner's half of the columns into its smem ----
    const int pc0 = (1 - z) * (Cfg::BN / 2);
    const uint32_t rpart = mapa_shared(smem_u32(part), (uint32_t)(rank ^ 1));
    fold_half(pc0, [&](int c0, double (&acc)[16]) {
#pragma unroll
      for (int c = 0; c < 16; ++c) st_dsmem_f64(rpart + (uint32_t)(((c0 + c) * Cfg::BM + rl) * 8), acc[c]);
    });
  }
  cluster_sync_all();
  if (warp >= 2) {  // ---- phase 2: my half = fold(mine) + partner's partial, scaled, stored ----
    const int oc0 = z * (Cfg::BN / 2);
    // my half tile, scaled, goes to smem rows (pitch 66 doubles: 16-B aligned rows, <= 4-way
    // bank conflicts) and each row leaves as one 512-byte bulk copy (async proxy)
    double* otile = part + (Cfg::BN / 2) * Cfg::BM;
    double* fcs = otile + Cfg::BM * 66;  // 2^eb of my half's columns
    if (warp == 2) {
      fcs[2 * lane] = oz_scale(1.0, eb0);
      fcs[2 * lane + 1] = oz_scale(1.0, eb1);
    }
    const double fr = oz_scale(1.0, era);  // 2^ea of my row: v 2^ea 2^eb is exact (powers of two)
    asm volatile("bar.sync 1, 128;" ::: "memory");  // epilogue warps only
    const double* cold = C + (long long)row * ldc + n0 + oc0;  // the previous segments' sum
    const bool add_old = accumulate && row < n;
    fold_half(oc0, [&](int c0, double (&acc)[16]) {
#pragma unroll
      for (int c = 0; c < 16; ++c) {
        const double v = (acc[c] + part[(c0 + c) * Cfg::BM + rl]) * fr * fcs[c0 + c];
        otile[rl * 66 + c0 + c] = (add_old && n0 + oc0 + c0 + c < N2) ? v + cold[c0 + c] : v;
      }
    });
    fence_proxy_async();  // generic-proxy smem writes -> visible to the bulk copy engine
    const int ncols = min(Cfg::BN / 2, N2 - (n0 + oc0));
    if (row < n && ncols > 0) {
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(C + (long long)row * ldc + n0 + oc0),
                   "r"(smem_u32(otile + rl * 66)), "r"((uint32_t)(ncols * 8))
                   : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");  // smem stays valid until read
    }
    tc_fence_before();
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"((uint32_t)Cfg::TMEM_COLS));
  }
}

// Digit planes of the real-doubled state in the tiled layout (TR = OZ_TR_A, KS = ld / 32 steps):
// one CTA per sample row of V (K complex = 2K reals); e = frexp exponent of max |x| (0 for an
// all-zero row).  Padding K bytes get zero digits; padding rows are never
// written (their products only reach output rows / columns that are not stored).
__global__ void ozaki_slice_rows_kernel(const double2* __restrict__ V, int K, int S, int8_t* __restrict__ planes,
                                        int ld, int* __restrict__ e_out) {
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
  // each thread slices 16 consecutive reals (a 16-byte run of every digit plane: one contiguous,
  // 16-byte aligned piece of the tiled layout) and stores it with one vector store per plane
  const int KS = ld / 32;
  const double sc = ldexp(1.0, -e);
  for (int c0 = 16 * threadIdx.x; c0 < ld; c0 += 16 * blockDim.x) {
    double t[16];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int kc = (c0 >> 1) + q;
      const double2 z = (2 * kc < 2 * K) ? v[kc] : make_double2(0.0, 0.0);
      t[2 * q] = z.x * sc;  // exact: a power-of-two scaling
      t[2 * q + 1] = z.y * sc;
    }
    int8_t* dst = planes + oz_tiled(b, c0, OZ_TR_A, KS, S);
    for (int i = 0; i < S; ++i) {
      uint32_t w[4] = {0u, 0u, 0u, 0u};
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        t[q] *= 128.0;
        const double d = trunc(t[q]);
        t[q] -= d;
        w[q >> 2] |= ((uint32_t)(uint8_t)(int8_t)(int)d) << (8 * (q & 3));
      }
      *reinterpret_cast<uint4*>(dst + i * 256) = make_uint4(w[0], w[1], w[2], w[3]);
    }
  }
}

// Digit planes of a site's B_r^T (2N rows x 2K): row 2c = (Gr, -Gi, ...), row 2c+1 = (Gi, Gr, ...)
// over the site's rows i; one CTA per B_r^T row r; tiled layout with TR = OZ_TR_B.
// G may be a column block of a wider site: element (i, c) at G[i * ldg + c], c < N (ldg = 0: N).
__global__ void ozaki_slice_site_kernel(const double2* __restrict__ G, int K, int N, int S, int8_t* __restrict__ planes,
                                        int ld, int* __restrict__ e_out, long long ldg = 0) {
  if (ldg == 0) ldg = N;
  __shared__ double red[32];
  const int r = blockIdx.x;
  const int c = r >> 1, q = r & 1;
  double m = 0.0;
  for (int i = threadIdx.x; i < K; i += blockDim.x) {
    const double2 g = G[(long long)i * ldg + c];
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
  const int KS = ld / 32;
  for (int kk = threadIdx.x; kk < ld; kk += blockDim.x) {
    double x = 0.0;
    if (kk < 2 * K) {
      const double2 g = G[(long long)(kk >> 1) * ldg + c];
      const int p = kk & 1;
      x = (p == 0) ? (q == 0 ? g.x : g.y) : (q == 0 ? -g.y : g.x);
    }
    ozaki_digits(x, e, S, planes + oz_tiled(r, kk, OZ_TR_B, KS, S));
  }
}

}  // namespace mps
