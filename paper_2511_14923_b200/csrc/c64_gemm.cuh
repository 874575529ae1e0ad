// c64_gemm.cuh — complex64 K1 on the 5th-gen tensor cores (tcgen05, kind::tf32), the
// "optional complex64 variant under a stated tolerance" of the north star.
//
// Precision: 3xTF32.  Every fp32 operand x is split into hi = rna_tf32(x) and lo = x - hi
// (exact in fp32); D += hi.hi + hi.lo + lo.hi accumulates in fp32 in TMEM, which recovers
// ~fp32 accuracy from the 10-bit-mantissa tensor path (parity bar 1e-4).
//
// Complex product: real-doubled 4M, like the FP64 4M kernel, so the accumulator holds C
// interleaved: A_r = V (n x 2K, K-major = V's own interleaved layout), B_r^T (2N x 2K,
// K-major) holds rows (Gr, -Gi, Gr, -Gi, ...) and (Gi, Gr, Gi, Gr, ...) per complex output
// column; it is built once per site (c64_site_planes_kernel).  State planes are written
// by the draw kernel (split_planes_kernel for a caller-supplied state).
//
// Kernel: one 128 x BN output tile per CTA, 6 warps: warp 0 issues TMA (4 boxes per stage:
// A hi/lo 128 x 32 fp32, B hi/lo BN x 32 fp32, 128B swizzle), warp 1 owns TMEM and one of its
// lanes issues tcgen05.mma (M=128, N=BN, K=8; 4 k-steps x 3 passes per stage) and commits
// stage release / accumulator-ready to mbarriers, warps 2-5 drain TMEM (tcgen05.ld 32x32b)
// to global fp32.  The k order (stage, k-step, pass) is fixed, so results do not depend on n.
#pragma once
#include "ptx.cuh"

namespace mps {

__device__ __forceinline__ uint64_t umma_desc_k_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);  // start address (16 B units)
  d |= (uint64_t)1 << 16;                    // leading byte offset: unused for swizzled K-major
  d |= (uint64_t)(1024 >> 4) << 32;          // stride byte offset: one 8-row x 128 B swizzle atom
  d |= (uint64_t)1 << 46;                    // descriptor version 1 (sm_100)
  d |= (uint64_t)2 << 61;                    // layout: SWIZZLE_128B
  return d;
}

// kind::tf32 instruction descriptor: D fp32, A/B tf32, both K-major, M x N
__host__ __device__ constexpr uint32_t idesc_tf32(int M, int N) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void umma_tf32(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
// multicast variants for a 2-CTA cluster sharing the B tile
__device__ __forceinline__ void umma_commit_mc(uint64_t* bar, uint16_t mask) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::
                   "r"(smem_u32(bar)),
               "h"(mask)
               : "memory");
}
__device__ __forceinline__ void tma_load_2d_mc(void* smem_dst, const CUtensorMap* map, int x, int y, uint64_t* bar,
                                               uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.multicast::cluster"
      " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_u32(bar)), "h"(mask)
      : "memory");
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void tmem_ld_32x32b_x32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// fp32 -> (hi, lo): hi = x rounded to tf32 (low 13 mantissa bits zero), lo = x - hi (exact)
__device__ __forceinline__ void split_tf32(float x, float& hi, float& lo) {
  uint32_t h;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(h) : "f"(x));
  hi = __uint_as_float(h);
  lo = __fsub_rn(x, hi);
}

template <int BN_, int STAGES_>
struct C64Cfg {
  static constexpr int BM = 128, BN = BN_, BK = 32, STAGES = STAGES_;
  static constexpr int A_BYTES = BM * BK * 4;  // 16 KiB per plane
  static constexpr int B_BYTES = BN * BK * 4;
  static constexpr int STAGE_BYTES = 2 * A_BYTES + 2 * B_BYTES;
  static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 + 2 * STAGES * 8 + 5 * 8 + 16;
  static constexpr int TMEM_COLS = BN;  // fp32 accumulator, BN <= 256 (power of 2)
  static constexpr int THREADS = 192;
};

// MC: launched as 2-CTA clusters along M; the two CTAs (same N tile) each fetch half of the
// B rows and multicast them to both, so each SM pulls 64 KiB instead of 96 KiB per stage
// from L2 (the kernel is L2-bandwidth-bound without it).  A slot is refilled only after
// both CTAs' MMAs released it (empty barriers count 2, commits multicast to the pair).
template <class Cfg, bool MC>
__global__ void __launch_bounds__(Cfg::THREADS, 1)
    c64_gemm_kernel(const __grid_constant__ CUtensorMap tm_ahi, const __grid_constant__ CUtensorMap tm_alo,
                    const __grid_constant__ CUtensorMap tm_bhi, const __grid_constant__ CUtensorMap tm_blo,
                    float* __restrict__ C, int n, int N2, int KB, long long ldc) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + Cfg::STAGES * Cfg::STAGE_BYTES);
  uint64_t* empty = full + Cfg::STAGES;
  uint64_t* tmem_full = empty + Cfg::STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_full + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m0 = blockIdx.x * Cfg::BM, n0 = blockIdx.y * Cfg::BN;

  const uint32_t crank = MC ? cluster_ctarank() : 0;
  griddep_launch_dependents();
  if (threadIdx.x == 0) {
    for (int s = 0; s < Cfg::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], MC ? 2 : 1);
    }
    mbar_init(tmem_full, 1);
    fence_barrier_init();
    prefetch_tmap(&tm_ahi);
    prefetch_tmap(&tm_alo);
    prefetch_tmap(&tm_bhi);
    prefetch_tmap(&tm_blo);
  }
  if (warp == 1) {  // TMEM allocation: one whole warp
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"((uint32_t)Cfg::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  if constexpr (MC) cluster_sync_all();  // peer barriers initialised before any remote arrive
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {  // ---- TMA producer ----
      griddep_wait();  // A planes come from the previous kernel
      for (int kb = 0; kb < KB; ++kb) {
        const int s = kb % Cfg::STAGES;
        mbar_wait(&empty[s], ((kb / Cfg::STAGES) & 1) ^ 1);
        uint8_t* st = smem + s * Cfg::STAGE_BYTES;
        mbar_arrive_expect_tx(&full[s], Cfg::STAGE_BYTES);
        tma_load_2d(st, &tm_ahi, kb * Cfg::BK, m0, &full[s]);
        tma_load_2d(st + Cfg::A_BYTES, &tm_alo, kb * Cfg::BK, m0, &full[s]);
        if constexpr (MC) {  // my half of the B rows, multicast to both CTAs of the pair
          const int half = Cfg::BN / 2;
          const uint32_t boff = crank * half * Cfg::BK * 4;
          tma_load_2d_mc(st + 2 * Cfg::A_BYTES + boff, &tm_bhi, kb * Cfg::BK, n0 + crank * half, &full[s], 0x3);
          tma_load_2d_mc(st + 2 * Cfg::A_BYTES + Cfg::B_BYTES + boff, &tm_blo, kb * Cfg::BK, n0 + crank * half,
                         &full[s], 0x3);
        } else {
          tma_load_2d(st + 2 * Cfg::A_BYTES, &tm_bhi, kb * Cfg::BK, n0, &full[s]);
          tma_load_2d(st + 2 * Cfg::A_BYTES + Cfg::B_BYTES, &tm_blo, kb * Cfg::BK, n0, &full[s]);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---- MMA issuer ----
      constexpr uint32_t idesc = idesc_tf32(Cfg::BM, Cfg::BN);
      for (int kb = 0; kb < KB; ++kb) {
        const int s = kb % Cfg::STAGES;
        mbar_wait(&full[s], (kb / Cfg::STAGES) & 1);
        tc_fence_after();
        const uint32_t st = smem_u32(smem + s * Cfg::STAGE_BYTES);
        const uint32_t ahi = st, alo = st + Cfg::A_BYTES, bhi = st + 2 * Cfg::A_BYTES, blo = bhi + Cfg::B_BYTES;
#pragma unroll
        for (int k = 0; k < Cfg::BK / 8; ++k) {  // K = 8 tf32 = 32 B per instruction
          const uint32_t off = k * 32;
          const uint64_t dah = umma_desc_k_sw128(ahi + off), dal = umma_desc_k_sw128(alo + off);
          const uint64_t dbh = umma_desc_k_sw128(bhi + off), dbl = umma_desc_k_sw128(blo + off);
          umma_tf32(tmem, dah, dbh, idesc, (kb | k) != 0);
          umma_tf32(tmem, dah, dbl, idesc, 1u);
          umma_tf32(tmem, dal, dbh, idesc, 1u);
        }
        if constexpr (MC)
          umma_commit_mc(&empty[s], 0x3);  // the slot is free for both CTAs' producers
        else
          umma_commit(&empty[s]);  // smem slot free once these MMAs have read it
      }
      umma_commit(tmem_full);  // accumulator complete
    }
  } else {
    // ---- epilogue: warps 2..5 drain TMEM lanes 32*(warp%4) .. +31 ----
    mbar_wait(tmem_full, 0);
    tc_fence_after();
    const int q = warp & 3;
    const int row = m0 + 32 * q + lane;
    float* crow = C + (long long)row * ldc;
#pragma unroll 1
    for (int c0 = 0; c0 < Cfg::BN; c0 += 32) {
      uint32_t r[32];
      tmem_ld_32x32b_x32(tmem + ((uint32_t)(32 * q) << 16) + c0, r);
      const int col = n0 + c0;
      if (row < n) {
        if (col + 32 <= N2 && (ldc & 3) == 0) {  // rows 16-B aligned: vector stores
#pragma unroll
          for (int j = 0; j < 32; j += 4)
            *reinterpret_cast<float4*>(crow + col + j) = make_float4(
                __uint_as_float(r[j]), __uint_as_float(r[j + 1]), __uint_as_float(r[j + 2]), __uint_as_float(r[j + 3]));
        } else if (col + 32 <= N2) {  // ldc = 2N is even: complex (8-B) stores are always aligned
#pragma unroll
          for (int j = 0; j < 32; j += 2)
            *reinterpret_cast<float2*>(crow + col + j) = make_float2(__uint_as_float(r[j]), __uint_as_float(r[j + 1]));
        } else {
#pragma unroll
          for (int j = 0; j < 32; ++j)
            if (col + j < N2) crow[col + j] = __uint_as_float(r[j]);
        }
      }
    }
    tc_fence_before();
  }
  __syncthreads();
  if constexpr (MC) cluster_sync_all();  // no CTA leaves while its peer may still signal it
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"((uint32_t)Cfg::TMEM_COLS));
  }
}

// Persistent variant: grid = min(tiles, SMs); CTA c walks tiles c, c + G, ... (m fastest).  Two
// TMEM accumulators (2 x BN columns): the MMA warp fills one while the epilogue warps drain the
// other, so a tile's epilogue overlaps the next tile's mainloop; the TMA ring runs across tiles.
template <class Cfg>
__global__ void __launch_bounds__(Cfg::THREADS, 1)
    c64_gemm_persistent_kernel(const __grid_constant__ CUtensorMap tm_ahi, const __grid_constant__ CUtensorMap tm_alo,
                               const __grid_constant__ CUtensorMap tm_bhi, const __grid_constant__ CUtensorMap tm_blo,
                               float* __restrict__ C, int n, int N2, int KB, long long ldc) {
  static_assert(2 * Cfg::BN <= 512, "two accumulators must fit TMEM");
  extern __shared__ __align__(16) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + Cfg::STAGES * Cfg::STAGE_BYTES);
  uint64_t* empty = full + Cfg::STAGES;
  uint64_t* acc_full = empty + Cfg::STAGES;  // [2]
  uint64_t* acc_empty = acc_full + 2;        // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);
  constexpr uint32_t TMEM_COLS = 2 * Cfg::BN <= 256 ? 256 : 512;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int MT = (n + Cfg::BM - 1) / Cfg::BM;
  const int ntiles = MT * ((N2 + Cfg::BN - 1) / Cfg::BN);
  const int my_tiles = (ntiles - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x;

  griddep_launch_dependents();
  if (threadIdx.x == 0) {
    for (int s = 0; s < Cfg::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&acc_full[a], 1);
      mbar_init(&acc_empty[a], 4);  // one arrive per epilogue warp
    }
    fence_barrier_init();
    prefetch_tmap(&tm_ahi);
    prefetch_tmap(&tm_alo);
    prefetch_tmap(&tm_bhi);
    prefetch_tmap(&tm_blo);
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {  // ---- TMA producer over all (tile, k-block) pairs ----
      griddep_wait();
      int g = 0;
      for (int q = 0; q < my_tiles; ++q) {
        const int tile = (int)blockIdx.x + q * (int)gridDim.x;
        const int m0 = (tile % MT) * Cfg::BM, n0 = (tile / MT) * Cfg::BN;
        for (int kb = 0; kb < KB; ++kb, ++g) {
          const int s = g % Cfg::STAGES;
          mbar_wait(&empty[s], ((g / Cfg::STAGES) & 1) ^ 1);
          uint8_t* st = smem + s * Cfg::STAGE_BYTES;
          mbar_arrive_expect_tx(&full[s], Cfg::STAGE_BYTES);
          tma_load_2d(st, &tm_ahi, kb * Cfg::BK, m0, &full[s]);
          tma_load_2d(st + Cfg::A_BYTES, &tm_alo, kb * Cfg::BK, m0, &full[s]);
          tma_load_2d(st + 2 * Cfg::A_BYTES, &tm_bhi, kb * Cfg::BK, n0, &full[s]);
          tma_load_2d(st + 2 * Cfg::A_BYTES + Cfg::B_BYTES, &tm_blo, kb * Cfg::BK, n0, &full[s]);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---- MMA issuer ----
      constexpr uint32_t idesc = idesc_tf32(Cfg::BM, Cfg::BN);
      int g = 0;
      for (int q = 0; q < my_tiles; ++q) {
        const int a = q & 1;
        mbar_wait(&acc_empty[a], ((q >> 1) & 1) ^ 1);  // the epilogue has drained this accumulator
        tc_fence_after();
        const uint32_t acc = tmem + a * Cfg::BN;
        for (int kb = 0; kb < KB; ++kb, ++g) {
          const int s = g % Cfg::STAGES;
          mbar_wait(&full[s], (g / Cfg::STAGES) & 1);
          tc_fence_after();
          const uint32_t st = smem_u32(smem + s * Cfg::STAGE_BYTES);
          const uint32_t ahi = st, alo = st + Cfg::A_BYTES, bhi = st + 2 * Cfg::A_BYTES, blo = bhi + Cfg::B_BYTES;
#pragma unroll
          for (int k = 0; k < Cfg::BK / 8; ++k) {
            const uint32_t off = k * 32;
            const uint64_t dah = umma_desc_k_sw128(ahi + off), dal = umma_desc_k_sw128(alo + off);
            const uint64_t dbh = umma_desc_k_sw128(bhi + off), dbl = umma_desc_k_sw128(blo + off);
            umma_tf32(acc, dah, dbh, idesc, (kb | k) != 0);
            umma_tf32(acc, dah, dbl, idesc, 1u);
            umma_tf32(acc, dal, dbh, idesc, 1u);
          }
          umma_commit(&empty[s]);
        }
        umma_commit(&acc_full[a]);
      }
    }
  } else {
    // ---- epilogue warps 2..5: drain accumulator q & 1 while the next tile accumulates ----
    const int qw = warp & 3;
    for (int q = 0; q < my_tiles; ++q) {
      const int a = q & 1;
      const int tile = (int)blockIdx.x + q * (int)gridDim.x;
      const int m0 = (tile % MT) * Cfg::BM, n0 = (tile / MT) * Cfg::BN;
      mbar_wait(&acc_full[a], (q >> 1) & 1);
      tc_fence_after();
      const int row = m0 + 32 * qw + lane;
      float* crow = C + (long long)row * ldc;
#pragma unroll 1
      for (int c0 = 0; c0 < Cfg::BN; c0 += 32) {
        uint32_t r[32];
        tmem_ld_32x32b_x32(tmem + a * Cfg::BN + ((uint32_t)(32 * qw) << 16) + c0, r);
        const int col = n0 + c0;
        if (row < n) {
          if (col + 32 <= N2 && (ldc & 3) == 0) {
#pragma unroll
            for (int j = 0; j < 32; j += 4)
              *reinterpret_cast<float4*>(crow + col + j) =
                  make_float4(__uint_as_float(r[j]), __uint_as_float(r[j + 1]), __uint_as_float(r[j + 2]),
                              __uint_as_float(r[j + 3]));
          } else if (col + 32 <= N2) {
#pragma unroll
            for (int j = 0; j < 32; j += 2)
              *reinterpret_cast<float2*>(crow + col + j) = make_float2(__uint_as_float(r[j]), __uint_as_float(r[j + 1]));
          } else {
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if (col + j < N2) crow[col + j] = __uint_as_float(r[j]);
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&acc_empty[a]);
    }
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS));
  }
}

// ---------------------------------------------------------------------------------------------
// CTA-pair variant (tcgen05.mma.cta_group::2): a 2-CTA cluster along M owns a 256 x BN tile.  CTA r
// loads its 128 A rows and its BN/2 B rows (hi / lo planes) into its own shared memory, both TMA
// loads completing on the LEADER's stage barrier; the leader's single MMA thread issues
// M = 256 MMAs that read A and B from both CTAs (each CTA's TMEM receives its 128 rows x BN); the
// commits multicast "slot free" / "accumulator ready" to both CTAs.  Per SM, a K = 8 step reads
// 4 KB of A and BN/2 x 32 B of B for 128 x BN x 8 MACs: half the B shared-memory traffic of the
// single-CTA kernel at the same tile width.  Same k order (stage, k-step, pass) as the other
// variants.
// ---------------------------------------------------------------------------------------------
template <int BN_, int STAGES_>
struct C64Cg2Cfg {
  static constexpr int BM = 128, BN = BN_, BK = 32, STAGES = STAGES_;
  static constexpr int A_BYTES = BM * BK * 4;             // per plane, this CTA's rows
  static constexpr int B_BYTES = (BN / 2) * BK * 4;       // per plane, this CTA's half of the B rows
  static constexpr int STAGE_BYTES = 2 * A_BYTES + 2 * B_BYTES;
  static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 + 2 * STAGES * 8 + 5 * 8 + 16;
  static constexpr int TMEM_COLS = BN;
  static constexpr int THREADS = 192;
};

__device__ __forceinline__ void umma_tf32_cg2(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void umma_commit_cg2(uint64_t* bar, uint16_t mask) {
  asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::
                   "r"(smem_u32(bar)),
               "h"(mask)
               : "memory");
}
// 2-D TMA load into this CTA's shared memory whose completion is signalled on the pair leader's
// mbarrier (bar_cluster: a shared::cluster address from mapa)
__device__ __forceinline__ void tma_load_2d_cg2(void* smem_dst, const CUtensorMap* map, int x, int y,
                                                uint32_t bar_cluster) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(bar_cluster)
      : "memory");
}

template <class Cfg>
__global__ void __launch_bounds__(Cfg::THREADS, 1)
    c64_gemm_cg2_kernel(const __grid_constant__ CUtensorMap tm_ahi, const __grid_constant__ CUtensorMap tm_alo,
                        const __grid_constant__ CUtensorMap tm_bhi, const __grid_constant__ CUtensorMap tm_blo,
                        float* __restrict__ C, int n, int N2, int KB, long long ldc) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + Cfg::STAGES * Cfg::STAGE_BYTES);
  uint64_t* empty = full + Cfg::STAGES;
  uint64_t* tmem_full = empty + Cfg::STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_full + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m0 = blockIdx.x * Cfg::BM, n0 = blockIdx.y * Cfg::BN;
  const uint32_t crank = cluster_ctarank();

  griddep_launch_dependents();
  if (threadIdx.x == 0) {
    for (int s = 0; s < Cfg::STAGES; ++s) {
      mbar_init(&full[s], 1);   // used on the leader: its arrive.expect_tx + both CTAs' TMA bytes
      mbar_init(&empty[s], 1);  // the leader's MMA commit, multicast to both CTAs
    }
    mbar_init(tmem_full, 1);
    fence_barrier_init();
    prefetch_tmap(&tm_ahi);
    prefetch_tmap(&tm_alo);
    prefetch_tmap(&tm_bhi);
    prefetch_tmap(&tm_blo);
  }
  if (warp == 1) {  // TMEM allocation for the pair: one warp in each CTA
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"((uint32_t)Cfg::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();  // both CTAs' barriers and TMEM ready before any cross-CTA signal
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {  // ---- TMA producer (both CTAs): my A rows and my half of the B rows ----
      griddep_wait();
      uint32_t lead_full;
      asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(lead_full) : "r"(smem_u32(full)));
      for (int kb = 0; kb < KB; ++kb) {
        const int s = kb % Cfg::STAGES;
        mbar_wait(&empty[s], ((kb / Cfg::STAGES) & 1) ^ 1);
        uint8_t* st = smem + s * Cfg::STAGE_BYTES;
        if (crank == 0) mbar_arrive_expect_tx(&full[s], 2 * Cfg::STAGE_BYTES);  // both CTAs' bytes
        const uint32_t fb = lead_full + (uint32_t)(s * 8);
        const int nb = n0 + (int)crank * (Cfg::BN / 2);
        tma_load_2d_cg2(st, &tm_ahi, kb * Cfg::BK, m0, fb);
        tma_load_2d_cg2(st + Cfg::A_BYTES, &tm_alo, kb * Cfg::BK, m0, fb);
        tma_load_2d_cg2(st + 2 * Cfg::A_BYTES, &tm_bhi, kb * Cfg::BK, nb, fb);
        tma_load_2d_cg2(st + 2 * Cfg::A_BYTES + Cfg::B_BYTES, &tm_blo, kb * Cfg::BK, nb, fb);
      }
    }
  } else if (warp == 1) {
    if (crank == 0 && lane == 0) {  // ---- MMA issuer: the leader only, M = 256 over the pair ----
      constexpr uint32_t idesc = idesc_tf32(2 * Cfg::BM, Cfg::BN);
      for (int kb = 0; kb < KB; ++kb) {
        const int s = kb % Cfg::STAGES;
        mbar_wait(&full[s], (kb / Cfg::STAGES) & 1);
        tc_fence_after();
        const uint32_t st = smem_u32(smem + s * Cfg::STAGE_BYTES);
        const uint32_t ahi = st, alo = st + Cfg::A_BYTES, bhi = st + 2 * Cfg::A_BYTES, blo = bhi + Cfg::B_BYTES;
#pragma unroll
        for (int k = 0; k < Cfg::BK / 8; ++k) {
          const uint32_t off = k * 32;
          const uint64_t dah = umma_desc_k_sw128(ahi + off), dal = umma_desc_k_sw128(alo + off);
          const uint64_t dbh = umma_desc_k_sw128(bhi + off), dbl = umma_desc_k_sw128(blo + off);
          umma_tf32_cg2(tmem, dah, dbh, idesc, (kb | k) != 0);
          umma_tf32_cg2(tmem, dah, dbl, idesc, 1u);
          umma_tf32_cg2(tmem, dal, dbh, idesc, 1u);
        }
        umma_commit_cg2(&empty[s], 0x3);  // both CTAs' slots are free once these MMAs read them
      }
      umma_commit_cg2(tmem_full, 0x3);  // both CTAs' accumulators complete
    }
  } else {
    // ---- epilogue (both CTAs): warps 2..5 drain TMEM lanes 32*(warp%4) .. +31 of this CTA's rows ----
    mbar_wait(tmem_full, 0);
    tc_fence_after();
    const int q = warp & 3;
    const int row = m0 + 32 * q + lane;
    float* crow = C + (long long)row * ldc;
#pragma unroll 1
    for (int c0 = 0; c0 < Cfg::BN; c0 += 32) {
      uint32_t r[32];
      tmem_ld_32x32b_x32(tmem + ((uint32_t)(32 * q) << 16) + c0, r);
      const int col = n0 + c0;
      if (row < n) {
        if (col + 32 <= N2 && (ldc & 3) == 0) {
#pragma unroll
          for (int j = 0; j < 32; j += 4)
            *reinterpret_cast<float4*>(crow + col + j) = make_float4(
                __uint_as_float(r[j]), __uint_as_float(r[j + 1]), __uint_as_float(r[j + 2]), __uint_as_float(r[j + 3]));
        } else if (col + 32 <= N2) {
#pragma unroll
          for (int j = 0; j < 32; j += 2)
            *reinterpret_cast<float2*>(crow + col + j) = make_float2(__uint_as_float(r[j]), __uint_as_float(r[j + 1]));
        } else {
#pragma unroll
          for (int j = 0; j < 32; ++j)
            if (col + j < N2) crow[col + j] = __uint_as_float(r[j]);
        }
      }
    }
    tc_fence_before();
  }
  __syncthreads();
  cluster_sync_all();  // no CTA releases TMEM while the pair's MMAs or its peer's epilogue may run
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"((uint32_t)Cfg::TMEM_COLS));
  }
}

// Persistent CTA-pair variant: each 2-CTA cluster walks pair tiles t = pair, pair + npairs, ... (m
// fastest).  Two TMEM accumulators per CTA (2 x BN = 512 columns): the leader's MMA fills one while
// both CTAs' epilogue warps drain the other, so a tile's epilogue overlaps the next tile's
// mainloop; the leader waits for all 8 epilogue warps of the pair (4 local arrivals + 4 remote)
// before reusing an accumulator.  Same k order, same bits as every other variant.
template <class Cfg>
__global__ void __launch_bounds__(Cfg::THREADS, 1)
    c64_gemm_cg2p_kernel(const __grid_constant__ CUtensorMap tm_ahi, const __grid_constant__ CUtensorMap tm_alo,
                         const __grid_constant__ CUtensorMap tm_bhi, const __grid_constant__ CUtensorMap tm_blo,
                         float* __restrict__ C, int n, int N2, int KB, long long ldc) {
  static_assert(2 * Cfg::BN <= 512, "two accumulators must fit TMEM");
  extern __shared__ __align__(16) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + Cfg::STAGES * Cfg::STAGE_BYTES);
  uint64_t* empty = full + Cfg::STAGES;
  uint64_t* acc_full = empty + Cfg::STAGES;  // [2] both CTAs: the leader's commit, multicast
  uint64_t* acc_empty = acc_full + 2;        // [2] leader: the pair's 8 epilogue warps
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);
  constexpr uint32_t TMEM_COLS = 2 * Cfg::BN <= 256 ? 256 : 512;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t crank = cluster_ctarank();
  const int MT2 = (n + 2 * Cfg::BM - 1) / (2 * Cfg::BM);  // pair tiles along M (256 rows each)
  const int ntiles = MT2 * ((N2 + Cfg::BN - 1) / Cfg::BN);
  const int pair = (int)blockIdx.x / 2, npairs = (int)gridDim.x / 2;
  const int my_tiles = pair < ntiles ? (ntiles - pair + npairs - 1) / npairs : 0;

  griddep_launch_dependents();
  if (threadIdx.x == 0) {
    for (int s = 0; s < Cfg::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&acc_full[a], 1);
      mbar_init(&acc_empty[a], 8);  // 4 epilogue warps per CTA of the pair
    }
    fence_barrier_init();
    prefetch_tmap(&tm_ahi);
    prefetch_tmap(&tm_alo);
    prefetch_tmap(&tm_bhi);
    prefetch_tmap(&tm_blo);
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {  // ---- TMA producer (both CTAs) over all (tile, k-block) pairs ----
      griddep_wait();
      uint32_t lead_full;
      asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(lead_full) : "r"(smem_u32(full)));
      int g = 0;
      for (int q = 0; q < my_tiles; ++q) {
        const int tile = pair + q * npairs;
        const int m0 = (tile % MT2) * 2 * Cfg::BM + (int)crank * Cfg::BM, n0 = (tile / MT2) * Cfg::BN;
        const int nb = n0 + (int)crank * (Cfg::BN / 2);
        for (int kb = 0; kb < KB; ++kb, ++g) {
          const int s = g % Cfg::STAGES;
          mbar_wait(&empty[s], ((g / Cfg::STAGES) & 1) ^ 1);
          uint8_t* st = smem + s * Cfg::STAGE_BYTES;
          if (crank == 0) mbar_arrive_expect_tx(&full[s], 2 * Cfg::STAGE_BYTES);
          const uint32_t fb = lead_full + (uint32_t)(s * 8);
          tma_load_2d_cg2(st, &tm_ahi, kb * Cfg::BK, m0, fb);
          tma_load_2d_cg2(st + Cfg::A_BYTES, &tm_alo, kb * Cfg::BK, m0, fb);
          tma_load_2d_cg2(st + 2 * Cfg::A_BYTES, &tm_bhi, kb * Cfg::BK, nb, fb);
          tma_load_2d_cg2(st + 2 * Cfg::A_BYTES + Cfg::B_BYTES, &tm_blo, kb * Cfg::BK, nb, fb);
        }
      }
    }
  } else if (warp == 1) {
    if (crank == 0 && lane == 0) {  // ---- MMA issuer: the leader ----
      constexpr uint32_t idesc = idesc_tf32(2 * Cfg::BM, Cfg::BN);
      int g = 0;
      for (int q = 0; q < my_tiles; ++q) {
        const int a = q & 1;
        mbar_wait(&acc_empty[a], ((q >> 1) & 1) ^ 1);  // both CTAs have drained this accumulator
        tc_fence_after();
        const uint32_t acc = tmem + a * Cfg::BN;
        for (int kb = 0; kb < KB; ++kb, ++g) {
          const int s = g % Cfg::STAGES;
          mbar_wait(&full[s], (g / Cfg::STAGES) & 1);
          tc_fence_after();
          const uint32_t st = smem_u32(smem + s * Cfg::STAGE_BYTES);
          const uint32_t ahi = st, alo = st + Cfg::A_BYTES, bhi = st + 2 * Cfg::A_BYTES, blo = bhi + Cfg::B_BYTES;
#pragma unroll
          for (int k = 0; k < Cfg::BK / 8; ++k) {
            const uint32_t off = k * 32;
            const uint64_t dah = umma_desc_k_sw128(ahi + off), dal = umma_desc_k_sw128(alo + off);
            const uint64_t dbh = umma_desc_k_sw128(bhi + off), dbl = umma_desc_k_sw128(blo + off);
            umma_tf32_cg2(acc, dah, dbh, idesc, (kb | k) != 0);
            umma_tf32_cg2(acc, dah, dbl, idesc, 1u);
            umma_tf32_cg2(acc, dal, dbh, idesc, 1u);
          }
          umma_commit_cg2(&empty[s], 0x3);
        }
        umma_commit_cg2(&acc_full[a], 0x3);
      }
    }
  } else {
    // ---- epilogue warps 2..5 of both CTAs: drain accumulator q & 1 of this CTA's 128 rows ----
    const int qw = warp & 3;
    uint32_t lead_empty;
    asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(lead_empty) : "r"(smem_u32(acc_empty)));
    for (int q = 0; q < my_tiles; ++q) {
      const int a = q & 1;
      const int tile = pair + q * npairs;
      const int m0 = (tile % MT2) * 2 * Cfg::BM + (int)crank * Cfg::BM, n0 = (tile / MT2) * Cfg::BN;
      mbar_wait(&acc_full[a], (q >> 1) & 1);
      tc_fence_after();
      const int row = m0 + 32 * qw + lane;
      float* crow = C + (long long)row * ldc;
#pragma unroll 1
      for (int c0 = 0; c0 < Cfg::BN; c0 += 32) {
        uint32_t r[32];
        tmem_ld_32x32b_x32(tmem + a * Cfg::BN + ((uint32_t)(32 * qw) << 16) + c0, r);
        const int col = n0 + c0;
        if (row < n) {
          if (col + 32 <= N2 && (ldc & 3) == 0) {
#pragma unroll
            for (int j = 0; j < 32; j += 4)
              *reinterpret_cast<float4*>(crow + col + j) =
                  make_float4(__uint_as_float(r[j]), __uint_as_float(r[j + 1]), __uint_as_float(r[j + 2]),
                              __uint_as_float(r[j + 3]));
          } else if (col + 32 <= N2) {
#pragma unroll
            for (int j = 0; j < 32; j += 2)
              *reinterpret_cast<float2*>(crow + col + j) = make_float2(__uint_as_float(r[j]), __uint_as_float(r[j + 1]));
          } else {
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if (col + j < N2) crow[col + j] = __uint_as_float(r[j]);
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0)  // this warp is done with accumulator a: tell the leader (local or remote arrive)
        asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(lead_empty + (uint32_t)(a * 8))
                     : "memory");
    }
  }
  __syncthreads();
  cluster_sync_all();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS));
  }
}

// Site planes: Gamma (K x N complex64) -> B_r^T hi / lo (2N rows x ld fp32, K-major, zero pad)
//   row 2c   : (Gr[i][c], -Gi[i][c]) at columns (2i, 2i+1)
//   row 2c+1 : (Gi[i][c],  Gr[i][c])
__global__ void c64_site_planes_kernel(const float2* __restrict__ G, int K, int N, float* __restrict__ bhi,
                                       float* __restrict__ blo, int ld) {
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long total = (long long)2 * N * ld;
  if (idx >= total) return;
  const int r = (int)(idx / ld), kk = (int)(idx % ld);
  float v = 0.f;
  if (kk < 2 * K) {
    const int c = r >> 1, q = r & 1, i = kk >> 1, p = kk & 1;
    const float2 g = G[(long long)i * N + c];
    v = (p == 0) ? (q == 0 ? g.x : g.y) : (q == 0 ? -g.y : g.x);
  }
  float h, l;
  split_tf32(v, h, l);
  bhi[idx] = h;
  blo[idx] = l;
}

// complex64 rows (rows x cols complex, contiguous) -> hi / lo fp32 planes (rows x ld, zero pad)
__global__ void split_planes_kernel(const float2* __restrict__ V, long long rows, int cols, float* __restrict__ hi,
                                    float* __restrict__ lo, int ld) {
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= rows * ld) return;
  const long long r = idx / ld;
  const int kk = (int)(idx % ld);
  float v = 0.f;
  if (kk < 2 * cols) {
    const float2 z = V[r * cols + (kk >> 1)];
    v = (kk & 1) ? z.y : z.x;
  }
  float h, l;
  split_tf32(v, h, l);
  hi[idx] = h;
  lo[idx] = l;
}

}  // namespace mps
