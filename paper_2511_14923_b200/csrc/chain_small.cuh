// chain_small.cuh — the whole mode chain of a small MPS in ONE persistent launch
// (at C1/C2 sizes the two-kernels-per-mode chain is bound by
// dependent-kernel latency, ~6.5 us per kernel at chi = 100, not by work).
//
// Eligible shapes: complex128, 3M product mode, every site chi_l <= 128 and chi_r D <= 1024.
//
// A cluster of 16 CTAs (non-portable size) owns a group of 16 sample rows (two DMMA row fragments)
// and walks every mode m of [m_begin, m_end) for it without leaving the kernel:
//   K1    CTA r computes C[16 rows, its 1/16 of the chi_r D columns] = V . Gamma^[m] with the 3M
//         DMMA product of site_gemm3m_kernel — same fragments, same k order, same epilogue
//         expression, operand sums formed with the same DADD — so C is bit-identical to the
//         per-mode chain (8 compute warps, one 8-column fragment each).  Gamma streams through a
//         6-slot ring (2 k-stages per slot, one 1-D bulk copy per k-stage) from a copy of the
//         site pre-arranged in the ring's swizzled fragment layout (chain_site_kernel); a producer
//         warp runs the ring ahead across modes, so the next site lands while this mode draws.
//   xchg  each lane st.async's its C entries straight into the shared memory of the row's owner
//         (CTA r owns row r), completing on the owner's mbarrier: no cluster-wide barrier.
//   K2+K3 CTA r runs displace_draw_kernel's pass 1 / draw / pass 2 on its row from shared memory
//         (same thread <-> j map, same reduction tree, same draw rule => same bits) and
//         st.async's v' into row r of every CTA's V tile (next mode's A operand).
// A third warp builds D(alpha) for the coming modes (double-buffered) off the critical path.
// Row groups are independent chains; clusters persist over groups.
#pragma once
#include <cstdint>

#include "c64_gemm.cuh"
#include "displace_draw.cuh"
#include "ptx.cuh"

namespace mps {

constexpr int SC_CL = 16;                         // CTAs per cluster == sample rows per group (non-portable size)
constexpr int SC_MF = SC_CL / 8;                  // DMMA row fragments per group
constexpr int SC_KMAX = 128;                      // chi_l bound
constexpr int SC_NMAX = 1024;                     // chi_r * D bound (complex columns)
constexpr int SC_FMAX = SC_NMAX / 8 / SC_CL;      // 8-column fragments per CTA (8)
constexpr int SC_FW = SC_FMAX / 8;                // per compute warp (1)
#ifndef SC_KS_DEF  // tuning knob of tools/chain_trace.py
#define SC_KS_DEF 3
#endif
constexpr int SC_KS = SC_KS_DEF;                  // k stages (8 complex k each) per ring slot: one mbarrier
                                                  // wait (a pipeline drain) per slot; 3 measured best at C2
                                                  // (profiles/r02_small_chain_ring_sweep.txt)
#ifndef SC_KSTAGES_DEF  // k stages of Gamma in flight (tuning knob)
#define SC_KSTAGES_DEF 12
#endif
constexpr int SC_STAGES = SC_KSTAGES_DEF / SC_KS; // ring slots (12 k stages = 96 KB of Gamma in flight)
#ifndef SC_KW
#define SC_KW 8
#endif
// compute warps: 8 (each one 8-column fragment x both 8-row fragments) or 16 (one 8 x 8 fragment
// each: twice the warps to hide the LDS -> DMMA latency of the 16-row K1 slice; every output element
// still accumulates over k in the same order, so the bits do not change)
constexpr int SC_COMPUTE = SC_KW * 32;
constexpr int SC_MFW = SC_KW == 16 ? 1 : SC_MF;   // row fragments per compute warp
constexpr int SC_THREADS = SC_COMPUTE + 64;       // + ring producer warp + D(alpha) warp
constexpr int SC_STAGE_BYTES = SC_KS * SC_FMAX * 1024;  // SC_KS x fc blocks of (8 k rows x 8 complex), swizzled
constexpr int SC_VP = SC_KMAX * 16 + 16;          // V row pitch: == 16 mod 128 -> conflict-free LDS.128
constexpr int SC_OFF_V = SC_STAGES * SC_STAGE_BYTES;
constexpr int SC_OFF_C = SC_OFF_V + SC_CL * SC_VP;      // owned C row, 2 buffers (step parity)
constexpr int SC_OFF_T = SC_OFF_C + 2 * SC_NMAX * 16;   // D(alpha), 2 buffers
constexpr int SC_OFF_BAR = SC_OFF_T + 2 * DMAX * DMAX * 16;
constexpr int SC_NBAR = 2 * SC_STAGES + 2 + 1 + 2 + 2;  // full, empty, c_full x2, v_full, t_full x2, t_free x2
constexpr int SC_SMEM = SC_OFF_BAR + SC_NBAR * 8 + 1024 /*align*/;
static_assert(DRAW_THREADS <= SC_COMPUTE, "the draw's 128-thread j map runs on the first compute warps");

struct ChainArgs {
  const double2* const* sites;  // device array: chain layout of Gamma^[m] (chain_site_kernel), per m
  const int* chi;               // device array chi_0 .. chi_M
  int m_begin, m_end, n;
  const double2* state_in;      // n x chi_{m_begin}, or null (chi_{m_begin} = 1: v = 1)
  double2* state_out;           // n x chi_{m_end}, or null
  DrawArgs d;                   // C, v_out, vs_out, C32 and the plane outputs are unused
};

// Gamma (K x N complex, row-major) -> blocks (kt, f) of 1 KB: row i (k = 8 kt + i) holds complex
// columns 8 f .. 8 f + 7, column c in 16-byte chunk c ^ i (the TMA 128B swizzle site_gemm3m_kernel
// reads); zero outside K x N.  One CTA stage is then a contiguous run of its fc blocks.
__global__ void chain_site_kernel(const double2* __restrict__ G, int K, int N, double2* __restrict__ out) {
  const int F = (N + 7) >> 3, KT = (K + 7) >> 3;
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (long long)KT * F * 64) return;
  const int blk = (int)(idx >> 6), e = (int)(idx & 63);
  const int kt = blk / F, f = blk % F, i = e >> 3, cc = e & 7;  // cc: chunk position
  const int c = cc ^ i;                                          // the column stored there
  const int k = 8 * kt + i, col = 8 * f + c;
  out[idx] = (k < K && col < N) ? G[(long long)k * N + col] : make_double2(0.0, 0.0);
}

#ifdef SC_TRACE  // debug build only (tools/chain_trace.py): clock64 stamps of CTA 0's phases
__device__ long long sc_trace[2][256][8];
#define SC_STAMP(who, q, k) \
  if (blockIdx.x == 0 && (q) < 256) sc_trace[who][q][k] = clock64();
#else
#define SC_STAMP(who, q, k)
#endif

__device__ __forceinline__ uint32_t sc_mapa(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
// 16-byte store into a peer CTA's shared memory, completing 16 tx bytes on the peer's mbarrier
__device__ __forceinline__ void sc_st_async(uint32_t addr, double x, double y, uint32_t bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];" ::"r"(addr),
               "d"(x), "d"(y), "r"(bar)
               : "memory");
}
__device__ __forceinline__ void sc_cluster_sync() {
  asm volatile("barrier.cluster.arrive.release;\nbarrier.cluster.wait.acquire;" ::: "memory");
}
__device__ __forceinline__ void sc_bar_compute() { asm volatile("bar.sync 1, %0;" ::"n"(SC_COMPUTE) : "memory"); }

template <int DT>
__global__ void __launch_bounds__(SC_THREADS, 1) small_chain_kernel(const __grid_constant__ ChainArgs P) {
  extern __shared__ __align__(16) uint8_t sc_raw[];
  uint8_t* smem = sc_raw + ((1024u - (smem_u32(sc_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + SC_OFF_BAR);
  uint64_t* empty = full + SC_STAGES;
  uint64_t* c_full = empty + SC_STAGES;  // [2]: this CTA's C row of step q landed (parity q & 1)
  uint64_t* v_full = c_full + 2;         // the next V tile landed
  uint64_t* t_full = v_full + 1;         // [2]: D(alpha) of step q built
  uint64_t* t_free = t_full + 2;         // [2]: the draw of step q is done with it
  uint8_t* Vt = smem + SC_OFF_V;
  __shared__ double red[DRAW_THREADS / 32][DMAX];
  __shared__ double p_s[DMAX];
  __shared__ int k_s;
  __shared__ double pk_s;
  __shared__ uint8_t st_s;

  const DrawArgs& A = P.d;
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int rank = (int)cluster_ctarank();
  const int cluster = blockIdx.x / SC_CL, nclusters = gridDim.x / SC_CL;
  const int D = DT ? DT : A.D;
  const int nmodes = P.m_end - P.m_begin;
  const int ngroups = (P.n + SC_CL - 1) / SC_CL;
  const int my_groups = cluster < ngroups ? (ngroups - cluster + nclusters - 1) / nclusters : 0;
  const int nsteps = my_groups * nmodes;  // step q: group cluster + (q / nmodes) nclusters, mode m_begin + q % nmodes
  const bool ident = !(A.disp || A.alpha || A.alpha_sigma >= 0.0);
  auto F_of = [&](int m) { return (P.chi[m + 1] * D + 7) >> 3; };
  auto row_of = [&](int q) { return (cluster + (q / nmodes) * nclusters) * SC_CL + rank; };

  if (tid == SC_COMPUTE) {
    for (int s = 0; s < SC_STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], SC_COMPUTE / 32);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&c_full[i], 1);
      mbar_init(&t_full[i], 1);
      mbar_init(&t_free[i], 1);
    }
    mbar_init(v_full, 1);
    fence_barrier_init();
    if (nsteps > 0) mbar_arrive_expect_tx(&c_full[0], (uint32_t)F_of(P.m_begin) * 128u);  // step 0's C row
  }
  __syncthreads();
  sc_cluster_sync();  // peers' barriers initialised (and step 0 expected) before any st.async lands
  // PDL: the Gamma ring (sites uploaded synchronously) may run ahead; every other warp reads inputs or
  // writes outputs that may belong to the previous kernel in the stream
  griddep_launch_dependents();
  if (warp != SC_COMPUTE / 32) griddep_wait();

  if (warp == SC_COMPUTE / 32) {
    // ===================== ring producer: Gamma stages of every step, in order =====================
    if (lane == 0) {
      uint32_t sidx = 0;
      for (int q = 0; q < nsteps; ++q) {
        const int m = P.m_begin + q % nmodes;
        const int KT = (P.chi[m] + 7) >> 3, F = F_of(m);
        const int f0 = rank * F / SC_CL, fc = (rank + 1) * F / SC_CL - f0;
        for (int kt = 0; kt < KT; kt += SC_KS, ++sidx) {
          const int slot = sidx % SC_STAGES, nks = min(SC_KS, KT - kt);
          if (sidx >= SC_STAGES) {
            mbar_wait(&empty[slot], ((sidx / SC_STAGES) - 1) & 1);
            fence_proxy_async();  // the consumers' ld.shared of the slot before the bulk-copy refill
          }
          mbar_arrive_expect_tx(&full[slot], (uint32_t)(nks * fc) * 1024u);
          if (fc)
            for (int ks = 0; ks < nks; ++ks)
              bulk_load_1d(smem + slot * SC_STAGE_BYTES + ks * fc * 1024, P.sites[m] + (size_t)((kt + ks) * F + f0) * 64,
                           fc * 1024u, &full[slot]);
        }
      }
    }
    __syncwarp();
  } else if (warp == SC_COMPUTE / 32 + 1) {
    // ===================== D(alpha) of this CTA's row, one step ahead =====================
    for (int q = 0; q < nsteps; ++q) {
      if (q >= 2) mbar_wait(&t_free[q & 1], ((q >> 1) - 1) & 1);
      const int b = row_of(q);
      if (!ident && b < P.n) {  // displace_draw_kernel's construction, unchanged
        const int m = P.m_begin + q % nmodes;
        double2* T = reinterpret_cast<double2*>(smem + SC_OFF_T) + (q & 1) * DMAX * DMAX;
        if (A.disp) {
          const double2* src = A.disp + ((long long)b * A.M + m) * D * D;
          for (int e = lane; e < D * D; e += 32) T[e] = src[e];
        } else {
          const unsigned long long gi = (unsigned long long)(A.first_index + b);
          const double2 a = A.alpha ? A.alpha[(long long)b * A.M + m] : stream_alpha(A.seed, gi, A.M, m, A.alpha_sigma);
          if (lane == 0) displacement_column0(a, D, T);
          __syncwarp();
          for (int d = 1; d < D; ++d) {
            if (lane < D) T[lane * D + d] = displacement_entry(a, D, T, lane, d);
            __syncwarp();
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&t_full[q & 1]);
    }
  } else {
    // ======================= compute warps: K1 tile, exchange, draw =======================
    const int g = lane >> 2, t = lane & 3;
    uint32_t sidx = 0, vph = 0;
    double u_pref = 0.0;
    int k_pref = 0;
    const uint32_t vt_addr = smem_u32(Vt), c_addr = smem_u32(smem + SC_OFF_C);
    const uint32_t cbar_addr = smem_u32(c_full), vbar_addr = smem_u32(v_full);
    for (int q = 0; q < nsteps; ++q) {
      const int m = P.m_begin + q % nmodes;
      const int K = P.chi[m], chi_r = P.chi[m + 1];
      const int KT = (K + 7) >> 3, F = F_of(m);
      const int f0 = rank * F / SC_CL, fc = (rank + 1) * F / SC_CL - f0;
      const int b = row_of(q);
      const bool valid = b < P.n;
      const bool first = (m == P.m_begin), last = (m == P.m_end - 1);
      SC_STAMP(0, q, 0);
      if (first) {  // new group: V <- state_in rows (or v = 1), zero elsewhere
        const int grp0 = b - rank;
        for (int e = tid; e < SC_CL * SC_KMAX; e += SC_COMPUTE) {
          const int r = e / SC_KMAX, j = e % SC_KMAX;
          double2 v = make_double2(0.0, 0.0);
          if (grp0 + r < P.n && j < K)
            v = P.state_in ? P.state_in[(long long)(grp0 + r) * K + j] : make_double2(1.0, 0.0);
          *reinterpret_cast<double2*>(Vt + r * SC_VP + j * 16) = v;
        }
        if (tid == 0) st_s = valid ? A.status[b] : 0;
      } else {
        mbar_wait(v_full, vph & 1);  // every row's v' of the previous mode
        ++vph;
      }
      if (tid == 0) {
        // Why no cluster barrier per mode: a peer's C entries for step q+1 need that peer's K1(q+1), which
        // needs every row's v'(q+1) (or, at a group start, follows the peer's draw(q), which needed this
        // CTA's K1(q) entries) -- so they land only after this point; the expects below therefore
        // precede every transaction they count.  C rows alternate between two buffers (step parity):
        // step q+2 can only be written after this CTA's own draw(q) has sent v'(q+1) or, at a group
        // start, after its K1(q+1) -- both after draw(q) stopped reading buffer q & 1.
        if (q + 1 < nsteps) {  // expect the next step's C row and (inside a group) its V tile
          const int m1 = P.m_begin + (q + 1) % nmodes;
          mbar_arrive_expect_tx(&c_full[(q + 1) & 1], (uint32_t)F_of(m1) * 128u);
          if (m1 != P.m_begin) mbar_arrive_expect_tx(v_full, (uint32_t)(SC_CL * ((chi_r + 7) & ~7) * 16));
        }
        if (valid && A.forced) k_pref = A.counts[(long long)b * A.ld_c + m];
        if (valid && !A.forced) {
          const unsigned long long gi = (unsigned long long)(A.first_index + b);
          u_pref = A.u ? A.u[(long long)b * A.ld_u + m]
                       : philox_double(numpy_key0(A.seed), gi / 64, (gi % 64) * (uint64_t)A.M + m);
        }
      }
      sc_bar_compute();

      if (tid == 0) SC_STAMP(0, q, 7);
      // ---- K1: 3M DMMA over this CTA's fragments (site_gemm3m_kernel's inner loop, DADD sums) ----
      const int fbase = (warp % 8) * SC_FW;
      const int mf0 = SC_MFW == SC_MF ? 0 : warp / 8;  // this warp's first row fragment
      double t1[SC_MFW][SC_FW][2], t2[SC_MFW][SC_FW][2], t3[SC_MFW][SC_FW][2];
#pragma unroll
      for (int mf = 0; mf < SC_MFW; ++mf)
#pragma unroll
        for (int j = 0; j < SC_FW; ++j)
#pragma unroll
          for (int e = 0; e < 2; ++e) t1[mf][j][e] = t2[mf][j][e] = t3[mf][j][e] = 0.0;
      // one k stage (two DMMA k steps) of this warp's fragment, in site_gemm3m_kernel's per-accumulator
      // k order.  The fragment test is hoisted out of the loop: a branch around mma.sync inside the
      // loop costs a WARPSYNC per step and keeps the scheduler from overlapping one step's LDS with
      // the previous step's DMMAs.
      auto kstage = [&](const uint8_t* st, int kt) {
#pragma unroll
        for (int step = 0; step < 2; ++step) {
          const int i = 2 * t + step;
          const double2 w = *reinterpret_cast<const double2*>(st + fbase * 1024 + i * 128 + ((g ^ i) << 4));
          double2 v[SC_MFW];
#pragma unroll
          for (int mf = 0; mf < SC_MFW; ++mf)
            v[mf] = *reinterpret_cast<const double2*>(Vt + (8 * (mf0 + mf) + g) * SC_VP + (8 * kt + i) * 16);
          const double ws = __dadd_rn(w.x, w.y);
#pragma unroll
          for (int mf = 0; mf < SC_MFW; ++mf) {
            dmma_8x8x4(t1[mf][0][0], t1[mf][0][1], v[mf].x, w.x);
            dmma_8x8x4(t2[mf][0][0], t2[mf][0][1], v[mf].y, w.y);
            dmma_8x8x4(t3[mf][0][0], t3[mf][0][1], __dadd_rn(v[mf].x, v[mf].y), ws);
          }
        }
      };
      if (fbase < fc) {
        for (int kt0 = 0; kt0 < KT; kt0 += SC_KS, ++sidx) {
          const int slot = sidx % SC_STAGES;
#ifdef SC_TRACE
          const long long w0 = clock64();
#endif
          mbar_wait(&full[slot], (sidx / SC_STAGES) & 1);
#ifdef SC_TRACE
          if (tid == 0 && blockIdx.x == 0 && q < 256) sc_trace[1][q][0] += clock64() - w0;
#endif
          const uint8_t* st = smem + slot * SC_STAGE_BYTES;
          if (kt0 + SC_KS <= KT) {
#pragma unroll
            for (int ks = 0; ks < SC_KS; ++ks) kstage(st + ks * fc * 1024, kt0 + ks);
          } else {
            for (int ks = 0; kt0 + ks < KT; ++ks) kstage(st + ks * fc * 1024, kt0 + ks);
          }
          __syncwarp();
          if (lane == 0) mbar_arrive(&empty[slot]);
        }
      } else {  // no fragment in this mode: keep the ring's slot accounting
        for (int kt0 = 0; kt0 < KT; kt0 += SC_KS, ++sidx) {
          const int slot = sidx % SC_STAGES;
          mbar_wait(&full[slot], (sidx / SC_STAGES) & 1);
          __syncwarp();
          if (lane == 0) mbar_arrive(&empty[slot]);
        }
      }
      SC_STAMP(0, q, 1);
      // epilogue: row 8 mf + g of the group is owned by CTA 8 mf + g — st.async the entries there
#pragma unroll
      for (int mf = 0; mf < SC_MFW; ++mf) {
        const uint32_t owner = (uint32_t)(8 * (mf0 + mf) + g);
        const uint32_t dst = sc_mapa(c_addr + (uint32_t)((q & 1) * SC_NMAX * 16), owner);
        const uint32_t bar = sc_mapa(cbar_addr + (uint32_t)((q & 1) * 8), owner);
#pragma unroll
        for (int nf = 0; nf < SC_FW; ++nf) {
          const int fi = fbase + nf;
          if (fi < fc) {
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              const int col = 8 * (f0 + fi) + 2 * t + e;
              sc_st_async(dst + (uint32_t)col * 16u, t1[mf][nf][e] - t2[mf][nf][e],
                          t3[mf][nf][e] - (t1[mf][nf][e] + t2[mf][nf][e]), bar);
            }
          }
        }
      }

      // ---- K2 + K3 on row b (displace_draw_kernel, C from shared memory) ----
      mbar_wait(&c_full[q & 1], (q >> 1) & 1);
      mbar_wait(&t_full[q & 1], (q >> 1) & 1);
      SC_STAMP(0, q, 2);
      const double2* Crow = reinterpret_cast<const double2*>(smem + SC_OFF_C) + (q & 1) * SC_NMAX;
      const double2* T = reinterpret_cast<const double2*>(smem + SC_OFF_T) + (q & 1) * DMAX * DMAX;
      const int jpad = (chi_r + 7) & ~7;
      // v' of j goes to row `rank` of every CTA's V tile, or to state_out after the last mode
      auto emit = [&](int j, double2 v) {
        if (last) {  // rows past n (padding of the last group) have no state_out row
          if (P.state_out && valid && j < chi_r) P.state_out[(long long)b * chi_r + j] = v;
          return;
        }
        const uint32_t vo = vt_addr + (uint32_t)(rank * SC_VP + j * 16);
#pragma unroll
        for (int p = 0; p < SC_CL; ++p) sc_st_async(sc_mapa(vo, (uint32_t)p), v.x, v.y, sc_mapa(vbar_addr, (uint32_t)p));
      };
      const long long crow = (long long)b * A.ld_c + m;
      const bool dead = !valid || (st_s & ST_FAILED) != 0;
      if (dead) {  // dead sample: zero state, count -1 (deterministic chain); invalid rows send zeros
        for (int j = tid; j < jpad; j += SC_COMPUTE) emit(j, make_double2(0.0, 0.0));
        if (valid && tid == 0 && !A.forced) A.counts[crow] = -1;
        if (valid && A.marg && tid < D) A.marg[crow * D + tid] = 0.0;
      } else {
        // pass 1 on warps 0-3 with the draw's 128-thread j map (the FP64 pipe is the bound, more warps
        // do not help): thread tid owns j = tid + 128 c
        constexpr int DR = DT ? DT : DMAX;
        if (warp < DRAW_THREADS / 32) {
          double acc[DR];
#pragma unroll
          for (int k = 0; k < DR; ++k) acc[k] = 0.0;
          for (int j = tid; j < chi_r; j += DRAW_THREADS) {
            const double2* src = Crow + j * D;
            bool done = false;
            if constexpr (DT > 0) {
              if (!ident) {  // d-outer / k-inner, as displace_draw_kernel (same per-k operation order)
                double2 e[DR];
#pragma unroll
                for (int k = 0; k < DR; ++k) e[k] = make_double2(0.0, 0.0);
#pragma unroll
                for (int d = 0; d < DR; ++d) {
                  const double2 cd = src[d];
#pragma unroll
                  for (int k = 0; k < DR; ++k) {
                    const double2 tk = lds_c128(&T[k * D + d]);
                    e[k].x = fma(tk.x, cd.x, e[k].x);
                    e[k].x = fma(-tk.y, cd.y, e[k].x);
                    e[k].y = fma(tk.x, cd.y, e[k].y);
                    e[k].y = fma(tk.y, cd.x, e[k].y);
                  }
                }
#pragma unroll
                for (int k = 0; k < DR; ++k) acc[k] = fma(e[k].x, e[k].x, fma(e[k].y, e[k].y, acc[k]));
                done = true;
              }
            }
            if (!done) {
              double2 c[DR];
#pragma unroll
              for (int d = 0; d < DR; ++d)
                if (DT || d < D) c[d] = src[d];
#pragma unroll
              for (int k = 0; k < DR; ++k) {
                if (!DT && k >= D) break;
                const double2 e = ident ? c[k] : disp_row<DT>(T, D, k, c);
                acc[k] = fma(e.x, e.x, fma(e.y, e.y, acc[k]));
              }
            }
          }
          if (tid == 0) SC_STAMP(0, q, 4);
          warp_tree_scatter(acc, red[warp], D);
        }
        sc_bar_compute();  // red[][] complete
        if (tid == 0) SC_STAMP(0, q, 5);
        if (warp == 0) {  // the draw (draw_row_warp, as displace_draw_kernel; u / forced k prefetched)
          const RowDraw r = draw_row_warp<DT>(red, DRAW_THREADS / 32, p_s, D, st_s, A.forced != 0,
                                              __shfl_sync(0xffffffffu, k_pref, 0), __shfl_sync(0xffffffffu, u_pref, 0),
                                              A.tie_eps);
          if (lane == 0) {
            st_s = r.status;
            k_s = r.k;
            pk_s = r.pk;
          }
          __syncwarp();
          named_bar_arrive(1, SC_COMPUTE);  // release pass 2; the bookkeeping stores are off its path
          if (A.marg && lane < D) A.marg[crow * D + lane] = (r.k >= 0) ? r.p / r.Ptot : 0.0;
          if (lane == 0) {
            A.status[b] = r.status;
            if (!A.forced) A.counts[crow] = r.k;
          }
        } else {
          sc_bar_compute();
        }
        if (tid == 0) SC_STAMP(0, q, 6);
        const int ks = k_s;
        const double pk = pk_s;
        for (int j = tid; j < jpad; j += SC_COMPUTE) {
          double2 e = make_double2(0.0, 0.0);
          if (j < chi_r && ks >= 0) {
            const double2* src = Crow + j * D;
            if (ident) {
              e = src[ks];
            } else {
#pragma unroll
              for (int d = 0; d < DR; ++d) {
                if (!DT && d >= D) break;
                const double2 c = src[d];
                const double2 tk = lds_c128(&T[ks * D + d]);
                e.x = fma(tk.x, c.x, e.x);
                e.x = fma(-tk.y, c.y, e.x);
                e.y = fma(tk.x, c.y, e.y);
                e.y = fma(tk.y, c.x, e.y);
              }
            }
            const double scale = row_scale(ks, pk);
            e = make_double2(e.x * scale, e.y * scale);
          }
          emit(j, e);
        }
      }
      SC_STAMP(0, q, 3);
      sc_bar_compute();  // every thread is done with T, st_s and red before they are reused
      if (tid == 0) mbar_arrive(&t_free[q & 1]);
    }
  }
  sc_cluster_sync();  // no CTA leaves while a peer may still st.async into it
}

}  // namespace mps
