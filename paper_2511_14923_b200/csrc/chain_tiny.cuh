// chain_tiny.cuh — the whole mode chain of a TINY MPS in one launch, one CTA per 8-row group and no
// cluster (BASELINE configs[0]: M = 8, chi = 16, D = 4).
//
// At chi <= 32 the 16-CTA cluster kernels (chain_small*.cuh) spend each mode on cross-CTA latency
// (C-row exchange, v' broadcast, peer skew: ~3 us per mode at C1) for a K1 of 8 rows x 64 columns
// x 16 k.  Here every site of the call's mode range sits in the CTA's shared memory (one bulk copy
// per site at launch, in chain_site_kernel's swizzled fragment layout), and one CTA of 8 warps walks
// an 8-row group (one DMMA row fragment) through all modes:
//   K1     warp w computes the 8-column fragments f = w, w + 8, ... of C = V . Gamma^[m] with
//          site_gemm3m_kernel's 3M DMMA product: same fragments, same per-accumulator k order, same
//          operand sums (DADD) and epilogue expression => C is bit-identical to the per-mode chain;
//   K2+K3  warp w then draws row w of the group: lane j < chi_r (<= 32) runs displace_draw_kernel's
//          pass 1 for its j (d-outer / k-inner FMAs), the xor-shuffle tree reduces over the lanes,
//          draw_row_warp applies the sampler.py:692-697 rule, and pass 2 writes v' into row w of the
//          V tile (or state_out after the last mode).  With chi_r <= 32 the 128-thread j map of the
//          per-mode draw puts every j in its warp 0 and adds exact zeros from warps 1-3, so this
//          one-warp reduction gives the same bits.
// Two CTA barriers per mode and nothing leaves the SM.  CTAs persist over groups (grid = min(groups,
// co-resident CTAs)), so the sites are loaded once per CTA.
#pragma once
#include <cstdint>

#include "chain_small.cuh"

namespace mps {

constexpr int TC_ROWS = 8;                          // sample rows per group (one DMMA row fragment)
constexpr int TC_W = 8;                             // warps: K1 fragments, then one row each
constexpr int TC_THREADS = TC_W * 32;
constexpr int TC_KMAX = 32;                         // chi_l bound (V tile width)
constexpr int TC_RMAX = 32;                         // chi_r bound (one lane per j in the draw)
constexpr int TC_NMAX = 256;                        // chi_r * D bound (C row)
constexpr int TC_MMAX = 64;                         // modes per call
constexpr int TC_VP = TC_KMAX * 16 + 16;            // V row pitch: == 16 mod 128 -> conflict-free LDS.128
constexpr int TC_OFF_V = 0;
constexpr int TC_OFF_C = TC_OFF_V + TC_ROWS * TC_VP;
constexpr int TC_OFF_T = TC_OFF_C + TC_ROWS * TC_NMAX * 16;
constexpr int TC_OFF_BAR = TC_OFF_T + TC_ROWS * DMAX * DMAX * 16;
constexpr int TC_OFF_SITES = (TC_OFF_BAR + TC_MMAX * 8 + 1023) & ~1023;
constexpr int TC_SMEM_MAX = 227 * 1024 - 4096;      // dynamic shared memory (static arrays + alignment slack)

__host__ __device__ constexpr int tc_site_bytes(int chi_l, int chi_r, int D) {
  return ((chi_l + 7) / 8) * ((chi_r * D + 7) / 8) * 1024;  // chain_site_kernel's layout, whole site
}

#ifdef TC_TRACE  // debug build only: clock64 stamps of CTA 0, warp 0, per mode
__device__ long long tc_trace[64][8];
#define TC_STAMP(q, k) \
  if (blockIdx.x == 0 && warp == 0 && lane == 0 && (q) < 64) tc_trace[q][k] = clock64();
#else
#define TC_STAMP(q, k)
#endif

template <int DT>
__global__ void __launch_bounds__(TC_THREADS, 1) tiny_chain_kernel(const __grid_constant__ ChainArgs P) {
  extern __shared__ __align__(16) uint8_t tc_raw[];
  uint8_t* smem = tc_raw + ((1024u - (smem_u32(tc_raw) & 1023u)) & 1023u);
  uint64_t* sbar = reinterpret_cast<uint64_t*>(smem + TC_OFF_BAR);  // site q of the range landed
  uint8_t* Vt = smem + TC_OFF_V;
  double2* Ct = reinterpret_cast<double2*>(smem + TC_OFF_C);
  __shared__ int soff[TC_MMAX];
  __shared__ double red[TC_W][DMAX];
  __shared__ double p_s[TC_W][DMAX];

  const DrawArgs& A = P.d;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3;
  const int D = DT ? DT : A.D;
  const int nmodes = P.m_end - P.m_begin;
  const int ngroups = (P.n + TC_ROWS - 1) / TC_ROWS;
  const bool ident = !(A.disp || A.alpha || A.alpha_sigma >= 0.0);
  double2* Tw = reinterpret_cast<double2*>(smem + TC_OFF_T) + warp * DMAX * DMAX;  // Q modes' D(alpha)
  const int Q = min(32, (DMAX * DMAX) / (D * D));  // modes per chunk of this warp's D(alpha) buffer

  // PDL: the next call's kernel may launch onto free SMs and stage its sites while this one runs
  griddep_launch_dependents();
  if (tid == 0) {
    int off = 0;
    for (int q = 0; q < nmodes; ++q) {
      const int m = P.m_begin + q;
      soff[q] = off;
      off += tc_site_bytes(P.chi[m], P.chi[m + 1], D);
      mbar_init(&sbar[q], 1);
    }
    fence_barrier_init();
    for (int q = 0; q < nmodes; ++q) {  // every site of the range, one bulk copy each
      const int m = P.m_begin + q;
      const uint32_t bytes = (uint32_t)tc_site_bytes(P.chi[m], P.chi[m + 1], D);
      mbar_arrive_expect_tx(&sbar[q], bytes);
      bulk_load_1d(smem + TC_OFF_SITES + soff[q], P.sites[m], bytes, &sbar[q]);
    }
  }
  // the sites and their metadata were written by synchronous uploads (mps_set_site); everything else
  // (inputs, status, state_in, outputs) may belong to the previous kernel in the stream
  griddep_wait();
  __syncthreads();

  for (int grp = blockIdx.x; grp < ngroups; grp += gridDim.x) {
    const int g0 = grp * TC_ROWS;
    const int b = g0 + warp;  // the row this warp draws
    const bool valid = b < P.n;
    {  // V <- state_in rows (or v = 1), zero elsewhere
      const int K0 = P.chi[P.m_begin];
      for (int e = tid; e < TC_ROWS * TC_KMAX; e += TC_THREADS) {
        const int r = e / TC_KMAX, j = e % TC_KMAX;
        double2 v = make_double2(0.0, 0.0);
        if (g0 + r < P.n && j < K0)
          v = P.state_in ? P.state_in[(long long)(g0 + r) * K0 + j] : make_double2(1.0, 0.0);
        *reinterpret_cast<double2*>(Vt + r * TC_VP + j * 16) = v;
      }
    }
    uint8_t st = valid ? A.status[b] : 0;  // this row's status (warp-uniform)
    double u_l = 0.0;  // lane l: the uniform (or forced outcome) of mode q0 + l of the current chunk
    int kf_l = 0;
    for (int q = 0; q < nmodes; ++q) {
      const int m = P.m_begin + q;
      const int K = P.chi[m], chi_r = P.chi[m + 1], N = chi_r * D;
      const int KT = (K + 7) >> 3, F = (N + 7) >> 3;
      const bool last = (q == nmodes - 1);
      const long long crow = (long long)b * A.ld_c + m;
      // ---- this row's uniforms / forced outcomes and D(alpha) for a chunk of Q modes at once ----
      // (lane-parallel: lane l takes mode q0 + l's uniform, lanes of group l / D build mode
      // q0 + p0 + l / D's matrix, so the Philox and the recurrences cost one latency per chunk, not
      // one per mode; same functions, same bits as displace_draw_kernel's construction)
      TC_STAMP(q, 0);
      if (q % Q == 0) {
        const int q0 = q, cnt = min(Q, nmodes - q);
        const unsigned long long gi = (unsigned long long)(A.first_index + b);
        u_l = 0.0;
        kf_l = 0;
        if (valid && lane < cnt) {
          const int mm = P.m_begin + q0 + lane;
          if (A.forced)
            kf_l = A.counts[(long long)b * A.ld_c + mm];
          else
            u_l = A.u ? A.u[(long long)b * A.ld_u + mm]
                      : philox_double(numpy_key0(A.seed), gi / 64, (gi % 64) * (uint64_t)A.M + mm);
        }
        if (valid && !ident) {
          if (A.disp) {
            const double2* src = A.disp + ((long long)b * A.M + P.m_begin + q0) * D * D;
            for (int e = lane; e < cnt * D * D; e += 32) Tw[e] = src[e];
          } else {
            const int per = 32 / D;  // modes per pass
            for (int p0 = 0; p0 < cnt; p0 += per) {
              const int qq = p0 + lane / D, k = lane % D;
              const bool act = lane / D < per && qq < cnt;
              double2* T = Tw + qq * D * D;
              double2 a = make_double2(0.0, 0.0);
              if (act) {
                const int mm = P.m_begin + q0 + qq;
                a = A.alpha ? A.alpha[(long long)b * A.M + mm] : stream_alpha(A.seed, gi, A.M, mm, A.alpha_sigma);
                if (k == 0) displacement_column0(a, D, T);
              }
              __syncwarp();
              for (int d = 1; d < D; ++d) {
                if (act) T[k * D + d] = displacement_entry(a, D, T, k, d);
                __syncwarp();
              }
            }
          }
        }
        __syncwarp();
      }
      const double u = __shfl_sync(0xffffffffu, u_l, q % Q);
      const int kf = __shfl_sync(0xffffffffu, kf_l, q % Q);
      const double2* Tq = Tw + (q % Q) * D * D;  // this mode's D(alpha)
      TC_STAMP(q, 1);
      __syncthreads();  // V of this mode (initial rows or every row's v') complete
      mbar_wait(&sbar[q], 0);
      TC_STAMP(q, 2);
      // ---- K1: 3M DMMA fragments (site_gemm3m_kernel's per-accumulator k order) ----
      const uint8_t* site = smem + TC_OFF_SITES + soff[q];
      for (int f = warp; f < F; f += TC_W) {
        double t1[2] = {0.0, 0.0}, t2[2] = {0.0, 0.0}, t3[2] = {0.0, 0.0};
        for (int kt = 0; kt < KT; ++kt) {
          const uint8_t* st8 = site + (kt * F + f) * 1024;
#pragma unroll
          for (int step = 0; step < 2; ++step) {
            const int i = 2 * t + step;
            const double2 w = *reinterpret_cast<const double2*>(st8 + i * 128 + ((g ^ i) << 4));
            const double2 v = *reinterpret_cast<const double2*>(Vt + g * TC_VP + (8 * kt + i) * 16);
            const double ws = __dadd_rn(w.x, w.y);
            dmma_8x8x4(t1[0], t1[1], v.x, w.x);
            dmma_8x8x4(t2[0], t2[1], v.y, w.y);
            dmma_8x8x4(t3[0], t3[1], __dadd_rn(v.x, v.y), ws);
          }
        }
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int col = 8 * f + 2 * t + e;
          Ct[g * TC_NMAX + col] = make_double2(t1[e] - t2[e], t3[e] - (t1[e] + t2[e]));
        }
      }
      TC_STAMP(q, 3);
      __syncthreads();  // C of the group complete; V free for this mode's v'
      TC_STAMP(q, 4);
      // ---- K2 + K3 on row b by warp `warp` ----
      const double2* Crow = Ct + warp * TC_NMAX;
      const int jpad = (chi_r + 7) & ~7;
      auto emit = [&](int j, double2 v) {
        if (last) {
          if (P.state_out && valid && j < chi_r) P.state_out[(long long)b * chi_r + j] = v;
          return;
        }
        *reinterpret_cast<double2*>(Vt + warp * TC_VP + j * 16) = v;
      };
      const bool dead = !valid || (st & ST_FAILED) != 0;
      if (dead) {
        for (int j = lane; j < jpad; j += 32) emit(j, make_double2(0.0, 0.0));
        if (valid && lane == 0 && !A.forced) A.counts[crow] = -1;
        if (valid && A.marg && lane < D) A.marg[crow * D + lane] = 0.0;
        continue;
      }
      constexpr int DR = DT ? DT : DMAX;
      double acc[DR];
#pragma unroll
      for (int k = 0; k < DR; ++k) acc[k] = 0.0;
      if (lane < chi_r) {  // pass 1 of j = lane
        const double2* src = Crow + lane * D;
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
                const double2 tk = lds_c128(&Tq[k * D + d]);
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
            const double2 e = ident ? c[k] : disp_row<DT>(Tq, D, k, c);
            acc[k] = fma(e.x, e.x, fma(e.y, e.y, acc[k]));
          }
        }
      }
      warp_tree_scatter(acc, red[warp], D);
      __syncwarp();
      TC_STAMP(q, 5);
      const RowDraw r = draw_row_warp<DT>(red + warp, 1, p_s[warp], D, st, A.forced != 0, kf, u, A.tie_eps);
      if (lane == 0) {
        A.status[b] = r.status;
        if (!A.forced) A.counts[crow] = r.k;
      }
      st = r.status;
      TC_STAMP(q, 6);
      const int ks = r.k;

      for (int j = lane; j < jpad; j += 32) {  // pass 2: gather + renormalise
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
              const double2 tk = lds_c128(&Tq[ks * D + d]);
              e.x = fma(tk.x, c.x, e.x);
              e.x = fma(-tk.y, c.y, e.x);
              e.y = fma(tk.x, c.y, e.y);
              e.y = fma(tk.y, c.x, e.y);
            }
          }
          const double scale = row_scale(ks, r.pk);
          e = make_double2(e.x * scale, e.y * scale);
        }
        emit(j, e);
      }
      // the normalised marginals leave after v' (p_s is rewritten only by this warp's next draw)
      if (A.marg && lane < D) A.marg[crow * D + lane] = (ks >= 0) ? r.p / r.Ptot : 0.0;
      TC_STAMP(q, 7);
    }
    __syncthreads();  // the group's last V / T reads are done before the next group overwrites them
  }
}

}  // namespace mps
