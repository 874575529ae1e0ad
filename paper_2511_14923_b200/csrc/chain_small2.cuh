// chain_small2.cuh — the small-chain kernel with the two 8-row halves of a group pipelined
// (DESIGN.md §3).
//
// small_chain_kernel walks a 16-row group mode by mode in lock step: K1 over all 16 rows, the C-row
// exchange, then every CTA's draw of its own row, then the state broadcast -- the cluster's FP64
// pipe idles while the rows draw, and the draws idle while K1 runs.  At C2 (chi = 100, n = 100:
// 7 groups) the step is exactly that chain, ~18 k cycles per mode.  Here the CTA is
// warp-specialised and the group is split into halves A (rows 0-7) and B (rows 8-15):
//   K1 warps (8)     K1_A(m) -> K1_B(m) -> K1_A(m+1) -> ...   one 8-column fragment x 8 rows each,
//                    the C entries st.async'ed to the row owners as each half finishes;
//   draw warps (4)   the owner's draw of its row: CTAs 0-7 draw half A while the K1 warps compute
//                    K1_B, CTAs 8-15 draw half B under K1_A of the next mode; v' goes to row r of
//                    every CTA's V tile (half r / 8 has its own "landed" barrier);
//   producer warp    the Gamma ring, streamed once per half (the second pass is an L2 hit);
//   D(alpha) warp    this CTA's row, one step ahead (double-buffered).
// Per output element K1 accumulates over k in site_gemm3m_kernel's order, the draw is
// displace_draw_kernel's 128-thread pass 1 / draw_row_warp / pass 2: every bit equals the per-mode
// chain and small_chain_kernel.
#pragma once
#include <cstdint>

#include "chain_small.cuh"

namespace mps {

constexpr int SC2_K1 = 256;                                      // 8 K1 warps
constexpr int SC2_DRAW = DRAW_THREADS;                           // 4 draw warps: the draw's j map
constexpr int SC2_THREADS = SC2_K1 + SC2_DRAW + 64;              // + ring producer + D(alpha) warp
constexpr int SC2_W_PROD = (SC2_K1 + SC2_DRAW) / 32, SC2_W_DALPHA = SC2_W_PROD + 1;
constexpr int SC2_NBAR = 2 * SC_STAGES + 2 + 2 + 2 + 2;          // full, empty, c_full[2], v_full[2], t_full[2], t_free[2]
constexpr int SC2_SMEM = SC_OFF_BAR + SC2_NBAR * 8 + 1024;

#ifdef SC_TRACE  // debug build only: clock64 stamps of cluster 0's CTA 0 (half A) and CTA 8 (half B)
__device__ long long sc2_trace[4][256][8];  // [0/1: K1 warp 0 of CTA 0 / 8][step][event], [2/3: draw warp 0]
#define SC2_STAMP(who, q, k)                                                              \
  if (blockIdx.x < SC_CL && (rank == 0 || rank == 8) && (q) < 256 && (threadIdx.x & 31) == 0) \
    sc2_trace[(who) + (rank == 8 ? 1 : 0)][q][k] = clock64();
#else
#define SC2_STAMP(who, q, k)
#endif

__device__ __forceinline__ void sc2_bar_k1() { asm volatile("bar.sync 2, %0;" ::"n"(SC2_K1) : "memory"); }
__device__ __forceinline__ void sc2_bar_draw() { asm volatile("bar.sync 3, %0;" ::"n"(SC2_DRAW) : "memory"); }

template <int DT>
__global__ void __launch_bounds__(SC2_THREADS, 1) small_chain2_kernel(const __grid_constant__ ChainArgs P) {
  extern __shared__ __align__(16) uint8_t sc_raw[];
  uint8_t* smem = sc_raw + ((1024u - (smem_u32(sc_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + SC_OFF_BAR);
  uint64_t* empty = full + SC_STAGES;
  uint64_t* c_full = empty + SC_STAGES;  // [2]: this CTA's C row of step q landed (parity q & 1)
  uint64_t* v_full = c_full + 2;         // [2]: half h of the next V tile landed
  uint64_t* t_full = v_full + 2;         // [2]: D(alpha) of step q built
  uint64_t* t_free = t_full + 2;         // [2]: the draw of step q is done with it
  uint8_t* Vt = smem + SC_OFF_V;
  __shared__ double red[DRAW_THREADS / 32][DMAX];
  __shared__ double p_s[DMAX];
  __shared__ int k_s;
  __shared__ double pk_s;
  __shared__ uint8_t st_s;  // status of this CTA's row (the draw warps')

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
  auto grp0_of = [&](int q) { return (cluster + (q / nmodes) * nclusters) * SC_CL; };

  if (tid == 0) {
    for (int s = 0; s < SC_STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], SC2_K1 / 32);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&c_full[i], 1);
      mbar_init(&v_full[i], 1);
      mbar_init(&t_full[i], 1);
      mbar_init(&t_free[i], 1);
    }
    fence_barrier_init();
    if (nsteps > 0) mbar_arrive_expect_tx(&c_full[0], (uint32_t)F_of(P.m_begin) * 128u);  // step 0's C row
  }
  __syncthreads();
  sc_cluster_sync();  // peers' barriers initialised (and step 0 expected) before any st.async lands
  // PDL: the Gamma ring (sites uploaded synchronously) may run ahead; every other warp reads inputs or
  // writes outputs that may belong to the previous kernel in the stream
  griddep_launch_dependents();
  if (warp != SC2_W_PROD) griddep_wait();

  if (warp == SC2_W_PROD) {
    // ============ ring producer: Gamma stages of every step, once per half, in order ============
    if (lane == 0) {
      uint32_t sidx = 0;
      for (int q = 0; q < nsteps; ++q) {
        const int m = P.m_begin + q % nmodes;
        const int KT = (P.chi[m] + 7) >> 3, F = F_of(m);
        const int f0 = rank * F / SC_CL, fc = (rank + 1) * F / SC_CL - f0;
        for (int h = 0; h < 2; ++h)
          for (int kt = 0; kt < KT; kt += SC_KS, ++sidx) {
            const int slot = sidx % SC_STAGES, nks = min(SC_KS, KT - kt);
            if (sidx >= SC_STAGES) {
              mbar_wait(&empty[slot], ((sidx / SC_STAGES) - 1) & 1);
              fence_proxy_async();  // the K1 warps' ld.shared of the slot before the bulk-copy refill
            }
            mbar_arrive_expect_tx(&full[slot], (uint32_t)(nks * fc) * 1024u);
            if (fc)
              for (int ks = 0; ks < nks; ++ks)
                bulk_load_1d(smem + slot * SC_STAGE_BYTES + ks * fc * 1024,
                             P.sites[m] + (size_t)((kt + ks) * F + f0) * 64, fc * 1024u, &full[slot]);
          }
      }
    }
    __syncwarp();
  } else if (warp == SC2_W_DALPHA) {
    // ===================== D(alpha) of this CTA's row, one step ahead =====================
    for (int q = 0; q < nsteps; ++q) {
      if (q >= 2) mbar_wait(&t_free[q & 1], ((q >> 1) - 1) & 1);
      const int b = grp0_of(q) + rank;
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
  } else if (warp < SC2_K1 / 32) {
    // ============== K1 warps: half A then half B of every mode, C entries to the owners ==============
    const int g = lane >> 2, t = lane & 3;
    uint32_t sidx = 0, vph[2] = {0u, 0u};
    const uint32_t c_addr = smem_u32(smem + SC_OFF_C), cbar_addr = smem_u32(c_full);
    const int fbase = warp;  // this warp's 8-column fragment (SC_FMAX = 8 per CTA)
    for (int q = 0; q < nsteps; ++q) {
      const int m = P.m_begin + q % nmodes;
      const int K = P.chi[m], chi_r = P.chi[m + 1];
      const int KT = (K + 7) >> 3, F = F_of(m);
      const int f0 = rank * F / SC_CL, fc = (rank + 1) * F / SC_CL - f0;
      const int grp0 = grp0_of(q);
      const bool first = (m == P.m_begin);
      for (int h = 0; h < 2; ++h) {
        if (first) {  // new group: rows of half h <- state_in (or v = 1), zero elsewhere
          if (q > 0) {
            // the previous group's last draws of half h are finished (one 16-byte token from each of
            // its 8 owners): their C buffers are free and their next C-row expects are armed, so this
            // half's K1 may send the new group's entries
            mbar_wait(&v_full[h], vph[h] & 1);
            ++vph[h];
          }
          sc2_bar_k1();  // every K1 warp is done reading these rows for the previous group
          for (int e = tid; e < 8 * SC_KMAX; e += SC2_K1) {
            const int r = 8 * h + e / SC_KMAX, j = e % SC_KMAX;
            double2 v = make_double2(0.0, 0.0);
            if (grp0 + r < P.n && j < K)
              v = P.state_in ? P.state_in[(long long)(grp0 + r) * K + j] : make_double2(1.0, 0.0);
            *reinterpret_cast<double2*>(Vt + r * SC_VP + j * 16) = v;
          }
          sc2_bar_k1();
        } else {
          if (warp == 0) SC2_STAMP(0, q, 4 * h + 0);
          mbar_wait(&v_full[h], vph[h] & 1);  // the 8 rows' v' of the previous mode
          ++vph[h];
        }
        if (warp == 0) SC2_STAMP(0, q, 4 * h + 1);
        // expect half h's next V tile (8 rows x jpad entries) -- or, before a new group, the 8 owners'
        // end-of-group tokens -- before any of its rows can be drawn: the draws of mode m need this
        // CTA's K1_h(m) entries, which come after this point
        if (tid == 0 && q + 1 < nsteps)
          mbar_arrive_expect_tx(&v_full[h], P.m_begin + (q + 1) % nmodes != P.m_begin
                                                ? (uint32_t)(8 * ((chi_r + 7) & ~7) * 16) : 8u * 16u);
        double t1[2] = {0.0, 0.0}, t2[2] = {0.0, 0.0}, t3[2] = {0.0, 0.0};
        auto kstage = [&](const uint8_t* st, int kt) {  // site_gemm3m_kernel's per-accumulator k order
#pragma unroll
          for (int step = 0; step < 2; ++step) {
            const int i = 2 * t + step;
            const double2 w = *reinterpret_cast<const double2*>(st + fbase * 1024 + i * 128 + ((g ^ i) << 4));
            const double2 v = *reinterpret_cast<const double2*>(Vt + (8 * h + g) * SC_VP + (8 * kt + i) * 16);
            const double ws = __dadd_rn(w.x, w.y);
            dmma_8x8x4(t1[0], t1[1], v.x, w.x);
            dmma_8x8x4(t2[0], t2[1], v.y, w.y);
            dmma_8x8x4(t3[0], t3[1], __dadd_rn(v.x, v.y), ws);
          }
        };
        if (fbase < fc) {
          for (int kt0 = 0; kt0 < KT; kt0 += SC_KS, ++sidx) {
            const int slot = sidx % SC_STAGES;
            mbar_wait(&full[slot], (sidx / SC_STAGES) & 1);
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
          // row 8 h + g of the group is owned by CTA 8 h + g: st.async the entries there
          const uint32_t owner = (uint32_t)(8 * h + g);
          const uint32_t dst = sc_mapa(c_addr + (uint32_t)((q & 1) * SC_NMAX * 16), owner);
          const uint32_t bar = sc_mapa(cbar_addr + (uint32_t)((q & 1) * 8), owner);
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int col = 8 * (f0 + fbase) + 2 * t + e;
            sc_st_async(dst + (uint32_t)col * 16u, t1[e] - t2[e], t3[e] - (t1[e] + t2[e]), bar);
          }
          if (warp == 0) SC2_STAMP(0, q, 4 * h + 2);
        } else {  // no fragment in this mode: keep the ring's slot accounting
          for (int kt0 = 0; kt0 < KT; kt0 += SC_KS, ++sidx) {
            const int slot = sidx % SC_STAGES;
            mbar_wait(&full[slot], (sidx / SC_STAGES) & 1);
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[slot]);
          }
        }
      }
      (void)chi_r;
    }
  } else {
    // ===================== draw warps: K2 + K3 of this CTA's row, every mode =====================
    const int dt = tid - SC2_K1, dw = dt >> 5;  // 128 threads: displace_draw_kernel's j map
    const int half = rank / 8;
    const uint32_t vt_addr = smem_u32(Vt), vbar_addr = smem_u32(v_full + half);
    for (int q = 0; q < nsteps; ++q) {
      const int m = P.m_begin + q % nmodes;
      const int chi_r = P.chi[m + 1];
      const int b = grp0_of(q) + rank;
      const bool valid = b < P.n;
      const bool first = (m == P.m_begin), last = (m == P.m_end - 1);
      double u = 0.0;
      int kf = 0;
      if (dw == 0 && valid) {  // the uniform / forced outcome of (b, m)
        if (A.forced) {
          kf = A.counts[(long long)b * A.ld_c + m];
        } else {
          const unsigned long long gi = (unsigned long long)(A.first_index + b);
          u = A.u ? A.u[(long long)b * A.ld_u + m]
                  : philox_double(numpy_key0(A.seed), gi / 64, (gi % 64) * (uint64_t)A.M + m);
        }
      }
      if (first && dt == 0) st_s = valid ? A.status[b] : 0;
      if (dw == 0) SC2_STAMP(2, q, 0);
      mbar_wait(&c_full[q & 1], (q >> 1) & 1);
      if (dw == 0) SC2_STAMP(2, q, 1);
      // expect the next step's C row: buffer (q + 1) & 1 was last read by draw(q - 1), already done
      if (dt == 0 && q + 1 < nsteps) mbar_arrive_expect_tx(&c_full[(q + 1) & 1], (uint32_t)F_of(P.m_begin + (q + 1) % nmodes) * 128u);
      mbar_wait(&t_full[q & 1], (q >> 1) & 1);
      sc2_bar_draw();  // st_s of a group's first mode visible to every draw thread
      if (dw == 0) SC2_STAMP(2, q, 5);
      const double2* Crow = reinterpret_cast<const double2*>(smem + SC_OFF_C) + (q & 1) * SC_NMAX;
      const double2* T = reinterpret_cast<const double2*>(smem + SC_OFF_T) + (q & 1) * DMAX * DMAX;
      const int jpad = (chi_r + 7) & ~7;
      auto emit = [&](int j, double2 v) {  // v' of j to row `rank` of every CTA's V tile, or state_out
        if (last) {
          if (P.state_out && valid && j < chi_r) P.state_out[(long long)b * chi_r + j] = v;
          return;
        }
        const uint32_t vo = vt_addr + (uint32_t)(rank * SC_VP + j * 16);
#pragma unroll
        for (int p = 0; p < SC_CL; ++p) sc_st_async(sc_mapa(vo, (uint32_t)p), v.x, v.y, sc_mapa(vbar_addr, (uint32_t)p));
      };
      const long long crow = (long long)b * A.ld_c + m;
      const bool dead = !valid || (st_s & ST_FAILED) != 0;
      if (dead) {
        for (int j = dt; j < jpad; j += SC2_DRAW) emit(j, make_double2(0.0, 0.0));
        if (valid && dt == 0 && !A.forced) A.counts[crow] = -1;
        if (valid && A.marg && dt < D) A.marg[crow * D + dt] = 0.0;
      } else {
        constexpr int DR = DT ? DT : DMAX;
        double acc[DR];
#pragma unroll
        for (int k = 0; k < DR; ++k) acc[k] = 0.0;
        for (int j = dt; j < chi_r; j += DRAW_THREADS) {
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
        warp_tree_scatter(acc, red[dw], D);
        sc2_bar_draw();  // red[][] complete
        if (dw == 0) SC2_STAMP(2, q, 2);
        if (dw == 0) {  // the draw (draw_row_warp, as displace_draw_kernel)
          const RowDraw r = draw_row_warp<DT>(red, DRAW_THREADS / 32, p_s, D, st_s, A.forced != 0,
                                              __shfl_sync(0xffffffffu, kf, 0), __shfl_sync(0xffffffffu, u, 0), A.tie_eps);
          if (lane == 0) {
            k_s = r.k;
            pk_s = r.pk;
            st_s = r.status;
          }
          __syncwarp();
          named_bar_arrive(3, SC2_DRAW);  // release pass 2; the bookkeeping stores are off its path
          if (A.marg && lane < D) A.marg[crow * D + lane] = (r.k >= 0) ? r.p / r.Ptot : 0.0;
          if (lane == 0) {
            A.status[b] = r.status;
            if (!A.forced) A.counts[crow] = r.k;
          }
        } else {
          sc2_bar_draw();
        }
        if (dw == 0) SC2_STAMP(2, q, 3);
        const int ks = k_s;
        const double pk = pk_s;
        for (int j = dt; j < jpad; j += SC2_DRAW) {
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
      sc2_bar_draw();  // every draw thread is done with T, red, C and k_s / pk_s before reuse
      if (dw == 0) SC2_STAMP(2, q, 4);
      if (dt == 0) mbar_arrive(&t_free[q & 1]);
      if (last && q + 1 < nsteps && dt < SC_CL) {
        // end of this group: a 16-byte token into row `rank`'s padding slot of every CTA's V tile
        // releases the next group's K1 of this half (it must not overwrite C buffers still being read)
        const uint32_t vo = vt_addr + (uint32_t)(rank * SC_VP + SC_KMAX * 16);
        sc_st_async(sc_mapa(vo, (uint32_t)dt), 0.0, 0.0, sc_mapa(vbar_addr, (uint32_t)dt));
      }
    }
  }
  sc_cluster_sync();  // no CTA leaves while a peer may still st.async into it
}

}  // namespace mps
