// displace_draw.cuh — K2+K3 for one mode: displacement einsum, |amplitude|^2 marginal,
// inverse-CDF draw, gather + renormalise, plus the
// counter-based streams (row a10) and D(alpha) construction (row a2).
//
// One CTA per sample b.  Pass 1 streams C[b] (chi_r x D complex, written by K1),
// forms E[j][k] = sum_d Disp[k][d] C[j][d] in registers and
// accumulates p[k] = sum_j |E[j][k]|^2 in a fixed order (thread-strided partials ->
// xor-shuffle tree -> warps summed in index order), so p is bit-identical for any
// batch size / grid.  Thread 0 draws k against u[b][m] with the sampler.py:692-697
// rule.  Pass 2 re-reads C[b] and writes v'[j] = E[j][k] / sqrt(p[k]) — the
// recomputation costs D MACs per j and saves storing E (16 n chi D bytes).

#pragma once
#include <cstdint>
#include <type_traits>

#include "c64_gemm.cuh"
#include "ptx.cuh"

namespace mps {

constexpr int DMAX = 16;
constexpr int DRAW_THREADS = 128;
constexpr double TIE_EPS = 1e-10;
constexpr uint8_t ST_FAILED = 1;
constexpr uint8_t ST_FLAGGED = 2;

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}

// ---------------------------------------------------------------------------
// numpy-compatible Philox4x64-10 (Random123 constants); numpy increments the
// 256-bit counter before each block, so output word q of key (k0, k1) is
// philox(ctr = q/4 + 1)[q % 4]; Generator.random() = (x >> 11) * 2^-53.
// ---------------------------------------------------------------------------
__host__ __device__ inline void philox4x64_10(uint64_t ctr[4], uint64_t k0, uint64_t k1) {
  const uint64_t M0 = 0xD2E7470EE14C6C93ull, M1 = 0xCA5A826395121157ull;
  const uint64_t W0 = 0x9E3779B97F4A7C15ull, W1 = 0xBB67AE8584CAA73Bull;
  for (int r = 0; r < 10; ++r) {
#ifdef __CUDA_ARCH__
    uint64_t hi0 = __umul64hi(M0, ctr[0]), lo0 = M0 * ctr[0];
    uint64_t hi1 = __umul64hi(M1, ctr[2]), lo1 = M1 * ctr[2];
#else
    unsigned __int128 p0 = (unsigned __int128)M0 * ctr[0], p1 = (unsigned __int128)M1 * ctr[2];
    uint64_t hi0 = (uint64_t)(p0 >> 64), lo0 = (uint64_t)p0, hi1 = (uint64_t)(p1 >> 64), lo1 = (uint64_t)p1;
#endif
    uint64_t c0 = hi1 ^ ctr[1] ^ k0, c2 = hi0 ^ ctr[3] ^ k1;
    ctr[0] = c0; ctr[1] = lo1; ctr[2] = c2; ctr[3] = lo0;
    k0 += W0; k1 += W1;
  }
}

// numpy turns the key list [seed, blk] into an array first; a seed >= 2^63 does not fit
// int64, so the list is converted through float64 (seed rounded to 53 bits, >= 2^64 -> 0).
// _stream_uniforms inherits that, and so do we, bit-for-bit.
__host__ __device__ inline uint64_t numpy_key0(uint64_t seed) {
  if (seed < (1ull << 63)) return seed;
  const double f = (double)seed;
  return f >= 18446744073709551616.0 ? 0ull : (uint64_t)f;
}

// The q-th double of numpy Generator(Philox(key=[k0, k1])).random(...)
__host__ __device__ inline double philox_double(uint64_t k0, uint64_t k1, uint64_t q) {
  uint64_t ctr[4] = {q / 4 + 1, 0, 0, 0};
  if (ctr[0] == 0) ctr[1] = 1;  // carry (unreachable for realistic q)
  philox4x64_10(ctr, k0, k1);
  return (double)(ctr[q & 3] >> 11) * (1.0 / 9007199254740992.0);
}

// uniforms of samples first..first+count-1, mode m: row i%64, column m of block i/64
__global__ void stream_uniforms_kernel(uint64_t seed, long long first, int count, int M, double* out,
                                       long long ld) {
  long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (long long)count * M) return;
  long long b = idx / M;
  int m = (int)(idx % M);
  unsigned long long i = (unsigned long long)(first + b);
  uint64_t q = (i % 64) * (uint64_t)M + m;
  out[b * ld + m] = philox_double(numpy_key0(seed), i / 64, q);
}

// alpha ~ CN(0, sigma^2) from the key (seed, 2^62 + i/64), 2M uniforms per sample row
__device__ inline double2 stream_alpha(uint64_t seed, unsigned long long i, int M, int m, double sigma) {
  const uint64_t blk = (1ull << 62) + i / 64;
  uint64_t q = (i % 64) * (uint64_t)(2 * M) + 2 * m;
  double u1 = philox_double(seed, blk, q), u2 = philox_double(seed, blk, q + 1);
  double rad = sigma * sqrt(-log1p(-u1));
  double ph = 2.0 * 3.141592653589793 * u2;
  double sn, cs;
  sincos(ph, &sn, &cs);
  return make_double2(rad * cs, rad * sn);
}

// sqrt(k) and 1/sqrt(k) (correctly rounded, as Python's math.sqrt and 1.0/x give them)
__constant__ double c_sqrt[17] = {0.0, 1.0, 1.4142135623730951, 1.7320508075688772, 2.0, 2.23606797749979, 2.449489742783178, 2.6457513110645907, 2.8284271247461903, 3.0, 3.1622776601683795, 3.3166247903554, 3.4641016151377544, 3.605551275463989, 3.7416573867739413, 3.872983346207417, 4.0};
__constant__ double c_rsqrt[17] = {0.0, 1.0, 0.7071067811865475, 0.5773502691896258, 0.5, 0.4472135954999579, 0.4082482904638631, 0.3779644730092272, 0.35355339059327373, 0.3333333333333333, 0.31622776601683794, 0.30151134457776363, 0.2886751345948129, 0.2773500981126146, 0.2672612419124244, 0.2581988897471611, 0.25};

// Exact truncated <k|D(alpha)|d> (oracle decision 6), row-major T[k*D + d].  The operation order
// mirrors the oracle's numpy expressions with explicit _rn intrinsics, so host and device agree to
// the last bit except where exp() differs by an ulp (a common factor of the whole matrix).
// cmul_rn is numpy's complex multiply a * b as its SIMD loops form it (numpy 2.x on FMA3 / AVX-512
// hosts: one fmaddsub of a.re * (b.re, b.im) against a.im * (b.im, b.re)), checked bit for bit
// against numpy 2.3 on random contiguous and strided pairs.  With it, a CPU emulation of the
// recurrence below reproduces oracle.displacement_matrix exactly when given numpy's exp()
// (tools/displacement_emulation.py, profiles/r02_conditioning.txt).  The plain two-rounding form
// disagreed with numpy on about half of the products.  At D = 16 and |alpha| ~ 2.4 the recurrence
// amplified that to ~1e-12 in D(alpha).
__device__ __forceinline__ double2 cmul_rn(double2 a, double2 b) {
  return make_double2(__fma_rn(a.x, b.x, -__dmul_rn(a.y, b.y)), __fma_rn(a.x, b.y, __dmul_rn(a.y, b.x)));
}

__device__ inline void displacement_column0(double2 a, int D, double2* T) {
  // T[0,0] = exp(-0.5 |a|^2); T[k,0] = T[k-1,0] * a / sqrt(k)  (numpy's complex / real
  // division multiplies by the reciprocal: Smith's algorithm with a zero imaginary part)
  const double e = exp(__dmul_rn(-0.5, __dadd_rn(__dmul_rn(a.x, a.x), __dmul_rn(a.y, a.y))));
  T[0] = make_double2(e, 0.0);
  for (int k = 1; k < D; ++k) {
    const double2 v = cmul_rn(T[(k - 1) * D], a);
    const double scl = c_rsqrt[k];
    T[k * D] = make_double2(__dmul_rn(v.x, scl), __dmul_rn(v.y, scl));
  }
}

__device__ inline double2 displacement_entry(double2 a, int D, const double2* T, int k, int d) {
  // T[k,d] = (sqrt(k) T[k-1,d-1] - conj(a) T[k,d-1]) * (1/sqrt(d));  row 0: (-conj(a) T[0,d-1]) * inv
  const double inv = c_rsqrt[d];
  const double2 t2 = cmul_rn(make_double2(a.x, -a.y), T[k * D + d - 1]);
  if (k == 0) return make_double2(__dmul_rn(-t2.x, inv), __dmul_rn(-t2.y, inv));
  const double sk = c_sqrt[k];
  const double2 t1 = T[(k - 1) * D + d - 1];
  return make_double2(__dmul_rn(__dsub_rn(__dmul_rn(sk, t1.x), t2.x), inv),
                      __dmul_rn(__dsub_rn(__dmul_rn(sk, t1.y), t2.y), inv));
}

__global__ void displacement_kernel(const double2* __restrict__ alpha, int count, int D, double2* __restrict__ out) {
  int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= count) return;
  double2 a = alpha[idx];
  double2* T = out + (long long)idx * D * D;
  displacement_column0(a, D, T);
  for (int d = 1; d < D; ++d)
    for (int k = 0; k < D; ++k) T[k * D + d] = displacement_entry(a, D, T, k, d);
}

struct DrawArgs {
  const double2* C;         // n x (chi_r*D)
  long long ldc;            // complex elements per C row
  int chi_r, D, m, M;
  long long first_index;
  const double* u;          // uniforms (n x ld_u) or null -> device stream
  long long ld_u;
  uint64_t seed;
  const double2* disp;      // n x M x D x D or null
  const double2* alpha;     // n x M or null
  double alpha_sigma;       // >= 0: device alpha stream when disp & alpha are null
  double2* v_out;           // n x chi_r
  double* vs_out;           // n x ld_vs sum plane (re + im) of v_out for the 3M GEMM, or null
  int ld_vs;
  // complex64 chain (C64 instantiation): C in fp32, next state as tf32 hi/lo planes of the
  // interleaved state (n x ld_a) or, for a stage's last mode, complex64 into v_out32
  const float2* C32;
  float2* v_out32;
  float* a_hi;
  float* a_lo;
  int ld_a;
  double tie_eps;           // |cdf - u| band that flags a draw (1e-10 c128, 1e-4 c64)
  int forced;               // 1: take the outcome from counts (input) instead of drawing
  int32_t* counts;          // n x ld_c
  long long ld_c;
  double* marg;             // n x ld_c x D or null
  uint8_t* status;          // n
};

// Broadcast read of a D(alpha) entry.  volatile: keeps ptxas from hoisting all D^2
// loop-invariant entries into registers across the j loop (which spills 2 KB).
__device__ __forceinline__ double2 lds_c128(const double2* p) {
  double2 v;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(smem_u32(p)));
  return v;
}

// E[k] = sum_d T[k][d] c[d] for one j (T in shared memory, broadcast reads)
template <int DT>
__device__ __forceinline__ double2 disp_row(const double2* T, int D, int k, const double2* c) {
  double2 e = make_double2(0.0, 0.0);
#pragma unroll
  for (int d = 0; d < (DT ? DT : DMAX); ++d) {
    if (!DT && d >= D) break;
    const double2 tk = lds_c128(&T[k * D + d]);
    e.x = fma(tk.x, c[d].x, e.x);
    e.x = fma(-tk.y, c[d].y, e.x);
    e.y = fma(tk.x, c[d].y, e.y);
    e.y = fma(tk.y, c[d].x, e.y);
  }
  return e;
}

// One CTA of DRAW_THREADS per sample; DT = compile-time D (0: runtime D <= DMAX).
// Pass 1 reads C[b] with 16-B loads (L1-resident per thread), pass 2 re-reads it
// (L2 hits: the row was touched microseconds earlier).  128 threads and <= 128 regs
// keep 4 CTAs per SM so one CTA's serial sections (D(alpha), the draw) hide behind
// the others' streaming.
// C element loads for both precisions (the c64 chain computes the draw in fp64 too)
template <bool C64>
__device__ __forceinline__ double2 load_c(const DrawArgs& A, long long idx) {
  if constexpr (C64) {
    const float2 v = A.C32[idx];
    return make_double2((double)v.x, (double)v.y);
  } else {
    return A.C[idx];
  }
}

// next-state store: c128 state (+ its 3M sum plane), or c64 as tf32 hi/lo planes / complex64
template <bool C64>
__device__ __forceinline__ void store_state(const DrawArgs& A, int b, int j, double2 v) {
  if constexpr (C64) {
    const float re = (float)v.x, im = (float)v.y;
    if (A.v_out32) {
      A.v_out32[(long long)b * A.chi_r + j] = make_float2(re, im);
    } else {
      float h, l;
      const long long o = (long long)b * A.ld_a + 2 * j;
      split_tf32(re, h, l);
      A.a_hi[o] = h;
      A.a_lo[o] = l;
      split_tf32(im, h, l);
      A.a_hi[o + 1] = h;
      A.a_lo[o + 1] = l;
    }
  } else {
    A.v_out[(long long)b * A.chi_r + j] = v;
    // __dadd_rn: no FMA contraction with the scaling, so the plane holds exactly the sum of
    // the stored (re, im) pair, as the GEMM's in-kernel add would form it
    if (A.vs_out) A.vs_out[(long long)b * A.ld_vs + j] = __dadd_rn(v.x, v.y);
  }
}

// complex64 chain: the einsum and the marginal partials run in fp32 (twice the fp64 rate;
// ~1e-7 relative, far inside the 1e-4 c64 bar); the draw itself stays in fp64.
template <int DT>
__device__ __forceinline__ float2 disp_row_f(const float2* T, int D, int k, const float2* c) {
  float2 e = make_float2(0.f, 0.f);
#pragma unroll
  for (int d = 0; d < (DT ? DT : DMAX); ++d) {
    if (!DT && d >= D) break;
    float2 tk;
    asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(tk.x), "=f"(tk.y) : "r"(smem_u32(&T[k * D + d])));
    e.x = fmaf(tk.x, c[d].x, e.x);
    e.x = fmaf(-tk.y, c[d].y, e.x);
    e.y = fmaf(tk.x, c[d].y, e.y);
    e.y = fmaf(tk.y, c[d].x, e.y);
  }
  return e;
}

// The draw of one sample row (the sampler.py:692-697 rule; teacher-forced: the given outcome),
// run by ALL 32 lanes of one warp.  Every floating-point operation of the serial form is kept:
// lane k < D sums p_k over the row's warp partials red[w][k] in warp order, every lane forms Ptot
// and its own prefix run_k with the serial loop's sequence of adds and divides once; the count,
// the min distance to a CDF boundary (fmin is exact) and the zero-probability walk-back
// (while (k > 0 && !(p[k] > 0)) --k) become ballots.  Writes p_s[0..D); returns the outcome
// (-1: failed), the updated status bits, Ptot and the renormalisation 1/sqrt(p(k)) in every lane,
// p(k) in every lane, and in lane k < D its own p(k).
//
// Latency (it sits on every chain's serial path, ~860 cycles at C1 in the round-2 form): the D-long
// prefix loop is unrolled (DT) with its loads hoisted; the tie flag is one ballot (the minimum of
// |cdf - u| over lanes < D - 1, or 1e300, is <= eps exactly when one of those terms is, or 1e300 is:
// fmin is exact and drops NaNs like the ballot does) instead of five shuffle rounds; and the
// renormalisation 1/sqrt(p(k)) is left to the caller's pass 2 (row_scale).  Same operations on the
// same operands: every result bit is unchanged.
struct RowDraw {
  int k;
  uint8_t status;
  double Ptot;
  double pk;  // p(k) in every lane (0 when k < 0): the renormalisation is row_scale(k, pk)
  double p;   // lane < D: p(lane)
};
// v' = E[:, k] / sqrt(p(k)) is formed as E * (1 / sqrt(p(k))) on every path.  Callers evaluate it
// where it is used (after their pass-2 FMAs are issued), so its ~300-cycle sqrt + reciprocal chain
// overlaps the gather instead of sitting between the draw and pass 2.
__device__ __forceinline__ double row_scale(int k, double pk) { return (k >= 0 && pk > 0.0) ? 1.0 / sqrt(pk) : 0.0; }

// The draw's partial marginals summed over the 32 lanes with the xor-shuffle butterfly's association
// (rounds 16, 8, 4, 2, 1 -- the fixed order every path shares), done as a reduce-scatter.  The N partials are padded to NP = 2^ceil(log2 N) (zeros for
// k >= N).  At round o the lanes i and i ^ o hold the same NP / (32 / o)-long set (their higher lane
// bits agree); the lower lane keeps the first half, the upper the second, each sends the half it drops
// and adds the partner's copy of the half it keeps.  Every kept value is own + partner of exactly the
// butterfly's pairs (addition commutes), so the totals carry the butterfly's bits, but a round moves
// half the set instead of all of it (N = 10: 16 shuffles instead of 50; N = 4: 6 instead of 20).  Once a
// set is one value the lower lane keeps the sum and the upper drops out.  Afterwards lane L holds the
// total of k = base (when alive); it writes out[k] for k < nvalid.  All indices are compile-time.
template <int N, typename T, typename O>
__device__ __forceinline__ void warp_tree_scatter(const T (&in)[N], O* out, int nvalid) {
  constexpr int NP = N <= 1 ? 1 : N <= 2 ? 2 : N <= 4 ? 4 : N <= 8 ? 8 : 16;
  static_assert(N <= 16, "at most 16 partials");
  const int lane = threadIdx.x & 31;
  T v[NP];
#pragma unroll
  for (int k = 0; k < NP; ++k) v[k] = k < N ? in[k] : T(0);
  int base = 0;
  bool alive = true;
#pragma unroll
  for (int r = 0; r < 5; ++r) {
    const int o = 16 >> r;
    const bool up = (lane & o) != 0;
    const int CM = NP >> r;  // compile-time after unrolling (0 once the set is a single value)
    if (CM >= 2) {
      const int H = CM / 2;
#pragma unroll
      for (int t = 0; t < NP / 2; ++t) {
        if (t < H) {
          const T x = up ? v[t] : v[H + t];
          const T y = __shfl_xor_sync(0xffffffffu, x, o);
          v[t] = (up ? v[H + t] : v[t]) + y;
        }
      }
      if (up) base += H;
    } else {
      const T y = __shfl_xor_sync(0xffffffffu, v[0], o);
      v[0] = v[0] + y;
      alive = alive && !up;
    }
  }
  if (alive && base < nvalid) out[base] = (O)v[0];
}
template <int DT>
__device__ inline RowDraw draw_row_warp(const double (*red)[DMAX], int nwarps, double* p_s, int D, uint8_t st0,
                                        bool forced, int k_forced, double u, double tie_eps) {
  const int lane = threadIdx.x & 31;
  double sacc = 0.0;
  if (lane < D) {
    for (int w = 0; w < nwarps; ++w) sacc += red[w][lane];
    p_s[lane] = sacc;
  }
  __syncwarp();
  double Ptot = 0.0, run = 0.0;
  if constexpr (DT > 0) {
    double pv[DT];
#pragma unroll
    for (int k = 0; k < DT; ++k) pv[k] = p_s[k];
#pragma unroll
    for (int k = 0; k < DT; ++k) {
      Ptot += pv[k];
      if (k <= lane) run += pv[k];
    }
  } else {
    for (int k = 0; k < D; ++k) {
      const double pv = p_s[k];
      Ptot += pv;
      if (k <= lane) run += pv;
    }
  }
  RowDraw r{-1, st0, Ptot, 0.0, sacc};
  const unsigned pos = __ballot_sync(0xffffffffu, lane < D && sacc > 0.0);
  if (!(Ptot > 0.0) || !isfinite(Ptot)) {
    r.status |= ST_FAILED;
  } else if (forced) {
    r.k = k_forced;
    if (r.k < 0 || r.k >= D) {
      r.status |= ST_FAILED;
      r.k = -1;
    }
  } else {
    const double cdf = (lane == D - 1) ? 1.0 : run / Ptot;
    const int cnt = __popc(__ballot_sync(0xffffffffu, lane < D && cdf <= u));
    const bool near = __any_sync(0xffffffffu, lane < D - 1 && fabs(cdf - u) <= tie_eps) || 1e300 <= tie_eps;
    const int kc = cnt < D - 1 ? cnt : D - 1;
    const unsigned below = pos & ((2u << kc) - 1u);
    r.k = below ? 31 - __clz(below) : 0;
    if (near) r.status |= ST_FLAGGED;
  }
  r.pk = __shfl_sync(0xffffffffu, sacc, r.k >= 0 ? r.k : 0);
  if (r.k < 0) r.pk = 0.0;
  return r;
}

// RING: the C row streams through a 2-slot shared-memory ring of 128-j chunks filled by 1-D TMA
// bulk copies (mbarrier per slot), for both passes; loads in flight cost no registers, so the
// kernel stops being bound on global-load latency.  Each thread still owns j = tid + 128 c, so
// the reduction order (and every result bit) is the same with and without the ring.
// ring slots of the draw kernel's C-row stream (a CTA keeps RING_SLOTS - 1 chunk loads in flight
// while it works on one); the c64 chunks are half the bytes, so it affords a deeper ring
#ifdef DRAW_TRACE  // debug build only (tools/draw_trace.py): per-CTA globaltimer stamps of one mode's launch
__device__ int dr_trace_m = -1;
__device__ long long dr_trace[8192][8];
__device__ __forceinline__ long long dr_now() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define DR_STAMP(k)                                                          \
  if (A.m == dr_trace_m && threadIdx.x == 0 && blockIdx.x < 8192) {         \
    dr_trace[blockIdx.x][k] = dr_now();                                      \
    if ((k) == 0) {                                                          \
      unsigned smid;                                                         \
      asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));                      \
      dr_trace[blockIdx.x][7] = smid;                                        \
    }                                                                        \
  }
#else
#define DR_STAMP(k)
#endif

#ifndef DRAW_SLOTS_C128
#define DRAW_SLOTS_C128 2
#endif
#ifndef DRAW_SLOTS_C64
#define DRAW_SLOTS_C64 2
#endif
template <bool C64>
__host__ __device__ constexpr int draw_ring_slots() { return C64 ? DRAW_SLOTS_C64 : DRAW_SLOTS_C128; }

template <int DT, bool C64, bool RING>
__global__ void __launch_bounds__(DRAW_THREADS, C64 ? 8 : 4)
    displace_draw_kernel(DrawArgs A) {
  using ElemT = typename std::conditional<C64, float2, double2>::type;
  extern __shared__ __align__(16) uint8_t ring_smem[];
  constexpr int NS = draw_ring_slots<C64>();
  __shared__ uint64_t ring_bar[NS];
  __shared__ double2 T[DMAX * DMAX];
  __shared__ float2 Tf[C64 ? DMAX * DMAX : 1];
  __shared__ double red[DRAW_THREADS / 32][DMAX];
  __shared__ double p_s[DMAX];
  __shared__ int k_s;
  __shared__ double pk_s;

  const int b = blockIdx.x;
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int D = DT ? DT : A.D;
  const unsigned long long gi = (unsigned long long)(A.first_index + b);
  const long long crow = (long long)b * A.ld_c + A.m;
  const long long cbase = (long long)b * A.ldc;
  const ElemT* Crow = (C64 ? reinterpret_cast<const ElemT*>(A.C32) : reinterpret_cast<const ElemT*>(A.C)) + cbase;
  const int nchunks = (A.chi_r + DRAW_THREADS - 1) / DRAW_THREADS;
  const int chunk_elems = DRAW_THREADS * D;

  // ring: chunk u (of the 2 * nchunks loads, pass 1 then pass 2) goes to slot u % NS
  auto ring_issue = [&](int u) {
    const int c = u % nchunks;
    const int j0 = c * DRAW_THREADS;
    const int nj = min(DRAW_THREADS, A.chi_r - j0);
    const uint32_t bytes = (uint32_t)(nj * D * (int)sizeof(ElemT));
    uint64_t* bar = &ring_bar[u % NS];
    mbar_arrive_expect_tx(bar, bytes);
    // pass 1 (u < nchunks) keeps the row's lines in L2 for pass 2's re-read, pass 2 lets them go:
    // DRAM reads drop from 1.16x to 1.00x the row bytes at C3 (profiles/r02_ncu_k23_draw_l2hints.txt)
    bulk_load_1d_hint(ring_smem + (size_t)(u % NS) * chunk_elems * sizeof(ElemT), Crow + (long long)j0 * D, bytes, bar,
                      u < nchunks);
  };
  auto ring_slot = [&](int u) -> const ElemT* {
    mbar_wait(&ring_bar[u % NS], (u / NS) & 1);
    return reinterpret_cast<const ElemT*>(ring_smem) + (size_t)(u % NS) * chunk_elems;
  };

  // ---- displacement matrix for (b, m): inputs only, so it runs before the PDL wait and
  //      overlaps the tail of the site GEMM that produces C ----
  DR_STAMP(0);
  griddep_launch_dependents();
  if (RING && tid == 0) {
    for (int i = 0; i < NS; ++i) mbar_init(&ring_bar[i], 1);
    fence_barrier_init();
  }
  const bool ident = !(A.disp || A.alpha || A.alpha_sigma >= 0.0);
  if (A.disp) {
    const double2* src = A.disp + ((long long)b * A.M + A.m) * D * D;
    for (int e = tid; e < D * D; e += DRAW_THREADS) T[e] = src[e];
  } else if (!ident && warp == 0) {
    const double2 a = A.alpha ? A.alpha[(long long)b * A.M + A.m] : stream_alpha(A.seed, gi, A.M, A.m, A.alpha_sigma);
    if (lane == 0) displacement_column0(a, D, T);
    __syncwarp();
    for (int d = 1; d < D; ++d) {  // column d from column d-1: no intra-step hazard
      if (lane < D) T[lane * D + d] = displacement_entry(a, D, T, lane, d);
      __syncwarp();
    }
  }
  if constexpr (C64) {
    __syncthreads();
    for (int e = tid; e < D * D; e += DRAW_THREADS) Tf[e] = make_float2((float)T[e].x, (float)T[e].y);
  }
  DR_STAMP(1);
  griddep_wait();  // the GEMM (and transitively the previous draw) is complete: C, status valid
  DR_STAMP(2);
#ifdef DRAW_NOOP  // timing experiment only (wrong results): the chain with the draw's work removed
  return;
#endif
  const bool dead = (A.status[b] & ST_FAILED) != 0;
  // with one chunk the row stays in slot 0 for pass 2 (no re-load); else loads 0 and 1 go out now
  if (RING && tid == 0 && !dead) {
    ring_issue(0);
    if (nchunks > 1)
      for (int u = 1; u < NS && u < 2 * nchunks; ++u) ring_issue(u);
  }
  __syncthreads();

  if (dead) {  // dead sample: zero state, count -1 (deterministic chain)
    for (int j = tid; j < A.chi_r; j += DRAW_THREADS) store_state<C64>(A, b, j, make_double2(0.0, 0.0));
    if (tid == 0 && !A.forced) A.counts[crow] = -1;
    if (A.marg && tid < D) A.marg[crow * D + tid] = 0.0;
    return;
  }

  // ---- pass 1: partial marginals (thread tid owns j = tid + 128 c) ----
  constexpr int DR = DT ? DT : DMAX;
  using AccT = typename std::conditional<C64, float, double>::type;
  AccT acc[DR];
#pragma unroll
  for (int k = 0; k < DR; ++k) acc[k] = AccT(0);
  for (int cidx = 0; cidx < nchunks; ++cidx) {
    const int j = cidx * DRAW_THREADS + tid;
    const ElemT* src = RING ? ring_slot(cidx) + tid * D : Crow + (long long)j * D;
    if (j < A.chi_r) {
      bool done = false;
      if constexpr (!C64 && DT > 0) {
        if (!ident) {
          // d-outer / k-inner: the D complex FMA chains E[k] = sum_d T[k][d] c[d] advance together
          // (same per-k operation order as disp_row, so the same bits), hiding the DFMA latency
          // that the k-outer form exposes as one 2D-long dependent chain at a time
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
        ElemT c[DR];
#pragma unroll
        for (int d = 0; d < DR; ++d)
          if (DT || d < D) c[d] = src[d];
#pragma unroll
        for (int k = 0; k < DR; ++k) {
          if (!DT && k >= D) break;
          if constexpr (C64) {
            const float2 e = ident ? c[k] : disp_row_f<DT>(Tf, D, k, c);
            acc[k] = fmaf(e.x, e.x, fmaf(e.y, e.y, acc[k]));
          } else {
            const double2 e = ident ? c[k] : disp_row<DT>(T, D, k, c);
            acc[k] = fma(e.x, e.x, fma(e.y, e.y, acc[k]));
          }
        }
      }
    }
    if (RING && nchunks > 1) {
      __syncthreads();  // every thread is done with this slot
      if (tid == 0 && cidx + NS < 2 * nchunks) {
        fence_proxy_async();  // those generic-proxy reads before the bulk-copy (async-proxy) refill
        ring_issue(cidx + NS);  // pass 1's next chunk, or pass 2's first
      }
    }
  }
  warp_tree_scatter(acc, red[warp], D);
  __syncthreads();
  DR_STAMP(3);
  if (warp == 0) {  // the draw, on warp 0 (draw_row_warp: the serial rule's exact operations)
    const long long ui = (long long)b * A.ld_u + A.m;
    const double u = A.forced ? 0.0
                     : A.u   ? A.u[ui]
                             : philox_double(numpy_key0(A.seed), gi / 64, (gi % 64) * (uint64_t)A.M + A.m);
    const RowDraw r = draw_row_warp<DT>(red, DRAW_THREADS / 32, p_s, D, A.status[b], A.forced != 0,
                                        A.forced ? A.counts[crow] : 0, u, A.tie_eps);
    if (lane == 0) {
      k_s = r.k;
      pk_s = r.pk;
    }
    __syncwarp();
    named_bar_arrive(1, DRAW_THREADS);  // release pass 2; the bookkeeping stores below are off its path
    if (A.marg && lane < D) A.marg[crow * D + lane] = (r.k >= 0) ? r.p / r.Ptot : 0.0;
    if (lane == 0) {
      A.status[b] = r.status;
      if (!A.forced) A.counts[crow] = r.k;
    }
  } else {
    named_bar_sync(1, DRAW_THREADS);
  }
  const int ks = k_s;
  const double scale = row_scale(ks, pk_s);
  DR_STAMP(4);

  // ---- pass 2: gather + renormalise ----
  for (int cidx = 0; cidx < nchunks; ++cidx) {
    const int j = cidx * DRAW_THREADS + tid;
    const ElemT* src = !RING           ? Crow + (long long)j * D
                       : (nchunks > 1) ? ring_slot(nchunks + cidx) + tid * D
                                       : reinterpret_cast<const ElemT*>(ring_smem) + tid * D;  // slot 0, still resident
    if (j < A.chi_r) {
      if (ks < 0) {
        store_state<C64>(A, b, j, make_double2(0.0, 0.0));
      } else if constexpr (C64) {
        const float fs = (float)scale;
        float2 e;
        if (ident) {
          e = src[ks];
        } else {
          float2 c[DR];
#pragma unroll
          for (int d = 0; d < DR; ++d)
            if (DT || d < D) c[d] = src[d];
          e = disp_row_f<DT>(Tf, D, ks, c);
        }
        store_state<true>(A, b, j, make_double2(e.x * fs, e.y * fs));
      } else {
        double2 e;
        if (ident) {
          e = src[ks];
        } else {
          e = make_double2(0.0, 0.0);
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
        store_state<false>(A, b, j, make_double2(e.x * scale, e.y * scale));
      }
    }
    if (RING && nchunks > 1) {
      __syncthreads();
      if (tid == 0 && nchunks + cidx + NS < 2 * nchunks) {
        fence_proxy_async();
        ring_issue(nchunks + cidx + NS);
      }
    }
  }
  DR_STAMP(5);
}

// chi = 1 complex64 starting state as tf32 planes (row pitch 4 floats): (1, 0, 0, 0) / zeros
__global__ void fill_ones_planes_kernel(float* hi, float* lo, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < 4 * n) {
    hi[i] = (i % 4 == 0) ? 1.0f : 0.0f;
    lo[i] = 0.0f;
  }
}

// chi = 1 starting state: v = (1, 0) per sample and its sum plane (row pitch 2 doubles)
__global__ void fill_ones_kernel(double2* v, double* vs, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    v[i] = make_double2(1.0, 0.0);
    vs[2 * i] = 1.0;
    vs[2 * i + 1] = 0.0;
  }
}

}  // namespace mps
