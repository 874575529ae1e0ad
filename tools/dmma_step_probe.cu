// DMMA step microbenchmarks (sm_100a): the small-chain K1 inner step (2 V rows + 1 Gamma fragment
// per k step, 3M: 6 DMMA.8x8x4) with operands from shared memory, without the ring, on 1..148 CTAs.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/dmma_step tools/dmma_step_probe.cu && /tmp/dmma_step 148
// Result (profiles/r01_dmma_probes.txt): 430 cycles per k-stage at 8 warps (ideal 384).
#include <cstdio>
#include <cstdint>
#include <cstdlib>
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};" : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}
// per step: 2 V rows (LDS.128) + 1 W (LDS.128), 3 DADD, 6 DMMA (the chain kernel's K1 step), MODE 1: no DADD (sums from smem)
template <int MODE>
__global__ void k(double* out, long long* cyc, int iters) {
  __shared__ __align__(16) double2 V[16][129];
  __shared__ __align__(16) double2 W[8][64];
  for (int i = threadIdx.x; i < 16 * 129; i += blockDim.x) (&V[0][0])[i] = make_double2(1e-3 * i, 2e-3 * i);
  for (int i = threadIdx.x; i < 8 * 64; i += blockDim.x) (&W[0][0])[i] = make_double2(3e-3 * i, 1e-3 * i);
  __syncthreads();
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  double t1[2][2] = {}, t2[2][2] = {}, t3[2][2] = {};
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int step = 0; step < 2; ++step) {
      const int i = 2 * t + step;
      const int kk = (8 * (it & 15) + i);
      double2 v[2];
      double as[2];
#pragma unroll
      for (int mf = 0; mf < 2; ++mf) {
        v[mf] = V[8 * mf + g][kk];
        as[mf] = MODE == 0 ? __dadd_rn(v[mf].x, v[mf].y) : v[mf].x;
      }
      const double2 w = W[i][(g ^ i) * 2 + (it & 1)];
      const double ws = MODE == 0 ? __dadd_rn(w.x, w.y) : w.y;
#pragma unroll
      for (int mf = 0; mf < 2; ++mf) {
        dmma(t1[mf][0], t1[mf][1], v[mf].x, w.x);
        dmma(t2[mf][0], t2[mf][1], v[mf].y, w.y);
        dmma(t3[mf][0], t3[mf][1], as[mf], ws);
      }
    }
  }
  long long t1c = clock64();
  double s = 0; for (int a = 0; a < 2; ++a) for (int b = 0; b < 2; ++b) s += t1[a][b] + t2[a][b] + t3[a][b];
  out[threadIdx.x + blockIdx.x * blockDim.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1c - t0;
}
int main(int argc, char** argv) {
  const int NB = argc > 1 ? atoi(argv[1]) : 1;
  double* o; long long* c; cudaMalloc(&o, 1 << 20); cudaMalloc(&c, 8);
  long long h; int iters = 2000;
  for (int w : {4, 8}) {
    k<0><<<NB, 32 * w>>>(o, c, iters); cudaDeviceSynchronize(); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("warps %d DADD sums: %.1f cycles per k-stage (12 DMMA/warp; ideal %d)\n", w, (double)h / iters, 12 * 16 * w / 4);
    k<1><<<NB, 32 * w>>>(o, c, iters); cudaDeviceSynchronize(); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("warps %d no DADD  : %.1f cycles per k-stage\n", w, (double)h / iters);
  }
  return 0;
}
