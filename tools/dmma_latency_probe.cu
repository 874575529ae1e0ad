// DMMA.8x8x4 latency / throughput probe: N independent accumulator chains per warp, W warps.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/dmma_lat tools/dmma_latency_probe.cu && /tmp/dmma_lat
// Result (profiles/r01_dmma_probes.txt): latency ~26 cycles; 16 cycles per DMMA per SM sub-partition.
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};" : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}
template <int CH>
__global__ void lat(double* out, long long* cyc, int iters) {
  double c0[CH], c1[CH];
  for (int i = 0; i < CH; ++i) c0[i] = c1[i] = threadIdx.x * 1e-3 + i;
  double a = 1.0000001, b = 0.9999999;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < CH; ++i) dmma(c0[i], c1[i], a, b);
  long long t1 = clock64();
  double s = 0; for (int i = 0; i < CH; ++i) s += c0[i] + c1[i];
  out[threadIdx.x + blockIdx.x * blockDim.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 1 << 20); cudaMalloc(&c, 8);
  long long h;
  int iters = 1000;
#define RUN(CH, W) lat<CH><<<1, 32 * W>>>(o, c, iters); cudaDeviceSynchronize(); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost); \
  printf("chains/warp %2d warps %d: %.1f cycles per DMMA per warp (chain step %.1f)\n", CH, W, (double)h / (iters * CH), (double)h / iters);
  RUN(1, 1) RUN(2, 1) RUN(4, 1) RUN(8, 1) RUN(16, 1) RUN(1, 4) RUN(4, 4) RUN(8, 4) RUN(8, 8) RUN(16, 8) RUN(6, 8) RUN(12, 4)
  return 0;
}
