// FP64 peak probe for B200 (sm_100a): DFMA and DMMA (mma.sync .f64) register-resident loops.
// Prints one JSON line per probe. Used once to fix the FP64 roofline denominator (profiles/fp64_peak.json).
#include <cstdio>
#include <cuda_runtime.h>

#define CHECK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("{\"error\": \"%s\"}\n", cudaGetErrorString(e)); return 1; } } while (0)

template <int ILP>
__global__ void dfma_loop(double* out, int iters, double a, double b) {
  double acc[ILP];
#pragma unroll
  for (int i = 0; i < ILP; ++i) acc[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i) acc[i] = fma(acc[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < ILP; ++i) s += acc[i];
  if (s == 12345.678) out[threadIdx.x] = s;
}

// m8n8k4: A 1 reg, B 1 reg, C 2 regs
template <int ILP>
__global__ void dmma_m8n8k4(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  double c[ILP][2];
#pragma unroll
  for (int i = 0; i < ILP; ++i) { c[i][0] = i; c[i][1] = -i; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < ILP; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[threadIdx.x] = s;
}

template <int ILP>
__global__ void dmma_m16n8k4(double* out, int iters) {
  double a0 = threadIdx.x * 1e-3, a1 = a0 + 1, b = 1.0 - threadIdx.x * 1e-4;
  double c[ILP][4];
#pragma unroll
  for (int i = 0; i < ILP; ++i) { c[i][0] = i; c[i][1] = -i; c[i][2] = 0; c[i][3] = 1; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i)
      asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3]) : "d"(a0), "d"(a1), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < ILP; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (s == 12345.678) out[threadIdx.x] = s;
}

template <int ILP>
__global__ void dmma_m16n8k8(double* out, int iters) {
  double a[4], b[2];
#pragma unroll
  for (int i = 0; i < 4; ++i) a[i] = threadIdx.x * 1e-3 + i;
  b[0] = 1.0; b[1] = 0.5;
  double c[ILP][4];
#pragma unroll
  for (int i = 0; i < ILP; ++i) { c[i][0] = i; c[i][1] = -i; c[i][2] = 0; c[i][3] = 1; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i)
      asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < ILP; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (s == 12345.678) out[threadIdx.x] = s;
}

template <int ILP>
__global__ void dmma_m16n8k16(double* out, int iters) {
  double a[8], b[4];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
#pragma unroll
  for (int i = 0; i < 4; ++i) b[i] = 1.0 - i * 0.25;
  double c[ILP][4];
#pragma unroll
  for (int i = 0; i < ILP; ++i) { c[i][0] = i; c[i][1] = -i; c[i][2] = 0; c[i][3] = 1; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                     "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < ILP; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (s == 12345.678) out[threadIdx.x] = s;
}

template <typename K>
static float time_kernel(K kern, int grid, int block, double* out, int iters, int reps) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  kern<<<grid, block>>>(out, iters);  // warm-up
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < reps; ++r) {
    cudaEventRecord(e0);
    kern<<<grid, block>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  return best;
}

int main() {
  int dev = 0, sms = 0, clk = 0;
  CHECK(cudaSetDevice(dev));
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  double* out; CHECK(cudaMalloc(&out, 4096 * sizeof(double)));
  const int reps = 5;
  for (int wpsm : {4, 8, 16}) {
    int block = 32 * wpsm, grid = sms;
    {
      int iters = 20000;
      auto k = [&](double* o, int it) { dfma_loop<8><<<grid, block>>>(o, it, 1.0000001, 1e-9); };
      (void)k;
      cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
      dfma_loop<8><<<grid, block>>>(out, iters, 1.0000001, 1e-9); cudaDeviceSynchronize();
      float best = 1e30f;
      for (int r = 0; r < reps; ++r) {
        cudaEventRecord(e0); dfma_loop<8><<<grid, block>>>(out, iters, 1.0000001, 1e-9); cudaEventRecord(e1);
        cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
      }
      double flops = 2.0 * 8 * iters * (double)grid * block;
      printf("{\"probe\": \"dfma\", \"warps_per_sm\": %d, \"tflops\": %.3f}\n", wpsm, flops / best / 1e9);
    }
    {
      int iters = 4000;
      float ms = time_kernel(dmma_m8n8k4<8>, grid, block, out, iters, reps);
      double flops = 2.0 * 8 * 8 * 4 * 8 * (double)iters * grid * wpsm;
      printf("{\"probe\": \"dmma_m8n8k4\", \"warps_per_sm\": %d, \"tflops\": %.3f}\n", wpsm, flops / ms / 1e9);
    }
    {
      int iters = 2000;
      float ms = time_kernel(dmma_m16n8k4<8>, grid, block, out, iters, reps);
      double flops = 2.0 * 16 * 8 * 4 * 8 * (double)iters * grid * wpsm;
      printf("{\"probe\": \"dmma_m16n8k4\", \"warps_per_sm\": %d, \"tflops\": %.3f}\n", wpsm, flops / ms / 1e9);
    }
    {
      int iters = 1000;
      float ms = time_kernel(dmma_m16n8k8<8>, grid, block, out, iters, reps);
      double flops = 2.0 * 16 * 8 * 8 * 8 * (double)iters * grid * wpsm;
      printf("{\"probe\": \"dmma_m16n8k8\", \"warps_per_sm\": %d, \"tflops\": %.3f}\n", wpsm, flops / ms / 1e9);
    }
    {
      int iters = 500;
      float ms = time_kernel(dmma_m16n8k16<8>, grid, block, out, iters, reps);
      double flops = 2.0 * 16 * 8 * 16 * 8 * (double)iters * grid * wpsm;
      printf("{\"probe\": \"dmma_m16n8k16\", \"warps_per_sm\": %d, \"tflops\": %.3f}\n", wpsm, flops / ms / 1e9);
    }
  }
  printf("{\"sms\": %d, \"clock_khz\": %d}\n", sms, clk);
  return 0;
}
