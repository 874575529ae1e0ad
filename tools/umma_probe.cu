// umma_probe.cu — tcgen05.mma issue-rate probe (not product code): one CTA per SM, one thread
// issues R back-to-back MMAs on resident shared-memory operands into a TMEM accumulator, for
// several (kind, N, swizzle) shapes; prints clk per MMA and the implied dense rate.  Used to pick
// the Ozaki (kind::i8) tile shape.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2511_14923_b200/csrc \
//        -o tools/umma_probe tools/umma_probe.cu -lcuda
#include <cstdio>
#include <cstdlib>
#include <cuda.h>
#include <cuda_runtime.h>

#include "c64_gemm.cuh"
#include "ozaki_gemm.cuh"

using namespace mps;

__device__ __forceinline__ uint64_t desc(uint32_t saddr, int sw, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)(sw == 128 ? 2 : sw == 64 ? 4 : 6) << 61;
  return d;
}

template <int KIND, int N, int SW>  // KIND 0: i8, 1: tf32
__global__ void __launch_bounds__(128, 1) probe(int R, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  uint8_t* s = sm + ((1024u - (smem_u32(sm) & 1023u)) & 1023u);
  for (int i = threadIdx.x; i < 96 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(s)[i] = 0;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&slot)), "r"(512u));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (threadIdx.x == 0) {
    const uint32_t a = smem_u32(s), b = smem_u32(s + 32 * 1024);
    const uint32_t sbo = SW * 8;  // 8-row atom
    constexpr uint32_t idesc = KIND == 0 ? idesc_i8(128, N) : idesc_tf32(128, N);
    const int ksteps = SW / 32;  // 32-byte K steps per swizzle row
    long long t0 = clock64();
    for (int r = 0; r < R; ++r) {
      const uint32_t off = (r % ksteps) * 32;
      const uint64_t da = desc(a + off, SW, sbo), db = desc(b + off, SW, sbo);
      if (KIND == 0)
        umma_i8(tmem, da, db, idesc, 1u);
      else
        umma_tf32(tmem, da, db, idesc, 1u);
    }
    umma_commit(&bar);
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    out[blockIdx.x] = (unsigned long long)(t1 - t0);
  }
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512u));
}

// the Ozaki mainloop pattern without TMA / barriers: per K step S(S+1)/2 products of plane i of A
// with plane j of B into accumulator d = i + j (S x N TMEM columns), stage layout of ozaki_gemm.cuh
template <int S, int N, bool SAME_ACC>
__global__ void __launch_bounds__(128, 1) probe_oz(int R, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  uint8_t* s = sm + ((1024u - (smem_u32(sm) & 1023u)) & 1023u);
  constexpr int A_BYTES = S * 128 * 32, B_BYTES = S * N * 32, STAGE = A_BYTES + B_BYTES, NST = 3;
  for (int i = threadIdx.x; i < NST * STAGE / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(s)[i] = 0;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&slot)), "r"(512u));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (threadIdx.x == 0) {
    constexpr uint32_t idesc = idesc_i8(128, N);
    long long t0 = clock64();
    for (int r = 0; r < R; ++r) {
      const uint32_t st = smem_u32(s + (r % NST) * STAGE);
#pragma unroll
      for (int d = 0; d < S; ++d)
#pragma unroll
        for (int i = 0; i <= d; ++i) {
          const uint64_t da = umma_desc_k_sw32(st + i * 256, S * 256);
          const uint64_t db = umma_desc_k_sw32(st + A_BYTES + (d - i) * 256, S * 256);
          umma_i8(tmem + (SAME_ACC ? 0 : d * N), da, db, idesc, 1u);
        }
    }
    umma_commit(&bar);
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    out[blockIdx.x] = (unsigned long long)(t1 - t0);
  }
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512u));
}

// smem port probe: MMAs (S=4, N=128 Ozaki pattern, 64 clk each at full rate) while another warp
// streams bulk copies from L2 into a separate smem region; copy_kb = KiB copied per k step.
__global__ void __launch_bounds__(128, 1) probe_port(int R, int copy_kb, const int8_t* src, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar, cbar[2];
  __shared__ uint32_t slot;
  uint8_t* s = sm + ((1024u - (smem_u32(sm) & 1023u)) & 1023u);
  constexpr int S = 4, N = 128, A_BYTES = S * 128 * 32, B_BYTES = S * N * 32, STAGE = A_BYTES + B_BYTES;
  uint8_t* wbuf = s + STAGE;  // 2 x 64 KiB copy targets
  for (int i = threadIdx.x; i < STAGE / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(s)[i] = 0;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    mbar_init(&cbar[0], 1);
    mbar_init(&cbar[1], 1);
    fence_barrier_init();
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&slot)), "r"(512u));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  long long t0 = clock64();
  if (threadIdx.x == 0) {
    constexpr uint32_t idesc = idesc_i8(128, N);
    const uint32_t st = smem_u32(s);
    for (int r = 0; r < R; ++r) {
#pragma unroll
      for (int d = 0; d < S; ++d)
#pragma unroll
        for (int i = 0; i <= d; ++i) {
          const uint64_t da = umma_desc_k_sw32(st + i * 256, S * 256);
          const uint64_t db = umma_desc_k_sw32(st + A_BYTES + (d - i) * 256, S * 256);
          umma_i8(tmem + d * N, da, db, idesc, 1u);
        }
    }
    umma_commit(&bar);
    mbar_wait(&bar, 0);
    out[2 * blockIdx.x] = (unsigned long long)(clock64() - t0);
  } else if (threadIdx.x == 32 && copy_kb > 0) {
    const uint32_t bytes = copy_kb * 1024;
    for (int r = 0; r < R; ++r) {
      const int b = r & 1;
      if (r >= 2) mbar_wait(&cbar[b], ((r >> 1) - 1) & 1);
      mbar_arrive_expect_tx(&cbar[b], bytes);
      bulk_load_1d(wbuf + b * 65536, src + (size_t)((blockIdx.x * 7 + r) % 64) * 65536, bytes, &cbar[b]);
    }
    for (int r = R; r < R + 2; ++r) mbar_wait(&cbar[r & 1], ((r >> 1) - 1) & 1);
    out[2 * blockIdx.x + 1] = (unsigned long long)(clock64() - t0);
  }
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512u));
}

void run_port(int copy_kb) {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned long long* d;
  cudaMalloc(&d, 2 * sms * sizeof(unsigned long long));
  cudaMemset(d, 0, 2 * sms * sizeof(unsigned long long));
  int8_t* src;
  cudaMalloc(&src, 64 * 65536);
  cudaMemset(src, 1, 64 * 65536);
  const int smem = 32 * 1024 + 2 * 65536 + 1024;
  cudaFuncSetAttribute(probe_port, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int R = 2000;
  probe_port<<<sms, 128, smem>>>(R, copy_kb, src, d);
  cudaError_t err = cudaDeviceSynchronize();
  unsigned long long h[2048];
  cudaMemcpy(h, d, 2 * sms * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
  double mma = 0, cp = 0;
  for (int i = 0; i < sms; ++i) { mma += h[2 * i]; cp += h[2 * i + 1]; }
  mma /= sms; cp /= sms;
  printf("{\"probe\": \"port\", \"copy_kb_per_kstep\": %d, \"mma_clk_per_kstep\": %.1f, \"copy_clk_per_kstep\": %.1f, "
         "\"copy_B_per_clk\": %.1f, \"err\": \"%s\"}\n", copy_kb, mma / R, cp / R, copy_kb * 1024.0 * R / (cp > 0 ? cp : 1),
         cudaGetErrorString(err));
  cudaFree(d);
  cudaFree(src);
}

template <int S, int N, bool SAME>
void run_oz() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned long long* d;
  cudaMalloc(&d, sms * sizeof(unsigned long long));
  const int smem = 3 * (S * 128 * 32 + S * N * 32) + 1024;
  cudaFuncSetAttribute(probe_oz<S, N, SAME>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int R = 1000;
  probe_oz<S, N, SAME><<<sms, 128, smem>>>(R, d);
  cudaError_t err = cudaDeviceSynchronize();
  unsigned long long h[1024];
  cudaMemcpy(h, d, sms * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
  double clk = 0;
  for (int i = 0; i < sms; ++i) clk += h[i];
  clk /= sms;
  const int P = S * (S + 1) / 2;
  printf("{\"probe\": \"ozaki_loop\", \"S\": %d, \"N\": %d, \"same_acc\": %d, \"clk_per_mma\": %.2f, \"err\": \"%s\"}\n",
         S, N, (int)SAME, clk / ((double)R * P), cudaGetErrorString(err));
  cudaFree(d);
}

template <int KIND, int N, int SW>
void run(const char* name) {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk_khz = 0;
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  unsigned long long* d;
  cudaMalloc(&d, sms * sizeof(unsigned long long));
  const int smem = 97 * 1024;
  cudaFuncSetAttribute(probe<KIND, N, SW>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int R = 20000;
  probe<KIND, N, SW><<<sms, 128, smem>>>(R, d);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  probe<KIND, N, SW><<<sms, 128, smem>>>(R, d);
  cudaEventRecord(e1);
  cudaError_t err = cudaDeviceSynchronize();
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long h[1024];
  cudaMemcpy(h, d, sms * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
  double clk = 0;
  for (int i = 0; i < sms; ++i) clk += h[i];
  clk /= sms;
  const int K = KIND == 0 ? 32 : 8;
  const double ops = 2.0 * 128 * N * K * (double)R * sms;
  printf("{\"probe\": \"%s\", \"N\": %d, \"swizzle\": %d, \"clk_per_mma\": %.2f, \"tops\": %.1f, \"err\": \"%s\"}\n",
         name, N, SW, clk / R, ops / (ms * 1e-3) / 1e12, cudaGetErrorString(err));
  cudaFree(d);
}

int main() {
  if (getenv("PORT_ONLY")) {
    for (int kb : {0, 8, 16, 32, 48, 64}) run_port(kb);
    return 0;
  }
  run<0, 64, 32>("i8");
  run<0, 64, 128>("i8");
  run<0, 128, 32>("i8");
  run<0, 128, 128>("i8");
  run<0, 256, 32>("i8");
  run<0, 256, 128>("i8");
  run<1, 64, 128>("tf32");
  run<1, 128, 128>("tf32");
  run<1, 256, 128>("tf32");
  for (int kb : {0, 8, 16, 32, 48, 64}) run_port(kb);
  return 0;
}
