// Launch-floor micro-benchmarks for the conv kernel's building blocks.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_2101_08458_b200/csrc tools/microbench.cu
#include <cuda_runtime.h>

#include <cstdio>

#include "kernels/ptx.cuh"

using namespace tzcdev;

__global__ void __launch_bounds__(384, 1) k_empty() {
  extern __shared__ uint8_t smem[];
  if (threadIdx.x == 1000) smem[0] = 1;
}

__global__ void __launch_bounds__(384, 1) k_tmem() {
  __shared__ uint32_t slot;
  if (warp_id() == 2) tmem_alloc<512>(&slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  uint32_t base = slot;
  __syncthreads();
  if (warp_id() == 2) {
    tc_fence_after();
    tmem_dealloc<512>(base);
  }
}

template <bool kHint>
__global__ void __launch_bounds__(384, 1) k_mbar_pingpong(int rounds) {
  __shared__ uint64_t bars[2];
  if (threadIdx.x == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    fence_barrier_init();
  }
  __syncthreads();
  const uint32_t w = warp_id();
  uint32_t ph = 0;
  for (int i = 0; i < rounds; ++i) {
    if (w == 0 && (threadIdx.x & 31) == 0) {
      mbar_arrive(&bars[0]);
      if (kHint)
        mbar_wait(&bars[1], ph);
      else {
        uint32_t addr = smem_u32(&bars[1]);
        asm volatile(
            "{\n\t.reg .pred P;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t@!P bra W_%=;\n\t}" ::"r"(
                addr),
            "r"(ph)
            : "memory");
      }
    } else if (w == 4 && (threadIdx.x & 31) == 0) {
      if (kHint)
        mbar_wait(&bars[0], ph);
      else {
        uint32_t addr = smem_u32(&bars[0]);
        asm volatile(
            "{\n\t.reg .pred P;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t@!P bra W_%=;\n\t}" ::"r"(
                addr),
            "r"(ph)
            : "memory");
      }
      mbar_arrive(&bars[1]);
    }
    ph ^= 1;
  }
}

template <typename F>
float time_it(F f, int reps) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  f();
  cudaDeviceSynchronize();
  cudaEventRecord(a);
  for (int i = 0; i < reps; ++i) f();
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return ms * 1000.f / reps;
}

int main() {
  const int smem = 197888;
  cudaFuncSetAttribute(k_empty, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  printf("empty 148x384, 0 smem:      %8.2f us\n", time_it([] { k_empty<<<148, 384>>>(); }, 200));
  printf("empty 148x384, 197KB smem:  %8.2f us\n", time_it([&] { k_empty<<<148, 384, smem>>>(); }, 200));
  printf("tmem alloc/dealloc 512:     %8.2f us\n", time_it([] { k_tmem<<<148, 384>>>(); }, 200));
  printf("mbar pingpong x100 (hint):  %8.2f us\n", time_it([] { k_mbar_pingpong<true><<<148, 384>>>(100); }, 50));
  printf("mbar pingpong x100 (spin):  %8.2f us\n", time_it([] { k_mbar_pingpong<false><<<148, 384>>>(100); }, 50));
  cudaError_t e = cudaDeviceSynchronize();
  printf("status: %s\n", cudaGetErrorString(e));
  return 0;
}
