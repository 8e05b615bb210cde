// Probe: the tcgen05.mma kind::i8 issue rate with operands already in SMEM
// (no TMA, no epilogue): one warp per CTA issues `iters` back-to-back
// M128 x N x K32 MMAs into one TMEM accumulator, 148 CTAs.  Prints cycles per
// MMA (clock64 around the loop) and the whole-GPU int8 rate from CUDA events
// — the tensor-core ceiling at the clocks this pool runs.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2101_08458_b200/csrc tools/i8_peak.cu
#include <cuda_runtime.h>

#include <cstdio>

#include "kernels/ptx.cuh"

using namespace tzcdev;

template <int N, bool PAIRK>
__global__ void __launch_bounds__(128, 1) peak(int iters, long long* cyc) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t done;
  __shared__ uint32_t slot;
  const uint32_t warp = warp_id();
  for (int i = threadIdx.x; i < (128 + N) * 128 / 16; i += blockDim.x) reinterpret_cast<uint4*>(sm)[i] = make_uint4(0, 0, 0, 0);
  if (threadIdx.x == 0) {
    mbar_init(&done, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<512>(&slot);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = slot;
  if (warp == 0) {
    const uint32_t a = smem_u32(sm), b = smem_u32(sm + 128 * 128);
    constexpr uint32_t ID = idesc_i8(128, N);
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if (elect_one()) umma<false>(tm, smem_desc_kmajor(a + 32 * k, 128), smem_desc_kmajor(b + 32 * k, 128), ID, 1u);
    }
    if (elect_one()) umma_commit(&done);
    __syncwarp();
    mbar_wait(&done, 0);
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) tmem_dealloc<512>(tm);
}

template <int N>
void run(int iters) {
  long long* d;
  cudaMalloc(&d, 148 * sizeof(long long));
  auto k = peak<N, false>;
  const int smem = 1024 + (128 + N) * 128;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  k<<<148, 128, smem>>>(iters, d);
  cudaDeviceSynchronize();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<<<148, 128, smem>>>(iters, d);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (long long x : h) avg += x;
  avg /= 148;
  const double mmas = 4.0 * iters;
  const double ops = 2.0 * 128 * N * 32 * mmas * 148;
  printf("N=%3d: %.1f cycles/MMA (clock64), %.0f TOPS whole GPU (events, %.3f ms) err=%s\n", N, avg / mmas,
         ops / (ms * 1e-3) / 1e12, ms, cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

int main() {
  run<64>(20000);
  run<128>(20000);
  run<256>(20000);
  run<256>(40000);
  return 0;
}
