// Probe: mbarrier hand-off round-trip latency between warps, with a plain
// mbarrier.arrive or a tcgen05.commit as the signal, 1 or 16 waiting warps,
// try_wait (suspend hint) or test_wait spinning.  Cycles per round trip.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2101_08458_b200/csrc tools/handoff_probe.cu
#include <cuda_runtime.h>

#include <cstdio>

#include "kernels/ptx.cuh"

using namespace tzcdev;

template <bool COMMIT, bool SPIN>
__global__ void pingpong(int iters, int nb, long long* out) {
  __shared__ uint64_t bx, by;
  __shared__ uint32_t slot;
  const uint32_t warp = warp_id(), lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    mbar_init(&bx, 1);
    mbar_init(&by, nb);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc<32>(&slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  auto wait = [&](uint64_t* b, uint32_t ph) {
    if (SPIN) mbar_wait_spin(b, ph);
    else mbar_wait(b, ph);
  };
  long long t0 = clock64();
  if (warp == 0) {  // "MMA" warp: signal X, wait for all B warps on Y
    for (int i = 0; i < iters; ++i) {
      if (COMMIT) {
        if (elect_one()) umma_commit(&bx);
        __syncwarp();
      } else if (lane == 0) {
        mbar_arrive(&bx);
      }
      wait(&by, i & 1);
    }
    if (lane == 0) out[blockIdx.x] = clock64() - t0;
  } else if ((int)warp <= nb) {  // "epilogue" warps
    for (int i = 0; i < iters; ++i) {
      wait(&bx, i & 1);
      __syncwarp();
      if (lane == 0) mbar_arrive(&by);
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) tmem_dealloc<32>(slot);
}

template <bool C, bool S>
void run(int nb) {
  long long* d;
  cudaMalloc(&d, 148 * sizeof(long long));
  const int iters = 2000;
  pingpong<C, S><<<148, 32 * 17>>>(iters, nb, d);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (long long x : h) avg += x;
  printf("signal=%s wait=%s waiters=%2d: %.0f cycles per round trip (%s)\n", C ? "tcgen05.commit" : "arrive",
         S ? "test_wait spin" : "try_wait", nb, avg / 148 / iters, cudaGetErrorString(e));
  cudaFree(d);
}

int main() {
  for (int nb : {1, 16}) {
    run<false, false>(nb);
    run<false, true>(nb);
    run<true, false>(nb);
    run<true, true>(nb);
  }
  return 0;
}
