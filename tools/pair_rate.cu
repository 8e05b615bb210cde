// Probe: the space-to-depth stem's pair-mode MMA stream in isolation, shaped
// like conv_ws_kernel's unit loop (MT sub-tiles x 8 K=32 MMAs, N = 64,
// SWIZZLE_NONE 16-byte pixels, LBO = 16 B), to find why the kernel's MMA phase
// runs at ~2x the 54-cycle rate tools/mma_rate.cu measured.  Variants:
//   mt      1, 2, 4 sub-tiles (distinct TMEM accumulators) per unit
//   fill    0 = zero SMEM operands, 1 = random bytes
//   wp      row pitch of the shifted window in pixels (115: the stem's S2D grid)
// Prints cycles per MMA (clock64 around the issue loop + final commit wait).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2101_08458_b200/csrc tools/pair_rate.cu
#include <cuda_runtime.h>

#include <cstdio>

#include "kernels/conv_ws.cuh"

using namespace tzcdev;

__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__global__ void __launch_bounds__(128, 1) pair_rate(int units, int mt, int wp, int fill, long long* cyc) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t done;
  __shared__ uint32_t slot;
  const uint32_t warp = warp_id();
  uint32_t h = threadIdx.x * 2654435761u + 7u;
  for (int i = threadIdx.x; i < 160 * 1024 / 4; i += blockDim.x) {
    h ^= h << 13; h ^= h >> 17; h ^= h << 5;
    reinterpret_cast<uint32_t*>(sm)[i] = fill ? h : 0u;
  }
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
    const uint32_t a_base = smem_u32(sm);                 // A: pixels at 16-byte pitch
    const uint32_t b_base = smem_u32(sm + 128 * 1024);    // B: [tap][64][16 B]
    const uint64_t a0 = smem_desc_none(a_base, 16, 128);
    const uint64_t b0 = smem_desc_none(b_base, 64 * 16, 128);
    constexpr uint32_t ID = idesc_i8(128, 64);
    uint32_t pa[8], pb[8];
    for (int r = 0, i = 0; r < 4; ++r)
      for (int s2 = 0; s2 < 4; s2 += 2, ++i) {
        pa[i] = (uint32_t)(r * wp + s2);
        pb[i] = (uint32_t)(((r * 4 + s2) * 64 * 16) >> 4);
      }
    const long long t0 = clock64();
    const unsigned long long g0 = gtime();
    for (int u = 0; u < units; ++u) {
      const uint32_t accb = tm + (uint32_t)((u & 1) * 256);
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        if (t < mt) {
          const uint64_t at = a0 + (uint64_t)(t * 128);
#pragma unroll
          for (int i = 0; i < 8; ++i)
            if (elect_one()) umma<false>(accb + t * 64, at + pa[i], b0 + pb[i], ID, i > 0 ? 1u : 0u);
        }
      }
    }
    if (elect_one()) umma_commit(&done);
    __syncwarp();
    mbar_wait(&done, 0);
    if (threadIdx.x == 0) {
      cyc[blockIdx.x] = clock64() - t0;
      cyc[148 + blockIdx.x] = (long long)(gtime() - g0);
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) tmem_dealloc<512>(tm);
}

int main() {
  long long* d;
  cudaMalloc(&d, 2 * 148 * sizeof(long long));
  const int smem = 1024 + 160 * 1024;
  cudaFuncSetAttribute(pair_rate, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int fill : {0, 1})
    for (int mt : {1, 2, 4})
      for (int wp : {115, 120}) {
        const int units = 4000 / mt;
        pair_rate<<<148, 128, smem>>>(units, mt, wp, fill, d);
        cudaError_t e = cudaDeviceSynchronize();
        long long h[296];
        cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
        double avg = 0, ns = 0;
        for (int i = 0; i < 148; ++i) avg += h[i], ns += h[148 + i];
        avg /= 148;
        ns /= 148;
        printf("fill %d mt %d wp %d: %.1f cycles/MMA, %.1f ns/MMA, SM clock %.0f MHz  (%s)\n", fill, mt, wp,
               avg / (units * mt * 8.0), ns / (units * mt * 8.0), avg / ns * 1e3, cudaGetErrorString(e));
      }
  return 0;
}
