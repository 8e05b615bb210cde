// Probe: single-thread tcgen05.mma issue rate for the shifted-window tile
// loop (3x3 taps x KB/32 K-steps per tile, one commit per tile), comparing
// how the descriptors reach the instruction:
//   mode 0: lane 0 only, descriptors from a shared-memory table (per-thread
//           registers -> R2UR + ELECT waterfall per MMA)
//   mode 1: whole warp runs the loop, descriptors from warp-uniform
//           arithmetic (uniform datapath), elect.sync around the MMA
//   mode 2: mode 1 with the tap loops fully unrolled (R, S compile-time)
// Prints SM cycles per MMA; the N=64 M=128 K=32 i8 MMA needs ~48 (SMEM-bound).
// Build: make -C tools mma-rate
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

#include "kernels/ptx.cuh"

using namespace tzcdev;

struct Tab {
  uint32_t a[64], b[64];
  int n;
};

template <int NB, int MODE>
__global__ void __launch_bounds__(640, 1) mma_rate(int tiles, int wp, int kb, long long* cycles,
                                                   const __grid_constant__ Tab ct) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t mbar[2], fin;
  __shared__ uint32_t slot;
  __shared__ uint64_t tab[2 * 64];
  const uint32_t warp = warp_id();
  const uint32_t lane = threadIdx.x & 31;
  const int ksteps = kb / 32;
  if (threadIdx.x == 0) {
    mbar_init(&mbar[0], 1);
    mbar_init(&mbar[1], 1);
    mbar_init(&fin, 1);
    fence_barrier_init();
    int i = 0;
    for (int r = 0; r < 3; ++r)
      for (int s = 0; s < 3; ++s)
        for (int k = 0; k < ksteps; ++k, ++i) {
          tab[2 * i] = (uint64_t)(((r * wp + s) * kb + 32 * k) >> 4);
          tab[2 * i + 1] = smem_desc_kmajor(smem_u32(sm) + 96 * 1024 + (r * 3 + s) * NB * kb + 32 * k, kb);
        }
  }
  if (warp == 1) tmem_alloc<256>(&slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  const uint32_t idesc = idesc_i8(128, NB);
  long long t0 = clock64();
  if (MODE == 0 && threadIdx.x == 0) {
    const uint64_t a0 = smem_desc_kmajor(smem_u32(sm), kb);
    const int per = 9 * ksteps;
    for (int t = 0; t < tiles; ++t) {
      for (int i = 0; i < per; ++i) umma<false>(tmem + (t & 1) * NB, a0 + tab[2 * i], tab[2 * i + 1], idesc, i > 0);
      umma_commit(&mbar[t & 1]);
    }
    umma_commit(&fin);
  } else if (MODE == 1 && warp == 0) {
    const uint32_t a_base = smem_u32(sm), b_base = smem_u32(sm) + 96 * 1024;
    for (int t = 0; t < tiles; ++t) {
      const uint32_t d = tmem + (t & 1) * NB;
      for (int r = 0; r < 3; ++r)
        for (int s = 0; s < 3; ++s)
          for (int k = 0; k < ksteps; ++k) {
            const uint64_t ad = smem_desc_kmajor(a_base + (r * wp + s) * kb + 32 * k, kb);
            const uint64_t bd = smem_desc_kmajor(b_base + (r * 3 + s) * NB * kb + 32 * k, kb);
            if (elect_one()) umma<false>(d, ad, bd, idesc, (r | s | k) ? 1u : 0u);
          }
      if (elect_one()) umma_commit(&mbar[t & 1]);
    }
    if (elect_one()) umma_commit(&fin);
  } else if (MODE == 2 && warp == 0) {
    const uint32_t a_base = smem_u32(sm), b_base = smem_u32(sm) + 96 * 1024;
    const uint64_t a0 = smem_desc_kmajor(a_base, kb), b0 = smem_desc_kmajor(b_base, kb);
    for (int t = 0; t < tiles; ++t) {
      const uint32_t d = tmem + (t & 1) * NB;
#pragma unroll
      for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int s = 0; s < 3; ++s)
#pragma unroll 2
          for (int k = 0; k < ksteps; ++k) {
            const uint64_t ad = a0 + (uint64_t)((uint32_t)((r * wp + s) * kb + 32 * k) >> 4);
            const uint64_t bd = b0 + (uint64_t)((uint32_t)((r * 3 + s) * NB * kb + 32 * k) >> 4);
            if (elect_one()) umma<false>(d, ad, bd, idesc, (r | s | k) ? 1u : 0u);
          }
      if (elect_one()) umma_commit(&mbar[t & 1]);
    }
    if (elect_one()) umma_commit(&fin);
  }
  else if (MODE >= 3 && warp == 0) {
    // MODE 6: pair-mode (SWIZZLE_NONE, LBO = 16 B: two consecutive 16-byte pixels per K=32) descriptors
    const uint64_t a0 = MODE == 6 ? (((uint64_t)(smem_u32(sm) >> 4) & 0x3FFF) | (1ull << 16) | (8ull << 32) | (1ull << 46))
                                  : smem_desc_kmajor(smem_u32(sm), kb);
    const uint64_t b0 = MODE == 6 ? (((uint64_t)((smem_u32(sm) + 96 * 1024) >> 4) & 0x3FFF) | ((uint64_t)(NB * 16 >> 4) << 16) |
                                     (8ull << 32) | (1ull << 46))
                                  : smem_desc_kmajor(smem_u32(sm) + 96 * 1024, kb);
    for (int t = 0; t < tiles; ++t) {
      const uint32_t d = tmem + (t & 1) * NB;
      if (MODE == 6) {
#pragma unroll 2
        for (int i = 0; i < ct.n; ++i)
          if (elect_one()) umma<false>(d, a0 + ct.a[i], b0 + ct.b[i], idesc, i > 0);
      } else if (MODE == 5) {
        for (int i = 0; i < ct.n; ++i)
          if (elect_one()) umma<false>(d, a0, b0, idesc, i > 0);
      } else if (MODE == 3) {
#pragma unroll 2
        for (int i = 0; i < ct.n; ++i)
          if (elect_one()) umma<false>(d, a0 + ct.a[i], b0 + ct.b[i], idesc, i > 0);
      } else {
#pragma unroll 4
        for (int i = 0; i < ct.n; ++i)
          if (elect_one()) umma<false>(d, a0 + ct.a[i], b0 + ct.b[i], idesc, i > 0);
      }
      if (elect_one()) umma_commit(&mbar[t & 1]);
    }
    if (elect_one()) umma_commit(&fin);
  }
  if (warp == 0) {
    mbar_wait(&fin, 0);
    if (blockIdx.x == 0 && lane == 0) cycles[0] = clock64() - t0;
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<256>(tmem);
  }
}

// Cost of the per-tile synchronisation of the MMA warp on barriers that are
// already complete: try_wait (suspend hint) / test_wait spin / fences.
__global__ void sync_cost(int iters, long long* cycles) {
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const uint32_t warp = warp_id();
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<32>(&slot);
  __syncthreads();
  if (threadIdx.x == 0) mbar_arrive(&bar);  // phase 0 complete
  __syncthreads();
  if (warp == 0) {
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) mbar_wait(&bar, 0);
    long long t1 = clock64();
    for (int i = 0; i < iters; ++i) {
      mbar_wait(&bar, 0);
      tc_fence_after();
    }
    long long t2 = clock64();
    for (int i = 0; i < iters; ++i) {
      uint32_t done = 0;
      while (!done)
        asm volatile("{\n\t.reg .pred P;\n\tmbarrier.test_wait.parity.shared::cta.b64 P, [%1], %2;\n\tselp.b32 %0, 1, 0, P;\n\t}"
                     : "=r"(done) : "r"(smem_u32(&bar)), "r"(0u) : "memory");
    }
    long long t3 = clock64();
    for (int i = 0; i < iters; ++i) {
      if (elect_one()) umma_commit(&bar);
      __syncwarp();
    }
    long long t4 = clock64();
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      cycles[0] = t1 - t0;
      cycles[1] = t2 - t1;
      cycles[2] = t3 - t2;
      cycles[3] = t4 - t3;
    }
  }
  __syncthreads();
  if (warp == 1) tmem_dealloc<32>(slot);
}

int main() {
  long long* dc;
  cudaMalloc(&dc, 64);
  const int tiles = 112;
  auto run = [&](auto kern, const char* name, int kb) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    Tab ct{};
    ct.n = 9 * (kb / 32);
    for (int r = 0, i = 0; r < 3; ++r)
      for (int s = 0; s < 3; ++s)
        for (int k = 0; k < kb / 32; ++k, ++i) {
          ct.a[i] = ((r * 58 + s) * kb + 32 * k) >> 4;
          ct.b[i] = ((r * 3 + s) * 64 * kb + 32 * k) >> 4;
        }
    kern<<<148, 640, 200 * 1024>>>(tiles, 58, kb, dc, ct);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      printf("%s: %s\n", name, cudaGetErrorString(e));
      exit(1);
    }
    long long c;
    cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost);
    const int n = tiles * 9 * (kb / 32);
    printf("%-22s kb %3d: %.1f cyc/MMA\n", name, kb, c / (double)n);
  };
  {
    sync_cost<<<148, 640>>>(1000, dc);
    cudaDeviceSynchronize();
    long long c[4];
    cudaMemcpy(c, dc, 32, cudaMemcpyDeviceToHost);
    printf("try_wait(done) %.1f  +fence %.1f  test_wait spin %.1f  commit %.1f cyc\n", c[0] / 1000.0, c[1] / 1000.0,
           c[2] / 1000.0, c[3] / 1000.0);
  }
  auto run_pair = [&](auto kern, const char* name, int wp, int salign) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    Tab ct{};
    ct.n = 8;
    for (int r = 0, i = 0; r < 4; ++r)
      for (int s2 = 0; s2 < 4; s2 += 2, ++i) {
        ct.a[i] = (uint32_t)(r * wp + s2 * salign);  // 16-byte pixels
        ct.b[i] = (uint32_t)(((r * 4 + s2) * 64 * 16) >> 4);
      }
    kern<<<148, 640, 200 * 1024>>>(tiles, wp, 16, dc, ct);
    cudaDeviceSynchronize();
    long long c;
    cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost);
    printf("%-22s wp %3d salign %d: %.1f cyc/MMA\n", name, wp, salign, c / (double)(tiles * 8));
  };
  run_pair(mma_rate<64, 6>, "pair N=64", 115, 1);
  run_pair(mma_rate<64, 6>, "pair N=64", 120, 1);
  run_pair(mma_rate<64, 6>, "pair N=64", 120, 4);
  run_pair(mma_rate<64, 6>, "pair N=64", 0, 0);
  for (int kb : {64}) {
    run(mma_rate<64, 0>, "N=64 lane0+table", kb);
    run(mma_rate<64, 1>, "N=64 uniform", kb);
    run(mma_rate<64, 2>, "N=64 uniform unrolled", kb);
    run(mma_rate<128, 0>, "N=128 lane0+table", kb);
    run(mma_rate<128, 2>, "N=128 uniform unrolled", kb);
    run(mma_rate<64, 3>, "N=64 param table u2", kb);
    run(mma_rate<64, 4>, "N=64 param table u4", kb);
    run(mma_rate<128, 4>, "N=128 param table u4", kb);
    run(mma_rate<64, 5>, "N=64 fixed desc", kb);
    run(mma_rate<128, 5>, "N=128 fixed desc", kb);
  }
  return 0;
}
