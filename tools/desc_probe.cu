// Probe: does a SWIZZLE_128B K-major UMMA descriptor whose start address is
// shifted by a whole number of 128-byte rows (not a multiple of the 8-row
// atom) read the rows TMA wrote there?  Needed for the shifted-window
// ("padded grid") 3x3 conv: all 9 taps are row-shifted views of one SMEM block.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -I../paper_2101_08458_b200/csrc desc_probe.cu
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#include "kernels/ptx.cuh"

using namespace tzcdev;

constexpr int ROWS = 256, KB = 128, N = 64;

__global__ void __launch_bounds__(128, 1) probe(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap tb,
                                               int shift, int base_off_mode, int32_t* out) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = sm;
  uint8_t* sB = sm + ROWS * KB;
  __shared__ uint64_t bar, mbar;
  __shared__ uint32_t slot;
  const uint32_t warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    mbar_init(&mbar, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<64>(&slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (threadIdx.x == 0) {
    mbar_expect_tx(&bar, ROWS * KB + N * KB);
    tma_load_2d(sA, &ta, &bar, 0, 0);
    tma_load_2d(sB, &tb, &bar, 0, 0);
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  if (threadIdx.x == 0) {
    const uint32_t a0 = smem_u32(sA) + shift * KB;
    const uint32_t b0 = smem_u32(sB);
    for (int k = 0; k < KB / 32; ++k) {
      uint64_t ad = smem_desc_kmajor(a0 + 32 * k, KB);
      if (base_off_mode == 1) ad |= (uint64_t)((a0 >> 7) & 7) << 49;
      const uint64_t bd = smem_desc_kmajor(b0 + 32 * k, KB);
      umma<false>(tmem, ad, bd, idesc_i8(128, N), k > 0);
    }
    umma_commit(&mbar);
  }
  mbar_wait(&mbar, 0);
  tc_fence_after();
  uint32_t v[32];
  for (int c = 0; c < N / 32; ++c) {
    tmem_ld32(tmem + ((warp * 32) << 16) + c * 32, v);
    tmem_ld_wait();
    for (int j = 0; j < 32; ++j) out[(warp * 32 + lane) * N + c * 32 + j] = (int32_t)v[j];
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<64>(tmem);
  }
}

// SWIZZLE_NONE K-major: A rows of 16 B at 16 B pitch (a dense [rows][16]
// array); one K=32 MMA reads row i's chunk 0 at start+16i and chunk 1 at
// start+16+16i (LBO = 16 B: the next row), i.e. taps (s, s+1) of a stride-1
// conv over 16-byte pixels.  B stored [chunk][n][16] (LBO = N*16, SBO = 128).
__device__ uint64_t desc_none(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  return d;  // layout type 0 = SWIZZLE_NONE
}

__global__ void __launch_bounds__(128, 1) probe16(const uint8_t* gA, const int8_t* gB, int shift, int32_t* out) {
  __shared__ __align__(1024) uint8_t sA[ROWS * 16];
  __shared__ __align__(1024) uint8_t sB[2 * N * 16];
  __shared__ uint64_t mbar;
  __shared__ uint32_t slot;
  const uint32_t warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  for (int i = threadIdx.x; i < ROWS * 16; i += 128) sA[i] = gA[i];
  for (int i = threadIdx.x; i < 2 * N * 16; i += 128) sB[i] = (uint8_t)gB[i];
  if (threadIdx.x == 0) {
    mbar_init(&mbar, 1);
    fence_barrier_init();
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == 1) tmem_alloc<64>(&slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (threadIdx.x == 0) {
    const uint64_t ad = desc_none(smem_u32(sA) + shift * 16, 16, 128);
    const uint64_t bd = desc_none(smem_u32(sB), N * 16, 128);
    umma<false>(tmem, ad, bd, idesc_i8(128, N), 0);
    umma_commit(&mbar);
  }
  mbar_wait(&mbar, 0);
  tc_fence_after();
  uint32_t v[32];
  for (int c = 0; c < N / 32; ++c) {
    tmem_ld32(tmem + ((warp * 32) << 16) + c * 32, v);
    tmem_ld_wait();
    for (int j = 0; j < 32; ++j) out[(warp * 32 + lane) * N + c * 32 + j] = (int32_t)v[j];
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<64>(tmem);
  }
}

// MMA throughput: issue `iters` MMAs (M=128, N=NB, K=32 i8) back to back on
// one SM; A start shifted by `shift` rows of `kb` bytes; swz: 128/64/0(none).
template <int NB>
__global__ void __launch_bounds__(128, 1) mma_rate(int shift, int kb, int swz, int iters, long long* cycles) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t mbar;
  __shared__ uint32_t slot;
  const uint32_t warp = threadIdx.x / 32;
  if (threadIdx.x == 0) {
    mbar_init(&mbar, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<256>(&slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (threadIdx.x == 0) {
    const uint32_t a0 = smem_u32(sm) + shift * kb;
    const uint32_t b0 = smem_u32(sm) + 64 * 1024;
    uint64_t ad, bd;
    if (swz == 0) {
      ad = 0; bd = 0;
      ad |= (uint64_t)((a0 >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)8 << 32) | ((uint64_t)1 << 46);
      bd |= (uint64_t)((b0 >> 4) & 0x3FFF) | ((uint64_t)((NB * 16) >> 4) << 16) | ((uint64_t)8 << 32) | ((uint64_t)1 << 46);
    } else {
      ad = smem_desc_kmajor(a0, swz);
      bd = smem_desc_kmajor(b0, swz);
    }
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) umma<false>(tmem, ad, bd, idesc_i8(128, NB), i > 0);
    umma_commit(&mbar);
    mbar_wait(&mbar, 0);
    cycles[0] = clock64() - t0;
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<256>(tmem);
  }
}

int main() {
  {
    long long* dc;
    cudaMalloc(&dc, 8);
    auto run = [&](auto kern, const char* name, int shift, int kb, int swz) {
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      kern<<<1, 128, 200 * 1024>>>(shift, kb, swz, 2000, dc);
      cudaDeviceSynchronize();
      long long c;
      cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost);
      printf("%-12s shift %3d kb %3d swz %3d: %.1f cycles/MMA\n", name, shift, kb, swz, c / 2000.0);
    };
    for (int sh : {0, 1, 3, 8}) {
      run(mma_rate<64>, "N=64", sh, 128, 128);
      run(mma_rate<128>, "N=128", sh, 128, 128);
      run(mma_rate<256>, "N=256", sh, 128, 128);
      run(mma_rate<64>, "N=64 sw64", sh, 64, 64);
      run(mma_rate<64>, "N=64 none", sh, 16, 0);
    }
  }
  cudaDriverEntryPointQueryResult q;
  void* fn = nullptr;
  cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &fn, 12000, cudaEnableDefault, &q);
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  std::vector<uint8_t> hA(ROWS * KB);
  std::vector<int8_t> hB(N * KB);
  srand(1);
  for (auto& x : hA) x = rand() & 0xff;
  for (auto& x : hB) x = (int8_t)(rand() & 0xff);
  void *dA, *dB;
  int32_t* dO;
  cudaMalloc(&dA, hA.size());
  cudaMalloc(&dB, hB.size());
  cudaMalloc(&dO, 128 * N * 4);
  cudaMemcpy(dA, hA.data(), hA.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(dB, hB.data(), hB.size(), cudaMemcpyHostToDevice);
  CUtensorMap ta, tb;
  cuuint64_t da[2] = {KB, ROWS}, db[2] = {KB, N}, sa[1] = {KB}, sb[1] = {KB};
  cuuint32_t ba[2] = {KB, ROWS}, bb[2] = {KB, N}, es[2] = {1, 1};
  enc(&ta, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, dA, da, sa, ba, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
      CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  enc(&tb, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, dB, db, sb, bb, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
      CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  const int smem = 1024 + ROWS * KB + N * KB;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  std::vector<int32_t> hO(128 * N);
  for (int mode = 0; mode < 2; ++mode)
    for (int shift : {0, 1, 2, 3, 5, 7, 8, 9, 58, 117}) {
      if (shift + 128 > ROWS) continue;
      probe<<<1, 128, smem>>>(ta, tb, shift, mode, dO);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) {
        printf("mode %d shift %d: %s\n", mode, shift, cudaGetErrorString(e));
        return 1;
      }
      cudaMemcpy(hO.data(), dO, hO.size() * 4, cudaMemcpyDeviceToHost);
      int bad = 0;
      for (int i = 0; i < 128; ++i)
        for (int j = 0; j < N; ++j) {
          int64_t acc = 0;
          for (int k = 0; k < KB; ++k) acc += (int)hA[(shift + i) * KB + k] * (int)hB[j * KB + k];
          bad += (int32_t)acc != hO[i * N + j];
        }
      printf("base_offset mode %d shift %3d: %s (%d mismatches)\n", mode, shift, bad ? "WRONG" : "ok", bad);
    }
  // ---- 16-byte-row probe
  {
    std::vector<uint8_t> a16(ROWS * 16);
    std::vector<int8_t> b16(2 * N * 16);
    for (auto& x : a16) x = rand() & 0xff;
    for (auto& x : b16) x = (int8_t)(rand() & 0xff);
    uint8_t* dA16;
    int8_t* dB16;
    cudaMalloc(&dA16, a16.size());
    cudaMalloc(&dB16, b16.size());
    cudaMemcpy(dA16, a16.data(), a16.size(), cudaMemcpyHostToDevice);
    cudaMemcpy(dB16, b16.data(), b16.size(), cudaMemcpyHostToDevice);
    for (int shift : {0, 1, 2, 3, 7, 9, 115}) {
      probe16<<<1, 128>>>(dA16, dB16, shift, dO);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("probe16 shift %d: %s\n", shift, cudaGetErrorString(e)); return 1; }
      cudaMemcpy(hO.data(), dO, hO.size() * 4, cudaMemcpyDeviceToHost);
      int bad = 0;
      for (int i = 0; i < 128; ++i)
        for (int j = 0; j < N; ++j) {
          int64_t acc = 0;
          for (int k = 0; k < 16; ++k) acc += (int)a16[(shift + i) * 16 + k] * (int)b16[0 * N * 16 + j * 16 + k];
          for (int k = 0; k < 16; ++k) acc += (int)a16[(shift + i + 1) * 16 + k] * (int)b16[1 * N * 16 + j * 16 + k];
          bad += (int32_t)acc != hO[i * N + j];
        }
      printf("none/16B rows, LBO=16 overlap, shift %3d: %s (%d mismatches)\n", shift, bad ? "WRONG" : "ok", bad);
    }
  }
  return 0;
}
