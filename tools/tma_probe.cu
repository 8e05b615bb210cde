// Probe: 2-D tiled TMA (the conv kernels' operand loads) throughput per SM.
// 148 CTAs, one thread keeps S slots in flight; each slot is filled by OPS
// tiled loads of a [rows x 128 B] box (SWIZZLE_128B) from an L2-resident
// (32 MB) or HBM (1 GB) matrix.  Prints bytes/clk/SM: whether several loads
// in flight overlap, and the per-SM ceiling of the operand path.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2101_08458_b200/csrc tools/tma_probe.cu -lcuda
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdio>

#include "kernels/ptx.cuh"

using namespace tzcdev;

__global__ void __launch_bounds__(128, 1) tmabw(const __grid_constant__ CUtensorMap tm, int rows_total, int box_rows,
                                                int ops, int slots, int iters, int mode, unsigned* sink) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bars[4][16];
  // mode 0: one thread, ring of `slots`; mode 1: one thread, issue all slots
  // then wait all (batches); mode 2: 4 threads (one per warp), each its own
  // ring of `slots` over a quarter of the iterations
  const int nthr = mode == 2 ? 4 : 1;
  if (threadIdx.x % 32 != 0 || (int)(threadIdx.x / 32) >= nthr) return;
  const int tid = threadIdx.x / 32;
  uint64_t* bar = bars[tid];
  for (int s = 0; s < slots; ++s) mbar_init(&bar[s], 1);
  fence_barrier_init();
  sm += tid * (box_rows * 128 * ops * slots);
  iters /= nthr;
  const int box_bytes = box_rows * 128;
  const int slot_bytes = box_bytes * ops;
  const int per_cta = rows_total / gridDim.x / (box_rows * ops) * (box_rows * ops);
  auto issue = [&](int s, long long i) {
    mbar_expect_tx(&bar[s], slot_bytes);
    const int r0 = blockIdx.x * per_cta + (int)((i * box_rows * ops) % per_cta);
    for (int o = 0; o < ops; ++o)
      tma_load_2d(sm + s * slot_bytes + o * box_bytes, &tm, &bar[s], 0, r0 + o * box_rows);
  };
  if (mode == 1) {
    uint32_t ph = 0;
    for (long long i = 0; i < iters; i += slots) {
      for (int s = 0; s < slots; ++s) issue(s, i + s);
      for (int s = 0; s < slots; ++s) mbar_wait(&bar[s], ph);
      ph ^= 1;
    }
  } else {
    for (int s = 0; s < slots; ++s) issue(s, s + tid * 7);
    uint32_t ph = 0;
    for (long long i = 0; i < iters; ++i) {
      const int s = (int)(i % slots);
      mbar_wait(&bar[s], ph);
      if (s == slots - 1) ph ^= 1;
      if (i + slots < iters) issue(s, i + slots + tid * 7);
    }
  }
  if (sm[5] == 0x7f && sm[77] == 0x11) sink[0] = 1;
}

int main() {
  uint8_t* src;
  unsigned* sink;
  const long long big = 1ll << 30;
  cudaMalloc(&src, big);
  cudaMemset(src, 1, big);
  cudaMalloc(&sink, 64);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &fn, 12000, cudaEnableDefault, &q);
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  for (long long region : {32ll << 20, 1ll << 30}) {
    const int rows_total = (int)(region / 128);
    for (int box_rows : {64, 128}) {
      CUtensorMap tm;
      cuuint64_t dims[2] = {128, (cuuint64_t)rows_total};
      cuuint64_t strides[1] = {128};
      cuuint32_t box[2] = {128, (cuuint32_t)box_rows};
      cuuint32_t es[2] = {1, 1};
      CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, src, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                       CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (r != CUDA_SUCCESS) {
        printf("encode failed %d\n", (int)r);
        return 1;
      }
      for (int mode : {0, 1, 2})
      for (int ops : {1}) {
        for (int slots : {2, 4}) {
          const int slot_bytes = box_rows * 128 * ops;
          if (slot_bytes * slots * (mode == 2 ? 4 : 1) > 200 * 1024) continue;
          const int iters = (int)((8ll << 20) / slot_bytes);
          const int smem = 1024 + slot_bytes * slots * (mode == 2 ? 4 : 1);
          cudaFuncSetAttribute(tmabw, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
          tmabw<<<148, 128, smem>>>(tm, rows_total, box_rows, ops, slots, iters, mode, sink);
          cudaDeviceSynchronize();
          cudaEvent_t e0, e1;
          cudaEventCreate(&e0);
          cudaEventCreate(&e1);
          float best = 1e9;
          for (int rep = 0; rep < 4; ++rep) {
            cudaEventRecord(e0);
            tmabw<<<148, 128, smem>>>(tm, rows_total, box_rows, ops, slots, iters, mode, sink);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (ms < best) best = ms;
          }
          const double bytes = 148.0 * slot_bytes * iters;
          printf("mode %d region %6.0f MB box %3d x 128 B, %d op(s)/slot, %d slots: %7.2f us  %6.0f GB/s  %5.1f B/clk/SM  %s\n", mode,
                 region / 1e6, box_rows, ops, slots, best * 1e3, bytes / (best * 1e-3) / 1e9,
                 bytes / 148 / (best * 1e-3) / 1.965e9, cudaGetErrorString(cudaGetLastError()));
        }
      }
    }
  }
  return 0;
}
