// Probe: TMA im2col load throughput per SM (the general kernel's A operand for
// strided / 3x3 convs) vs a tiled load of the same bytes.  148 CTAs, 4 issuing
// warps (one lane each) with 2 slots each; every load is one 128-pixel x 128-B
// im2col box (16 KB) at successive output positions.  Input NHWC u8, C = 128,
// 56 x 56 (+pad), N = 256 (~100 MB, L2-resident slices per CTA are re-read).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2101_08458_b200/csrc tools/im2col_probe.cu -lcuda
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdio>

#include "kernels/ptx.cuh"

using namespace tzcdev;

__global__ void __launch_bounds__(128, 1) i2c(const __grid_constant__ CUtensorMap tm, int ow_n, int oh_n, int n_img,
                                              int stride, int iters, int taps, unsigned* sink) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bars[4][2];
  if (threadIdx.x % 32 != 0) return;
  const int tid = threadIdx.x / 32;
  uint64_t* bar = bars[tid];
  for (int s = 0; s < 2; ++s) mbar_init(&bar[s], 1);
  fence_barrier_init();
  sm += tid * 2 * 16384;
  const int ohow = ow_n * oh_n;
  auto issue = [&](int s, long long i) {
    mbar_expect_tx(&bar[s], 16384);
    const long long tile = (blockIdx.x + 148ll * (i / taps)) * 4 + tid;
    const int tap = (int)(i % taps);
    const long long m0 = (tile * 128) % ((long long)ohow * n_img);
    const int img = (int)(m0 / ohow), rem = (int)(m0 % ohow);
    const int oh = rem / ow_n, ow = rem % ow_n;
    tma_load_im2col_4d(sm + s * 16384, &tm, &bar[s], 0, ow * stride, oh * stride, img, (uint16_t)(tap % 3),
                       (uint16_t)(tap / 3));
  };
  issue(0, 0);
  issue(1, 1);
  uint32_t ph = 0;
  for (long long i = 0; i < iters; ++i) {
    const int s = (int)(i & 1);
    mbar_wait(&bar[s], ph);
    if (s == 1) ph ^= 1;
    if (i + 2 < iters) issue(s, i + 2);
  }
  if (sm[5] == 0x7f && sm[77] == 0x11) sink[0] = 1;
}

int main() {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPointByVersion("cuTensorMapEncodeIm2col", &fn, 12000, cudaEnableDefault, &q);
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeIm2col_v12000>(fn);
  unsigned* sink;
  cudaMalloc(&sink, 64);
  for (int stride : {1, 2}) {
    for (int r : {1, 3}) {
      const int N = 256, C = 128, H = 56 + (r - 1), W = 56 + (r - 1);
      uint8_t* x;
      cudaMalloc(&x, (size_t)N * H * W * C);
      cudaMemset(x, 1, (size_t)N * H * W * C);
      CUtensorMap tm;
      cuuint64_t dims[4] = {(cuuint64_t)C, (cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)N};
      cuuint64_t strides[3] = {(cuuint64_t)C, (cuuint64_t)W * C, (cuuint64_t)H * W * C};
      int lower[2] = {0, 0};
      int upper[2] = {-(r - 1), -(r - 1)};
      cuuint32_t es[4] = {1, (cuuint32_t)stride, (cuuint32_t)stride, 1};
      CUresult rc = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, x, dims, strides, lower, upper, 128, 128, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (rc != CUDA_SUCCESS) {
        printf("encode failed %d\n", (int)rc);
        return 1;
      }
      const int oh = (H - r) / stride + 1, ow = (W - r) / stride + 1;
      const int iters = 512, taps = r * r;
      const int smem = 1024 + 4 * 2 * 16384;
      cudaFuncSetAttribute(i2c, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      i2c<<<148, 128, smem>>>(tm, ow, oh, N, stride, iters, taps, sink);
      cudaDeviceSynchronize();
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      float best = 1e9;
      for (int rep = 0; rep < 4; ++rep) {
        cudaEventRecord(e0);
        i2c<<<148, 128, smem>>>(tm, ow, oh, N, stride, iters, taps, sink);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
      }
      const double bytes = 148.0 * 4 * 16384 * iters;
      printf("im2col stride %d, %dx%d taps: %7.2f us  %6.0f GB/s  %5.1f B/clk/SM  %s\n", stride, r, r, best * 1e3,
             bytes / (best * 1e-3) / 1e9, bytes / 148 / (best * 1e-3) / 1.965e9, cudaGetErrorString(cudaGetLastError()));
      cudaFree(x);
    }
  }
  return 0;
}
