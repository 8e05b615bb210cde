// K5 layout adapters: the reference's channel-blocked conv2d_tdsl layouts
// (/root/reference/proj/src/workloads.cpp:65-92) -> the NHWC / [K,R,S,C]
// layouts the TMA-fed kernel consumes.  cb = 4 blocks put 4-byte channel
// runs in memory, below TMA's 16-byte minimum box row, so the
// exact reference program is served by one memory-bound gather pass.  Output
// needs no adapter: the epilogue writes blocked layouts directly
// (tzc_out_layout).  Byte moves only — bit-exact by construction.
#include <cuda_runtime.h>

#include <cstdint>

#include "../tzc_b200_internal.hpp"

namespace tzcdev {

template <typename T>
__global__ void unblock_data_kernel(const T* __restrict__ src, T* __restrict__ dst, int C, int H, int W,
                                    int cb) {
  const int64_t total = (int64_t)C * H * W;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    // dst NHWC index i = (h*W + w)*C + c
    const int c = (int)(i % C);
    const int64_t hw = i / C;
    const int co = c / cb, ci = c - co * cb;
    dst[i] = src[((int64_t)co * H * W + hw) * cb + ci];
  }
}

template <typename T>
__global__ void unblock_kernel_kernel(const T* __restrict__ src, T* __restrict__ dst, int K, int C, int R, int S,
                                      int kb, int cb) {
  const int64_t total = (int64_t)K * R * S * C;
  const int CO = C / cb;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    // dst [K,R,S,C]
    const int c = (int)(i % C);
    int64_t t = i / C;
    const int s = (int)(t % S);
    t /= S;
    const int r = (int)(t % R);
    const int k = (int)(t / R);
    const int ko = k / kb, ki = k - ko * kb, co = c / cb, ci = c - co * cb;
    dst[i] = src[(((((int64_t)ko * CO + co) * R + r) * S + s) * kb + ki) * cb + ci];
  }
}

}  // namespace tzcdev

namespace tzcb200 {

static int blocks_for(int64_t n) { return (int)std::min<int64_t>((n + 255) / 256, 8 * 148); }

Status unblock_data(const void* src, void* dst, int c, int h, int w, int cb, int eb, cudaStream_t st) {
  if (c <= 0 || h <= 0 || w <= 0 || cb <= 0 || c % cb) return Status(TZC_E_SHAPE, "unblock_data: bad geometry");
  int64_t n = (int64_t)c * h * w;
  if (eb == 1)
    tzcdev::unblock_data_kernel<uint8_t><<<blocks_for(n), 256, 0, st>>>((const uint8_t*)src, (uint8_t*)dst, c, h, w, cb);
  else if (eb == 2)
    tzcdev::unblock_data_kernel<uint16_t><<<blocks_for(n), 256, 0, st>>>((const uint16_t*)src, (uint16_t*)dst, c, h, w, cb);
  else
    return Status(TZC_E_SHAPE, "unblock_data: elem_bytes must be 1 or 2");
  g_launches.fetch_add(1, std::memory_order_relaxed);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? Status() : Status(TZC_E_DEVICE, cudaGetErrorString(e));
}

Status unblock_kernel(const void* src, void* dst, int k, int c, int r, int s, int kb, int cb, int eb,
                      cudaStream_t st) {
  if (k <= 0 || c <= 0 || kb <= 0 || cb <= 0 || k % kb || c % cb) return Status(TZC_E_SHAPE, "unblock_kernel: bad geometry");
  int64_t n = (int64_t)k * r * s * c;
  if (eb == 1)
    tzcdev::unblock_kernel_kernel<uint8_t><<<blocks_for(n), 256, 0, st>>>((const uint8_t*)src, (uint8_t*)dst, k, c, r, s, kb, cb);
  else if (eb == 2)
    tzcdev::unblock_kernel_kernel<uint16_t><<<blocks_for(n), 256, 0, st>>>((const uint16_t*)src, (uint16_t*)dst, k, c, r, s, kb, cb);
  else
    return Status(TZC_E_SHAPE, "unblock_kernel: elem_bytes must be 1 or 2");
  g_launches.fetch_add(1, std::memory_order_relaxed);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? Status() : Status(TZC_E_DEVICE, cudaGetErrorString(e));
}

}  // namespace tzcb200
