// K5 layout adapters: the reference's channel-blocked conv2d_tdsl layouts
// (/root/reference/proj/src/workloads.cpp:65-92) -> the NHWC / [K,R,S,C]
// layouts the TMA-fed kernel consumes.  cb = 4 blocks put 4-byte channel
// runs in memory, below TMA's 16-byte minimum box row, so the
// exact reference program is served by one memory-bound gather pass.  Output
// needs no adapter: the epilogue writes blocked layouts directly
// (tzc_out_layout).  Byte moves only — bit-exact by construction.
#include <algorithm>
#include <cuda_runtime.h>

#include <cstdint>

#include "../tzc_b200_internal.hpp"
#include "ptx.cuh"

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

// ---- K7: explicit im2col for thin-channel convs (the C = 3 stem) ---------------
// A row m = (n, oh, ow) gets K index (r*S + s)*C + c, zero-padded to kp
// columns (kp a multiple of 64 bytes so the GEMM K block is legal).  The
// padded columns multiply zero-padded weight columns: the sum is unchanged
// (the reference's own pad legality argument, rewriter.cpp:175-204).
namespace tzcdev {

// One thread per output pixel row: copy the R contiguous (S*C)-element runs
// of its receptive field into a shared-memory row (odd word stride: no bank
// conflicts), zero the tail, then the block writes its 256 contiguous rows
// with coalesced 16-byte stores.
constexpr int kIm2colRows = 128;

template <typename T>
__global__ void __launch_bounds__(kIm2colRows) im2col_pad_kernel(const T* __restrict__ x, T* __restrict__ a, int64_t M,
                                                               int Hp, int Wp, int C, int R, int S, int stride, int OH,
                                                               int OW, int rsc, int kp) {
  extern __shared__ uint32_t srow[];
  const int row_words = (kp * (int)sizeof(T)) / 4;  // kp*sizeof(T) is a multiple of 64 bytes
  const int pitch = row_words | 1;                   // odd pitch: conflict-free
  const int64_t m0 = (int64_t)blockIdx.x * kIm2colRows;
  const int t = threadIdx.x;
  const int64_t m = m0 + t;
  uint32_t* my = srow + t * pitch;
  for (int w = 0; w < row_words; ++w) my[w] = 0u;
  if (m < M) {
    const int64_t n = m / ((int64_t)OH * OW);
    const int rem = (int)(m - n * OH * OW);
    const int oh = rem / OW, ow = rem - oh * OW;
    T* row = reinterpret_cast<T*>(my);
    const int seg = S * C;
    for (int r = 0; r < R; ++r) {
      const T* src = x + ((n * Hp + (int64_t)oh * stride + r) * Wp + (int64_t)ow * stride) * C;
      for (int j = 0; j < seg; ++j) row[r * seg + j] = src[j];
    }
  }
  __syncthreads();
  // coalesced copy-out of [rows, row_words] words
  const int64_t rows = min((int64_t)kIm2colRows, M - m0);
  uint4* dst = reinterpret_cast<uint4*>(a + m0 * kp);
  const int vec_per_row = row_words / 4;
  for (int i = t; i < rows * vec_per_row; i += kIm2colRows) {
    const int rr = i / vec_per_row, vv = i - rr * vec_per_row;
    const uint32_t* s = srow + rr * pitch + vv * 4;
    dst[i] = make_uint4(s[0], s[1], s[2], s[3]);
  }
}

template <typename T>
__global__ void weight_pad_kernel(const T* __restrict__ w, T* __restrict__ b, int K, int R, int S, int C,
                                  int64_t wsk, int64_t wst, int kp) {
  const int64_t total = (int64_t)K * kp;
  const int rsc = R * S * C;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int k = (int)(i / kp);
    const int kk = (int)(i - (int64_t)k * kp);
    T v = T(0);
    if (kk < rsc) {
      const int tap = kk / C, c = kk - tap * C;
      v = w[k * wsk + tap * wst + c];
    }
    b[i] = v;
  }
}

}  // namespace tzcdev

namespace tzcb200 {

Status im2col_pad(const Problem& pb, const void* x, void* a, int kp, cudaStream_t st) {
  const int rsc = pb.r * pb.s * pb.c;
  const int eb = pb.f16 ? 2 : 1;
  const int pitch = ((kp * eb) / 4) | 1;
  const size_t smem = (size_t)tzcdev::kIm2colRows * pitch * 4;
  const int64_t blocks = (pb.m + tzcdev::kIm2colRows - 1) / tzcdev::kIm2colRows;
  if (smem > 200 * 1024 || blocks > INT32_MAX) return Status(TZC_E_INJECT, "im2col row too wide");
  if (pb.f16) {
    cudaFuncSetAttribute(tzcdev::im2col_pad_kernel<uint16_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    tzcdev::im2col_pad_kernel<uint16_t><<<(int)blocks, tzcdev::kIm2colRows, smem, st>>>(
        (const uint16_t*)x, (uint16_t*)a, pb.m, pb.hp, pb.wp, pb.c, pb.r, pb.s, pb.stride, pb.oh, pb.ow, rsc, kp);
  } else {
    cudaFuncSetAttribute(tzcdev::im2col_pad_kernel<uint8_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    tzcdev::im2col_pad_kernel<uint8_t><<<(int)blocks, tzcdev::kIm2colRows, smem, st>>>(
        (const uint8_t*)x, (uint8_t*)a, pb.m, pb.hp, pb.wp, pb.c, pb.r, pb.s, pb.stride, pb.oh, pb.ow, rsc, kp);
  }
  g_launches.fetch_add(1, std::memory_order_relaxed);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? Status() : Status(TZC_E_DEVICE, cudaGetErrorString(e));
}

Status weight_pad(const Problem& pb, const void* w, void* b, int kp, cudaStream_t st) {
  const int64_t n = (int64_t)pb.ngemm * kp;
  if (pb.f16)
    tzcdev::weight_pad_kernel<uint16_t><<<blocks_for(n), 256, 0, st>>>((const uint16_t*)w, (uint16_t*)b, pb.ngemm, pb.r,
                                                                       pb.s, pb.c, pb.w_stride_k, pb.w_stride_tap, kp);
  else
    tzcdev::weight_pad_kernel<uint8_t><<<blocks_for(n), 256, 0, st>>>((const uint8_t*)w, (uint8_t*)b, pb.ngemm, pb.r,
                                                                      pb.s, pb.c, pb.w_stride_k, pb.w_stride_tap, kp);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? Status() : Status(TZC_E_DEVICE, cudaGetErrorString(e));
}

}  // namespace tzcb200

// ---- space-to-depth for stride-2 thin-channel convs (the C=3 stem) -------------
// A stride-2 R x S conv over C channels equals a stride-1 ceil(R/2) x ceil(S/2)
// conv over the 2x2 space-to-depth input with 4C channels (zero-padded here
// to 16 so each pixel is one 16-byte row):
//   x4[n,i,j,(a*2+b)*C+c] = x[n,2i+a,2j+b,c],  w4[k,i,j,(a*2+b)*C+c] = w[k,2i+a,2j+b,c]
// (out-of-range taps / pixels are zero).  Pure byte moves: exact.
namespace tzcdev {

// One thread per 16-byte S2D pixel.  For C = 3 with an even row pitch each
// (a, row) contributes 6 contiguous bytes at an even offset: three 16-bit
// loads; otherwise byte loads.
__global__ void s2d_data_kernel(const uint8_t* __restrict__ x, uint4* __restrict__ x4, int64_t npix4, int Hp, int Wp,
                                int C, int Hp4, int Wp4) {
  const bool fast3 = C == 3 && ((int64_t)Wp * 3) % 2 == 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < npix4; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t n = i / ((int64_t)Hp4 * Wp4);
    const int rem = (int)(i - n * Hp4 * Wp4);
    const int h4 = rem / Wp4, w4 = rem - h4 * Wp4;
    uint32_t wd[4] = {0, 0, 0, 0};
    if (fast3) {
      uint32_t u[6] = {0, 0, 0, 0, 0, 0};  // 16-bit pieces: row a -> u[3a..3a+2]
#pragma unroll
      for (int a = 0; a < 2; ++a) {
        const int h = 2 * h4 + a;
        if (h >= Hp) continue;
        const uint16_t* src = reinterpret_cast<const uint16_t*>(x + ((n * Hp + h) * Wp + 2 * w4) * 3);
        const bool two = 2 * w4 + 1 < Wp;
        u[3 * a + 0] = __ldg(src);
        u[3 * a + 1] = __ldg(src + 1);
        u[3 * a + 2] = two ? __ldg(src + 2) : 0u;
        if (!two) u[3 * a + 1] &= 0x00ffu;  // pixel (2*w4+1) is outside the input
      }
      // channel order (a*2+b)*3+c: bytes 0..5 = row 0 (b=0,1), bytes 6..11 = row 1
      wd[0] = u[0] | (u[1] << 16);
      wd[1] = u[2] | (u[3] << 16);
      wd[2] = u[4] | (u[5] << 16);
    } else {
      uint8_t v[16];
#pragma unroll
      for (int t = 0; t < 16; ++t) v[t] = 0;
      for (int a = 0; a < 2; ++a)
        for (int b = 0; b < 2; ++b) {
          const int h = 2 * h4 + a, w = 2 * w4 + b;
          if (h < Hp && w < Wp) {
            const uint8_t* src = x + ((n * Hp + h) * Wp + w) * C;
            for (int c = 0; c < C; ++c) v[(a * 2 + b) * C + c] = src[c];
          }
        }
      for (int t = 0; t < 4; ++t) wd[t] = v[4 * t] | (v[4 * t + 1] << 8) | (v[4 * t + 2] << 16) | ((uint32_t)v[4 * t + 3] << 24);
    }
    x4[i] = make_uint4(wd[0], wd[1], wd[2], wd[3]);
  }
}

// C = 3 stem, one block per S2D row (n, h4): the two input rows are read
// with coalesced 16-bit loads into shared memory, then every thread emits
// 16-byte S2D pixels with one vector store.  Memory-bound; replaces the
// per-pixel kernel's 64-bit index math and six scattered loads per pixel.
__global__ void s2d_rows_c3_kernel(const uint8_t* __restrict__ x, uint4* __restrict__ x4, int Hp, int Wp, int Hp4,
                                   int Wp4, int rows) {
  // grid-stride over S2D rows (n, h4); thread t of the block emits pixels
  // w4 = t, t + 128, ... with six independent 16-bit loads each (no shared
  // memory round trip, 32-bit index math once per row)
  for (int row = blockIdx.x; row < rows; row += gridDim.x) {
    const int n = row / Hp4, h4 = row - n * Hp4;
    const uint16_t* r0 = reinterpret_cast<const uint16_t*>(x + ((int64_t)n * Hp + 2 * h4) * Wp * 3);
    const uint16_t* r1 = r0 + Wp * 3 / 2;  // Hp, Wp even (host): row 2*h4+1 exists, 2-byte aligned
    uint4* dst = x4 + (int64_t)row * Wp4;
#pragma unroll 2
    for (int w4 = threadIdx.x; w4 < Wp4; w4 += blockDim.x) {
      const uint32_t a0 = __ldg(r0 + 3 * w4), a1 = __ldg(r0 + 3 * w4 + 1), a2 = __ldg(r0 + 3 * w4 + 2);
      const uint32_t b0 = __ldg(r1 + 3 * w4), b1 = __ldg(r1 + 3 * w4 + 1), b2 = __ldg(r1 + 3 * w4 + 2);
      dst[w4] = make_uint4(a0 | (a1 << 16), a2 | (b0 << 16), b1 | (b2 << 16), 0u);
    }
  }
}

// The int8 C = 3 stem in ONE launch: the first blocks rearrange the weights
// (s2d_weight_kernel's work, one launch fewer on the stem's critical path),
// the rest build the S2D pixel rows, one warp per row.  Each thread emits two
// neighbouring S2D pixels from 32-bit loads: the 12 input bytes of a pixel
// pair start 4-byte aligned in row 2*h4 (Hp, Wp even) and 2 bytes off in row
// 2*h4+1 when Wp % 4 == 2 (funnel-shifted from the aligned words around
// them); 7 loads per 2 pixels instead of 12 16-bit ones.  The last pixel
// (pair) of a row keeps the 16-bit loads (no read past the row's end).
__device__ __forceinline__ uint4 s2d_pixel16(const uint16_t* r0, const uint16_t* r1, int w4) {
  const uint32_t a0 = __ldg(r0 + 3 * w4), a1 = __ldg(r0 + 3 * w4 + 1), a2 = __ldg(r0 + 3 * w4 + 2);
  const uint32_t b0 = __ldg(r1 + 3 * w4), b1 = __ldg(r1 + 3 * w4 + 1), b2 = __ldg(r1 + 3 * w4 + 2);
  return make_uint4(a0 | (a1 << 16), a2 | (b0 << 16), b1 | (b2 << 16), 0u);
}
template <typename T>
__device__ __forceinline__ void s2d_weight_elems(const T* __restrict__ w, T* __restrict__ w4, int K, int R, int S,
                                                 int C, int64_t wsk, int64_t wst, int R4, int S4, int64_t first,
                                                 int64_t step) {
  const int64_t total = (int64_t)K * R4 * S4 * 16;
  for (int64_t i = first; i < total; i += step) {
    const int ch = (int)(i % 16);
    int64_t t = i / 16;
    const int j = (int)(t % S4);
    t /= S4;
    const int ii = (int)(t % R4);
    const int k = (int)(t / R4);
    T v = 0;
    if (ch < 4 * C) {
      const int ab = ch / C, c = ch - ab * C;
      const int r = 2 * ii + ab / 2, s = 2 * j + ab % 2;
      if (r < R && s < S) v = w[k * wsk + (int64_t)(r * S + s) * wst + c];
    }
    w4[i] = v;
  }
}
__global__ void s2d_stem_c3_kernel(const uint8_t* __restrict__ x, uint4* __restrict__ x4, int Hp, int Wp, int Hp4,
                                   int Wp4, int rows, int row_blocks, const uint8_t* __restrict__ w,
                                   uint8_t* __restrict__ w4, int K, int R, int S, int64_t wsk, int64_t wst, int R4,
                                   int S4) {
  const int wblocks = gridDim.x - row_blocks;  // the first blocks: they run in the first wave, not the tail
  if ((int)blockIdx.x < wblocks) {
    s2d_weight_elems<uint8_t>(w, w4, K, R, S, 3, wsk, wst, R4, S4, (int64_t)blockIdx.x * blockDim.x + threadIdx.x,
                              (int64_t)wblocks * blockDim.x);
    return;
  }
  const int rb = blockIdx.x - wblocks;
  const bool odd1 = (Wp * 3) % 4 != 0;  // row 2*h4+1 starts 2 bytes past a 4-byte boundary
  const int pairs = Wp4 / 2 - 1;        // pairs with whole-word loads (the last pair / pixel is 16-bit)
  // one warp per S2D row (a row has ~Wp/4 pairs: a whole block per row left
  // most of its threads idle)
  const int wpb = blockDim.x / 32, lane = threadIdx.x & 31;
  for (int row = rb * wpb + threadIdx.x / 32; row < rows; row += row_blocks * wpb) {
    const int n = row / Hp4, h4 = row - n * Hp4;
    const uint8_t* r0b = x + ((int64_t)n * Hp + 2 * h4) * Wp * 3;
    const uint8_t* r1b = r0b + Wp * 3;
    const uint32_t* r0 = reinterpret_cast<const uint32_t*>(r0b);
    const uint32_t* r1 = reinterpret_cast<const uint32_t*>(r1b - (odd1 ? 2 : 0));
    uint4* dst = x4 + (int64_t)row * Wp4;
    for (int j = lane; j < pairs; j += 32) {
      const uint32_t a0 = __ldg(r0 + 3 * j), a1 = __ldg(r0 + 3 * j + 1), a2 = __ldg(r0 + 3 * j + 2);
      uint32_t b0, b1, b2;
      if (odd1) {
        const uint32_t m0 = __ldg(r1 + 3 * j), m1 = __ldg(r1 + 3 * j + 1), m2 = __ldg(r1 + 3 * j + 2),
                       m3 = __ldg(r1 + 3 * j + 3);
        b0 = __funnelshift_r(m0, m1, 16);
        b1 = __funnelshift_r(m1, m2, 16);
        b2 = __funnelshift_r(m2, m3, 16);
      } else {
        b0 = __ldg(r1 + 3 * j);
        b1 = __ldg(r1 + 3 * j + 1);
        b2 = __ldg(r1 + 3 * j + 2);
      }
      dst[2 * j] = make_uint4(a0, (a1 & 0xFFFFu) | (b0 << 16), (b0 >> 16) | (b1 << 16), 0u);
      dst[2 * j + 1] = make_uint4((a1 >> 16) | (a2 << 16), (a2 >> 16) | (b1 & 0xFFFF0000u), b2, 0u);
    }
    // the row's last pair / odd pixel: 16-bit loads
    const uint16_t* h0 = reinterpret_cast<const uint16_t*>(r0b);
    const uint16_t* h1 = reinterpret_cast<const uint16_t*>(r1b);
    for (int w4i = 2 * pairs + lane; w4i < Wp4; w4i += 32) dst[w4i] = s2d_pixel16(h0, h1, w4i);
  }
}

// fp16 C = 3 stem: 32-byte S2D pixels (halfs (a*2+b)*3+c, 4 zero halfs);
// the input pixel pair (2*w4, 2*w4+1) of a row is 12 contiguous bytes at a
// 4-byte aligned offset (Wp even): three 32-bit loads per row.
__global__ void s2d_rows_c3_f16_kernel(const uint8_t* __restrict__ x, uint4* __restrict__ x4, int Hp, int Wp, int Hp4,
                                       int Wp4, int rows) {
  for (int row = blockIdx.x; row < rows; row += gridDim.x) {
    const int n = row / Hp4, h4 = row - n * Hp4;
    const uint32_t* r0 = reinterpret_cast<const uint32_t*>(x + ((int64_t)n * Hp + 2 * h4) * Wp * 6);
    const uint32_t* r1 = r0 + Wp * 3 / 2;
    uint4* dst = x4 + (int64_t)row * Wp4 * 2;
#pragma unroll 2
    for (int w4 = threadIdx.x; w4 < Wp4; w4 += blockDim.x) {
      const uint32_t a0 = __ldg(r0 + 3 * w4), a1 = __ldg(r0 + 3 * w4 + 1), a2 = __ldg(r0 + 3 * w4 + 2);
      const uint32_t b0 = __ldg(r1 + 3 * w4), b1 = __ldg(r1 + 3 * w4 + 1), b2 = __ldg(r1 + 3 * w4 + 2);
      dst[2 * w4] = make_uint4(a0, a1, a2, b0);
      dst[2 * w4 + 1] = make_uint4(b1, b2, 0u, 0u);
    }
  }
}

__global__ void zero_tail_kernel(uint4* p, int64_t from, int64_t to) {
  for (int64_t i = from + threadIdx.x; i < to; i += blockDim.x) p[i] = make_uint4(0, 0, 0, 0);
}

template <typename T>
__global__ void s2d_weight_kernel(const T* __restrict__ w, T* __restrict__ w4, int K, int R, int S, int C, int64_t wsk,
                                  int64_t wst, int R4, int S4) {
  const int64_t total = (int64_t)K * R4 * S4 * 16;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int ch = (int)(i % 16);
    int64_t t = i / 16;
    const int j = (int)(t % S4);
    t /= S4;
    const int ii = (int)(t % R4);
    const int k = (int)(t / R4);
    T v = 0;
    if (ch < 4 * C) {
      const int ab = ch / C, c = ch - ab * C;
      const int r = 2 * ii + ab / 2, s = 2 * j + ab % 2;
      if (r < R && s < S) v = w[k * wsk + (int64_t)(r * S + s) * wst + c];
    }
    w4[i] = v;
  }
}

}  // namespace tzcdev

namespace tzcb200 {

Status s2d_stem(const Problem& pb, const void* x, const void* w, void* x4, void* w4, int hp4, int wp4, int r4, int s4,
                cudaStream_t st, bool one_launch) {
  const int64_t npix4 = (int64_t)pb.n * hp4 * wp4;
  if (pb.f16) {  // C = 3, even extents (s2d_eligible)
    const int rows = pb.n * hp4;
    tzcdev::s2d_rows_c3_f16_kernel<<<std::min(rows, 148 * 16), 128, 0, st>>>((const uint8_t*)x, (uint4*)x4, pb.hp,
                                                                             pb.wp, hp4, wp4, rows);
  } else if (one_launch && pb.c == 3 && pb.hp % 2 == 0 && pb.wp % 2 == 0 && reinterpret_cast<uintptr_t>(x) % 4 == 0 &&
             wp4 >= 2) {
    // rows + weights in one launch (the weights' blocks run beside the rows')
    const int rows = pb.n * hp4;
    const int row_blocks = std::min((rows + 3) / 4, 148 * 16);  // 4 warps = 4 rows per block
    const int64_t nw = (int64_t)pb.ngemm * r4 * s4 * 16;
    const int wblocks = (int)std::min<int64_t>((nw + 255) / 256, 64);
    tzcdev::s2d_stem_c3_kernel<<<row_blocks + wblocks, 128, 0, st>>>(
        (const uint8_t*)x, (uint4*)x4, pb.hp, pb.wp, hp4, wp4, rows, row_blocks, (const uint8_t*)w, (uint8_t*)w4,
        pb.ngemm, pb.r, pb.s, pb.w_stride_k, pb.w_stride_tap, r4, s4);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    const int64_t padded = (npix4 + 7) / 8 * 8;
    if (padded > npix4) {
      tzcdev::zero_tail_kernel<<<1, 32, 0, st>>>((uint4*)x4, npix4, padded);
      g_launches.fetch_add(1, std::memory_order_relaxed);
    }
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? Status() : Status(TZC_E_DEVICE, cudaGetErrorString(e));
  } else if (pb.c == 3 && pb.hp % 2 == 0 && pb.wp % 2 == 0 && reinterpret_cast<uintptr_t>(x) % 2 == 0) {
    const int rows = pb.n * hp4;
    tzcdev::s2d_rows_c3_kernel<<<std::min(rows, 148 * 16), 128, 0, st>>>((const uint8_t*)x, (uint4*)x4, pb.hp, pb.wp,
                                                                         hp4, wp4, rows);
  } else {
    tzcdev::s2d_data_kernel<<<blocks_for(npix4), 256, 0, st>>>((const uint8_t*)x, (uint4*)x4, npix4, pb.hp, pb.wp, pb.c,
                                                               hp4, wp4);
  }
  g_launches.fetch_add(1, std::memory_order_relaxed);
  const int64_t padded = (npix4 + 7) / 8 * 8;
  if (padded > npix4 && !pb.f16) {  // fp16 pixels are 32 B: the tail is zeroed as 2 uint4 each below
    tzcdev::zero_tail_kernel<<<1, 32, 0, st>>>((uint4*)x4, npix4, padded);
    g_launches.fetch_add(1, std::memory_order_relaxed);
  } else if (padded > npix4) {
    tzcdev::zero_tail_kernel<<<1, 32, 0, st>>>((uint4*)x4, 2 * npix4, 2 * padded);
    g_launches.fetch_add(1, std::memory_order_relaxed);
  }
  const int64_t nw = (int64_t)pb.ngemm * r4 * s4 * 16;
  if (pb.f16)
    tzcdev::s2d_weight_kernel<uint16_t><<<blocks_for(nw), 256, 0, st>>>(
        (const uint16_t*)w, (uint16_t*)w4, pb.ngemm, pb.r, pb.s, pb.c, pb.w_stride_k, pb.w_stride_tap, r4, s4);
  else
    tzcdev::s2d_weight_kernel<uint8_t><<<blocks_for(nw), 256, 0, st>>>(
        (const uint8_t*)w, (uint8_t*)w4, pb.ngemm, pb.r, pb.s, pb.c, pb.w_stride_k, pb.w_stride_tap, r4, s4);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? Status() : Status(TZC_E_DEVICE, cudaGetErrorString(e));
}

}  // namespace tzcb200
