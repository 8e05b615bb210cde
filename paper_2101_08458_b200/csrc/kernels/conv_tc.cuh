// tcgen05 implicit-GEMM Conv2D / GEMM kernel for sm_100a.
//
// This is the device body behind the reference's tensorized Conv2D/Matmul
// execution path (the Intrinsic branch of Evaluator::exec,
// /root/reference/proj/src/vm.cpp:343-390, reached from eval_tir
// vm.cpp:510-516).  One launch executes the whole injected nest of a
// tcgen05-tensorized op: every (M-tile, N-tile, K-block) "intrinsic call"
// of the reference's TIR becomes one TMA-fed, TMEM-accumulated MMA step.
//
// GEMM view: M = N_img*OH*OW output pixels (matmul: rows of A), N = output
// channels (matmul: columns), K = R*S*C (matmul: K).
//
// Warp roles (256 threads, one CTA per SM, persistent over work units):
//   warp 0      TMA producer (A tile: 2-D tiled or im2col; B tile: 3-D
//               tiled (C, K_out, tap) or MN-major 2-D for fp16 matmul)
//   warp 1      MMA issuer (lane 0 issues tcgen05.mma, commits to mbarriers)
//   warp 2      TMEM allocator
//   warps 4..7  epilogue: tcgen05.ld -> C-seed wrap-add -> requant / cast ->
//               128-bit global stores in the op's (possibly channel-blocked)
//               output layout
// Pipelines: STAGES-deep smem ring (full/empty mbarriers), 2 TMEM
// accumulator buffers (tmem_full/tmem_empty), static persistent schedule.
#pragma once
#include <cuda.h>
#include <cuda_fp16.h>

#include <cstdint>

#include "ptx.cuh"

namespace tzcdev {

enum EpKind : int32_t { EP_I32 = 0, EP_REQUANT_I8 = 1, EP_F32 = 2, EP_CAST_F16 = 3, EP_PARTIAL = 4 };
enum AMode : int32_t { A_TILED = 0, A_IM2COL = 1 };

struct alignas(64) ConvKernelParams {
  CUtensorMap tmA;
  CUtensorMap tmB;
  int32_t M, Ngemm;
  int32_t num_kb;    // K blocks of a full reduction
  int32_t c_blocks;  // K blocks per filter tap
  int32_t S;         // filter width (tap -> (r, s))
  int32_t OW, OHOW, stride;
  int32_t tiles_m, tiles_n, num_tiles, splits;
  // epilogue
  void* out;
  const void* seed;   // nullable; accumulator dtype, output layout
  void* partial;      // split-K workspace [splits][M][Ngemm] (acc dtype)
  int64_t out_stride_m, out_stride_blk;
  int32_t out_nb;
  int32_t ep_kind;
  float scale;
};

template <int BN, int KB>
struct ConvCfg {
  static constexpr int BM = 128;
  static constexpr int A_BYTES = BM * KB;
  static constexpr int B_BYTES = BN * KB;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int STAGES_RAW = (200 * 1024) / STAGE_BYTES;
  static constexpr int STAGES = STAGES_RAW > 8 ? 8 : STAGES_RAW;
  static constexpr uint32_t TMEM_COLS = (2 * BN <= 32) ? 32 : (2 * BN <= 64) ? 64 : (2 * BN <= 128) ? 128 : (2 * BN <= 256) ? 256 : 512;
  static constexpr int SMEM_BYTES = 1024 /*align slack*/ + STAGES * STAGE_BYTES + 256;
};

// ---- epilogue math (bit-exact restatement of the reference semantics) ----
// cast<i8>(cast<fp32>(c) * s): vm.cpp:79-84 (float_to_int: NaN->0,
// saturate to int64, trunc toward zero) then wrap to 8 bits (dtype.cpp:40-48).
__device__ __forceinline__ uint32_t requant_byte(int32_t c, float s) {
  float f = __fmul_rn(__int2float_rn(c), s);
  long long q;
  if (f != f)
    q = 0;
  else if (f >= 9223372036854775808.0f)
    q = 0x7fffffffffffffffLL;
  else if (f <= -9223372036854775808.0f)
    q = (-0x7fffffffffffffffLL - 1);
  else
    q = __float2ll_rz(f);
  return static_cast<uint32_t>(q) & 0xffu;
}

__device__ __forceinline__ void st_v4(void* p, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("st.global.v4.b32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(a), "r"(b), "r"(c), "r"(d)
               : "memory");
}
__device__ __forceinline__ uint4 ld_v4(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.v4.b32 {%0, %1, %2, %3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

// Stores 16 consecutive accumulator columns v[0..16) of row m, column n.
template <bool kF16>
__device__ __forceinline__ void store16(const ConvKernelParams& p, int m, int n, const uint32_t* v) {
  int64_t off = (p.out_nb == p.Ngemm) ? (int64_t)m * p.out_stride_m + n
                                      : (int64_t)(n / p.out_nb) * p.out_stride_blk +
                                            (int64_t)m * p.out_stride_m + (n % p.out_nb);
  uint32_t a[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) a[i] = v[i];
  if (p.seed != nullptr) {
    const uint4* s = reinterpret_cast<const uint4*>(static_cast<const uint32_t*>(p.seed) + off);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      uint4 t = ld_v4(s + j);
      if constexpr (kF16) {  // fp32 accumulator: seed + sum
        a[4 * j + 0] = __float_as_uint(__uint_as_float(t.x) + __uint_as_float(a[4 * j + 0]));
        a[4 * j + 1] = __float_as_uint(__uint_as_float(t.y) + __uint_as_float(a[4 * j + 1]));
        a[4 * j + 2] = __float_as_uint(__uint_as_float(t.z) + __uint_as_float(a[4 * j + 2]));
        a[4 * j + 3] = __float_as_uint(__uint_as_float(t.w) + __uint_as_float(a[4 * j + 3]));
      } else {  // int32 two's-complement wrap-add (vm.cpp:486-491)
        a[4 * j + 0] += t.x;
        a[4 * j + 1] += t.y;
        a[4 * j + 2] += t.z;
        a[4 * j + 3] += t.w;
      }
    }
  }
  switch (p.ep_kind) {
    case EP_REQUANT_I8: {
      uint32_t w[4];
#pragma unroll
      for (int j = 0; j < 4; ++j)
        w[j] = requant_byte((int32_t)a[4 * j], p.scale) | (requant_byte((int32_t)a[4 * j + 1], p.scale) << 8) |
               (requant_byte((int32_t)a[4 * j + 2], p.scale) << 16) |
               (requant_byte((int32_t)a[4 * j + 3], p.scale) << 24);
      st_v4(static_cast<int8_t*>(p.out) + off, w[0], w[1], w[2], w[3]);
      break;
    }
    case EP_CAST_F16: {
      uint32_t w[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        __half lo = __float2half_rn(__uint_as_float(a[2 * j]));
        __half hi = __float2half_rn(__uint_as_float(a[2 * j + 1]));
        w[j] = (uint32_t)__half_as_ushort(lo) | ((uint32_t)__half_as_ushort(hi) << 16);
      }
      uint16_t* o = static_cast<uint16_t*>(p.out) + off;
      st_v4(o, w[0], w[1], w[2], w[3]);
      st_v4(o + 8, w[4], w[5], w[6], w[7]);
      break;
    }
    default: {  // EP_I32 / EP_F32: raw 32-bit accumulator image
      uint32_t* o = static_cast<uint32_t*>(p.out) + off;
#pragma unroll
      for (int j = 0; j < 4; ++j) st_v4(o + 4 * j, a[4 * j], a[4 * j + 1], a[4 * j + 2], a[4 * j + 3]);
    }
  }
}

template <int BN, int KB, bool kF16, int kAMode, bool kBMN>
__global__ void __launch_bounds__(256, 1) conv_tc_kernel(const __grid_constant__ ConvKernelParams p) {
  using Cfg = ConvCfg<BN, KB>;
  constexpr int BM = Cfg::BM;
  constexpr int STAGES = Cfg::STAGES;
  constexpr int KE = kF16 ? KB / 2 : KB;  // K elements per block
  constexpr int MMAS = KB / 32;           // K=32 (i8) / K=16 (f16): 32 bytes per MMA
  constexpr uint32_t IDESC = kF16 ? idesc_f16(BM, BN, kBMN) : idesc_i8(BM, BN);

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * Cfg::A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + STAGES * Cfg::B_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const uint32_t warp = warp_id();
  const uint32_t lane = threadIdx.x & 31;

  if (warp == 0 && lane == 0) {
    tma_prefetch(&p.tmA);
    tma_prefetch(&p.tmB);
  }
  if (warp == 1 && lane == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 4);
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc<Cfg::TMEM_COLS>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  const int num_units = p.num_tiles * p.splits;

  if (warp == 0) {
    // ===================== TMA producer =====================
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int u = blockIdx.x; u < num_units; u += gridDim.x) {
        const int tile = u / p.splits, split = u - tile * p.splits;
        const int m_tile = tile / p.tiles_n, n_tile = tile - m_tile * p.tiles_n;
        const int kb0 = (int)((int64_t)split * p.num_kb / p.splits);
        const int kb1 = (int)((int64_t)(split + 1) * p.num_kb / p.splits);
        const int m0 = m_tile * BM, n0 = n_tile * BN;
        int img = 0, oh = 0, ow = 0;
        if constexpr (kAMode == A_IM2COL) {
          img = m0 / p.OHOW;
          const int rem = m0 - img * p.OHOW;
          oh = rem / p.OW;
          ow = rem - oh * p.OW;
        }
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          const int tap = kb / p.c_blocks;
          const int cb = kb - tap * p.c_blocks;
          uint8_t* dA = sA + stage * Cfg::A_BYTES;
          uint8_t* dB = sB + stage * Cfg::B_BYTES;
          mbar_expect_tx(&full[stage], Cfg::STAGE_BYTES);
          if constexpr (kAMode == A_IM2COL) {
            const int r = tap / p.S, s = tap - r * p.S;
            tma_load_im2col_4d(dA, &p.tmA, &full[stage], cb * KE, ow * p.stride, oh * p.stride, img,
                               (uint16_t)s, (uint16_t)r);
          } else {
            tma_load_2d(dA, &p.tmA, &full[stage], kb * KE, m0);
          }
          if constexpr (kBMN) {
#pragma unroll
            for (int j = 0; j < BN / 64; ++j)
              tma_load_2d(dB + j * (KE * 128), &p.tmB, &full[stage], n0 + 64 * j, kb * KE);
          } else {
            tma_load_3d(dB, &p.tmB, &full[stage], cb * KE, n0, tap);
          }
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer =====================
    int stage = 0;
    uint32_t phase = 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int u = blockIdx.x; u < num_units; u += gridDim.x) {
      const int split = u % p.splits;
      const int kb0 = (int)((int64_t)split * p.num_kb / p.splits);
      const int kb1 = (int)((int64_t)(split + 1) * p.num_kb / p.splits);
      mbar_wait(&tempty[acc], acc_phase ^ 1);
      tc_fence_after();
      const uint32_t tmem_d = tmem_base + acc * BN;
      for (int kb = kb0; kb < kb1; ++kb) {
        mbar_wait(&full[stage], phase);
        tc_fence_after();
        if (lane == 0) {
          const uint32_t a_base = smem_u32(sA + stage * Cfg::A_BYTES);
          const uint32_t b_base = smem_u32(sB + stage * Cfg::B_BYTES);
#pragma unroll
          for (int k = 0; k < MMAS; ++k) {
            const uint64_t adesc = smem_desc_kmajor(a_base + 32 * k, KB);
            uint64_t bdesc;
            if constexpr (kBMN)
              bdesc = smem_desc_mnmajor_sw128(b_base + k * 16 * 128, KE * 128);
            else
              bdesc = smem_desc_kmajor(b_base + 32 * k, KB);
            umma<kF16>(tmem_d, adesc, bdesc, IDESC, (kb > kb0 || k > 0) ? 1u : 0u);
          }
          umma_commit(&empty[stage]);
          if (kb == kb1 - 1) umma_commit(&tfull[acc]);
        }
        __syncwarp();
        if (++stage == STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
  } else if (warp >= 4) {
    // ===================== epilogue =====================
    const uint32_t q = warp & 3;  // TMEM lane quarter this warp may access
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int u = blockIdx.x; u < num_units; u += gridDim.x) {
      const int tile = u / p.splits, split = u - tile * p.splits;
      const int m_tile = tile / p.tiles_n, n_tile = tile - m_tile * p.tiles_n;
      const int m = m_tile * BM + q * 32 + lane;
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
#pragma unroll 1
      for (int c = 0; c < BN / 32; ++c) {
        uint32_t v[32];
        tmem_ld32(tmem_base + ((q * 32) << 16) + acc * BN + c * 32, v);
        tmem_ld_wait();
        const int n = n_tile * BN + c * 32;
        if (m < p.M) {
          if (p.ep_kind == EP_PARTIAL) {
            uint32_t* o = static_cast<uint32_t*>(p.partial) + ((int64_t)split * p.M + m) * p.Ngemm + n;
#pragma unroll
            for (int j = 0; j < 8; ++j)
              if (n + 4 * j < p.Ngemm) st_v4(o + 4 * j, v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
          } else {
            if (n < p.Ngemm) store16<kF16>(p, m, n, v);
            if (n + 16 < p.Ngemm) store16<kF16>(p, m, n + 16, v + 16);
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
  }
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<Cfg::TMEM_COLS>(tmem_base);
  }
}

// Split-K fix-up: out = epilogue(seed + sum_s partial[s]).  Integer partial
// sums are combined with wrapping int32 adds, which is associative, so the
// result is bit-identical to any reduction order (F8); fp32 partials are
// combined in split order.
template <bool kF16>
__global__ void splitk_reduce_kernel(const __grid_constant__ ConvKernelParams p) {
  const int64_t groups = (int64_t)p.M * (p.Ngemm / 16);
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < groups;
       g += (int64_t)gridDim.x * blockDim.x) {
    const int m = (int)(g / (p.Ngemm / 16));
    const int n = (int)(g - (int64_t)m * (p.Ngemm / 16)) * 16;
    uint32_t v[16];
    for (int i = 0; i < 16; ++i) v[i] = 0;
    for (int s = 0; s < p.splits; ++s) {
      const uint4* src =
          reinterpret_cast<const uint4*>(static_cast<const uint32_t*>(p.partial) + ((int64_t)s * p.M + m) * p.Ngemm + n);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        uint4 t = ld_v4(src + j);
        if constexpr (kF16) {
          v[4 * j + 0] = __float_as_uint(__uint_as_float(v[4 * j + 0]) + __uint_as_float(t.x));
          v[4 * j + 1] = __float_as_uint(__uint_as_float(v[4 * j + 1]) + __uint_as_float(t.y));
          v[4 * j + 2] = __float_as_uint(__uint_as_float(v[4 * j + 2]) + __uint_as_float(t.z));
          v[4 * j + 3] = __float_as_uint(__uint_as_float(v[4 * j + 3]) + __uint_as_float(t.w));
        } else {
          v[4 * j + 0] += t.x;
          v[4 * j + 1] += t.y;
          v[4 * j + 2] += t.z;
          v[4 * j + 3] += t.w;
        }
      }
    }
    store16<kF16>(p, m, n, v);
  }
}

}  // namespace tzcdev
