// Weight-stationary, shifted-window tcgen05 kernel for stride-1 convolutions
// (and the C=3 stem after a space-to-depth rewrite).
//
// Computing on the *padded* pixel grid q = (n*Hp + oh)*Wp + ow turns every
// filter tap (r, s) into a row shift of one matrix: the A rows of tap (r, s)
// for pixels [q0, q0+128) are input pixels [q0 + r*Wp + s, ...).  So one TMA
// load of SR = 128 + (R-1)*Wp + (S-1) input rows per channel block feeds all
// R*S taps; each tap is a UMMA descriptor whose start address is shifted by
// whole rows (hardware-verified for SWIZZLE_128B/64B: the swizzle follows the
// absolute SMEM address, tools/desc_probe.cu).  The im2col path re-streams
// every input pixel R*S times through L2; this one streams it ~1.x times.
// The (R-1) extra columns / rows of the padded grid are computed and dropped
// by the epilogue (waste (Hp*Wp)/(OH*OW): 7% at 56x56, 15% at 28x28).
//
// The whole weight tensor (all taps, all channel blocks, N <= 256) is loaded
// into SMEM once per CTA and stays there for every tile (weight-stationary):
// per tile only the A super-tile moves.
//
// Pair mode (kPair): 16-byte pixels (the space-to-depth stem: 4 x 4 taps of
// 12(+4) channels).  SWIZZLE_NONE rows at 16-byte pitch; one K=32 MMA covers
// taps (r, s) and (r, s+1) by setting the descriptor's leading-byte offset
// to 16 B — the next row — (hardware-verified, tools/desc_probe.cu).
//
// Work unit = MT consecutive 128-row tiles (host-chosen, p.mt; 2*MT*BN TMEM
// columns): one A super-tile of MT*128 + halo rows feeds MT accumulators, so
// the halo re-read ((R-1)*Wp+(S-1) rows) and the per-unit barrier / commit /
// epilogue hand-off costs are paid once per MT tiles.
#pragma once
#include "conv_tc.cuh"

namespace tzcdev {

// smem descriptor, SWIZZLE_NONE K-major: LBO = distance between the two
// 16-byte K chunks of an MMA, SBO = distance between 8-row groups.
__device__ __forceinline__ uint64_t smem_desc_none(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFF);
  d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFF) << 16;
  d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFF) << 32;
  d |= static_cast<uint64_t>(1) << 46;
  return d;
}

template <int BN, int KB, bool kF16, bool kPair, int kEpm>
__global__ void __launch_bounds__(EpiCfg<BN>::THREADS, 1) conv_ws_kernel(const __grid_constant__ ConvKernelParams p) {
  constexpr int BM = 128;
  constexpr int KE = kF16 ? KB / 2 : KB;
  constexpr uint32_t IDESC = kF16 ? idesc_f16(BM, BN, false) : idesc_i8(BM, BN);
  constexpr uint32_t TMEM_COLS = 512;  // 2 accumulators x MT tiles x BN (MT <= 256 / BN)
  const int taps = p.R * p.S;
  const int c_blocks = p.c_blocks;
  const int b_tile = BN * KB;                                     // one (tap, channel block) of weights
  const int b_bytes = taps * c_blocks * b_tile;
  const int a_slot = ((p.a_nbox * p.a_box_bytes + 1023) / 1024) * 1024;
  extern __shared__ uint8_t smem_raw[];
  TZC_TRACE_DECL
  TZC_TRACE_INIT;
  TZC_CHK_INIT(p);
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sB = smem;
  uint8_t* sA = smem + ((b_bytes + 1023) / 1024) * 1024;
  const int a_slots = p.splits;  // host-chosen ring depth (stored in `splits`; no split-K in this kernel)
  uint64_t* afull = reinterpret_cast<uint64_t*>(sA + a_slots * a_slot);
  uint64_t* aempty = afull + a_slots;
  uint64_t* bfull = aempty + a_slots;
  uint64_t* tfull = bfull + 1;
  uint64_t* tempty = tfull + 4;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 4);
  const int NACC = p.nacc;  // TMEM accumulator ring: NACC x MT x BN <= 512 columns

  const uint32_t warp = warp_id();
  const uint32_t lane = threadIdx.x & 31;
  if (threadIdx.x == 0) TZC_TRACE_POINT(0);
  if (warp == 0 && lane == 0) {
    tma_prefetch(&p.tmA);
    tma_prefetch(&p.tmB);
  }
  if (warp == 1 && lane == 0) {
    for (int s = 0; s < a_slots; ++s) {
      mbar_init(&afull[s], 1);
      mbar_init(&aempty[s], 1);
    }
    mbar_init(bfull, 1);
    for (int a = 0; a < NACC; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], EpiCfg<BN>::WARPS / p.epi_groups);
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc<TMEM_COLS>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  pdl_launch_dependents();
  pdl_wait();

  const int num_tiles = p.num_tiles;  // work units of MT tiles
  const int MT = p.mt;
  if (warp == 0) {
    if (lane == 0) {
      // stationary weights: every (tap, channel block) tile, once
      mbar_expect_tx(bfull, b_bytes);
      if constexpr (kPair) {
        for (int t = 0; t < taps; t += 2)  // box (16 ch, BN, 2 taps) == [tap][n][16 B]
          tma_load_3d(sB + t * b_tile, &p.tmB, bfull, 0, 0, t);
      } else {
        for (int t = 0; t < taps; ++t)
          for (int cb = 0; cb < c_blocks; ++cb) tma_load_3d(sB + (t * c_blocks + cb) * b_tile, &p.tmB, bfull, cb * KE, 0, t);
      }
      int slot = 0;
      uint32_t phase = 0;
      for (int tile = blockIdx.x, it = 0; tile < num_tiles; tile += gridDim.x, ++it) {
        const int q0 = tile * MT * BM;
        for (int cb = 0; cb < c_blocks; ++cb) {
          mbar_wait(&aempty[slot], phase ^ 1);
          if (it < 10) TZC_TRACE_POINT(10 + 5 * it);
          uint8_t* dA = sA + slot * a_slot;
          mbar_expect_tx(&afull[slot], p.a_nbox * p.a_box_bytes);
          const int row0 = kPair ? q0 >> 3 : q0;  // pair mode: 8 pixels per 128-byte TMA row
          for (int b = 0; b < p.a_nbox; ++b)
            tma_load_2d_p(dA + b * p.a_box_bytes, &p.tmA, &afull[slot], cb * KE, row0 + b * p.box_rows, p.pol_a);
          if (++slot == a_slots) {
            slot = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer =====================
    // The whole warp runs this loop on warp-uniform values (descriptors from
    // the kernel-parameter table), so ptxas keeps them in uniform registers
    // and issues UTCIMMA back to back; a lane-0 loop pays ~125 cycles per MMA
    // in R2UR + elect waterfalls, above the 48-cycle N=64 MMA (tools/mma_rate.cu).
    const uint32_t b_base = smem_u32(sB);
    constexpr int MT_PAIR_MAX = 4;
    uint32_t pa[8], pb[8];
    if constexpr (kPair) {  // host guarantees n_mma == 8 (4 x 4 taps) in pair mode
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        pa[i] = p.mma_a[i];
        pb[i] = p.mma_b[i];
      }
    }
    mbar_wait(bfull, 0);
    int slot = 0;
    uint32_t phase = 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int tile = blockIdx.x, it = 0; tile < num_tiles; tile += gridDim.x, ++it) {
      mbar_wait(&tempty[acc], acc_phase ^ 1);
      tc_fence_after();
      const uint32_t tmem_acc = tmem_base + acc * (MT * BN);
      if (lane == 0 && it < 10) TZC_TRACE_POINT(11 + 5 * it);
      for (int cb = 0; cb < c_blocks; ++cb) {
        mbar_wait(&afull[slot], phase);
        tc_fence_after();
        if (lane == 0 && it < 10 && cb == 0) TZC_TRACE_POINT(12 + 5 * it);
        {
          const uint32_t a_base = smem_u32(sA + slot * a_slot);
          const uint64_t a0 = kPair ? smem_desc_none(a_base, 16, 128) : smem_desc_kmajor(a_base, KB);
          const uint32_t b_cb = b_base + (kPair ? 0u : (uint32_t)(cb * b_tile));
          const uint64_t b0 = kPair ? smem_desc_none(b_cb, BN * 16, 128) : smem_desc_kmajor(b_cb, KB);
          const int n_mma = p.n_mma;
          if constexpr (kPair) {
            // the space-to-depth stem: 4 x 4 taps, two per MMA = 8 MMAs per
            // tile, offsets held in uniform registers for the whole kernel
            // (a constant-bank load per MMA put its latency on the issue path)
#pragma unroll
            for (int t = 0; t < MT_PAIR_MAX; ++t) {
              if (t < MT) {
                const uint64_t at = a0 + (uint64_t)(t * 128);
                const uint32_t tmem_d = tmem_acc + t * BN;
#pragma unroll
                for (int i = 0; i < 8; ++i)
                  if (elect_one()) umma<kF16>(tmem_d, at + pa[i], b0 + pb[i], IDESC, i > 0 ? 1u : 0u);
              }
            }
          } else if (MT == 1) {
#pragma unroll 2
            for (int i = 0; i < n_mma; ++i)
              if (elect_one()) umma<kF16>(tmem_acc, a0 + p.mma_a[i], b0 + p.mma_b[i], IDESC, (cb > 0 || i > 0) ? 1u : 0u);
          } else {
            // (tap, K step) outer, tile t of the unit inner: each offset pair
            // is read from the parameter bank once per MT MMAs (t-outer paid
            // two constant loads per MMA on the issue path: 69 cycles per N=64
            // MMA against the 48-cycle SMEM bound).  Each accumulator still
            // receives its MMAs in order i = 0, 1, ... (identical sums).
#pragma unroll 1
            for (int i = 0; i < n_mma; ++i) {
              const uint64_t ai = a0 + p.mma_a[i];
              const uint64_t bi = b0 + p.mma_b[i];
              const uint32_t accum = (cb > 0 || i > 0) ? 1u : 0u;
#pragma unroll
              for (int t = 0; t < 4; ++t)  // tile t: A rows shifted by t*128 (16-byte descriptor units)
                if (t < MT && elect_one()) umma<kF16>(tmem_acc + t * BN, ai + (uint64_t)(t * 8 * KB), bi, IDESC, accum);
            }
          }
          if (elect_one()) {
            umma_commit(&aempty[slot]);
            if (cb == c_blocks - 1) umma_commit(&tfull[acc]);
          }
          if (lane == 0 && it < 10 && cb == c_blocks - 1) TZC_TRACE_POINT(70 + it);
        }
        __syncwarp();
        if (++slot == a_slots) {
          slot = 0;
          phase ^= 1;
        }
      }
      if (++acc == NACC) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
  } else if (warp >= 4) {
    // ===================== epilogue: padded grid -> output rows =====================
    // EG (p.epi_groups) groups of 16/EG warps; group g drains accumulator
    // buffer g for EG == 2 (ping-pong over alternate units).  A group's W =
    // 4/EG warps per TMEM lane quarter split the unit's MT tiles x BN columns:
    // W >= MT: G = W/MT column groups per tile; W < MT: MT/W whole tiles each.
    const int EG = p.epi_groups;
    const uint32_t q4 = warp & 3;
    const int W = 4 / EG;
    const int g = EG == 2 ? (int)((warp - 4) >> 3) : 0;
    const int h = (int)((warp - 4) >> 2) % W;
    const int hw = p.Hp * p.Wp;
    const int G = W >= MT ? W / MT : 1;
    const int TPW = W >= MT ? 1 : MT / W;  // tiles per warp
    const int cols = BN / G, col0 = (h % G) * cols;
    int acc = g;
    uint32_t acc_phase = 0;
    for (int tile = blockIdx.x + g * (int)gridDim.x, it = g; tile < num_tiles; tile += EG * gridDim.x, it += EG) {
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      if (threadIdx.x == 128 && it < 10) TZC_TRACE_POINT(13 + 5 * it);
#pragma unroll 1
      for (int i = 0; i < TPW; ++i) {
        const int t = W >= MT ? h / G : h * TPW + i;
        const int q = (tile * MT + t) * BM + q4 * 32 + lane;
        int m = -1;
        if (q < p.P) {  // exact magic-number division (q < 2^22 host-checked)
          const int n = (int)(((uint64_t)q * p.magic_hw) >> 40), rem = q - n * hw;
          const int oh = (int)(((uint64_t)rem * p.magic_wp) >> 40), ow = rem - oh * p.Wp;
          if (oh < p.OH && ow < p.OWv) m = (n * p.OH + oh) * p.OWv + ow;
        }
        if (p.debug_flags & 2) m = -1;
        const uint32_t tq = tmem_base + ((q4 * 32) << 16) + acc * (MT * BN) + t * BN + col0;
        if (!(p.debug_flags & 1)) {
          const bool fast = p.vec_ok && BN <= p.Ngemm;
          if (cols == 16) {
            epi_chunk<16, kF16, kEpm, BN>(p, tq, m, col0, fast);
          } else if (kEpm == EPM_REQUANT && p.simple && !p.range_check && cols == 64) {
            // the bench / serving requant: both 32-column TMEM loads in flight
            // before one wait (the lean simple path leaves room for 64
            // accumulator registers; the general paths keep one chunk)
            uint32_t va[32], vb[32];
            tmem_ld32(tq, va);
            tmem_ld32(tq + 32, vb);
            tmem_ld_wait();
            if (m >= 0) {
              epi_simple_impl<32, BN, false>(p, m, col0, va, 0u, 0, 0);
              epi_simple_impl<32, BN, false>(p, m, col0 + 32, vb, 0u, 0, 0);
            }
          } else {
#pragma unroll 1
            for (int c = 0; c < cols / 32; ++c) epi_chunk<32, kF16, kEpm, BN>(p, tq + 32 * c, m, col0 + 32 * c, fast);
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
      if (threadIdx.x == 128 && it < 10) TZC_TRACE_POINT(14 + 5 * it);
      if (EG == 2) {
        acc_phase ^= 1;
      } else if (++acc == NACC) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
  }
  __syncwarp();
  __syncthreads();
  TZC_TRACE_FLUSH;
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<TMEM_COLS>(tmem_base);
  }
}

}  // namespace tzcdev
