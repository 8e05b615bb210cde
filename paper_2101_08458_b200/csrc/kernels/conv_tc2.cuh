// conv_tc2_kernel: the general tiled / TMA-im2col conv-GEMM on CTA pairs
// (cta_group::2), for the int8 requant epilogue (direct or TMA-store).
//
// Why: a single-CTA 128 x BN tile pulls 128 + BN operand rows per K block
// through L2 -> SMEM (~6300 B/cycle chip-wide); a pair computes one 256 x BN
// tile with ONE M=256 MMA stream, each CTA holding its 128 A rows and HALF
// of the B rows (the MMA reads B[0, BN/2) from CTA 0 and B[BN/2, BN) from
// CTA 1), so a CTA pulls 128 + BN/2 rows: -33 % L2 -> SMEM bytes at BN=256,
// -25 % at BN=128.  Measured: 2-3 us faster per deep-K layer (3x3 at 14x14
// and 7x7), slower on K <= 1 KiB layers, and no gain in the multi-branch
// suite, so it is opt-in (set_option "pair").
//
// Roles (both CTAs run all of them except the MMA issuer):
//   warp 0   TMA producer: waits its own `empty` slot, loads its A / B half,
//            completion counted on the LEADER's `full` barrier
//   warp 1   (leader only) MMA issuer: tcgen05.mma.cta_group::2, commits
//            multicast to both CTAs' `empty` / `tfull` barriers
//   warp 2   TMEM allocation (cta_group::2, both CTAs)
//   warps 4+ epilogue on this CTA's 128 accumulator rows; arrival on the
//            leader's `tempty` barrier (2 x 16 warps)
// The tile order, requant and TMA-store epilogue are those of
// conv_tc_kernel (conv_tc.cuh); units are pair tiles (m_pair, n_tile).
#pragma once
#include "conv_tc.cuh"

namespace tzcdev {

template <int BN>
struct Pair2Cfg {
  static constexpr int KB = 128;
  static constexpr int A_BYTES = 128 * KB;
  static constexpr int B_BYTES = (BN / 2) * KB;  // this CTA's half of the B tile
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int STAGING_BYTES = 128 * BN;
  static constexpr int TMEM_COLS = 2 * BN;
};

template <int BN, int kAMode>
__global__ void __launch_bounds__(EpiCfg<BN>::THREADS, 1) conv_tc2_kernel(const __grid_constant__ ConvKernelParams p) {
  using Cfg = Pair2Cfg<BN>;
  constexpr int BM = 128, KB = 128, KE = 128, MMAS = KB / 32;
  constexpr uint32_t IDESC = idesc_i8(256, BN);
  const int STAGES = p.stages;

  extern __shared__ uint8_t smem_raw[];
  TZC_CHK_INIT(p);
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sStage = smem;
  uint8_t* sA = smem + Cfg::STAGING_BYTES;
  uint8_t* sB = sA + STAGES * Cfg::A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + STAGES * Cfg::B_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const uint32_t warp = warp_id();
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const int pair = (int)(blockIdx.x >> 1), npairs = (int)(gridDim.x >> 1);

  if (warp == 0 && lane == 0) {
    tma_prefetch(&p.tmA);
    tma_prefetch(&p.tmB);
  }
  if (warp == 1 && lane == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);   // leader: its producer's expect_tx arrival (+ both CTAs' bytes)
      mbar_init(&empty[s], 1);  // the leader's multicast commit
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 32);  // 16 epilogue warps x 2 CTAs (leader's copy)
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc_cg2<Cfg::TMEM_COLS>(tmem_slot);
  tc_fence_before();
  cluster_sync();  // peer barriers initialised before any remote arrive / complete_tx
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  pdl_launch_dependents();
  pdl_wait();

  const int num_units = p.num_tiles;  // pair tiles

  if (warp == 0 || (warp == 3 && p.producers == 2)) {
    // two producer warps, alternate K blocks (as conv_tc_kernel: loads issued
    // from one waiting thread complete ~serially, tools/tma_probe.cu)
    if (lane == 0) {
      const uint32_t pj = warp == 0 ? 0u : 1u;
      const uint32_t np = p.producers == 2 ? 2u : 1u;
      uint32_t g = 0;
      const uint32_t full0 = mapa_shared(smem_u32(full), 0);  // the leader's full[0]
      int stage = 0;
      uint32_t phase = 0;
      for (int u = pair; u < num_units; u += npairs) {
        const int m_pair = (int)fdiv(u, p.fd_tiles_n), n_tile = u - m_pair * p.tiles_n;
        const int m0 = (2 * m_pair + (int)rank) * BM, n0 = n_tile * BN + (int)rank * (BN / 2);
        int img = 0, oh = 0, ow = 0;
        if constexpr (kAMode == A_IM2COL) {
          img = (int)fdiv(m0, p.fd_ohow);
          const int rem = m0 - img * p.OHOW;
          oh = (int)fdiv(rem, p.fd_ow);
          ow = rem - oh * p.OW;
        }
        for (int kb = 0; kb < p.num_kb; ++kb, ++g) {
          if (np == 2 && (g & 1u) != pj) {
            if (++stage == STAGES) {
              stage = 0;
              phase ^= 1;
            }
            continue;
          }
          mbar_wait(&empty[stage], phase ^ 1);
          const int tap = (int)fdiv(kb, p.fd_cblocks);
          const int cb = kb - tap * p.c_blocks;
          uint8_t* dA = sA + stage * Cfg::A_BYTES;
          uint8_t* dB = sB + stage * Cfg::B_BYTES;
          const uint32_t fb = full0 + stage * 8;
          if (rank == 0) mbar_expect_tx(&full[stage], 2 * Cfg::STAGE_BYTES);
          if constexpr (kAMode == A_IM2COL) {
            const int r = (int)fdiv(tap, p.fd_s), s = tap - r * p.S;
            tma_load_im2col_4d_cg2(dA, &p.tmA, fb, cb * KE, ow * p.stride, oh * p.stride, img, (uint16_t)s,
                                   (uint16_t)r);
          } else {
            tma_load_2d_cg2(dA, &p.tmA, fb, kb * KE, m0, p.pol_a ? p.pol_a : kL2EvictFirst);
          }
          tma_load_3d_cg2(dB, &p.tmB, fb, cb * KE, n0, tap);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (rank == 0) {
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int u = pair; u < num_units; u += npairs) {
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t tmem_d = tmem_base + acc * BN;
        for (int kb = 0; kb < p.num_kb; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t a_base = smem_u32(sA + stage * Cfg::A_BYTES);
          const uint32_t b_base = smem_u32(sB + stage * Cfg::B_BYTES);
#pragma unroll
          for (int k = 0; k < MMAS; ++k) {
            const uint64_t adesc = smem_desc_kmajor(a_base + 32 * k, KB);
            const uint64_t bdesc = smem_desc_kmajor(b_base + 32 * k, KB);
            if (elect_one()) umma_i8_cg2(tmem_d, adesc, bdesc, IDESC, (kb > 0 || k > 0) ? 1u : 0u);
          }
          if (elect_one()) {
            umma_commit_cg2(&empty[stage], 3);
            if (kb == p.num_kb - 1) umma_commit_cg2(&tfull[acc], 3);
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
    }
  } else if (warp >= 4) {
    // 16 warps: 4 per TMEM lane quarter, BN/4 columns each (conv_tc_kernel, EG = 1)
    const uint32_t q = warp & 3;
    const uint32_t h = (warp - 4) >> 2;
    constexpr int HALF = BN / 4;
    constexpr int CW = EpiCfg<BN>::CW;
    constexpr int RB = BN < 128 ? BN : 128;
    const uint32_t tempty0 = mapa_shared(smem_u32(tempty), 0);
    uint8_t* stq = sStage + q * (32 * BN);
    const uint32_t bar = 1 + q;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int u = pair; u < num_units; u += npairs) {
      const int m_pair = (int)fdiv(u, p.fd_tiles_n), n_tile = u - m_pair * p.tiles_n;
      const int m_tile = 2 * m_pair + (int)rank;
      const int m = m_tile * BM + q * 32 + lane;
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const uint32_t tq = tmem_base + ((q * 32) << 16) + acc * BN;
      if (p.tma_store) {
        if (h == 0 && lane == 0) bulk_wait_read0();  // the previous store has read the staging
        named_bar_sync(bar, 128);
#pragma unroll 1
        for (int c = 0; c < HALF / CW; ++c) {
          const int col = h * HALF + c * CW;
          epi_chunk<CW, false, EPM_REQUANT, BN>(p, tq + col, m < p.M ? m : -1, n_tile * BN + col, true,
                                                smem_u32(stq), (int)lane, col);
        }
        fence_proxy_async_smem();
        named_bar_sync(bar, 128);
        if (h == 0 && lane == 0 && m_tile * BM < p.M) {
#pragma unroll
          for (int b = 0; b < BN / RB; ++b)
            tma_store_2d(&p.tmO, stq + b * (32 * RB), n_tile * BN + b * RB, m_tile * BM + q * 32);
          bulk_commit();
        }
      } else {  // direct row stores (whole N tile in range: host-checked)
#pragma unroll 1
        for (int c = 0; c < HALF / CW; ++c) {
          const int col = h * HALF + c * CW;
          epi_chunk<CW, false, EPM_REQUANT, BN>(p, tq + col, m < p.M ? m : -1, n_tile * BN + col, true);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(tempty0 + acc * 8);
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
    if (p.tma_store && h == 0 && lane == 0) bulk_wait0();
  }
  __syncwarp();
  __syncthreads();
  cluster_sync();  // the peer is done with its TMEM and with remote arrivals
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc_cg2<Cfg::TMEM_COLS>(tmem_base);
  }
}

}  // namespace tzcdev
