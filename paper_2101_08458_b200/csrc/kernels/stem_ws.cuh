// The C = 3, stride-2 stem (ResNet's 7x7 / 2 over 3 channels) as ONE kernel:
// space-to-depth fused into the producer side of the shifted-window,
// weight-stationary tcgen05 kernel (conv_ws.cuh pair mode).
//
// Space-to-depth turns the stride-2 7x7 conv over 3 channels into a stride-1
// 4x4 conv over 16-byte pixels (4 phases x 3 channels + 4 zero bytes):
//   x4[n,i,j][(a*2+b)*3+c] = x[n, 2i+a, 2j+b, c]
//   w4[k,i,j][(a*2+b)*3+c] = w[k, 2i+a, 2j+b, c]      (zero outside 7x7)
// exact because padded channels meet zero weights (the reference's own pad
// argument, /root/reference/proj/src/rewriter.cpp:175-204).  The earlier
// path materialised x4 in HBM with a separate kernel (read 41 MB, write 54 MB,
// re-read 54 MB at batch 256) and w4 with a third launch.  Here:
//
//   warp 0      TMA producer: per work unit, the CONTIGUOUS raw byte range
//               its S2D rows need (1-D tensor map over the input bytes,
//               256-byte boxes from a 16-byte aligned start, OOB zero fill)
//   warp 1      MMA issuer: per 128-row tile 8 K=32 MMAs, each covering taps
//               (r, s) and (r, s+1) (descriptor LBO = next pixel / next tap)
//   warps 2, 3  transform: raw staging -> 16-byte S2D pixels of the unit's
//               A super-tile (SWIZZLE_NONE, the layout pair-mode MMAs read);
//               explicit LDS, 4 independent pixels per thread per step
//   warps 4..   epilogue (as conv_ws)
// and in the prologue every warp but the producer rearranges the raw
// [K,7,7,3] weights into the stationary S2D weight tile in SMEM.
#pragma once
#include "conv_tc.cuh"

#ifndef TZC_STEM_SPIN
#define TZC_STEM_SPIN 0
#endif

namespace tzcdev {

// SWIZZLE_NONE K-major descriptor (conv_ws.cuh keeps its own copy).
__device__ __forceinline__ uint64_t stem_desc_none(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFF);
  d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFF) << 16;
  d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFF) << 32;
  d |= static_cast<uint64_t>(1) << 46;
  return d;
}

// 32-bit shared-memory load at a shared-window address (explicit LDS: a
// plain C++ load through the dynamic-smem pointer compiled to a generic LD,
// which went through the LSU's global queue and made the transform 3x slower).
__device__ __forceinline__ uint32_t lds32(uint32_t addr) {
  uint32_t v;
  asm("ld.shared.b32 %0, [%1];" : "=r"(v) : "r"(addr));
  return v;
}

// 8 bytes of the raw staging starting at byte offset o (word-aligned reads).
__device__ __forceinline__ uint2 raw8(uint32_t base, uint32_t o) {
  const uint32_t a = base + (o & ~3u), sh = (o & 3u) * 8u;
  uint32_t w0, w1, w2;
  asm volatile("ld.shared.b32 %0, [%1];" : "=r"(w0) : "r"(a));
  asm volatile("ld.shared.b32 %0, [%1];" : "=r"(w1) : "r"(a + 4));
  asm volatile("ld.shared.b32 %0, [%1];" : "=r"(w2) : "r"(a + 8));
  return make_uint2(__funnelshift_r(w0, w1, sh), __funnelshift_r(w1, w2, sh));
}

__device__ __forceinline__ void stem_wait(uint64_t* bar, uint32_t parity) {
#if TZC_STEM_SPIN
  mbar_wait_spin(bar, parity);
#else
  mbar_wait(bar, parity);
#endif
}

template <int BN, int kEpm>
__global__ void __launch_bounds__(EpiCfg<BN>::THREADS, 1) stem_ws_kernel(const __grid_constant__ ConvKernelParams p) {
  constexpr int BM = 128;
  constexpr uint32_t IDESC = idesc_i8(BM, BN);
  constexpr uint32_t TMEM_COLS = 512;
  constexpr int TAPS = 16;                 // 4 x 4 S2D taps
  constexpr int B_TILE = BN * 16;          // one tap of weights: BN rows x 16 bytes
  constexpr int B_BYTES = TAPS * B_TILE;
  const int a_slot = ((p.SR * 16 + 1023) / 1024) * 1024;
  const int a_slots = p.splits;            // A ring depth
  const int r_slots = p.raw_slots;
  extern __shared__ uint8_t smem_raw[];
  TZC_TRACE_DECL
  TZC_TRACE_INIT;
  TZC_CHK_INIT(p);
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sB = smem;
  uint8_t* sA = sB + ((B_BYTES + 1023) / 1024) * 1024;
  uint8_t* sR = sA + a_slots * a_slot;
  uint64_t* rfull = reinterpret_cast<uint64_t*>(sR + r_slots * p.raw_slot);
  uint64_t* rempty = rfull + r_slots;
  uint64_t* afull = rempty + r_slots;
  uint64_t* aempty = afull + a_slots;
  uint64_t* bready = aempty + a_slots;
  uint64_t* tfull = bready + 1;
  uint64_t* tempty = tfull + 4;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 4);
  const int NACC = p.nacc;
  constexpr int kBuildWarps = EpiCfg<BN>::WARPS + 3;  // warps 1..3 + the epilogue warps

  const uint32_t warp = warp_id();
  const uint32_t lane = threadIdx.x & 31;
  if (warp == 0 && lane == 0) tma_prefetch(&p.tmA);
  if (warp == 1 && lane == 0) {
    for (int s = 0; s < r_slots; ++s) {
      mbar_init(&rfull[s], 1);
      mbar_init(&rempty[s], 2);  // the two transform warps
    }
    for (int s = 0; s < a_slots; ++s) {
      mbar_init(&afull[s], 2);
      mbar_init(&aempty[s], 1);
    }
    mbar_init(bready, kBuildWarps);
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

  const int units = p.num_tiles;
  const int MT = p.mt;
  const int hw4 = p.Hp * p.Wp;  // S2D grid (padded): Hp4 x Wp4 per image
  const int row_bytes = p.raw_wp * p.raw_c;

  if (warp == 0) {
    // ===================== raw TMA producer =====================
    if (lane == 0) {
      int slot = 0;
      uint32_t phase = 0;
      for (int u = blockIdx.x; u < units; u += gridDim.x) {
        const int q0 = u * MT * BM;
        const int n0 = (int)(((uint64_t)q0 * p.magic_hw) >> 40), rem = q0 - n0 * hw4;
        const int i0 = (int)(((uint64_t)rem * p.magic_wp) >> 40);
        // TMA box starts must be 16-byte aligned: stage from the aligned-down offset
        const int base = (((n0 * p.raw_hp + 2 * i0) * p.raw_wp) * p.raw_c) & ~15;
        stem_wait(&rempty[slot], phase ^ 1);
        if (u / (int)gridDim.x < 10) TZC_TRACE_POINT(10 + 5 * (u / (int)gridDim.x));
        if (!(p.debug_flags & 8)) mbar_expect_tx(&rfull[slot], p.raw_boxes * 256);
        uint8_t* dst = sR + slot * p.raw_slot;
        if (p.debug_flags & 8) {
          mbar_arrive(&rfull[slot]);  // debug: no loads (expect_tx of 0 bytes below)
        } else {
          for (int b = 0; b < p.raw_boxes; ++b)
            tma_load_1d_hint(dst + 256 * b, &p.tmA, &rfull[slot], base + 256 * b, kL2EvictFirst);
        }
        if (++slot == r_slots) {
          slot = 0;
          phase ^= 1;
        }
      }
    }
    return;  // the producer does not join the weight build (its loads are in flight)
  }

  // ---- prologue (warps 1..): stationary S2D weights, built from raw [K,R,S,C]
  {
    const int t = threadIdx.x - 32, nt = blockDim.x - 32;
    const uint8_t* w = static_cast<const uint8_t*>(p.wraw);
    for (int ch = (p.debug_flags & 32) ? TAPS * BN : t; ch < TAPS * BN; ch += nt) {  // 16-byte chunk (tap, k)
      const int tap = ch / BN, k = ch - tap * BN;
      const int r4 = tap >> 2, s4 = tap & 3;
      uint32_t b[12];
#pragma unroll
      for (int ph = 0; ph < 4; ++ph) {
        const int r = 2 * r4 + (ph >> 1), s = 2 * s4 + (ph & 1);
        const bool in = r < p.w_r && s < p.w_s;
        const uint8_t* src = w + k * p.w_sk + (int64_t)(r * p.w_s + s) * p.w_st;
#pragma unroll
        for (int c = 0; c < 3; ++c) b[3 * ph + c] = (in && c < p.raw_c) ? __ldg(src + c) : 0u;
      }
      st_shared_v4(smem_u32(sB + tap * B_TILE + k * 16), b[0] | (b[1] << 8) | (b[2] << 16) | (b[3] << 24),
                   b[4] | (b[5] << 8) | (b[6] << 16) | (b[7] << 24), b[8] | (b[9] << 8) | (b[10] << 16) | (b[11] << 24),
                   0u);
    }
    fence_proxy_async_smem();  // generic-proxy writes -> visible to the tensor core (async proxy)
    __syncwarp();
    if (lane == 0) mbar_arrive(bready);
  }

  // S2D transform of the k-th work unit of this CTA into its A slot by
  // nthr threads (thread tid takes pixels tid, tid + nthr, ...).
  // Every pixel independently: p = j0 + px -> (row r, column j) by a 32-bit
  // magic multiply, (n, i) = (n0, i0 + r) carried over image ends; the row
  // h+1 / pixel x+1 edge cases are masks, so the loads of all of a thread's
  // pixels are in flight together.
  auto transform_unit = [&](int k, int tid, int nthr) {
    // the geometry in registers: kernel-parameter (constant bank) loads on
    // the transform's critical path cost more than the arithmetic
    const int gH = p.Hp, gW = p.Wp, gSR = p.SR, gP = p.P, ghp = p.raw_hp, gwp = p.raw_wp, gdbg = p.debug_flags;
    const uint32_t gm = p.magic_wp32;
    const int u = blockIdx.x + k * (int)gridDim.x;
    const int rslot = k % r_slots, aslot = k % a_slots;
    const uint32_t rphase = (uint32_t)(k / r_slots) & 1u, aphase = (uint32_t)(k / a_slots) & 1u;
    const int q0 = u * MT * BM;
    const int n0 = (int)(((uint64_t)q0 * p.magic_hw) >> 40), rem0 = q0 - n0 * hw4;
    const int i0 = (int)(((uint64_t)rem0 * p.magic_wp) >> 40);
    const int base = (((n0 * ghp + 2 * i0) * gwp) * p.raw_c) & ~15;  // as the producer staged it
    if (!(gdbg & 256)) {
      stem_wait(&rfull[rslot], rphase);
      stem_wait(&aempty[aslot], aphase ^ 1u);
    }
    if (threadIdx.x == 64 && k < 10) TZC_TRACE_POINT(100 + k);
    const uint32_t rs = smem_u32(sR + rslot * p.raw_slot);
    const uint32_t as = smem_u32(sA + aslot * a_slot);
    // Row by row of the S2D grid: each transform warp takes whole rows of the
    // unit (warp-uniform (n, i), no division per pixel) and each lane a run of
    // 4 consecutive pixels, whose 2 x 24 raw bytes are contiguous (7 words
    // per raw row).  Everything at the edges is a mask, never a branch: the
    // unit's first / last partial row (px outside [0, SR)), the row end
    // (jj >= Wp4), a missing raw pixel x+1 (odd widths), a missing raw row
    // h+1 (odd heights) and rows past the last image (zeros).
    const int j0 = rem0 - i0 * gW;
    const int rows = (j0 + gSR + gW - 1) / gW;  // S2D rows the unit touches
    for (int r = (gdbg & 16) ? rows : tid / 32; r < rows; r += nthr / 32) {
      int i = i0 + r, n = n0;
      while (i >= gH) {  // the unit crosses into the next image (uniform)
        i -= gH;
        ++n;
      }
      const int h = 2 * i;
      const bool live = q0 + r * gW - j0 < gP;  // this S2D row is inside the batch
      const uint32_t m1 = (live && h + 1 < ghp) ? 0xffffffffu : 0u;
      const uint32_t m0 = live ? 0xffffffffu : 0u;
      const int jj = 4 * (int)lane;               // first column of this lane's run
      const int px0 = r * gW - j0 + jj;           // its pixel index in the unit
      if (jj >= gW || px0 >= gSR || px0 + 4 <= 0) continue;
      const int o = live ? ((n * ghp + h) * gwp + 2 * jj) * 3 - base : 0;
      const int o1 = o + row_bytes;
      const uint32_t sh = (uint32_t)(o & 3) * 8u, sh1 = (uint32_t)(o1 & 3) * 8u;
      const uint32_t ad = rs + ((uint32_t)o & ~3u), ad1 = rs + ((uint32_t)o1 & ~3u);
      uint32_t a[6], b[6];  // the two raw rows' 24 bytes of this run, as words
      {
        uint32_t w[7], u[7];
#pragma unroll
        for (int q = 0; q < 7; ++q) w[q] = lds32(ad + 4 * q);
#pragma unroll
        for (int q = 0; q < 7; ++q) u[q] = lds32(ad1 + 4 * q);
#pragma unroll
        for (int q = 0; q < 6; ++q) {
          a[q] = __funnelshift_r(w[q], w[q + 1], sh) & m0;
          b[q] = __funnelshift_r(u[q], u[q + 1], sh1) & m1;
        }
      }
      // pixel e of the run: row bytes [6e, 6e+6) of each raw row (bytes 0..2
      // raw pixel x = 2(jj+e), bytes 3..5 raw pixel x+1)
      uint32_t v[4][3];
      v[0][0] = a[0];
      v[0][1] = __byte_perm(a[1], b[0], 0x5410);
      v[0][2] = __byte_perm(b[0], b[1], 0x5432);
      v[1][0] = __byte_perm(a[1], a[2], 0x5432);
      v[1][1] = __byte_perm(a[2], b[1], 0x7632);
      v[1][2] = b[2];
      v[2][0] = a[3];
      v[2][1] = __byte_perm(a[4], b[3], 0x5410);
      v[2][2] = __byte_perm(b[3], b[4], 0x5432);
      v[3][0] = __byte_perm(a[4], a[5], 0x5432);
      v[3][1] = __byte_perm(a[5], b[4], 0x7632);
      v[3][2] = b[5];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int px = px0 + e;
        if (px < 0 || px >= gSR || jj + e >= gW) continue;
        if (2 * (jj + e) + 1 >= gwp) {  // raw pixel x+1 is outside (odd width): zero its 3 bytes per row
          v[e][0] &= 0x00ffffffu;        // row h:   x+1 c0
          v[e][1] &= 0xffff0000u;        // row h:   x+1 c1 c2
          v[e][2] &= 0x000000ffu;        // row h+1: x+1 c0 c1 c2
        }
        st_shared_v4(as + 16u * (uint32_t)px, v[e][0], v[e][1], v[e][2], 0u);
      }
    }
    if (threadIdx.x == 64 && k < 10) TZC_TRACE_POINT(110 + k);
    if (!(gdbg & 64)) fence_proxy_async_smem();  // generic-proxy writes -> visible to the tensor core (async proxy)
    __syncwarp();
    if (lane == 0) {
      mbar_arrive(&afull[aslot]);
      mbar_arrive(&rempty[rslot]);
    }
  };

  if (warp == 2 || warp == 3) {
    // ===================== S2D transform (warps 2, 3) =====================
    const int nk = units > (int)blockIdx.x ? (units - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x : 0;
    for (int k = 0; k < nk; ++k) transform_unit(k, (int)(warp - 2) * 32 + (int)lane, 64);
  } else if (warp == 1) {
    // ===================== MMA issuer =====================
    const uint32_t b_base = smem_u32(sB);
    uint32_t pa[8], pb[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      pa[i] = p.mma_a[i];
      pb[i] = p.mma_b[i];
    }
    stem_wait(bready, 0);
    tc_fence_after();
    int slot = 0, acc = 0;
    uint32_t phase = 0, acc_phase = 0;
    for (int u = blockIdx.x, it = 0; u < units; u += gridDim.x, ++it) {
      if (lane == 0 && it < 10) TZC_TRACE_POINT(80 + it);
      stem_wait(&tempty[acc], acc_phase ^ 1);
      if (lane == 0 && it < 10) TZC_TRACE_POINT(90 + it);
      tc_fence_after();
      const uint32_t tmem_acc = tmem_base + acc * (MT * BN);
      stem_wait(&afull[slot], phase);
      if (lane == 0 && it < 10) TZC_TRACE_POINT(12 + 5 * it);
      tc_fence_after();
      const uint64_t a0 = stem_desc_none(smem_u32(sA + slot * a_slot), 16, 128);
      const uint64_t b0 = stem_desc_none(b_base, B_TILE, 128);
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        if (t < MT) {
          const uint64_t at = a0 + (uint64_t)(t * 128);  // tile t: 128 pixels further (16-byte units)
          const uint32_t tmem_d = tmem_acc + t * BN;
#pragma unroll
          for (int i = 0; i < 8; ++i)
            if (elect_one() && !(p.debug_flags & 1)) umma<false>(tmem_d, at + pa[i], b0 + pb[i], IDESC, i > 0 ? 1u : 0u);
        }
      }
      if (elect_one()) {
        umma_commit(&aempty[slot]);
        umma_commit(&tfull[acc]);
      }
      if (lane == 0 && it < 10) TZC_TRACE_POINT(70 + it);
      __syncwarp();
      if (++slot == a_slots) {
        slot = 0;
        phase ^= 1;
      }
      if (++acc == NACC) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
  } else if (warp >= 4) {
    // ===================== epilogue: padded S2D grid -> output rows =====================
    const int EG = p.epi_groups;
    const uint32_t q4 = warp & 3;
    const int W = 4 / EG;
    const int g = EG == 2 ? (int)((warp - 4) >> 3) : 0;
    const int h = (int)((warp - 4) >> 2) % W;
    const int G = W >= MT ? W / MT : 1;
    const int TPW = W >= MT ? 1 : MT / W;
    const int cols = BN / G, col0 = (h % G) * cols;
    const bool fast = p.vec_ok && BN <= p.Ngemm;
    const int nk = units > (int)blockIdx.x ? (units - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x : 0;
    int acc = g;
    uint32_t acc_phase = 0;
    for (int k = 0; k < nk; ++k) {
      if (EG == 2 && (k & 1) != g) continue;
      const int u = blockIdx.x + k * (int)gridDim.x;
      stem_wait(&tfull[acc], acc_phase);
      if (threadIdx.x == 128 && k < 10) TZC_TRACE_POINT(13 + 5 * k);
      tc_fence_after();
#pragma unroll 1
      for (int i = 0; i < TPW; ++i) {
        const int t = W >= MT ? h / G : h * TPW + i;
        const int q = (u * MT + t) * BM + (int)q4 * 32 + (int)lane;
        int m = -1;
        if (q < p.P) {
          const int n = (int)(((uint64_t)q * p.magic_hw) >> 40), rem = q - n * hw4;
          const int oh = (int)(((uint64_t)rem * p.magic_wp) >> 40), ow = rem - oh * p.Wp;
          if (oh < p.OH && ow < p.OWv) m = (n * p.OH + oh) * p.OWv + ow;
        }
        const uint32_t tq = tmem_base + ((q4 * 32) << 16) + acc * (MT * BN) + t * BN + col0;
        if (p.debug_flags & 2) {
        } else if (cols == 16) {
          epi_chunk<16, false, kEpm, BN>(p, tq, m, col0, fast);
        } else {
#pragma unroll 1
          for (int c = 0; c < cols / 32; ++c) epi_chunk<32, false, kEpm, BN>(p, tq + 32 * c, m, col0 + 32 * c, fast);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
      if (threadIdx.x == 128 && k < 10) TZC_TRACE_POINT(14 + 5 * k);
      if (EG == 2) {
        acc_phase ^= 1;
      } else if (++acc == NACC) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
  }
  __syncwarp();
  // the producer warp returned early: a named barrier over the other warps
  named_bar_sync(1, blockDim.x - 32);
  TZC_TRACE_FLUSH;
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<TMEM_COLS>(tmem_base);
  }
}

}  // namespace tzcdev
