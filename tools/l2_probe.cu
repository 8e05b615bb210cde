// Probe: L2 -> shared-memory bulk-copy bandwidth per SM (the operand path of
// the conv kernels).  148 CTAs, one thread each keeps S chunks of CH bytes in
// flight with cp.async.bulk (1-D TMA) from an L2-resident region, waiting on
// one mbarrier per slot.  Modes: 0 = every CTA reads its own slice of the
// region (distinct lines), 1 = every CTA reads the SAME chunks in the same
// order (the weight operand: all SMs fetch one B block at once), 2 = same
// chunks, but CTA b starts at chunk offset b (rotated).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2101_08458_b200/csrc tools/l2_probe.cu
#include <cuda_runtime.h>

#include <cstdio>

#include "kernels/ptx.cuh"

using namespace tzcdev;

template <int MODE, bool SPIN>
__global__ void __launch_bounds__(32, 1) l2bw(const uint8_t* src, long long region, int ch, int slots, int iters,
                                              unsigned* sink) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar[16];
  if (threadIdx.x != 0) return;
  for (int s = 0; s < slots; ++s) mbar_init(&bar[s], 1);
  fence_barrier_init();
  const long long nch = region / ch;
  const long long per_cta = nch / gridDim.x;
  auto chunk = [&](long long i) -> long long {
    if (MODE == 0) return (blockIdx.x * per_cta + i % per_cta) * ch;
    if (MODE == 1) return (i % nch) * ch;
    return ((i + blockIdx.x) % nch) * ch;
  };
  auto issue = [&](int s, long long i) {
    mbar_expect_tx(&bar[s], ch);
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(sm + s * ch)),
        "l"(src + chunk(i)), "r"(ch), "r"(smem_u32(&bar[s]))
        : "memory");
  };
  for (int s = 0; s < slots; ++s) issue(s, s);
  uint32_t ph = 0;
  for (long long i = 0; i < iters; ++i) {
    const int s = (int)(i % slots);
    if (SPIN)
      mbar_wait_spin(&bar[s], ph);
    else
      mbar_wait(&bar[s], ph);
    if (s == slots - 1) ph ^= 1;
    if (i + slots < iters) issue(s, i + slots);
  }
  if (sm[5] == 0x7f && sm[77] == 0x11) sink[0] = 1;
}

template <int MODE, bool SPIN = false>
void run(const uint8_t* src, long long region, int ch, int slots, int iters, unsigned* sink) {
  auto k = l2bw<MODE, SPIN>;
  const int smem = 1024 + ch * slots;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  k<<<148, 32, smem>>>(src, region, ch, slots, iters, sink);
  cudaDeviceSynchronize();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e9;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    k<<<148, 32, smem>>>(src, region, ch, slots, iters, sink);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  const double bytes = 148.0 * ch * iters;
  printf("%s mode %d region %6.1f MB chunk %6d slots %2d: %7.2f us  %6.0f GB/s  %5.1f B/clk/SM (@1.965GHz) err=%s\n", SPIN ? "spin" : "wait", MODE,
         region / 1e6, ch, slots, best * 1e3, bytes / (best * 1e-3) / 1e9, bytes / 148 / (best * 1e-3) / 1.965e9,
         cudaGetErrorString(cudaGetLastError()));
}

int main() {
  uint8_t* src;
  unsigned* sink;
  const long long big = 1ll << 30;
  cudaMalloc(&src, big);
  cudaMemset(src, 1, big);
  cudaMalloc(&sink, 64);
  for (int ch : {8192, 16384, 32768, 65536}) {
    for (int slots : {2, 3}) {
      if (ch * slots > 200 * 1024) continue;
      const int iters = (int)((8ll << 20) / ch);  // 8 MB per CTA
      run<0, false>(src, 32ll << 20, ch, slots, iters, sink);
      run<0, true>(src, 32ll << 20, ch, slots, iters, sink);
      run<0, true>(src, 1ll << 30, ch, slots, iters, sink);
    }
  }
  return 0;
}
