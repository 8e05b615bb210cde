// Cycle trace of one conv_tc launch (CTA 0).  Build:
//   make -C tools trace   (see tools/Makefile)
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#include "tzc_b200.h"

extern "C" void tzc_trace_dump(unsigned long long* out);

int main(int argc, char** argv) {
  int m = argc > 1 ? atoi(argv[1]) : 128, n = argc > 2 ? atoi(argv[2]) : 256, k = argc > 3 ? atoi(argv[3]) : 128;
  void *a, *b, *o;
  cudaMalloc(&a, (size_t)m * k);
  cudaMalloc(&b, (size_t)n * k);
  cudaMalloc(&o, (size_t)m * n * 4);
  cudaMemset(a, 1, (size_t)m * k);
  cudaMemset(b, 1, (size_t)n * k);
  tzc_gemm_desc d{};
  d.profile = TZC_PROFILE_U8I8;
  d.m = m; d.n = n; d.k = k;
  d.out.nb = n; d.out.stride_m = n;
  tzc_epilogue ep{TZC_EP_REQUANT_I8, 1.0f / 16384};
  for (int it = 0; it < 3; ++it) {
    int rc = tzc_b200_gemm_i8(&d, (const uint8_t*)a, (const int8_t*)b, nullptr, o, &ep, nullptr);
    if (rc) { printf("rc=%d %s\n", rc, tzc_b200_last_error()); return 1; }
    unsigned long long t[64];
    tzc_trace_dump(t);
    printf("iter %d:", it);
    const char* names[] = {"start", "setup", "tma_issued", "first_full", "mma_commit", "epi_start", "epi_end", "end"};
    for (int i = 1; i < 8; ++i) printf(" %s=%lld", names[i], (long long)(t[i] - t[0]));
    printf("\n   chunks:");
    for (int c = 0; c < 8; ++c) printf(" [%lld %lld %lld]", (long long)(t[8 + 3 * c] - t[0]), (long long)(t[9 + 3 * c] - t[0]), (long long)(t[10 + 3 * c] - t[0]));
    printf("\n");
  }
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
