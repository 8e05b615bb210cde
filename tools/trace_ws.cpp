// Cycle trace of one conv launch (shifted-window or general kernel), CTA 0, first 10 tiles:
// args: n hp c k r stride [debug_flags] [shifted_window 0/1]
// [producer A issued, MMA tile start, MMA first A ready, epi start, epi end]
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <algorithm>
#include <string>
#include <vector>

#include "tzc_b200.h"

extern "C" void tzc_trace_dump(unsigned long long* out);
extern "C" void tzc_debug_flags(int f);
extern "C" void tzc_trace_cta(unsigned long long* out);

int main(int argc, char** argv) {
  int n = argc > 1 ? atoi(argv[1]) : 256, hp = argc > 2 ? atoi(argv[2]) : 230, c = argc > 3 ? atoi(argv[3]) : 3;
  int k = argc > 4 ? atoi(argv[4]) : 64, r = argc > 5 ? atoi(argv[5]) : 7, st = argc > 6 ? atoi(argv[6]) : 2;
  void *x, *w, *o;
  size_t xb = (size_t)n * hp * hp * c, wb = (size_t)k * r * r * c;
  int oh = (hp - r) / st + 1;
  cudaMalloc(&x, xb);
  cudaMalloc(&w, wb);
  cudaMalloc(&o, (size_t)n * oh * oh * k);
  cudaMemset(x, 1, xb);
  cudaMemset(w, 1, wb);
  tzc_conv_desc d{};
  d.profile = TZC_PROFILE_U8I8;
  d.n = n; d.hp = hp; d.wp = hp; d.c = c; d.k = k; d.r = r; d.s = r; d.stride = st;
  d.w_stride_k = (int64_t)r * r * c; d.w_stride_tap = c;
  d.out.nb = k; d.out.stride_m = k;
  tzc_epilogue ep{TZC_EP_REQUANT_I8, 1.0f / 4096};
  if (argc > 7) tzc_debug_flags(atoi(argv[7]));
  if (argc > 8) tzc_b200_set_option("shifted_window", atoi(argv[8]));
  if (const char* env = getenv("TZC_OPTS")) {  // "name=value,name=value"
    std::string s(env);
    size_t i = 0;
    while (i < s.size()) {
      size_t j = s.find(',', i);
      if (j == std::string::npos) j = s.size();
      const std::string kv = s.substr(i, j - i);
      const size_t eq = kv.find('=');
      if (eq != std::string::npos) tzc_b200_set_option(kv.substr(0, eq).c_str(), atoi(kv.substr(eq + 1).c_str()));
      i = j + 1;
    }
  }
  // warm the clocks first: a few hundred launches (~50-100 ms) so the traced
  // launches run at the sustained SM clock, not the idle one (a trace taken
  // right after start-up ran at ~1 GHz)
  for (int wu = 0; wu < 400; ++wu) tzc_b200_conv2d_i8(&d, (const uint8_t*)x, (const int8_t*)w, nullptr, o, &ep, nullptr);
  cudaDeviceSynchronize();
  for (int it = 0; it < 3; ++it) {
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    int rc = tzc_b200_conv2d_i8(&d, (const uint8_t*)x, (const int8_t*)w, nullptr, o, &ep, nullptr);
    cudaEventRecord(b);
    if (rc) { printf("rc=%d %s\n", rc, tzc_b200_last_error()); return 1; }
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    unsigned long long t[128];
    tzc_trace_dump(t);
    printf("iter %d: %.1f us total\n", it, ms * 1000);
    {
      static unsigned long long ct[2][1024];
      tzc_trace_cta(&ct[0][0]);
      unsigned long long s0 = ~0ull, s1 = 0, e0 = ~0ull, e1 = 0;
      int nc = 0;
      for (int b = 0; b < 1024; ++b) {
        if (!ct[0][b] || ct[1][b] < ct[0][b]) continue;
        ++nc;
        s0 = std::min(s0, ct[0][b]); s1 = std::max(s1, ct[0][b]);
        e0 = std::min(e0, ct[1][b]); e1 = std::max(e1, ct[1][b]);
      }
      printf("  CTAs %d: start spread %.2f us, end min %.2f max %.2f us after first start\n", nc, (s1 - s0) / 1e3,
             (e0 - s0) / 1e3, (e1 - s0) / 1e3);
      std::vector<double> ends;
      for (int b = 0; b < 1024; ++b)
        if (ct[0][b] && ct[1][b] >= ct[0][b]) ends.push_back((ct[1][b] - s0) / 1e3);
      std::sort(ends.begin(), ends.end());
      if (!ends.empty())
        printf("  end percentiles: p10 %.2f p50 %.2f p90 %.2f us\n", ends[ends.size() / 10], ends[ends.size() / 2],
               ends[ends.size() * 9 / 10]);
      cudaMemset(nullptr, 0, 0);
    }
    for (int i = 0; i < 10; ++i)
      printf("  tile %d: prodA=%lld mmaStart=%lld aReady=%lld issued=%lld epiStart=%lld epiEnd=%lld\n", i, (long long)(t[10 + 5 * i] - t[0]),
             (long long)(t[11 + 5 * i] - t[0]), (long long)(t[12 + 5 * i] - t[0]), (long long)(t[70 + i] - t[0]), (long long)(t[13 + 5 * i] - t[0]),
             (long long)(t[14 + 5 * i] - t[0]));
    for (int i = 0; i < 10; ++i)
      printf("  tile %d: mmaLoopTop=%lld temptyOk=%lld xformStart=%lld xformEnd=%lld\n", i, (long long)(t[80 + i] - t[0]),
             (long long)(t[90 + i] - t[0]), (long long)(t[100 + i] - t[0]), (long long)(t[110 + i] - t[0]));
  }
  {
    unsigned long long t[128];
    tzc_trace_dump(t);
    printf("  tile 4 epilogue (thread 128): start=%lld waitread=%lld bar1=%lld c0=%lld c1=%lld c2=%lld c3=%lld bar2=%lld tma=%lld end=%lld\n",
           (long long)(t[13 + 5 * 4] - t[0]), (long long)(t[119] - t[0]), (long long)(t[120] - t[0]), (long long)(t[121] - t[0]),
           (long long)(t[122] - t[0]), (long long)(t[123] - t[0]), (long long)(t[124] - t[0]), (long long)(t[125] - t[0]),
           (long long)(t[126] - t[0]), (long long)(t[14 + 5 * 4] - t[0]));
  }
  return 0;
}
