// extern "C" boundary (include/tzc_b200.h): validates descriptors, maps
// them onto the kernel Problem, and turns tzcb200::Status / C++ exceptions
// into return codes + a thread-local message.  No exception crosses.
#include <cuda_runtime.h>

#include <cstring>
#include <map>
#include <mutex>
#include <vector>
#include <exception>
#include <string>

#include "../tzc_b200_internal.hpp"

namespace tzcb200 {

namespace {
thread_local std::string g_last_error;

}  // namespace

void set_last_error(const std::string& m) { g_last_error = m; }

namespace {

int report(const Status& st) {
  if (!st.ok()) g_last_error = st.msg;
  return st.code;
}

Status check_layout(const tzc_out_layout& o, int ngemm, int64_t m) {
  if (o.nb <= 0 || ngemm % o.nb != 0) return Status(TZC_E_SHAPE, "out layout: nb must divide the channel count");
  if (o.stride_m < o.nb) return Status(TZC_E_SHAPE, "out layout: stride_m must be >= nb");
  if (o.nb != ngemm && o.stride_blk < (m - 1) * o.stride_m + o.nb)
    return Status(TZC_E_SHAPE, "out layout: stride_blk must separate channel blocks");
  return Status();
}

// TMA operands need 16-byte aligned base addresses; outputs / seeds do not
// (the epilogue falls back to element stores).
Status check_ptr(const void* p, const char* what, bool nullable, bool tma = true) {
  if (!p) return nullable ? Status() : Status(TZC_E_MISSING_INPUT, std::string(what) + " is NULL");
  if (tma && reinterpret_cast<uintptr_t>(p) % 16 != 0)
    return Status(TZC_E_INJECT, std::string(what) + " must be 16-byte aligned (TMA)");
  return Status();
}

}  // namespace

Status problem_from_conv(const tzc_conv_desc& d, Problem* pb) {
  if (d.profile != TZC_PROFILE_U8I8 && d.profile != TZC_PROFILE_F16) return Status(TZC_E_TYPE, "unknown profile");
  if (d.n <= 0 || d.hp <= 0 || d.wp <= 0 || d.c <= 0 || d.k <= 0 || d.r <= 0 || d.s <= 0 || d.stride <= 0)
    return Status(TZC_E_SHAPE, "conv extents must be positive");
  if (d.hp < d.r || d.wp < d.s) return Status(TZC_E_SHAPE, "filter does not fit the (pre-padded) input");
  Problem p;
  p.f16 = d.profile == TZC_PROFILE_F16;
  p.n = d.n;
  p.hp = d.hp;
  p.wp = d.wp;
  p.c = d.c;
  p.r = d.r;
  p.s = d.s;
  p.stride = d.stride;
  p.oh = (d.hp - d.r) / d.stride + 1;
  p.ow = (d.wp - d.s) / d.stride + 1;
  p.taps = d.r * d.s;
  p.m = (int64_t)d.n * p.oh * p.ow;
  p.ngemm = d.k;
  p.w_stride_k = d.w_stride_k;
  p.w_stride_tap = d.w_stride_tap;
  p.out = d.out;
  const int e = p.f16 ? 2 : 1;
  const bool k7 = ((int64_t)d.c * e) % 16 != 0;  // thin channels: explicit im2col path, no TMA on x/w
  if (!k7 && ((d.w_stride_k * e) % 16 || (p.taps > 1 && (d.w_stride_tap * e) % 16)))
    return Status(TZC_E_INJECT, "weight strides must be multiples of 16 bytes (TMA)");
  if (!k7 && d.r == 1 && d.s == 1 && d.stride == 1) {
    // 1x1 unit-stride conv is a plain GEMM over the pixel rows
    p.a_mode = 0;
    p.a_kdim = d.c;
    p.a_rows = (int64_t)d.n * d.hp * d.wp;
    p.a_row_stride = d.c;
  } else {
    p.a_mode = 1;
  }
  Status st = check_layout(d.out, d.k, p.m);
  if (!st.ok()) return st;
  *pb = p;
  return Status();
}

Status problem_from_gemm(const tzc_gemm_desc& d, Problem* pb) {
  if (d.profile != TZC_PROFILE_U8I8 && d.profile != TZC_PROFILE_F16) return Status(TZC_E_TYPE, "unknown profile");
  if (d.m <= 0 || d.n <= 0 || d.k <= 0) return Status(TZC_E_SHAPE, "matmul extents must be positive");
  if (d.b_kn && d.profile != TZC_PROFILE_F16) return Status(TZC_E_INJECT, "[K,N] B operand is only supported for fp16");
  Problem p;
  p.f16 = d.profile == TZC_PROFILE_F16;
  p.a_mode = 0;
  p.c = d.k;
  p.taps = 1;
  p.wp = d.m;
  p.m = d.m;
  p.ngemm = d.n;
  p.a_kdim = d.k;
  p.a_rows = d.m;
  p.a_row_stride = d.k;
  p.w_stride_k = d.k;
  p.w_stride_tap = d.k;
  p.b_kn = d.b_kn;
  p.out = d.out;
  const int e = p.f16 ? 2 : 1;
  if ((int64_t)d.k * e % 16) return Status(TZC_E_INJECT, "K row must be a multiple of 16 bytes (TMA)");
  if (d.b_kn && (int64_t)d.n * e % 16) return Status(TZC_E_INJECT, "[K,N] row must be a multiple of 16 bytes (TMA)");
  Status st = check_layout(d.out, d.n, d.m);
  if (!st.ok()) return st;
  *pb = p;
  return Status();
}

}  // namespace tzcb200

using namespace tzcb200;

#define TZC_GUARD_BEGIN try {
#define TZC_GUARD_END                                   \
  }                                                     \
  catch (const std::exception& ex) {                    \
    return report(Status(TZC_E_INTERNAL, ex.what()));   \
  }                                                     \
  catch (...) {                                         \
    return report(Status(TZC_E_INTERNAL, "unknown exception")); \
  }

namespace {

template <typename D>
std::string key_of(const D& d, char kind) {
  return std::string(1, kind) + std::string(reinterpret_cast<const char*>(&d), sizeof(D));
}

int run_conv(const tzc_conv_desc* d, int profile, const void* x, const void* w, const void* seed, void* out,
             const tzc_epilogue* ep, void* stream) {
  if (!d || !ep) return report(Status(TZC_E_MISSING_INPUT, "NULL descriptor"));
  if (d->profile != profile) return report(Status(TZC_E_TYPE, "descriptor profile does not match the entry point"));
  Problem pb;
  Status st = problem_from_conv(*d, &pb);
  if (st.ok()) st = check_ptr(x, "x", false);
  if (st.ok()) st = check_ptr(w, "w", false);
  if (st.ok()) st = check_ptr(seed, "c_seed", true, false);
  if (st.ok()) st = check_ptr(out, "out", false, false);
  if (!st.ok()) return report(st);
  return report(run_problem(pb, options_for(key_of(*d, 'c')), x, w, seed, out, *ep, static_cast<cudaStream_t>(stream)));
}

int run_gemm(const tzc_gemm_desc* d, int profile, const void* a, const void* b, const void* seed, void* out,
             const tzc_epilogue* ep, void* stream) {
  if (!d || !ep) return report(Status(TZC_E_MISSING_INPUT, "NULL descriptor"));
  if (d->profile != profile) return report(Status(TZC_E_TYPE, "descriptor profile does not match the entry point"));
  Problem pb;
  Status st = problem_from_gemm(*d, &pb);
  if (st.ok()) st = check_ptr(a, "a", false);
  if (st.ok()) st = check_ptr(b, "b", false);
  if (st.ok()) st = check_ptr(seed, "c_seed", true, false);
  if (st.ok()) st = check_ptr(out, "out", false, false);
  if (!st.ok()) return report(st);
  return report(run_problem(pb, options_for(key_of(*d, 'g')), a, b, seed, out, *ep, static_cast<cudaStream_t>(stream)));
}

}  // namespace

extern "C" {

int tzc_b200_conv2d_i8(const tzc_conv_desc* d, const uint8_t* x, const int8_t* w, const int32_t* c_seed, void* out,
                       const tzc_epilogue* ep, void* stream) {
  TZC_GUARD_BEGIN
  return run_conv(d, TZC_PROFILE_U8I8, x, w, c_seed, out, ep, stream);
  TZC_GUARD_END
}

int tzc_b200_conv2d_f16(const tzc_conv_desc* d, const uint16_t* x, const uint16_t* w, const float* c_seed, void* out,
                        const tzc_epilogue* ep, void* stream) {
  TZC_GUARD_BEGIN
  return run_conv(d, TZC_PROFILE_F16, x, w, c_seed, out, ep, stream);
  TZC_GUARD_END
}

int tzc_b200_gemm_i8(const tzc_gemm_desc* d, const uint8_t* a, const int8_t* b, const int32_t* c_seed, void* out,
                     const tzc_epilogue* ep, void* stream) {
  TZC_GUARD_BEGIN
  return run_gemm(d, TZC_PROFILE_U8I8, a, b, c_seed, out, ep, stream);
  TZC_GUARD_END
}

int tzc_b200_gemm_f16(const tzc_gemm_desc* d, const uint16_t* a, const uint16_t* b, const float* c_seed, void* out,
                      const tzc_epilogue* ep, void* stream) {
  TZC_GUARD_BEGIN
  return run_gemm(d, TZC_PROFILE_F16, a, b, c_seed, out, ep, stream);
  TZC_GUARD_END
}

int tzc_b200_plan_conv(const tzc_conv_desc* d, tzc_plan* plan) {
  TZC_GUARD_BEGIN
  if (!d || !plan) return report(Status(TZC_E_MISSING_INPUT, "NULL argument"));
  Problem pb;
  Status st = problem_from_conv(*d, &pb);
  if (st.ok()) st = plan_problem(pb, options_for(key_of(*d, 'c')), plan);
  return report(st);
  TZC_GUARD_END
}

int tzc_b200_plan_gemm(const tzc_gemm_desc* d, tzc_plan* plan) {
  TZC_GUARD_BEGIN
  if (!d || !plan) return report(Status(TZC_E_MISSING_INPUT, "NULL argument"));
  Problem pb;
  Status st = problem_from_gemm(*d, &pb);
  if (st.ok()) st = plan_problem(pb, options_for(key_of(*d, 'g')), plan);
  return report(st);
  TZC_GUARD_END
}

}  // extern "C"

extern "C" {

int tzc_b200_set_option(const char* name, int64_t value) {
  if (!name) return report(Status(TZC_E_MISSING_INPUT, "NULL option name"));
  return report(set_default_option(name, value));
}

int tzc_b200_set_splits(int32_t splits) {
  if (splits < 0) return report(Status(TZC_E_SHAPE, "splits must be >= 0"));
  return report(set_default_option("splits", splits));
}

int tzc_b200_unblock_data(const void* src, void* dst, int32_t c, int32_t h, int32_t w, int32_t cb, int32_t elem_bytes,
                          void* stream) {
  TZC_GUARD_BEGIN
  if (!device_ok()) return report(Status(TZC_E_DEVICE, "no usable sm_100 (B200) device"));
  return report(unblock_data(src, dst, c, h, w, cb, elem_bytes, static_cast<cudaStream_t>(stream)));
  TZC_GUARD_END
}

int tzc_b200_unblock_kernel(const void* src, void* dst, int32_t k, int32_t c, int32_t r, int32_t s, int32_t kb,
                            int32_t cb, int32_t elem_bytes, void* stream) {
  TZC_GUARD_BEGIN
  if (!device_ok()) return report(Status(TZC_E_DEVICE, "no usable sm_100 (B200) device"));
  return report(unblock_kernel(src, dst, k, c, r, s, kb, cb, elem_bytes, static_cast<cudaStream_t>(stream)));
  TZC_GUARD_END
}

const char* tzc_b200_last_error(void) { return g_last_error.c_str(); }

uint64_t tzc_b200_launch_count(void) { return g_launches.load(); }

int tzc_b200_last_launch(tzc_launch_info* info) {
  if (!info) return report(Status(TZC_E_SHAPE, "null tzc_launch_info"));
  if (!tzcb200::last_launch(info)) return report(Status(TZC_E_SHAPE, "no launch on this thread yet"));
  return TZC_OK;
}

int tzc_b200_device_ok(void) {
  try {
    return device_ok();
  } catch (...) {
    return 0;
  }
}

const char* tzc_b200_version(void) { return "tzc-b200 0.1.0 (sm_100a, tcgen05 kind::i8/kind::f16)"; }

}  // extern "C"

// ---- measured-time tuner (the device analogue of tzc::tune, proj/src/tuner.cpp:111-274) ----
namespace {

// Candidate option sets; index 0 is the default plan.  Each is one kernel-plan
// decision of the reference's GPU sketch space re-cast for this backend:
// tile width (BN), split-K (split_reduction), kernel family (shifted window vs
// TMA im2col), tiles per work unit, epilogue grouping, store path, CTA pairs.
const char* const kCandidates[] = {
    "",           "bn=64",          "bn=128",         "bn=256",        "splits=2",      "splits=4",
    "shifted_window=0", "ws_mt=1",  "ws_mt=2",        "ws_mt=4",       "pingpong_kb=2", "pingpong_kb=16",
    "tma_store=1", "pair=1;pair_min_kb=1;pair_min_round=0", "ws_1x1=1", "ws_epi_groups=2", "l2_hints=0",
    "pair=0", "pair=1;pair_min_kb=1;pair_bn=0;pair_min_round=0", "b_res=0"};
constexpr int kNumCandidates = sizeof(kCandidates) / sizeof(kCandidates[0]);

template <typename Run>
int tune_problem(const std::string& key, Run run, int reps, int apply, char* log, int64_t loglen, cudaStream_t st) {
  if (reps < 1) reps = 10;
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(st, &cap) == cudaSuccess && cap != cudaStreamCaptureStatusNone)
    return report(Status(TZC_E_VALIDATION, "tune: the stream is being captured"));
  cudaEvent_t e0, e1;
  if (cudaEventCreate(&e0) != cudaSuccess || cudaEventCreate(&e1) != cudaSuccess)
    return report(Status(TZC_E_DEVICE, "tune: cudaEventCreate failed"));
  std::string text;
  double best_us = 0, default_us = 0;
  int best = -1;
  for (int c = 0; c < kNumCandidates; ++c) {
    Options o = options_for("");
    float ms = 0;
    Status s = parse_option_spec(kCandidates[c], &o, nullptr);
    {
      for (int w = 0; w < 2 && s.ok(); ++w) s = run(o, st);
      if (s.ok()) cudaEventRecord(e0, st);
      for (int r = 0; r < reps && s.ok(); ++r) s = run(o, st);
      if (s.ok()) cudaEventRecord(e1, st);
      if (s.ok() && cudaEventSynchronize(e1) != cudaSuccess) s = Status(TZC_E_DEVICE, "tune: launch failed");
      if (s.ok()) cudaEventElapsedTime(&ms, e0, e1);
    }
    char line[160];
    if (!s.ok()) {
      if (c == 0) {
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        return report(s);
      }
      std::snprintf(line, sizeof line, "candidate %d %s skipped\n", c, kCandidates[c]);
      text += line;
      continue;
    }
    const double us = 1000.0 * ms / reps;
    std::snprintf(line, sizeof line, "candidate %d %s %.2f us\n", c, c ? kCandidates[c] : "default", us);
    text += line;
    if (c == 0) default_us = us;
    // a non-default plan must beat the default by 1% to be kept
    if (best < 0 || (us < best_us && us < 0.99 * default_us)) best = c, best_us = us;
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  char line[160];
  std::snprintf(line, sizeof line, "best %d %s %.2f us (default %.2f us)\n", best, best ? kCandidates[best] : "default",
                best_us, default_us);
  text += line;
  if (apply) set_problem_options(key, best ? kCandidates[best] : "");
  if (log && loglen > 0) {
    const size_t n = std::min<size_t>(text.size(), (size_t)loglen - 1);
    std::memcpy(log, text.data(), n);
    log[n] = 0;
  }
  return best;
}

}  // namespace

extern "C" {

int tzc_b200_tune_conv(const tzc_conv_desc* d, const void* x, const void* w, const void* c_seed, void* out,
                       const tzc_epilogue* ep, int32_t reps, int32_t apply, char* log, int64_t loglen, void* stream) {
  TZC_GUARD_BEGIN
  if (!d || !ep) return report(Status(TZC_E_MISSING_INPUT, "NULL descriptor"));
  Problem pb;
  Status st = problem_from_conv(*d, &pb);
  if (st.ok()) st = check_ptr(x, "x", false);
  if (st.ok()) st = check_ptr(w, "w", false);
  if (st.ok()) st = check_ptr(c_seed, "c_seed", true, false);
  if (st.ok()) st = check_ptr(out, "out", false, false);
  if (!st.ok()) return report(st);
  const tzc_epilogue e = *ep;
  return tune_problem(
      key_of(*d, 'c'), [&](const Options& o, cudaStream_t s) { return run_problem(pb, o, x, w, c_seed, out, e, s); }, reps, apply, log,
      loglen, static_cast<cudaStream_t>(stream));
  TZC_GUARD_END
}

int tzc_b200_tune_gemm(const tzc_gemm_desc* d, const void* a, const void* b, const void* c_seed, void* out,
                       const tzc_epilogue* ep, int32_t reps, int32_t apply, char* log, int64_t loglen, void* stream) {
  TZC_GUARD_BEGIN
  if (!d || !ep) return report(Status(TZC_E_MISSING_INPUT, "NULL descriptor"));
  Problem pb;
  Status st = problem_from_gemm(*d, &pb);
  if (st.ok()) st = check_ptr(a, "a", false);
  if (st.ok()) st = check_ptr(b, "b", false);
  if (st.ok()) st = check_ptr(c_seed, "c_seed", true, false);
  if (st.ok()) st = check_ptr(out, "out", false, false);
  if (!st.ok()) return report(st);
  const tzc_epilogue e = *ep;
  return tune_problem(
      key_of(*d, 'g'), [&](const Options& o, cudaStream_t s) { return run_problem(pb, o, a, b, c_seed, out, e, s); }, reps, apply, log,
      loglen, static_cast<cudaStream_t>(stream));
  TZC_GUARD_END
}

int tzc_b200_clear_tuning(void) {
  clear_problem_options();
  return TZC_OK;
}

}  // extern "C"

extern "C" {

// Installs (spec = "name=value;...") or clears (spec = "" or NULL) the plan
// options used for every launch of this exact descriptor.
int tzc_b200_set_problem_options_conv(const tzc_conv_desc* d, const char* spec) {
  TZC_GUARD_BEGIN
  if (!d) return report(Status(TZC_E_MISSING_INPUT, "NULL descriptor"));
  return report(set_problem_options(key_of(*d, 'c'), spec ? spec : ""));
  TZC_GUARD_END
}

int tzc_b200_set_problem_options_gemm(const tzc_gemm_desc* d, const char* spec) {
  TZC_GUARD_BEGIN
  if (!d) return report(Status(TZC_E_MISSING_INPUT, "NULL descriptor"));
  return report(set_problem_options(key_of(*d, 'g'), spec ? spec : ""));
  TZC_GUARD_END
}

int tzc_b200_save_tuning(const char* path, int32_t* count) {
  TZC_GUARD_BEGIN
  if (!path) return report(Status(TZC_E_MISSING_INPUT, "NULL path"));
  int n = 0;
  Status st = save_problem_options(path, &n);
  if (st.ok() && count) *count = n;
  return report(st);
  TZC_GUARD_END
}

int tzc_b200_load_tuning(const char* path, int32_t* count) {
  TZC_GUARD_BEGIN
  if (!path) return report(Status(TZC_E_MISSING_INPUT, "NULL path"));
  int n = 0;
  Status st = load_problem_options(path, &n);
  if (st.ok() && count) *count = n;
  return report(st);
  TZC_GUARD_END
}

// The tuner's candidate plans, one option spec per line (line 0 = default = "").
int tzc_b200_tune_candidates(char* buf, int64_t buflen) {
  std::string s;
  for (int c = 0; c < kNumCandidates; ++c) s += std::string(kCandidates[c]) + "\n";
  if (!buf || (int64_t)s.size() + 1 > buflen) return report(Status(TZC_E_SHAPE, "text buffer too small"));
  std::memcpy(buf, s.c_str(), s.size() + 1);
  return TZC_OK;
}

}  // extern "C"
