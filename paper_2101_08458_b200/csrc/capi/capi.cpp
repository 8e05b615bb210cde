// extern "C" boundary (include/tzc_b200.h): validates descriptors, maps
// them onto the kernel Problem, and turns tzcb200::Status / C++ exceptions
// into return codes + a thread-local message.  No exception crosses.
#include <cuda_runtime.h>

#include <cstring>
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
  return report(run_problem(pb, x, w, seed, out, *ep, static_cast<cudaStream_t>(stream)));
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
  return report(run_problem(pb, a, b, seed, out, *ep, static_cast<cudaStream_t>(stream)));
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
  if (st.ok()) st = plan_problem(pb, plan);
  return report(st);
  TZC_GUARD_END
}

int tzc_b200_plan_gemm(const tzc_gemm_desc* d, tzc_plan* plan) {
  TZC_GUARD_BEGIN
  if (!d || !plan) return report(Status(TZC_E_MISSING_INPUT, "NULL argument"));
  Problem pb;
  Status st = problem_from_gemm(*d, &pb);
  if (st.ok()) st = plan_problem(pb, plan);
  return report(st);
  TZC_GUARD_END
}

int tzc_b200_set_option(const char* name, int64_t value) {
  if (!name) return report(Status(TZC_E_MISSING_INPUT, "NULL option name"));
  const std::string n(name);
  if (n == "splits") {
    if (value < 0) return report(Status(TZC_E_SHAPE, "splits must be >= 0"));
    set_forced_splits((int)value);
    return TZC_OK;
  }
  if (n == "shifted_window") {
    set_ws_enabled(value ? 1 : 0);
    return TZC_OK;
  }
  if (n == "ws_epi_groups") {
    set_ws_epi_groups((int)value);
    return TZC_OK;
  }
  if (n == "tail_split") {
    set_tail_split((int)value);
    return TZC_OK;
  }
  if (n == "split_min_kb") {
    set_split_min_kb((int)value);
    return TZC_OK;
  }
  if (n == "pingpong_kb") {
    set_pingpong_kb((int)value);
    return TZC_OK;
  }
  if (n == "ws_mt") {
    set_ws_mt((int)value);
    return TZC_OK;
  }
  if (n == "ws_1x1_k") {
    set_ws_1x1_k((int)value);
    return TZC_OK;
  }
  if (n == "ws_1x1") {
    set_ws_1x1((int)value);
    return TZC_OK;
  }
  if (n == "bn") {
    set_forced_bn((int)value);
    return TZC_OK;
  }
  if (n == "tma_store_k") {
    set_tma_store_k((int)value);
    return TZC_OK;
  }
  if (n == "pair_min_kb") {
    set_pair_min_kb((int)value);
    return TZC_OK;
  }
  if (n == "pair") {
    set_pair((int)value);
    return TZC_OK;
  }
  if (n == "st256") {
    set_st256((int)value);
    return TZC_OK;
  }
  if (n == "l2_hints") {
    set_l2_hints((int)value);
    return TZC_OK;
  }
  if (n == "tma_store") {
    set_tma_store((int)value);
    return TZC_OK;
  }
  return report(Status(TZC_E_VALIDATION, "unknown option '" + n + "'"));
}

int tzc_b200_set_splits(int32_t splits) {
  if (splits < 0) return report(Status(TZC_E_SHAPE, "splits must be >= 0"));
  set_forced_splits(splits);
  return TZC_OK;
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

int tzc_b200_device_ok(void) {
  try {
    return device_ok();
  } catch (...) {
    return 0;
  }
}

const char* tzc_b200_version(void) { return "tzc-b200 0.1.0 (sm_100a, tcgen05 kind::i8/kind::f16)"; }

}  // extern "C"
