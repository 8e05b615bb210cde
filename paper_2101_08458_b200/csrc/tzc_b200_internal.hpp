// Internal (C++) interface between the C ABI (capi/), the tzc host library
// (host/) and the CUDA kernels (kernels/).  Not installed.
#pragma once
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <string>

#include "tzc_b200.h"

namespace tzcb200 {

struct Status {
  int code = TZC_OK;
  std::string msg;
  Status() = default;
  Status(int c, std::string m) : code(c), msg(std::move(m)) {}
  bool ok() const { return code == TZC_OK; }
};

// One device problem in GEMM form (see kernels/conv_tc.cuh for the kernel).
struct Problem {
  int f16 = 0;
  int a_mode = 0;  // 0 = 2-D tiled A, 1 = im2col A
  // conv geometry (GEMM: n = 1, hp = 1, wp = M, r = s = stride = 1)
  int n = 1, hp = 1, wp = 1, c = 0, r = 1, s = 1, stride = 1, oh = 1, ow = 1, taps = 1;
  int64_t m = 0;   // GEMM rows
  int ngemm = 0;   // GEMM columns (output channels)
  // tiled A: [a_rows][a_kdim] with a_row_stride elements between rows
  int64_t a_kdim = 0, a_rows = 0, a_row_stride = 0;
  // B: element (n, tap, c) at n*w_stride_k + tap*w_stride_tap + c
  int64_t w_stride_k = 0, w_stride_tap = 0;
  int b_kn = 0;    // fp16 matmul: B stored [K, N]
  tzc_out_layout out{};
  // split-K factor requested by the op's schedule (split_reduction); 0 = the
  // process-wide setting.  A forced split runs on the general kernel.
  int forced_splits = 0;
};

Status plan_problem(const Problem& pb, tzc_plan* plan);
bool needs_k7(const Problem& pb);
Problem k7_gemm(const Problem& pb, int* kp_out);
Status run_problem(const Problem& pb, const void* a, const void* b, const void* seed, void* out,
                   const tzc_epilogue& ep, cudaStream_t stream);
void set_forced_splits(int s);
void set_ws_enabled(int on);
void set_tma_store(int on);
void set_tma_store_k(int k);
void set_l2_hints(int h);
void set_st256(int on);
void set_pair(int on);
void set_pair_min_kb(int kb);
void set_forced_bn(int bn);
void set_ws_1x1(int on);
void set_ws_1x1_k(int k);
void set_ws_mt(int mt);
void set_pingpong_kb(int kb);
void set_split_min_kb(int kb);
void set_tail_split(int on);
void set_ws_epi_groups(int g);
int device_ok();
int num_sms();

Status problem_from_conv(const tzc_conv_desc& d, Problem* pb);
Status problem_from_gemm(const tzc_gemm_desc& d, Problem* pb);

Status unblock_data(const void* src, void* dst, int c, int h, int w, int cb, int eb, cudaStream_t st);
Status unblock_kernel(const void* src, void* dst, int k, int c, int r, int s, int kb, int cb, int eb,
                      cudaStream_t st);

Status im2col_pad(const Problem& pb, const void* x, void* a, int kp, cudaStream_t st);
Status weight_pad(const Problem& pb, const void* w, void* b, int kp, cudaStream_t st);

Status s2d_stem(const Problem& pb, const void* x, const void* w, void* x4, void* w4, int hp4, int wp4, int r4, int s4,
                cudaStream_t st);

extern std::atomic<uint64_t> g_launches;
void set_last_error(const std::string& msg);

}  // namespace tzcb200
