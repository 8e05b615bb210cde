// Internal (C++) interface between the C ABI (capi/), the tzc host library
// (host/) and the CUDA kernels (kernels/).  Not installed.
#pragma once
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <string>
#include <utility>
#include <vector>

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

// Plan knobs, named as tzc_b200_set_option names them.  Every launch plans
// from one snapshot (the process defaults plus the per-descriptor overrides
// the tuner installs), taken once per call and passed down by value, so a
// concurrent set_option never changes a plan half-way through a call.
// Options choose the kernel plan only, never the results.
struct Options {
  int splits = 0;               // forced split-K factor (0 = automatic)
  int shifted_window = 1;       // weight-stationary kernel for eligible stride-1 convs
  int ws_epi_groups = 0;        // shifted window: 1 or 2 (ping-pong) epilogue groups; 0 = by shape (2 for 3x3)
  int tail_split = 0;           // split the under-filled last round of tiles along K
  int split_min_kb = 0;         // automatic split-K keeps >= this many K blocks per split (0: off)
  int splitk_inkernel = 1;      // split-K partials combined inside the kernel (last-arriver fix-up)
  // general kernel: ping-pong epilogue groups (2 x 8 warps on alternate
  // accumulators) for tiles of up to this many K blocks.  Off by default since
  // the requant fast path: one 16-warp group is faster on every thin-K layer
  // (c3_1x1_128_512 34.8 -> 31.9 us) and the suite +1.1-1.3 % on one box.
  int pingpong_kb = 0;
  int ws_mt = 0;                // shifted window: force 1/2/4 tiles per work unit (0 = automatic)
  int ws_1x1_k = 64;            // shifted window for 1x1 convs with K <= this many bytes
  int ws_1x1 = 0;               // ... for every 1x1 stride-1 conv
  int bn = 0;                   // force the N tile (0 = automatic)
  int tma_store_k = 64;         // tma_store == 2: TMA-store epilogue for GEMM K <= this many bytes
  // CTA-pair (cta_group::2) kernel for eligible int8 requant layers with >=
  // pair_min_kb K blocks and N tiles >= pair_bn: each CTA loads half of B, so
  // operand bytes per MMA drop 12 -> 8 KB at BN = 256 (the general kernel is
  // bound by the ~60 B/clk/SM L2->SMEM operand stream; tools/tma_probe.cu).
  // Measured with two producer warps: 4-9% faster for BN = 256 layers with
  // >= 8 K blocks, slower for BN = 128 and for 4-block layers.
  int pair_min_kb = 8;
  int pair = 1;
  int pair_bn = 256;
  // ... and only when the pair tiles fill >= this many rounds of SM pairs: with
  // fewer (batch 32) a cluster's two-SM footprint backfills the SMs other graph
  // branches leave idle worse (batch 32: 682-690 TOPS without pairs, 655-677 with)
  int pair_min_round = 1;
  int l2_a_max_out_mb = 64;     // general kernel: A evict-first hint only for outputs <= this many MB (0: always)
  int s2d_one = 1;              // int8 C=3 stem: S2D rows + weight rearrangement in one launch
  int producers = 2;            // TMA producer warps of the general / pair kernels (1 or 2)
  int st256 = 1;                // 256-bit epilogue stores where aligned
  int l2_hints = 1;             // 1: A loads evict-first; 2: B loads evict-last
  int tma_store = 0;            // int8 TMA-store epilogue: 0 never, 1 always, 2 by K
  // general kernel: keep the CTA's whole B tile in SMEM when it fits: 0 never,
  // 1 always, 2 for 1x1 layers (c3_1x1s2_256_512 38.2 -> 35.9 us, c3_1x1_256_128
  // 55.4 -> 53.8; 3x3 im2col layers lose ring depth: c3_3x3s2_128 34.8 -> 35.9)
  int b_res = 2;
  int stem_fused = 0;           // C = 3 stride-2 int8 stem: space-to-depth fused into the kernel (stem_ws.cuh;
                                // correct, but slower than the separate S2D pass: DESIGN.md §8 finding 10)
};
// Validates and applies one named option; false (with *err) for an unknown
// name or an illegal value.
bool apply_option(Options* o, const std::string& name, int64_t value, std::string* err);
const char* const* option_names();  // null-terminated
// Snapshot of the process defaults (tzc_b200_set_option) plus the overrides
// installed for `key` (a descriptor's bytes; "" = none).
Options options_for(const std::string& key);
Status parse_option_spec(const std::string& spec, Options* o, std::vector<std::pair<std::string, int64_t>>* items);
Status set_default_option(const std::string& name, int64_t value);
Status set_problem_options(const std::string& key, const std::string& spec);
// the plan cache file (one line per installed descriptor)
Status save_problem_options(const std::string& path, int* count);
Status load_problem_options(const std::string& path, int* count);
void clear_problem_options();

Status plan_problem(const Problem& pb, const Options& o, tzc_plan* plan);
bool needs_k7(const Problem& pb);
Problem k7_gemm(const Problem& pb, int* kp_out);
Status run_problem(const Problem& pb, const Options& o, const void* a, const void* b, const void* seed, void* out,
                   const tzc_epilogue& ep, cudaStream_t stream);
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
                cudaStream_t st, bool one_launch = true);

extern std::atomic<uint64_t> g_launches;
// the calling thread's most recent launch (tzc_b200_last_launch)
bool last_launch(tzc_launch_info* out);
void set_last_error(const std::string& msg);

}  // namespace tzcb200
