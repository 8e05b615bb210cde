/* tzc_b200.h — C ABI of the B200 (sm_100a) backend for the UNIT/tzc
 * tensorized-instruction compiler.
 *
 * This is the drop-in boundary for the reference's hot path: executing a
 * tensorized Conv2D/Matmul body.  In the reference that is
 *   TensorValue eval_tir(const TensorIR&, const Inputs&)
 *     /root/reference/proj/include/tzc/vm.hpp:58  (impl proj/src/vm.cpp:510-516)
 * whose Intrinsic branch (proj/src/vm.cpp:343-390) gathers register images,
 * runs the instruction semantics and scatters the result.  Here one call runs
 * the whole injected nest of a tcgen05-tensorized op on the GPU.
 *
 * Two levels:
 *  (1) device level — caller-owned DEVICE buffers, stream-ordered, no
 *      allocation beyond a cached split-K workspace:
 *        tzc_b200_conv2d_i8 / _f16, tzc_b200_gemm_i8 / _f16, tzc_b200_plan_*
 *  (2) op level — the reference-facing plugin: a .tdsl op text plus an
 *      instruction name (exactly what `tzc verify op.tdsl --intrinsic X`
 *      takes, proj/src/cli.cpp:227-283) and HOST buffers in the op's declared
 *      layouts; parses/inspects/plans with this repo's tzc host library and
 *      runs level (1):   tzc_b200_run_op
 *
 * Conventions: every function returns 0 on success and a negative code on
 * failure; tzc_b200_last_error() (thread-local) holds the message.  Codes map
 * onto the reference's error taxonomy (proj/include/tzc/errors.hpp:12-40).
 * No C++ exceptions cross this boundary.  Streams are cudaStream_t passed as
 * void* (NULL = legacy default stream).
 */
#ifndef TZC_B200_H
#define TZC_B200_H

#include <stdint.h>

#if defined(__GNUC__)
#define TZC_API __attribute__((visibility("default")))
#else
#define TZC_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (errors.hpp:26-38 kinds, plus DeviceError) ------------- */
enum {
  TZC_OK = 0,
  TZC_E_SYNTAX = -1,        /* SyntaxError */
  TZC_E_VALIDATION = -2,    /* ValidationError */
  TZC_E_TYPE = -3,          /* TypeError */
  TZC_E_RULE = -4,          /* RuleError */
  TZC_E_UNKNOWN_INTR = -5,  /* UnknownIntrinsic */
  TZC_E_SCHEDULE = -6,      /* ScheduleError */
  TZC_E_DIVISIBILITY = -7,  /* DivisibilityError */
  TZC_E_PAD = -8,           /* PadUnsupported */
  TZC_E_INJECT = -9,        /* InjectError: op/layout not expressible by a kernel */
  TZC_E_SHAPE = -10,        /* ShapeError */
  TZC_E_MISSING_INPUT = -11,/* MissingInput */
  TZC_E_NO_MAPPING = -12,   /* NoFeasibleMapping */
  TZC_E_IO = -13,           /* IoError */
  TZC_E_DEVICE = -20,       /* CUDA / driver failure, or no sm_100 device */
  TZC_E_INTERNAL = -30
};

/* Element profiles of the reference workloads (proj/include/tzc/workloads.hpp:40-45). */
enum { TZC_PROFILE_U8I8 = 0, /* u8 data x i8 weight -> i32 (tcgen05 kind::i8) */
       TZC_PROFILE_F16 = 1   /* fp16 x fp16 -> fp32     (tcgen05 kind::f16) */ };

/* Fused epilogues.  The reference expresses requantize/cast as a second op
 * over the accumulator:
 *   REQUANT_I8:  Q[..] = cast<i8>(cast<fp32>(C[..]) * s)
 *                (fp32 RNE, fp32 multiply RNE, trunc toward zero with int64
 *                 saturation, wrap mod 256: proj/src/vm.cpp:79-84,136-164)
 *   CAST_F16:    H[..] = cast<fp16>(C[..])  (binary16 RNE, dtype.cpp:53-101)
 * where C = c_seed + sum (the accumulate-form "+=" op, int32 wrap-around). */
enum { TZC_EP_I32 = 0, TZC_EP_REQUANT_I8 = 1, TZC_EP_F32 = 2, TZC_EP_CAST_F16 = 3 };

typedef struct tzc_epilogue {
  int32_t kind;  /* TZC_EP_* */
  float scale;   /* s of REQUANT_I8 */
} tzc_epilogue;

/* Output (and C-seed) layout in the GEMM view (m = output pixel / matmul
 * row, n = output channel / matmul column): element (m, n) lives at
 *     (n / nb) * stride_blk + m * stride_m + (n % nb)        [elements]
 *  NHWC / row-major:                      nb = N, stride_m = N
 *  conv2d_tdsl blocked [K/kb, OH, OW, kb]: nb = kb, stride_m = kb,
 *                                          stride_blk = OH*OW*kb
 *  (proj/src/workloads.cpp:65-92).  nb must be 16 or a multiple of 32. */
typedef struct tzc_out_layout {
  int32_t nb;
  int32_t pad_;
  int64_t stride_m;
  int64_t stride_blk;
} tzc_out_layout;

/* Valid Conv2D over a spatially pre-padded NHWC input (the reference has no
 * halo semantics; ResNet pad=1 is materialised, SURVEY.md §7 hard part 3):
 *   out[n,oh,ow,k] (+)= sum_{r,s,c} x[n, oh*stride+r, ow*stride+s, c] * w[k,r,s,c]
 * with OH = (hp-r)/stride+1, OW = (wp-s)/stride+1.  Weight element (k,r,s,c)
 * lives at k*w_stride_k + (r*s_+s)*w_stride_tap + c (c contiguous), which
 * covers both [K,R,S,C] (w_stride_k = R*S*C, w_stride_tap = C) and the
 * (lane_block,red_block)=(K,C) form of conv2d_tdsl, [R,S,K,C]
 * (w_stride_k = C, w_stride_tap = K*C). */
typedef struct tzc_conv_desc {
  int32_t profile;
  int32_t n, hp, wp, c;
  int32_t k, r, s, stride;
  int32_t pad_;
  int64_t w_stride_k, w_stride_tap;
  tzc_out_layout out;
} tzc_conv_desc;

/* Matmul (matmul_tdsl, proj/src/workloads.cpp:41-63):
 *   C[x,y] (+)= sum_k A[x,k] * B(y,k)
 * A is [M,K] row-major.  b_kn = 0: B is [N,K] (the int8 profile layout);
 * b_kn = 1: B is [K,N] (the fp16 profile layout; MN-major UMMA operand). */
typedef struct tzc_gemm_desc {
  int32_t profile;
  int32_t m, n, k;
  int32_t b_kn;
  int32_t pad_;
  tzc_out_layout out;
} tzc_gemm_desc;

/* The kernel configuration chosen for a problem (the device analogue of the
 * reference's TensorizedOp/GPU sketch: tile = pragma window, stages = buffer
 * depth, splits = split_reduction; proj/include/tzc/rewriter.hpp:56-69,
 * 118-124). */
typedef struct tzc_plan {
  int32_t bm, bn, bk_bytes, stages;
  int32_t a_mode;          /* 0 = 2-D tiled TMA, 1 = TMA im2col */
  int32_t splits;          /* split-K factor (1 = none) */
  int32_t grid, smem_bytes;
  int32_t tiles_m, tiles_n;
  int64_t workspace_bytes; /* split-K partial buffer */
} tzc_plan;

/* ---- level 1: device buffers ------------------------------------------------ */
TZC_API int tzc_b200_conv2d_i8(const tzc_conv_desc* d, const uint8_t* x, const int8_t* w,
                       const int32_t* c_seed /* nullable => 0 */, void* out,
                       const tzc_epilogue* ep, void* stream);
TZC_API int tzc_b200_conv2d_f16(const tzc_conv_desc* d, const uint16_t* x, const uint16_t* w,
                        const float* c_seed, void* out, const tzc_epilogue* ep, void* stream);
TZC_API int tzc_b200_gemm_i8(const tzc_gemm_desc* d, const uint8_t* a, const int8_t* b,
                     const int32_t* c_seed, void* out, const tzc_epilogue* ep, void* stream);
TZC_API int tzc_b200_gemm_f16(const tzc_gemm_desc* d, const uint16_t* a, const uint16_t* b,
                      const float* c_seed, void* out, const tzc_epilogue* ep, void* stream);

/* The plan a launch of this descriptor would use (descriptor only: the
 * CTA-pair choice, which needs the fused requant epilogue, and the resident-B
 * ring are decided at launch; tzc_b200_last_launch reports what ran). */
TZC_API int tzc_b200_plan_conv(const tzc_conv_desc* d, tzc_plan* plan);

/* What the calling thread's most recent conv/GEMM launch actually ran (the
 * executed tile, not a plan query): kernel 0 = general (TMA tiled / im2col),
 * 1 = shifted-window, 2 = space-to-depth stem (shifted-window, pair mode),
 * 3 = CTA pair (cta_group::2, M = 256 rows per MMA), 4 = K7 GEMM (thin
 * channels), 5 = the stem with space-to-depth fused into the kernel.  Returns TZC_E_SHAPE if this thread has launched nothing. */
typedef struct tzc_launch_info {
  int32_t kernel;
  int32_t cta_group;       /* 1 or 2 */
  int32_t bm, bn, bk_bytes;
  int32_t a_mode;
  int32_t grid;
  int32_t splits;
} tzc_launch_info;
TZC_API int tzc_b200_last_launch(tzc_launch_info* info);
TZC_API int tzc_b200_plan_gemm(const tzc_gemm_desc* d, tzc_plan* plan);
/* Force a split-K factor for subsequent launches (0 = automatic). */
TZC_API int tzc_b200_set_splits(int32_t splits);
/* Process-wide tuning options (all default to the measured-best setting;
 * results never change, only the kernel plan):
 *   "splits"         force a split-K factor (0 = automatic)
 *   "split_min_kb"   automatic split-K when a grid underfills the GPU, keeping
 *                    >= this many K blocks per split (default: off)
 *   "tail_split"     split the under-filled last round of tiles (default 0)
 *   "shifted_window" weight-stationary shifted-window kernel for eligible
 *                    stride-1 convs (default 1; 0 = always TMA im2col)
 *   "ws_1x1"         force the shifted-window kernel for every 1x1 stride-1 conv
 *   "ws_1x1_k"       ... and use it for 1x1 stride-1 convs with K <= this many
 *                    bytes (default 64)
 *   "ws_mt"          force its 128-row tiles per work unit (1, 2, 4; 0 = auto)
 *   "ws_epi_groups"  1 or 2 epilogue groups in the shifted-window kernel
 *   "pingpong_kb"    ping-pong epilogue groups for tiles of <= this many K blocks
 *   "bn"             force the N tile (64, 128, 256; 0 = automatic)
 *   "tma_store"      int8 requant outputs staged in SMEM and written by TMA:
 *                    0 never (default), 1 always, 2 when the GEMM K is at
 *                    most "tma_store_k" bytes (default 64)
 *   "l2_hints"       TMA load L2 policies: bit 0 = activations evict-first
 *                    (default 1), bit 1 = weights evict-last
 *   "st256"          256-bit epilogue stores on the 2^-k requant path (1)
 *   "pair"           CTA-pair kernel (tcgen05 cta_group::2, 256-row tiles, B
 *                    split across the pair) for eligible int8 requant layers
 *                    (default 0) with >= "pair_min_kb" K blocks (default 16) */
TZC_API int tzc_b200_set_option(const char* name, int64_t value);

/* K5 layout adapter for the reference's channel-blocked conv2d_tdsl layouts
 * (cb = 4 rows are below TMA's 16-byte minimum):
 *   data[C/cb,H,W,cb] -> NHWC[1,H,W,C];  elem_bytes 1 (u8) or 2 (fp16). */
TZC_API int tzc_b200_unblock_data(const void* src, void* dst, int32_t c, int32_t h, int32_t w,
                          int32_t cb, int32_t elem_bytes, void* stream);
/*   kernel[K/kb,C/cb,R,S,kb,cb] -> [K,R,S,C]. */
TZC_API int tzc_b200_unblock_kernel(const void* src, void* dst, int32_t k, int32_t c, int32_t r,
                            int32_t s, int32_t kb, int32_t cb, int32_t elem_bytes, void* stream);

/* Measured-time tuner (the device analogue of tzc::tune, proj/include/tzc/
 * tuner.hpp:71-72 / proj/src/tuner.cpp:111-274, which ranks candidates by a
 * VM cost model): times each candidate kernel plan of this problem (tile
 * width, split-K, kernel family, tiles per unit, epilogue grouping, store
 * path, CTA pairs) with CUDA events over `reps` launches on `stream` (L2-warm,
 * the caller's buffers; results never change between plans), writes one
 * "candidate <i> <options> <us> us" line per candidate plus a "best" line into
 * `log`, and returns the winning index (0 = the default plan; a non-default
 * plan must be >= 1% faster).  With apply != 0 the winner is installed for
 * every later launch of an identical descriptor (also inside CUDA graphs
 * captured afterwards).  The stream must not be capturing. */
TZC_API int tzc_b200_tune_conv(const tzc_conv_desc* d, const void* x, const void* w, const void* c_seed, void* out,
                               const tzc_epilogue* ep, int32_t reps, int32_t apply, char* log, int64_t loglen,
                               void* stream);
TZC_API int tzc_b200_tune_gemm(const tzc_gemm_desc* d, const void* a, const void* b, const void* c_seed, void* out,
                               const tzc_epilogue* ep, int32_t reps, int32_t apply, char* log, int64_t loglen,
                               void* stream);
/* Drops every installed per-problem plan. */
TZC_API int tzc_b200_clear_tuning(void);
/* Installs ("name=value;...") or clears ("" / NULL) the plan options for every
 * launch of this exact descriptor — how a suite-level search (bench.py
 * --tune 2) applies its per-layer choices. */
TZC_API int tzc_b200_set_problem_options_conv(const tzc_conv_desc* d, const char* spec);
TZC_API int tzc_b200_set_problem_options_gemm(const tzc_gemm_desc* d, const char* spec);
/* The plan cache on disk: writes every installed per-descriptor plan (tuned or
 * set) to `path`, one line each, or installs the plans a saved file holds
 * (all lines are validated before any is installed).  `count` (nullable)
 * receives the number of plans.  A process started with
 * TZC_B200_PLAN_CACHE=<path> loads that file before its first launch. */
TZC_API int tzc_b200_save_tuning(const char* path, int32_t* count);
TZC_API int tzc_b200_load_tuning(const char* path, int32_t* count);
/* The candidate option specs tzc_b200_tune_* times, one per line (line 0 = default). */
TZC_API int tzc_b200_tune_candidates(char* buf, int64_t buflen);

/* ---- level 2: op text + host buffers (reference-facing plugin) -------------- */
/* Runs `op_tdsl` tensorized with `intrinsic` (a builtin name such as
 * "tcgen05_i8_m128n256k32" or a .intr path) on the GPU.  Inputs are HOST
 * buffers packed at their declared width in declaration order of `names`;
 * for accumulate-form ops the output's initial image is passed under the
 * output's name (as eval_tir expects, proj/src/vm.cpp:414-440).  If
 * `requant_tdsl` is non-NULL it must be the reference-expressible epilogue op
 * over the output (Q = cast<i8>(cast<fp32>(C) * s) or H = cast<fp16>(C)); it
 * is fused and `host_out` receives its result instead of C. */
TZC_API int tzc_b200_run_op(const char* op_tdsl, const char* intrinsic, const char* requant_tdsl,
                    int32_t n_inputs, const char* const* names, const void* const* host_inputs,
                    void* host_out, int64_t out_bytes);

/* The reference's lowering chain, `lower` -> `inject_intrinsic` -> `eval_tir`
 * (proj/include/tzc/rewriter.hpp:85-95, vm.hpp:50; driven the same way by
 * `tzc verify`, proj/src/cli.cpp:227-283).  `schedule` is schedule text
 * (proj/src/rewriter.cpp:30-131 grammar) or NULL for tile_and_reorder's
 * schedule of the first device-realisable mapping.  The nest must hold one
 * tcgen05 call; other instructions return TZC_E_INJECT (no CPU VM).  Buffers
 * as for tzc_b200_run_op. */
TZC_API int tzc_b200_eval_tir(const char* op_tdsl, const char* schedule, const char* intrinsic,
                              const char* requant_tdsl, int32_t n_inputs, const char* const* names,
                              const void* const* host_inputs, void* host_out, int64_t out_bytes);

/* ---- host-library introspection (op text in, text out; no GPU needed) --------- */
/* print_tensor_ir(lower(op, schedule)), injected with `intrinsic` when it is
 * non-NULL (schedule NULL: the tensorized IR of the first device mapping):
 * the reference's golden-snapshot text (proj/src/tensor_ir.cpp print format). */
TZC_API int tzc_b200_lower(const char* op_tdsl, const char* schedule, const char* intrinsic, char* buf, int64_t buflen);
/* parse_compute + infer_types + print_compute (proj/src/compute_op.cpp:285-313). */
TZC_API int tzc_b200_parse(const char* op_tdsl, char* buf, int64_t buflen);
/* inspect(): one "<mapping>" line per feasible mapping, in the reference's
 * order (proj/src/inspector.cpp:178-216); grouped != 0 adds the fused
 * data-parallel groups this backend maps onto tcgen05's M / N. */
TZC_API int tzc_b200_inspect(const char* op_tdsl, const char* intrinsic, int32_t grouped, char* buf, int64_t buflen);
/* tensorize(): chosen mapping, reference schedule text and the kernel plan. */
TZC_API int tzc_b200_describe(const char* op_tdsl, const char* intrinsic, char* buf, int64_t buflen);
/* The reference's TNSR tensor container (proj/src/vm.cpp:686-822):
 * tensor_to_text(load_tensor(path), max_elems), and load + save (a format check). */
TZC_API int tzc_b200_tensor_text(const char* path, int64_t max_elems, char* buf, int64_t buflen);
TZC_API int tzc_b200_tensor_roundtrip(const char* src_path, const char* dst_path);
/* builtin_names(), one per line. */
TZC_API int tzc_b200_builtins(char* buf, int64_t buflen);
/* print_intrinsic(resolve_intrinsic(ref)): the .intr text (proj/src/intrinsics.cpp:298-314). */
TZC_API int tzc_b200_print_intrinsic(const char* intrinsic, char* buf, int64_t buflen);

/* ---- misc --------------------------------------------------------------------- */
TZC_API const char* tzc_b200_last_error(void);
/* Number of kernels this library has launched since load (all devices). */
TZC_API uint64_t tzc_b200_launch_count(void);
/* 1 if a device with compute capability 10.0 is present and usable. */
TZC_API int tzc_b200_device_ok(void);
TZC_API const char* tzc_b200_version(void);

#ifdef __cplusplus
}
#endif
#endif /* TZC_B200_H */
