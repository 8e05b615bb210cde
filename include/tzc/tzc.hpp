// tzc host library (B200 backend) — the reference's operator and
// instruction-registration C++ API, re-implemented for this backend.
//
// A tensor op (.tdsl text) plus an instruction description (.intr text or a
// builtin name) is the entry point, exactly as in the reference
// (/root/reference/proj/include/tzc/*.hpp).  The names, argument meaning and
// error kinds follow the reference so existing callers keep compiling; the
// tensorized body executes on sm_100a through include/tzc_b200.h instead of
// the reference VM.
//
//   reference header (proj/include/tzc/)      here
//   errors.hpp   Error + 13 kinds             same names and kinds
//   dtype.hpp    DType, wrap_int, binary16    same
//   expr.hpp     Expr, linearize, ...          same (surface subset + vector nodes)
//   compute_op.hpp / parser.hpp               ComputeOp, parse_compute, validate,
//                                              infer_types, reduce_form, print_compute
//   intrinsics.hpp                             Intrinsic, OperandRule, builtin(),
//                                              parse/load/resolve/print_intrinsic;
//                                              + tcgen05 kind::i8 / kind::f16 builtins
//   inspector.hpp                              inspect_compute, match_operation,
//                                              check_feasible, enumerate_mappings,
//                                              inspect; + fused dp groups (F6)
//   rewriter.hpp (tile_and_reorder)            tile_and_reorder -> TensorizedOp with a
//                                              device KernelPlan (tiles, TMA layouts)
//   rewriter.hpp (Schedule, lower,              same; Pad is realised in-kernel (TMA OOB)
//     inject_intrinsic) / tensor_ir.hpp        print_tensor_ir = the reference's snapshot text
//   vm.hpp (TensorValue, random_inputs,        same value types; eval_tir runs tcgen05 nests
//           compare, eval_tir)                 on the B200 (run_tensorized), nothing on a CPU VM
#ifndef TZC_B200_TZC_HPP
#define TZC_B200_TZC_HPP

#include <cstdint>
#include <functional>
#include <iosfwd>
#include <map>
#include <memory>
#include <optional>
#include <stdexcept>
#include <string>
#include <tuple>
#include <vector>

#if defined(__GNUC__)
#pragma GCC visibility push(default)
#endif

namespace tzc {

// ============================ errors =====================================
class Error : public std::runtime_error {
 public:
  Error(std::string kind, const std::string& msg) : std::runtime_error(kind + ": " + msg), kind_(std::move(kind)) {}
  const std::string& kind() const { return kind_; }

 private:
  std::string kind_;
};

#define TZC_ERROR_KIND(NAME) \
  struct NAME : Error {      \
    explicit NAME(const std::string& m) : Error(#NAME, m) {} \
  }
TZC_ERROR_KIND(SyntaxError);
TZC_ERROR_KIND(ValidationError);
TZC_ERROR_KIND(TypeError);
TZC_ERROR_KIND(RuleError);
TZC_ERROR_KIND(UnknownIntrinsic);
TZC_ERROR_KIND(ScheduleError);
TZC_ERROR_KIND(DivisibilityError);
TZC_ERROR_KIND(PadUnsupported);
TZC_ERROR_KIND(InjectError);
TZC_ERROR_KIND(ShapeError);
TZC_ERROR_KIND(MissingInput);
TZC_ERROR_KIND(NoFeasibleMapping);
TZC_ERROR_KIND(IoError);
TZC_ERROR_KIND(DeviceError);  // backend addition: CUDA / driver failure
#undef TZC_ERROR_KIND

struct InternalError : std::logic_error {
  explicit InternalError(const std::string& m) : std::logic_error("InternalError: " + m) {}
};
inline void internal_check(bool ok, const char* msg) {
  if (!ok) throw InternalError(msg);
}

// ============================ scalar types ===============================
struct DType {
  enum class Kind : uint8_t { Invalid = 0, Int, UInt, Float };
  Kind kind = Kind::Invalid;
  int bits = 0;
  int lanes = 1;
  constexpr DType() = default;
  constexpr DType(Kind k, int b, int l = 1) : kind(k), bits(b), lanes(l) {}
  bool defined() const { return kind != Kind::Invalid; }
  bool is_int() const { return kind == Kind::Int || kind == Kind::UInt; }
  bool is_signed() const { return kind == Kind::Int; }
  bool is_float() const { return kind == Kind::Float; }
  bool is_scalar() const { return lanes == 1; }
  DType scalar() const { return DType(kind, bits, 1); }
  DType with_lanes(int l) const { return DType(kind, bits, l); }
  friend bool operator==(const DType& a, const DType& b) {
    return a.kind == b.kind && a.bits == b.bits && a.lanes == b.lanes;
  }
  friend bool operator!=(const DType& a, const DType& b) { return !(a == b); }
};
inline constexpr DType kU8{DType::Kind::UInt, 8}, kI8{DType::Kind::Int, 8}, kU16{DType::Kind::UInt, 16},
    kI16{DType::Kind::Int, 16}, kU32{DType::Kind::UInt, 32}, kI32{DType::Kind::Int, 32},
    kF16{DType::Kind::Float, 16}, kF32{DType::Kind::Float, 32};

std::string dtype_name(const DType& t);
DType dtype_from_name(const std::string& name);  // SyntaxError on unknown names
int64_t wrap_int(int64_t v, const DType& t);     // two's complement at t.bits
uint16_t f64_to_f16_bits(double x);              // binary16 RNE, single rounding
double f16_bits_to_f64(uint16_t bits);
double round_f16(double x);
inline double round_f32(double x) { return static_cast<double>(static_cast<float>(x)); }

// ============================ expressions ================================
struct Expr;
using ExprPtr = std::shared_ptr<const Expr>;
struct Expr {
  enum class Kind : uint8_t { IntImm, FloatImm, Var, Load, Cast, Add, Mul, FloorDiv, FloorMod, Ramp, Broadcast, Concat };
  Kind kind;
  DType dtype;
  int64_t ival = 0;
  double fval = 0.0;
  std::string name;
  std::vector<ExprPtr> args;
  int64_t lanes_arg = 0;
};

ExprPtr int_imm(int64_t v, DType t = kI32);
ExprPtr float_imm(double v, DType t = kF32);
ExprPtr var(const std::string& name);
ExprPtr load(const std::string& tensor, std::vector<ExprPtr> indices, DType t = DType());
ExprPtr cast(DType t, ExprPtr src);
ExprPtr add(ExprPtr a, ExprPtr b);
ExprPtr mul(ExprPtr a, ExprPtr b);
ExprPtr floordiv(ExprPtr a, ExprPtr b);
ExprPtr floormod(ExprPtr a, ExprPtr b);
ExprPtr ramp(ExprPtr base, int64_t stride, int64_t lanes);
ExprPtr broadcast(ExprPtr value, int64_t lanes);
ExprPtr concat(std::vector<ExprPtr> parts);

inline bool is_const(const ExprPtr& e) { return e->kind == Expr::Kind::IntImm || e->kind == Expr::Kind::FloatImm; }
inline bool is_leaf(const ExprPtr& e) { return is_const(e) || e->kind == Expr::Kind::Load; }
int64_t lanes_of(const ExprPtr& e);

bool expr_equal(const ExprPtr& a, const ExprPtr& b, bool compare_dtype = true);
ExprPtr substitute(const ExprPtr& e, const std::map<std::string, ExprPtr>& subst);
void collect_vars(const ExprPtr& e, std::vector<std::string>* out);
bool contains_var(const ExprPtr& e, const std::string& name);

struct AffineForm {
  std::map<std::string, int64_t> coeff;
  int64_t constant = 0;
};
std::optional<AffineForm> linearize(const ExprPtr& e);
std::string expr_to_string(const ExprPtr& e);

// ============================ tensor ops =================================
enum class LoopKind : uint8_t { DataParallel, Reduction };
struct LoopVar {
  std::string name;
  int64_t extent = 0;
  LoopKind kind = LoopKind::DataParallel;
};
enum class Role : uint8_t { Input, Output };
struct TensorDecl {
  std::string name;
  std::vector<int64_t> shape;
  DType dtype;
  Role role = Role::Input;
  int64_t size() const {
    int64_t n = 1;
    for (int64_t d : shape) n *= d;
    return n;
  }
};
struct ComputeOp {
  std::vector<TensorDecl> tensors;
  std::vector<LoopVar> loops;
  std::string out;
  std::vector<ExprPtr> indices;
  ExprPtr value;
  bool update = false;
  const TensorDecl* find_tensor(const std::string& name) const;
  const LoopVar* find_loop(const std::string& name) const;
  const TensorDecl& output() const;
  std::vector<LoopVar> loops_of_kind(LoopKind k) const;
};

ComputeOp parse_compute(const std::string& text);  // validated, not typed
void validate(const ComputeOp& op);
ComputeOp infer_types(const ComputeOp& op);
struct ReduceForm {
  ExprPtr init;
  ExprPtr term;
};
ReduceForm reduce_form(const ComputeOp& op);
bool op_equal(const ComputeOp& a, const ComputeOp& b, bool compare_dtype = true);
std::string print_compute(const ComputeOp& op);

// ============================ instructions ===============================
struct OperandRule {
  enum class Kind : uint8_t { Vectorize, Broadcast, UnrollConcat, Passthrough };
  Kind kind = Kind::Passthrough;
  std::string loop;
  int64_t count = 0;
  static std::string kind_name(Kind k);
};
struct Intrinsic {
  std::string name;
  ComputeOp semantics;  // type-resolved
  std::vector<std::pair<std::string, std::vector<OperandRule>>> operand_rules;
  std::string target_mnemonic;
  bool requires_inplace_acc = false;
  const std::vector<OperandRule>* rules_for(const std::string& tensor) const;
  std::string accumulator() const;
};
void validate_intrinsic(const Intrinsic& intr);
// Builtins: the reference's vdot_16x4, vdot_4x4, wmma_16x16x16 plus the
// sm_100a tensor-core descriptions this backend executes:
//   tcgen05_i8_m128n{64,128,256}k32   d[m,n] += i32(a[m,k]) * i32(b[n,k])   u8 x s8
//   tcgen05_f16_m128n{64,128,256}k16  d[m,n] += f32(a[m,k]) * f32(b[n,k])   (K-major B)
//   tcgen05_f16_m128n{64,128,256}k16_mn                           ... b[k,n] (MN-major B)
const Intrinsic& builtin(const std::string& name);
std::vector<std::string> builtin_names();
Intrinsic parse_intrinsic(const std::string& text, const std::string& name);
Intrinsic load_intrinsic(const std::string& path);
Intrinsic resolve_intrinsic(const std::string& ref);
std::string print_intrinsic(const Intrinsic& intr);

// ============================ inspector ==================================
struct BindMap {
  std::map<std::string, ExprPtr> reg_to_op;
  std::vector<std::pair<ExprPtr, ExprPtr>> pairs;  // (instruction leaf, op leaf)
};
struct MatchResult {
  bool ok = false;
  BindMap bind;
  std::string reason;
};
MatchResult inspect_compute(const ExprPtr& instr_value, const ExprPtr& op_value);
MatchResult match_operation(const ComputeOp& op, const Intrinsic& intr);

struct LoopMapping {
  std::vector<std::pair<std::string, std::string>> f;  // op loop -> instruction loop (instruction order)
  bool needs_padding = false;
  std::map<std::string, std::vector<std::string>> broadcast_axes;
  // Backend extension: additional op loops fused, outermost
  // first, in front of f's op loop onto the same instruction loop, e.g. the
  // (n, oh) of a convolution's pixel axis fused with ow onto tcgen05's M.
  std::map<std::string, std::vector<std::string>> fused;
  std::string instr_loop_of(const std::string& op_loop) const;
  std::string op_loop_of(const std::string& instr_loop) const;
  std::string to_string() const;  // "{y->i, k->j}", fused groups as "(n,oh,ow)->m"
};
bool check_feasible(const ComputeOp& op, const Intrinsic& intr, const BindMap& bind,
                    const std::vector<std::pair<std::string, std::string>>& f,
                    std::map<std::string, std::vector<std::string>>* broadcast_out = nullptr);
std::vector<LoopMapping> enumerate_mappings(const ComputeOp& op, const Intrinsic& intr, const BindMap& bind);
// Mappings whose dp instruction loops may take fused groups of op loops (the
// product extent is what must be a multiple; tails are TMA out-of-bounds).
std::vector<LoopMapping> enumerate_group_mappings(const ComputeOp& op, const Intrinsic& intr, const BindMap& bind);
struct InspectionReport {
  MatchResult match;
  std::vector<LoopMapping> mappings;
};
InspectionReport inspect(const ComputeOp& op, const Intrinsic& intr);

// ============================ device lowering ============================
// How one op is executed by the sm_100a kernel (the analogue of the
// reference's tensorize schedule + injected call).
struct KernelPlan {
  enum class Family : uint8_t { Matmul, ConvNHWC, ConvBlocked, ConvBlocked3D };
  Family family = Family::Matmul;
  bool f16 = false;
  // geometry in the kernel's GEMM view
  int64_t n = 1, hp = 1, wp = 1, c = 0, k = 0, r = 1, s = 1, stride = 1;
  int64_t m = 0;                  // matmul rows
  bool b_kn = false;              // fp16 matmul B stored [K, N]
  int64_t w_stride_k = 0, w_stride_tap = 0;
  int64_t cb = 0, kb = 0;         // ConvBlocked: channel blocks of data / output
  int64_t out_nb = 0, out_stride_m = 0, out_stride_blk = 0;
  std::string data, weight, out;  // op tensor names bound to a, b, d
  int64_t splits = 0;             // device split-K from the schedule's split_reduction (0 = planner's choice)
  int64_t dp = 1, kd = 1, od = 1; // ConvBlocked3D: input depth, depth taps, output depth
  // the instruction's tile: M rows per MMA (256 = cta_group::2, the CTA-pair
  // kernel) and N columns per MMA, which the launch uses as its N tile
  int64_t tile_m = 128, tile_n = 0;
  std::string describe() const;
};
struct Transform;
using Schedule = std::vector<Transform>;
// ============================ schedules ==================================
// (declared ahead of TensorizedOp, which carries one)
struct Transform {
  enum class Kind : uint8_t { Pad, Split, Reorder, Fuse, Parallel, Unroll, SplitReduction, Pragma };
  Kind kind = Kind::Split;
  std::string a, b;
  std::vector<std::string> names;
  int64_t factor = 0;
  static std::string kind_name(Kind k);
};
std::string print_schedule(const Schedule& s);     // one transform per line
Schedule parse_schedule(const std::string& text);  // SyntaxError on bad lines
Schedule load_schedule(const std::string& path);   // IoError when unreadable

// The reference's pad_to_multiple (proj/include/tzc/rewriter.hpp:44-49):
// raises `loop` to the next multiple of `multiple`, growing every tensor
// dimension it indexes (zero extension).  A reduction loop may only be
// padded when a multiplicative factor of the reduction term reads a
// zero-extended index for every added iteration; otherwise PadUnsupported.
// On the device the zero extension is TMA out-of-bounds fill, not a copy.
ComputeOp pad_to_multiple(const ComputeOp& op, const std::string& loop, int64_t multiple);

// The reference's TensorizedOp (proj/include/tzc/rewriter.hpp:56-65) plus the
// device plan this backend executes.
struct TensorizedOp {
  ComputeOp op;        // possibly padded
  ComputeOp original;  // before padding (equal to op when nothing was padded)
  LoopMapping mapping;
  Schedule schedule;   // pads + (fuses) + splits + reorder + pragma
  std::vector<std::string> outer_dp, outer_red, pragma_axes;
  // Backend: the sm_100a kernel realising the pragma nest; has_plan is false
  // for instructions this backend does not execute (the CPU descriptions).
  KernelPlan plan;
  bool has_plan = false;
};
// Pure schedule construction for any instruction, as in the reference:
// DivisibilityError when a mapped extent is not a multiple of its instruction
// extent and allow_pad is false (the reference default).  For tcgen05
// instructions the device plan is derived too (InjectError when the op's
// layout has no sm_100a kernel); fused pixel groups (F6) are split with
// device-clipped tails instead of padded.
TensorizedOp tile_and_reorder(const ComputeOp& op, const Intrinsic& intr, const LoopMapping& mapping,
                              bool allow_pad = false);
// Convenience: match, pick the first device-realisable mapping, tile.
TensorizedOp tensorize(const ComputeOp& op, const Intrinsic& intr);

// ============================ schedules + tensor IR ======================
// The reference's lowering chain (proj/include/tzc/rewriter.hpp:14-116,
// proj/include/tzc/tensor_ir.hpp:13-78): a Schedule applied to an op gives
// the imperative TensorIR nest; inject_intrinsic replaces its tensorize
// pragma nest with one instruction call; eval_tir executes it — here on the
// B200 only (tcgen05 descriptions), never on a CPU interpreter.
enum class LoopAnn : uint8_t { Serial, Parallel, Unrolled, Tensorize };
std::string loop_ann_name(LoopAnn a);

struct Stmt;
using StmtPtr = std::shared_ptr<const Stmt>;
struct Stmt {
  enum class Kind : uint8_t { For, Store, Intrinsic, Seq };
  Kind kind = Kind::Seq;
  std::string var;  // For
  int64_t extent = 0;
  LoopAnn ann = LoopAnn::Serial;
  StmtPtr body;
  std::string tensor;             // Store / Intrinsic destination
  std::vector<ExprPtr> indices;   // Store
  ExprPtr value;                  // Store
  std::string intrinsic;          // Intrinsic
  ExprPtr dst_index;              // Intrinsic: lane scatter pattern
  std::vector<ExprPtr> args;      // Intrinsic: one vector operand per input register
  std::vector<StmtPtr> stmts;     // Seq
};
StmtPtr make_for(std::string var, int64_t extent, StmtPtr body, LoopAnn ann = LoopAnn::Serial);
StmtPtr make_store(std::string tensor, std::vector<ExprPtr> indices, ExprPtr value);
StmtPtr make_intrinsic(std::string name, std::string dst_tensor, ExprPtr dst_index, std::vector<ExprPtr> args);
StmtPtr make_seq(std::vector<StmtPtr> stmts);

struct TensorIR {
  std::vector<TensorDecl> tensors;
  std::vector<std::string> temps;
  std::string output;
  bool seed_output = false;
  StmtPtr root;
  std::vector<Intrinsic> intrinsics;
  // Backend extension: the op the nest was lowered from and the mapping the
  // injected call realises; eval_tir turns them into the device KernelPlan.
  std::shared_ptr<const ComputeOp> source;
  LoopMapping mapping;
  const TensorDecl* find_tensor(const std::string& name) const;
  const Intrinsic* find_intrinsic(const std::string& name) const;
};
std::string print_tensor_ir(const TensorIR& ir);  // the reference's golden-snapshot format
void visit_stmts(const StmtPtr& s, const std::function<void(const Stmt&)>& f);
int count_stmts(const StmtPtr& s, Stmt::Kind kind);

struct LinearSplit {
  ExprPtr residual;  // never null
  std::map<std::string, int64_t> coeff;
};
std::optional<LinearSplit> split_linear(const ExprPtr& e, const std::vector<std::string>& vars);

struct LowerOptions {
  bool literal_unroll = false;
  // Backend extension: a split whose factor does not divide the extent gets
  // ceil(extent / factor) outer iterations instead of a ScheduleError; the
  // device clips the tail (TMA out-of-bounds zero fill on loads, masked
  // stores).  tensorized_ir sets it for fused pixel groups (F6).
  bool clip_tails = false;
};
// Leading Pad transforms reshape the op (pad_to_multiple), the rest works on
// axes — the reference's lower (proj/src/rewriter.cpp:509-646).
TensorIR lower(const ComputeOp& op, const Schedule& schedule, const LowerOptions& opts = {});
TensorIR inject_intrinsic(const TensorIR& ir, const Intrinsic& intr, const LoopMapping& mapping);
// lower(tile_and_reorder schedule) + inject for the first device-realisable mapping.
TensorIR tensorized_ir(const ComputeOp& op, const Intrinsic& intr);

// ============================ values =====================================
struct TensorValue {
  DType dtype;
  std::vector<int64_t> shape;
  std::vector<int64_t> idata;
  std::vector<double> fdata;
  static TensorValue zeros(DType t, std::vector<int64_t> shape);
  int64_t size() const;
  bool is_float() const { return dtype.is_float(); }
};
using Inputs = std::map<std::string, TensorValue>;
TensorValue random_tensor(const TensorDecl& decl, uint64_t seed);
Inputs random_inputs(const ComputeOp& op, uint64_t seed);
struct Deviation {
  double max_rel = 0.0;
  int64_t mismatches = 0;
  bool bitexact = true;
};
Deviation compare(const TensorValue& ref, const TensorValue& got, double rtol);

// The reference's tensor container (proj/include/tzc/vm.hpp:108-116,
// proj/src/vm.cpp:686-822): "TNSR", version u8 = 1, dtype code u8
// (u8 i8 u16 i16 u32 i32 fp16 fp32 = 0..7), rank u8, little-endian u64
// extents, raw little-endian elements at the declared width.  IoError on
// malformed input.
void write_tensor(std::ostream& os, const TensorValue& v);
TensorValue read_tensor(std::istream& is);
void save_tensor(const std::string& path, const TensorValue& v);
TensorValue load_tensor(const std::string& path);
std::string tensor_to_text(const TensorValue& v, int64_t max_elems = 64);

// Zero-extends `v` into `shape` / slices the leading region back out (the
// reference's embed / slice, proj/include/tzc/vm.hpp:103-106; host helpers
// around padded pipelines).
TensorValue embed(const TensorValue& v, const std::vector<int64_t>& shape);
TensorValue slice(const TensorValue& v, const std::vector<int64_t>& shape);

// ============================ cost ledger ================================
// The reference's operation counters (proj/include/tzc/vm.hpp:62-99).  They
// are pure functions of the nest's loop extents (no data-dependent control
// flow), so both entry points compute them without evaluating any tensor
// value: measure_static from the extents, measure by walking the executed
// iteration space.  On this backend they describe the nest (work
// conservation, tuner ranking on the reference's CPU sketches); device time
// comes from CUDA events (tzc_b200_tune_*).
struct CostReport {
  int64_t scalar_mac_count = 0;  // executed scalar stores weighted by their value's Mul count
  int64_t load_count = 0;        // scalar loads + gathered vector lanes
  int64_t store_count = 0;       // scalar stores + scattered vector lanes
  std::map<std::string, int64_t> intrinsic_calls;
  int64_t intrinsic_call_count = 0;
  int64_t parallel_credit = 1;   // max parallel loop extent
  int64_t unroll_depth = 1;      // product of unrolled loop extents
  std::string to_string() const;
};
CostReport measure(const TensorIR& ir, const Inputs& inputs);
CostReport measure_static(const TensorIR& ir);
struct CostModel {
  int64_t cores = 24;
  int64_t unroll_target = 4;
};
using CostKey = std::tuple<int64_t, int64_t, int64_t>;
CostKey cost_key(const CostReport& r, const CostModel& m = {});
std::string cost_key_to_string(const CostKey& k);

// Executes a tensorized op on the B200 (the role eval_tir plays on the
// reference VM).  Inputs as for eval_tir: declared inputs plus, for
// accumulate-form ops, the output's initial image under the output's name.
// `epilogue_op` (optional) is the reference-expressible requantize / cast
// op over the output, fused into the kernel.
TensorValue run_tensorized(const TensorizedOp& t, const Inputs& inputs, const ComputeOp* epilogue_op = nullptr);

// The reference's eval_tir (proj/include/tzc/vm.hpp:50, src/vm.cpp:510-516):
// executes an injected TensorIR.  Only nests whose single call is a tcgen05
// description run (on the B200); anything else throws InjectError — there is
// no CPU interpreter behind this entry point.
TensorValue eval_tir(const TensorIR& ir, const Inputs& inputs, const ComputeOp* epilogue_op = nullptr);
// Measured-time plan search for a tensorized matmul / NHWC conv on the B200
// (tzc_b200_tune_*): one "candidate <i> <options> <us> us" line per candidate
// plan and a "best" line; the winner is installed for that device problem.
std::string tune_tensorized(const TensorizedOp& t, const Inputs& inputs, int reps = 10);
// The device plan eval_tir executes for `ir` (InjectError as above).
TensorizedOp device_plan(const TensorIR& ir);

// Packed-buffer form used by the C ABI (tzc_b200_run_op): buffers at the
// declared element width, row-major.
void run_tensorized_packed(const TensorizedOp& t, const std::map<std::string, const void*>& host_inputs,
                           void* host_out, int64_t out_bytes, const ComputeOp* epilogue_op = nullptr);

// ============================ workloads ==================================
// The reference's generators and banks (proj/include/tzc/workloads.hpp:13-64):
// surface .tdsl texts, channel-blocked data [C/cb,H,W,cb], kernel
// [K/kb,C/cb,R,S,kb,cb], output [K/kb,OH,OW,kb]; valid convolutions.
struct ConvShape {
  std::string name;
  int64_t in_c = 0;
  int64_t in_hw = 0;
  int64_t out_c = 0;
  int64_t kernel = 0;
  int64_t stride = 1;
  int64_t out_hw() const { return (in_hw - kernel) / stride + 1; }
};
struct DtypeProfile {
  DType data;
  DType weight;
  DType acc;
};
inline DtypeProfile int8_profile() { return {kU8, kI8, kI32}; }
inline DtypeProfile fp16_profile() { return {kF16, kF16, kF32}; }
std::string matmul_tdsl(int64_t m, int64_t n, int64_t k, const DtypeProfile& p = int8_profile());
std::string conv2d_tdsl(const ConvShape& c, int64_t lane_block, int64_t red_block,
                        const DtypeProfile& p = int8_profile());
std::string conv3d_tdsl(const ConvShape& c, int64_t lane_block, int64_t red_block,
                        const DtypeProfile& p = int8_profile());
// Backend addition: batched NHWC (pre-padded) conv, [K,R,S,C] weights.
std::string conv2d_nhwc_tdsl(int64_t n, int64_t hp, int64_t wp, int64_t c, int64_t k, int64_t r, int64_t s,
                             int64_t stride = 1, const DtypeProfile& p = int8_profile());
const std::vector<ConvShape>& table1_bank();
const std::vector<ConvShape>& resnet18_3d_bank();
// Backend addition: the 23 distinct ResNet-50 v1.5 convolutions (SURVEY.md
// App. A) with the pad materialised in in_hw.
const std::vector<ConvShape>& resnet50_bank();
struct BankEntry {
  ConvShape shape;
  std::string tdsl;
  bool is_3d = false;
};
// "table1" | "resnet18_3d" (| "resnet50": NHWC, batch 1); ShapeError otherwise.
std::vector<BankEntry> bank_by_name(const std::string& name);

// ============================ sketches + tuner ===========================
// The reference's search API (proj/include/tzc/rewriter.hpp:100-131,
// proj/include/tzc/tuner.hpp:12-72).  Target::Gpu runs the measured-time
// search on the B200 for tcgen05 descriptions: every candidate device plan
// (tile width, split-K = split_reduction, kernel family, tiles per unit,
// epilogue grouping, CTA pairs) is timed with CUDA events and ranked by time;
// CostKey = (median ns, 0, 0).  The CPU sketch space (threading / unrolling
// for the reference's CPU VM) is out of scope for this backend
// (SURVEY.md §2 row 7): its entry points throw InjectError.
struct CpuSketch {
  int l1 = 0;
  int64_t f1 = 1;
  int l2 = 0;
  int64_t f2 = 1;
  std::string to_string() const;
};
struct GpuSketch {
  int64_t p = 1;
  bool fuse_hw = false;
  int64_t split_k = 1;
  std::string to_string() const;
};
Schedule apply_cpu_sketch(const TensorizedOp& t, const CpuSketch& sketch);
Schedule apply_gpu_sketch(const TensorizedOp& t, const GpuSketch& sketch);
int64_t cpu_fused_parallel_extent(const TensorizedOp& t, const CpuSketch& s);
int64_t cpu_unroll_factor(const TensorizedOp& t, const CpuSketch& s);
struct CpuLimits {
  int64_t parallel_bound = 3000;
  int64_t unroll_bound = 8;
};
struct GpuLimits {
  int64_t p_max = 2;
  std::vector<int64_t> split_factors = {64};
  bool allow_fuse = true;
};
std::vector<CpuSketch> enumerate_cpu_space(const TensorizedOp& t, const CpuLimits& limits = {});
std::vector<GpuSketch> enumerate_gpu_space(const TensorizedOp& t, const GpuLimits& limits = {});
enum class Target : uint8_t { Cpu, Gpu };
struct TuneOptions {
  Target target = Target::Cpu;
  int budget = 16;
  uint64_t seed = 0;
  bool allow_pad = true;
  CpuLimits cpu_limits{};
  GpuLimits gpu_limits{};
  CostModel cost_model{};
  int64_t verify_limit = 1 << 22;
  bool force_verify = false;
  std::ostream* log = nullptr;
};
struct Candidate {
  int id = -1;
  LoopMapping mapping;
  std::string sketch;
  Schedule schedule;
  CostReport cost;
  CostKey key{};
  bool verified = false;
};
struct TuneResult {
  Candidate best;
  std::vector<Candidate> evaluated;
};
TuneResult tune(const ComputeOp& op, const Intrinsic& intr, const TuneOptions& opts = {});

}  // namespace tzc

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif

#endif
