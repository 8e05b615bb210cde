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
  std::string describe() const;
};
struct TensorizedOp {
  ComputeOp op;
  LoopMapping mapping;
  std::vector<std::string> schedule;  // split / reorder / pragma lines (reference schedule text)
  std::vector<std::string> outer_dp, outer_red, pragma_axes;
  KernelPlan plan;
};
// Throws DivisibilityError only when padding is not allowed and the device
// cannot cover a tail; InjectError when the op's layout has no kernel.
TensorizedOp tile_and_reorder(const ComputeOp& op, const Intrinsic& intr, const LoopMapping& mapping,
                              bool allow_pad = true);
// Convenience: match, pick the first device-realisable mapping, tile.
TensorizedOp tensorize(const ComputeOp& op, const Intrinsic& intr);

// ============================ schedules + tensor IR ======================
// The reference's lowering chain (proj/include/tzc/rewriter.hpp:14-116,
// proj/include/tzc/tensor_ir.hpp:13-78): a Schedule applied to an op gives
// the imperative TensorIR nest; inject_intrinsic replaces its tensorize
// pragma nest with one instruction call; eval_tir executes it — here on the
// B200 only (tcgen05 descriptions), never on a CPU interpreter.
struct Transform {
  enum class Kind : uint8_t { Pad, Split, Reorder, Fuse, Parallel, Unroll, SplitReduction, Pragma };
  Kind kind = Kind::Split;
  std::string a, b;
  std::vector<std::string> names;
  int64_t factor = 0;
  static std::string kind_name(Kind k);
};
using Schedule = std::vector<Transform>;
std::string print_schedule(const Schedule& s);     // one transform per line
Schedule parse_schedule(const std::string& text);  // SyntaxError on bad lines
Schedule load_schedule(const std::string& path);   // IoError when unreadable

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
// Pad transforms throw PadUnsupported: this backend realises padding with
// TMA out-of-bounds zero fill inside the kernel (tile_and_reorder's plan).
TensorIR lower(const ComputeOp& op, const Schedule& schedule, const LowerOptions& opts = {});
TensorIR lower(const ComputeOp& op, const std::vector<std::string>& schedule_lines, const LowerOptions& opts = {});
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

}  // namespace tzc

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif

#endif
