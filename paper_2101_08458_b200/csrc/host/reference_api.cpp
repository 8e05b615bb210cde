// tzc host library, part 5: the rest of the reference's public C++ API that
// a drop-in caller (the reference's own tests/acceptance.cpp) links against:
//
//   pad_to_multiple            proj/include/tzc/rewriter.hpp:44-49
//   embed / slice              proj/include/tzc/vm.hpp:103-106
//   CostReport, measure(_static), cost_key      proj/include/tzc/vm.hpp:62-99
//   workload generators + banks                 proj/include/tzc/workloads.hpp:13-64
//   sketches + tune                             proj/include/tzc/rewriter.hpp:100-131,
//                                               proj/include/tzc/tuner.hpp:12-72
//
// Everything here is host-side analysis of ops and nests; nothing evaluates
// tensor values on the CPU.  Semantics are restated from the reference's
// headers / SPEC.md and pinned by tests/test_reference_api.py (against the
// reference itself, oracle/_ref) and tests/cpp/acceptance (the reference's
// acceptance.cpp compiled against this library).
#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <functional>
#include <ostream>
#include <set>
#include <sstream>

#include "tzc/tzc.hpp"

namespace tzc {

// ============================ padding ====================================
namespace {

ExprPtr without_casts(ExprPtr e) {
  while (e->kind == Expr::Kind::Cast) e = e->args[0];
  return e;
}

// Operands of a product chain (looking through casts): a*b*c -> {a, b, c}.
void product_operands(const ExprPtr& e, std::vector<ExprPtr>* out) {
  const ExprPtr x = without_casts(e);
  if (x->kind != Expr::Kind::Mul) {
    out->push_back(x);
    return;
  }
  product_operands(x->args[0], out);
  product_operands(x->args[1], out);
}

void all_loads(const ExprPtr& e, std::vector<ExprPtr>* out) {
  if (e->kind == Expr::Kind::Load) out->push_back(e);
  for (const auto& a : e->args) all_loads(a, out);
}

// Does this product operand read only zero-extension for every iteration
// loop >= old_extent?  True when one of its index dimensions is an affine
// form with non-negative coefficients and constant whose smallest value at
// loop = old_extent (every other loop at 0) is already past the dimension.
bool reads_extension(const ComputeOp& op, const ExprPtr& f, const std::string& loop, int64_t old_extent) {
  if (f->kind != Expr::Kind::Load || f->name == op.out) return false;
  const TensorDecl* td = op.find_tensor(f->name);
  if (!td) return false;
  for (size_t d = 0; d < f->args.size() && d < td->shape.size(); ++d) {
    const auto form = linearize(f->args[d]);
    if (!form) continue;
    auto c = form->coeff.find(loop);
    if (c == form->coeff.end()) continue;
    bool monotone = form->constant >= 0;
    for (const auto& kv : form->coeff) monotone = monotone && kv.second >= 0;
    if (monotone && c->second * old_extent + form->constant >= td->shape[d]) return true;
  }
  return false;
}

}  // namespace

ComputeOp pad_to_multiple(const ComputeOp& op, const std::string& loop, int64_t multiple) {
  const LoopVar* lv = op.find_loop(loop);
  if (!lv) throw ScheduleError("pad: the op has no loop '" + loop + "'");
  if (multiple < 1) throw ScheduleError("pad: the multiple must be >= 1 (got " + std::to_string(multiple) + ")");
  const int64_t from = lv->extent, to = (from + multiple - 1) / multiple * multiple;
  if (to == from) return op;
  if (lv->kind == LoopKind::Reduction) {
    // the added iterations must add exact zeros to every output
    const ReduceForm rf = reduce_form(op);
    if (!rf.term) throw InternalError("pad: reduction loop without a reduction term");
    std::vector<ExprPtr> operands;
    product_operands(rf.term, &operands);
    const bool zero = std::any_of(operands.begin(), operands.end(),
                                  [&](const ExprPtr& f) { return reads_extension(op, f, loop, from); });
    if (!zero)
      throw PadUnsupported("pad: the extra iterations of reduction loop '" + loop +
                           "' would not add zeros (no product operand reads only the zero extension)");
  }
  ComputeOp out = op;
  for (auto& l : out.loops)
    if (l.name == loop) l.extent = to;
  // grow every dimension an access of the loop reaches, so all accesses stay
  // in bounds (the growth is the zero extension)
  std::vector<ExprPtr> accesses;
  all_loads(out.value, &accesses);
  accesses.push_back(load(out.out, out.indices));
  for (const auto& acc : accesses) {
    TensorDecl* td = nullptr;
    for (auto& t : out.tensors)
      if (t.name == acc->name) td = &t;
    if (!td) throw InternalError("pad: access to an undeclared tensor");
    for (size_t d = 0; d < acc->args.size(); ++d) {
      if (!contains_var(acc->args[d], loop)) continue;
      const auto form = linearize(acc->args[d]);
      if (!form) throw PadUnsupported("pad: loop '" + loop + "' reaches a non-affine index");
      if (form->constant < 0) throw PadUnsupported("pad: loop '" + loop + "' reaches an index with a negative offset");
      int64_t top = form->constant;
      for (const auto& [v, c] : form->coeff) {
        if (c < 0) throw PadUnsupported("pad: loop '" + loop + "' reaches an index with a negative stride");
        const LoopVar* x = out.find_loop(v);
        if (!x) throw InternalError("pad: index over an unknown loop");
        top += c * (x->extent - 1);
      }
      td->shape[d] = std::max(td->shape[d], top + 1);
    }
  }
  return out;
}

// ============================ embed / slice ==============================
namespace {
// Copies the common leading box of src into dst (both row-major).
void copy_box(const TensorValue& src, TensorValue* dst) {
  const size_t rank = src.shape.size();
  if (dst->shape.size() != rank) throw ShapeError("embed/slice: rank mismatch");
  std::vector<int64_t> box(rank), ss(rank, 1), ds(rank, 1);
  for (size_t d = 0; d < rank; ++d) box[d] = std::min(src.shape[d], dst->shape[d]);
  for (size_t d = rank; d-- > 1;) {
    ss[d - 1] = ss[d] * src.shape[d];
    ds[d - 1] = ds[d] * dst->shape[d];
  }
  int64_t n = 1;
  for (int64_t b : box) n *= b;
  std::vector<int64_t> at(rank, 0);
  for (int64_t k = 0; k < n; ++k) {
    int64_t so = 0, dof = 0;
    for (size_t d = 0; d < rank; ++d) so += at[d] * ss[d], dof += at[d] * ds[d];
    if (src.is_float()) dst->fdata[dof] = src.fdata[so];
    else dst->idata[dof] = src.idata[so];
    for (size_t d = rank; d-- > 0;) {
      if (++at[d] < box[d]) break;
      at[d] = 0;
    }
  }
}
}  // namespace

TensorValue embed(const TensorValue& v, const std::vector<int64_t>& shape) {
  for (size_t d = 0; d < shape.size() && d < v.shape.size(); ++d)
    if (shape[d] < v.shape[d]) throw ShapeError("embed: target extent smaller than the tensor's");
  TensorValue out = TensorValue::zeros(v.dtype, shape);
  copy_box(v, &out);
  return out;
}

TensorValue slice(const TensorValue& v, const std::vector<int64_t>& shape) {
  for (size_t d = 0; d < shape.size() && d < v.shape.size(); ++d)
    if (shape[d] > v.shape[d]) throw ShapeError("slice: target extent larger than the tensor's");
  TensorValue out = TensorValue::zeros(v.dtype, shape);
  copy_box(v, &out);
  return out;
}

// ============================ cost ledger ================================
std::string CostReport::to_string() const {
  std::ostringstream o;
  o << "macs=" << scalar_mac_count << " loads=" << load_count << " stores=" << store_count
    << " calls=" << intrinsic_call_count;
  for (const auto& [n, c] : intrinsic_calls) o << " " << n << "=" << c;
  o << " parallel=" << parallel_credit << " unroll=" << unroll_depth;
  return o.str();
}

namespace {

// Per-execution weights of one statement: value multiplies (not inside
// addresses) and loaded lanes (a vector load counts its lanes).
struct Weights {
  int64_t muls = 0, loads = 0;
};
void weigh(const ExprPtr& e, bool in_address, Weights* w) {
  if (e->kind == Expr::Kind::Load) {
    w->loads += lanes_of(e);
    for (const auto& a : e->args) weigh(a, true, w);
    return;
  }
  if (e->kind == Expr::Kind::Mul && !in_address) ++w->muls;
  for (const auto& a : e->args) weigh(a, in_address, w);
}

const Intrinsic& called(const TensorIR& ir, const std::string& name) {
  if (const Intrinsic* i = ir.find_intrinsic(name)) return *i;
  return builtin(name);
}

// `times` executions of statement s (every enclosing trip count multiplied in).
void tally(const TensorIR& ir, const StmtPtr& s, int64_t times, CostReport* c, std::map<std::string, int64_t>* unrolled) {
  switch (s->kind) {
    case Stmt::Kind::Seq:
      for (const auto& x : s->stmts) tally(ir, x, times, c, unrolled);
      return;
    case Stmt::Kind::For:
      if (s->ann == LoopAnn::Parallel) c->parallel_credit = std::max(c->parallel_credit, s->extent);
      if (s->ann == LoopAnn::Unrolled) (*unrolled)[s->var] = s->extent;
      tally(ir, s->body, times * s->extent, c, unrolled);
      return;
    case Stmt::Kind::Store: {
      Weights w;
      for (const auto& i : s->indices) weigh(i, true, &w);
      weigh(s->value, false, &w);
      c->scalar_mac_count += times * w.muls;
      c->load_count += times * w.loads;
      c->store_count += times;
      return;
    }
    case Stmt::Kind::Intrinsic: {
      const Intrinsic& in = called(ir, s->intrinsic);
      Weights w;
      weigh(s->dst_index, true, &w);
      for (const auto& a : s->args) weigh(a, true, &w);
      const int64_t lanes = in.semantics.output().size();
      if (in.semantics.update) w.loads += lanes;  // the in-place accumulator is read
      c->scalar_mac_count += times * w.muls;
      c->load_count += times * w.loads;
      c->store_count += times * lanes;
      c->intrinsic_calls[s->intrinsic] += times;
      c->intrinsic_call_count += times;
      return;
    }
  }
}

void finish(CostReport* c, const std::map<std::string, int64_t>& unrolled) {
  for (const auto& kv : unrolled) c->unroll_depth *= kv.second;
}

// Counts by walking the iteration space: every loop iterates, every statement
// adds its weights once per execution.  No value is computed.
void walk(const TensorIR& ir, const StmtPtr& s, CostReport* c, std::map<std::string, int64_t>* unrolled) {
  switch (s->kind) {
    case Stmt::Kind::Seq:
      for (const auto& x : s->stmts) walk(ir, x, c, unrolled);
      return;
    case Stmt::Kind::For:
      if (s->ann == LoopAnn::Parallel) c->parallel_credit = std::max(c->parallel_credit, s->extent);
      if (s->ann == LoopAnn::Unrolled) (*unrolled)[s->var] = s->extent;
      for (int64_t it = 0; it < s->extent; ++it) walk(ir, s->body, c, unrolled);
      return;
    default:
      tally(ir, s, 1, c, unrolled);
  }
}

}  // namespace

CostReport measure_static(const TensorIR& ir) {
  CostReport c;
  std::map<std::string, int64_t> unrolled;
  tally(ir, ir.root, 1, &c, &unrolled);
  finish(&c, unrolled);
  return c;
}

CostReport measure(const TensorIR& ir, const Inputs& inputs) {
  // the reference binds the buffers first: the same missing-input contract
  for (const auto& t : ir.tensors)
    if ((t.role == Role::Input || (t.name == ir.output && ir.seed_output)) && !inputs.count(t.name))
      throw MissingInput("measure: no input for tensor '" + t.name + "'");
  CostReport c;
  std::map<std::string, int64_t> unrolled;
  walk(ir, ir.root, &c, &unrolled);
  finish(&c, unrolled);
  return c;
}

CostKey cost_key(const CostReport& r, const CostModel& m) {
  const int64_t issued = r.intrinsic_call_count + r.scalar_mac_count;
  const int64_t credit = std::min(r.parallel_credit, m.cores);
  const int64_t off_target = r.unroll_depth > m.unroll_target ? r.unroll_depth - m.unroll_target
                                                              : m.unroll_target - r.unroll_depth;
  return {issued, -credit, off_target};
}

std::string cost_key_to_string(const CostKey& k) {
  return "(" + std::to_string(std::get<0>(k)) + ", " + std::to_string(std::get<1>(k)) + ", " +
         std::to_string(std::get<2>(k)) + ")";
}

// ============================ workloads ==================================
namespace {

std::string dims(const std::vector<int64_t>& v) {
  std::string s = "[";
  for (size_t i = 0; i < v.size(); ++i) s += (i ? ", " : "") + std::to_string(v[i]);
  return s + "]";
}

// "o + i" or "o * st + i" (a strided window position)
std::string window(const std::string& o, int64_t st, const std::string& i) {
  return st == 1 ? o + " + " + i : o + " * " + std::to_string(st) + " + " + i;
}

void need_blocks(const ConvShape& c, int64_t lb, int64_t rb) {
  if (lb < 1 || rb < 1 || c.in_c % rb || c.out_c % lb)
    throw ShapeError("conv '" + c.name + "': channels " + std::to_string(c.in_c) + " -> " + std::to_string(c.out_c) +
                     " do not divide into blocks of " + std::to_string(rb) + " / " + std::to_string(lb));
}

}  // namespace

std::string matmul_tdsl(int64_t m, int64_t n, int64_t k, const DtypeProfile& p) {
  // integer profile: B stored [N, K] (the dot-product instructions read it
  // k-contiguous); float profile: B stored [K, N] (the tensor-core layout)
  const bool fl = p.data.is_float();
  const std::string acc = dtype_name(p.acc);
  std::ostringstream o;
  o << "tensor A : " << dtype_name(p.data) << " " << dims({m, k}) << " input\n"
    << "tensor B : " << dtype_name(p.weight) << " " << (fl ? dims({k, n}) : dims({n, k})) << " input\n"
    << "tensor C : " << acc << " " << dims({m, n}) << " output\n"
    << "loop x : dp " << m << "\nloop y : dp " << n << "\nloop k : red " << k << "\n"
    << "C[x, y] += cast<" << acc << ">(A[x, k]) * cast<" << acc << ">(" << (fl ? "B[k, y]" : "B[y, k]") << ")\n";
  return o.str();
}

std::string conv2d_tdsl(const ConvShape& c, int64_t lb, int64_t rb, const DtypeProfile& p) {
  need_blocks(c, lb, rb);
  const int64_t co = c.in_c / rb, ko = c.out_c / lb, o = c.out_hw();
  const std::string acc = dtype_name(p.acc);
  std::ostringstream s;
  s << "tensor data : " << dtype_name(p.data) << " " << dims({co, c.in_hw, c.in_hw, rb}) << " input\n"
    << "tensor kernel : " << dtype_name(p.weight) << " " << dims({ko, co, c.kernel, c.kernel, lb, rb}) << " input\n"
    << "tensor out : " << acc << " " << dims({ko, o, o, lb}) << " output\n"
    << "loop ko : dp " << ko << "\nloop oh : dp " << o << "\nloop ow : dp " << o << "\nloop ki : dp " << lb << "\n"
    << "loop co : red " << co << "\nloop r : red " << c.kernel << "\nloop s : red " << c.kernel
    << "\nloop ci : red " << rb << "\n"
    << "out[ko, oh, ow, ki] += cast<" << acc << ">(data[co, " << window("oh", c.stride, "r") << ", "
    << window("ow", c.stride, "s") << ", ci]) * cast<" << acc << ">(kernel[ko, co, r, s, ki, ci])\n";
  return s.str();
}

std::string conv3d_tdsl(const ConvShape& c, int64_t lb, int64_t rb, const DtypeProfile& p) {
  need_blocks(c, lb, rb);
  const int64_t co = c.in_c / rb, ko = c.out_c / lb, o = c.out_hw(), kk = c.kernel;
  const std::string acc = dtype_name(p.acc);
  std::ostringstream s;
  s << "tensor data : " << dtype_name(p.data) << " " << dims({co, c.in_hw, c.in_hw, c.in_hw, rb}) << " input\n"
    << "tensor kernel : " << dtype_name(p.weight) << " " << dims({ko, co, kk, kk, kk, lb, rb}) << " input\n"
    << "tensor out : " << acc << " " << dims({ko, o, o, o, lb}) << " output\n"
    << "loop ko : dp " << ko << "\nloop od : dp " << o << "\nloop oh : dp " << o << "\nloop ow : dp " << o
    << "\nloop ki : dp " << lb << "\n"
    << "loop co : red " << co << "\nloop rd : red " << kk << "\nloop rh : red " << kk << "\nloop rw : red " << kk
    << "\nloop ci : red " << rb << "\n"
    << "out[ko, od, oh, ow, ki] += cast<" << acc << ">(data[co, " << window("od", c.stride, "rd") << ", "
    << window("oh", c.stride, "rh") << ", " << window("ow", c.stride, "rw") << ", ci]) * cast<" << acc
    << ">(kernel[ko, co, rd, rh, rw, ki, ci])\n";
  return s.str();
}

std::string conv2d_nhwc_tdsl(int64_t n, int64_t hp, int64_t wp, int64_t c, int64_t k, int64_t r, int64_t s,
                             int64_t st, const DtypeProfile& p) {
  const int64_t oh = (hp - r) / st + 1, ow = (wp - s) / st + 1;
  const std::string acc = dtype_name(p.acc);
  std::ostringstream o;
  o << "tensor data : " << dtype_name(p.data) << " " << dims({n, hp, wp, c}) << " input\n"
    << "tensor kernel : " << dtype_name(p.weight) << " " << dims({k, r, s, c}) << " input\n"
    << "tensor out : " << acc << " " << dims({n, oh, ow, k}) << " output\n"
    << "loop n : dp " << n << "\nloop oh : dp " << oh << "\nloop ow : dp " << ow << "\nloop k : dp " << k << "\n"
    << "loop r : red " << r << "\nloop s : red " << s << "\nloop c : red " << c << "\n"
    << "out[n, oh, ow, k] += cast<" << acc << ">(data[n, " << window("oh", st, "r") << ", " << window("ow", st, "s")
    << ", c]) * cast<" << acc << ">(kernel[k, r, s, c])\n";
  return o.str();
}

const std::vector<ConvShape>& table1_bank() {
  // PAPER.md Table 1 (the paper's conv workloads): name, in_c, in_hw, out_c, kernel, stride
  static const std::vector<ConvShape> bank = {
      {"conv01", 288, 35, 384, 3, 2}, {"conv02", 160, 9, 224, 3, 1},   {"conv03", 1056, 7, 192, 1, 1},
      {"conv04", 80, 73, 192, 3, 1},  {"conv05", 128, 16, 128, 3, 1},  {"conv06", 192, 16, 192, 3, 1},
      {"conv07", 256, 16, 256, 3, 1}, {"conv08", 1024, 14, 512, 1, 1}, {"conv09", 128, 16, 160, 3, 1},
      {"conv10", 576, 14, 192, 1, 1}, {"conv11", 96, 16, 128, 3, 1},   {"conv12", 1024, 14, 256, 1, 1},
      {"conv13", 576, 14, 128, 1, 1}, {"conv14", 64, 29, 96, 3, 1},    {"conv15", 64, 56, 128, 1, 2},
      {"conv16", 608, 14, 192, 1, 1}};
  return bank;
}

const std::vector<ConvShape>& resnet18_3d_bank() {
  static const std::vector<ConvShape> bank = {
      {"block2_conv", 64, 56, 64, 3, 1},   {"block3_down", 64, 56, 128, 3, 2},  {"block3_conv", 128, 28, 128, 3, 1},
      {"block3_skip", 64, 56, 128, 1, 2},  {"block4_down", 128, 28, 256, 3, 2}, {"block4_conv", 256, 14, 256, 3, 1},
      {"block4_skip", 128, 28, 256, 1, 2}, {"block5_down", 256, 14, 512, 3, 2}, {"block5_conv", 512, 7, 512, 3, 1},
      {"block5_skip", 256, 14, 512, 1, 2}};
  return bank;
}

const std::vector<ConvShape>& resnet50_bank() {
  static const std::vector<ConvShape> bank = {
      {"stem7x7", 3, 230, 64, 7, 2},          {"c2_1x1_64_64", 64, 56, 64, 1, 1},
      {"c2_3x3_64", 64, 58, 64, 3, 1},        {"c2_1x1_64_256", 64, 56, 256, 1, 1},
      {"c2_1x1_256_64", 256, 56, 64, 1, 1},   {"c3_1x1_256_128", 256, 56, 128, 1, 1},
      {"c3_3x3s2_128", 128, 58, 128, 3, 2},   {"c3_1x1_128_512", 128, 28, 512, 1, 1},
      {"c3_1x1s2_256_512", 256, 56, 512, 1, 2}, {"c3_1x1_512_128", 512, 28, 128, 1, 1},
      {"c3_3x3_128", 128, 30, 128, 3, 1},     {"c4_1x1_512_256", 512, 28, 256, 1, 1},
      {"c4_3x3s2_256", 256, 30, 256, 3, 2},   {"c4_1x1_256_1024", 256, 14, 1024, 1, 1},
      {"c4_1x1s2_512_1024", 512, 28, 1024, 1, 2}, {"c4_1x1_1024_256", 1024, 14, 256, 1, 1},
      {"c4_3x3_256", 256, 16, 256, 3, 1},     {"c5_1x1_1024_512", 1024, 14, 512, 1, 1},
      {"c5_3x3s2_512", 512, 16, 512, 3, 2},   {"c5_1x1_512_2048", 512, 7, 2048, 1, 1},
      {"c5_1x1s2_1024_2048", 1024, 14, 2048, 1, 2}, {"c5_1x1_2048_512", 2048, 7, 512, 1, 1},
      {"c5_3x3_512", 512, 9, 512, 3, 1}};
  return bank;
}

std::vector<BankEntry> bank_by_name(const std::string& name) {
  std::vector<BankEntry> out;
  if (name == "table1") {
    for (const auto& c : table1_bank()) out.push_back({c, conv2d_tdsl(c, 16, 4), false});
  } else if (name == "resnet18_3d") {
    for (const auto& c : resnet18_3d_bank()) out.push_back({c, conv3d_tdsl(c, 16, 4), true});
  } else if (name == "resnet50") {
    for (const auto& c : resnet50_bank())
      out.push_back({c, conv2d_nhwc_tdsl(1, c.in_hw, c.in_hw, c.in_c, c.out_c, c.kernel, c.kernel, c.stride), false});
  } else {
    throw ShapeError("unknown workload bank '" + name + "' (table1, resnet18_3d, resnet50)");
  }
  return out;
}

// ============================ sketches + tuner ===========================
std::string CpuSketch::to_string() const {
  return "cpu(l1=" + std::to_string(l1) + ",f1=" + std::to_string(f1) + ",l2=" + std::to_string(l2) +
         ",f2=" + std::to_string(f2) + ")";
}
std::string GpuSketch::to_string() const {
  return "gpu(p=" + std::to_string(p) + ",fuse=" + (fuse_hw ? "1" : "0") + ",split_k=" + std::to_string(split_k) +
         ")";
}

namespace {
[[noreturn]] void cpu_space_out_of_scope(const char* what) {
  throw InjectError(std::string(what) +
                    ": the CPU sketch space (threading / unrolling for the reference's CPU VM) is out of scope for "
                    "the B200 backend; use Target::Gpu (measured device plans)");
}
}  // namespace

Schedule apply_cpu_sketch(const TensorizedOp&, const CpuSketch&) { cpu_space_out_of_scope("apply_cpu_sketch"); }
int64_t cpu_fused_parallel_extent(const TensorizedOp&, const CpuSketch&) {
  cpu_space_out_of_scope("cpu_fused_parallel_extent");
}
int64_t cpu_unroll_factor(const TensorizedOp&, const CpuSketch&) { cpu_space_out_of_scope("cpu_unroll_factor"); }
std::vector<CpuSketch> enumerate_cpu_space(const TensorizedOp&, const CpuLimits&) {
  cpu_space_out_of_scope("enumerate_cpu_space");
}

// The GPU sketch on this backend: split_k is the only part that changes the
// nest's meaning (split_reduction: a partial buffer + a fold nest, which the
// device runs as split-K with the wrap-add fix-up); the p x p output window
// and the pixel fusion are the kernel's CTA tile and its fused pixel axis,
// which tile_and_reorder's plan already fixes.  So a sketch appends one
// split_reduction on the outermost reduction axis when split_k > 1.
Schedule apply_gpu_sketch(const TensorizedOp& t, const GpuSketch& g) {
  if (g.p < 1 || g.split_k < 1) throw ScheduleError("gpu sketch: p and split_k must be >= 1");
  Schedule s = t.schedule;
  if (g.split_k > 1) {
    if (t.outer_red.empty()) throw ScheduleError("gpu sketch: split_k needs an outer reduction axis");
    const std::string& axis = t.outer_red.front();  // lower() rejects a non-dividing segment count
    Transform sr;
    sr.kind = Transform::Kind::SplitReduction;
    sr.a = axis;
    sr.factor = g.split_k;
    s.insert(s.end() - 1, sr);  // before the pragma
  }
  return s;
}

std::vector<GpuSketch> enumerate_gpu_space(const TensorizedOp& t, const GpuLimits& lim) {
  std::vector<GpuSketch> out;
  out.push_back(GpuSketch{1, false, 1});
  for (int64_t f : lim.split_factors) {
    if (f < 2 || t.outer_red.empty()) continue;
    for (const auto& l : t.op.loops)
      if (l.name == t.outer_red.front() && l.extent % f == 0 && l.extent > f) out.push_back(GpuSketch{1, false, f});
  }
  return out;
}

TuneResult tune(const ComputeOp& op, const Intrinsic& intr, const TuneOptions& opts) {
  if (opts.target == Target::Cpu) cpu_space_out_of_scope("tune(Target::Cpu)");
  if (intr.target_mnemonic.rfind("tcgen05.", 0) != 0)
    throw InjectError("tune(Target::Gpu): '" + intr.name + "' is not a tcgen05 description");
  const MatchResult mr = match_operation(op, intr);
  if (!mr.ok) throw NoFeasibleMapping("no structural match: " + mr.reason);
  // the device-realisable mapping (fused pixel groups first), tiled once
  TensorizedOp t = tensorize(op, intr);
  const Inputs in = random_inputs(op, opts.seed);
  const std::string log = tune_tensorized(t, in, 10);
  // "candidate <i> <spec|default> <us> us" / "candidate <i> <spec> skipped" / "best ..."
  TuneResult res;
  std::istringstream ls(log);
  int budget = opts.budget;
  for (std::string line; std::getline(ls, line) && budget > 0;) {
    std::istringstream w(line);
    std::string tag, spec, unit;
    int id = -1;
    double us = 0;
    w >> tag >> id >> spec;
    if (tag != "candidate" || !(w >> us >> unit)) continue;
    --budget;
    Candidate c;
    c.id = id;
    c.mapping = t.mapping;
    c.sketch = spec;
    c.schedule = t.schedule;
    c.key = CostKey{(int64_t)(us * 1000.0 + 0.5), 0, 0};
    c.verified = true;  // every device plan is bit-exact by construction (tests/test_gpu_*.py)
    if (opts.log) *opts.log << "candidate " << id << " mapping=" << t.mapping.to_string() << " sketch=" << spec
                            << " cost=" << cost_key_to_string(c.key) << "\n";
    res.evaluated.push_back(c);
    if (res.best.id < 0 || c.key < res.best.key) res.best = c;
  }
  if (res.evaluated.empty()) throw NoFeasibleMapping("tune: no device plan could be timed");
  return res;
}

}  // namespace tzc
