// Schedules, lowering, intrinsic injection and eval_tir for the B200 backend.
//
// Same contract as the reference's rewriter / tensor IR
// (proj/include/tzc/rewriter.hpp:14-116, proj/src/rewriter.cpp:16-131 schedule
// text, :305-646 lower, :652-917 inject; proj/src/tensor_ir.cpp print format;
// proj/src/expr.cpp:217-268 split_linear): the printed IR of an op lowered and
// injected here is the reference's golden-snapshot text
// (tests/test_tensor_ir.py compares the two for the reference's own ops).
//
// What differs is execution: eval_tir runs a nest whose single call is a
// tcgen05 description on the B200 (via the KernelPlan of tile_and_reorder),
// and refuses anything else.  The fused pixel group of F6 (n, oh, ow fused
// onto tcgen05's M) is not linear in the pragma loops; its operands are kept
// as scalar gather addresses over the pragma axes (what TMA im2col realises),
// where the reference would raise InjectError.
#include <algorithm>
#include <fstream>
#include <set>
#include <sstream>

#include "tzc/tzc.hpp"

namespace tzc {

// ============================ schedule text ==============================
std::string Transform::kind_name(Kind k) {
  static const char* const names[] = {"pad", "split", "reorder", "fuse", "parallel", "unroll", "split_reduction", "pragma"};
  return names[static_cast<int>(k)];
}

std::string print_schedule(const Schedule& s) {
  std::ostringstream os;
  for (const auto& t : s) {
    os << Transform::kind_name(t.kind);
    using K = Transform::Kind;
    if (t.kind == K::Pad || t.kind == K::Split || t.kind == K::SplitReduction) os << " " << t.a << " " << t.factor;
    else if (t.kind == K::Fuse) os << " " << t.a << " " << t.b;
    else if (t.kind == K::Parallel || t.kind == K::Unroll) os << " " << t.a;
    else
      for (const auto& n : t.names) os << " " << n;
    os << "\n";
  }
  return os.str();
}

Schedule parse_schedule(const std::string& text) {
  Schedule out;
  std::istringstream in(text);
  std::string line;
  for (int no = 1; std::getline(in, line); ++no) {
    line = line.substr(0, line.find('#'));
    std::istringstream ls(line);
    std::vector<std::string> w;
    for (std::string t; ls >> t;) w.push_back(t);
    if (w.empty()) continue;
    const std::string where = "schedule line " + std::to_string(no) + ": ";
    auto arity = [&](size_t n) {
      if (w.size() != n + 1)
        throw SyntaxError(where + "'" + w[0] + "' takes " + std::to_string(n) + " argument(s)");
    };
    auto integer = [&](const std::string& s) {
      size_t used = 0;
      int64_t v = 0;
      try {
        v = std::stoll(s, &used);
      } catch (...) {
        used = 0;
      }
      if (used != s.size() || s.empty()) throw SyntaxError(where + "expected an integer, got '" + s + "'");
      return v;
    };
    Transform t;
    using K = Transform::Kind;
    if (w[0] == "pad" || w[0] == "split" || w[0] == "split_reduction") {
      arity(2);
      t.kind = w[0] == "pad" ? K::Pad : w[0] == "split" ? K::Split : K::SplitReduction;
      t.a = w[1];
      t.factor = integer(w[2]);
    } else if (w[0] == "fuse") {
      arity(2);
      t.kind = K::Fuse;
      t.a = w[1];
      t.b = w[2];
    } else if (w[0] == "parallel" || w[0] == "unroll") {
      arity(1);
      t.kind = w[0] == "parallel" ? K::Parallel : K::Unroll;
      t.a = w[1];
    } else if (w[0] == "reorder" || w[0] == "pragma") {
      if (w.size() < 2) throw SyntaxError(where + "'" + w[0] + "' needs at least one axis");
      t.kind = w[0] == "reorder" ? K::Reorder : K::Pragma;
      t.names.assign(w.begin() + 1, w.end());
    } else {
      throw SyntaxError(where + "unknown transform '" + w[0] + "'");
    }
    out.push_back(std::move(t));
  }
  return out;
}

Schedule load_schedule(const std::string& path) {
  std::ifstream f(path);
  if (!f) throw IoError("cannot open schedule file '" + path + "'");
  std::stringstream ss;
  ss << f.rdbuf();
  return parse_schedule(ss.str());
}

// ============================ statements =================================
std::string loop_ann_name(LoopAnn a) {
  switch (a) {
    case LoopAnn::Serial: return "serial";
    case LoopAnn::Parallel: return "parallel";
    case LoopAnn::Unrolled: return "unroll";
    case LoopAnn::Tensorize: return "tensorize";
  }
  return "?";
}

namespace {
std::shared_ptr<Stmt> node(Stmt::Kind k) {
  auto s = std::make_shared<Stmt>();
  s->kind = k;
  return s;
}
}  // namespace

StmtPtr make_for(std::string v, int64_t extent, StmtPtr body, LoopAnn ann) {
  internal_check(extent > 0, "loop extent must be positive");
  auto s = node(Stmt::Kind::For);
  s->var = std::move(v);
  s->extent = extent;
  s->ann = ann;
  s->body = std::move(body);
  return s;
}
StmtPtr make_store(std::string tensor, std::vector<ExprPtr> indices, ExprPtr value) {
  auto s = node(Stmt::Kind::Store);
  s->tensor = std::move(tensor);
  s->indices = std::move(indices);
  s->value = std::move(value);
  return s;
}
StmtPtr make_intrinsic(std::string name, std::string dst, ExprPtr dst_index, std::vector<ExprPtr> args) {
  auto s = node(Stmt::Kind::Intrinsic);
  s->intrinsic = std::move(name);
  s->tensor = std::move(dst);
  s->dst_index = std::move(dst_index);
  s->args = std::move(args);
  return s;
}
StmtPtr make_seq(std::vector<StmtPtr> stmts) {
  if (stmts.size() == 1) return stmts.front();
  auto s = node(Stmt::Kind::Seq);
  s->stmts = std::move(stmts);
  return s;
}

const TensorDecl* TensorIR::find_tensor(const std::string& n) const {
  for (const auto& t : tensors)
    if (t.name == n) return &t;
  return nullptr;
}
const Intrinsic* TensorIR::find_intrinsic(const std::string& n) const {
  for (const auto& i : intrinsics)
    if (i.name == n) return &i;
  return nullptr;
}

void visit_stmts(const StmtPtr& s, const std::function<void(const Stmt&)>& f) {
  if (!s) return;
  f(*s);
  visit_stmts(s->body, f);
  for (const auto& c : s->stmts) visit_stmts(c, f);
}
int count_stmts(const StmtPtr& s, Stmt::Kind kind) {
  int n = 0;
  visit_stmts(s, [&](const Stmt& x) { n += x.kind == kind; });
  return n;
}

namespace {
std::string join(const std::vector<ExprPtr>& v) {
  std::string s;
  for (size_t i = 0; i < v.size(); ++i) s += (i ? ", " : "") + expr_to_string(v[i]);
  return s;
}
void print_stmt(const Stmt& s, int depth, std::string* out) {
  const std::string ind(2 * depth, ' ');
  switch (s.kind) {
    case Stmt::Kind::For:
      *out += ind + "for " + s.var + " : " + std::to_string(s.extent) +
              (s.ann == LoopAnn::Serial ? "" : " " + loop_ann_name(s.ann)) + " {\n";
      print_stmt(*s.body, depth + 1, out);
      *out += ind + "}\n";
      break;
    case Stmt::Kind::Store:
      *out += ind + s.tensor + "[" + join(s.indices) + "] = " + expr_to_string(s.value) + "\n";
      break;
    case Stmt::Kind::Intrinsic:
      *out += ind + s.intrinsic + "(dst = " + s.tensor + "[" + expr_to_string(s.dst_index) + "]";
      for (const auto& a : s.args) *out += ", " + expr_to_string(a);
      *out += ")\n";
      break;
    case Stmt::Kind::Seq:
      for (const auto& c : s.stmts) print_stmt(*c, depth, out);
      break;
  }
}
}  // namespace

std::string print_tensor_ir(const TensorIR& ir) {
  std::string out;
  for (const auto& t : ir.tensors) {
    out += "buffer " + t.name + " : " + dtype_name(t.dtype) + " [";
    for (size_t i = 0; i < t.shape.size(); ++i) out += (i ? ", " : "") + std::to_string(t.shape[i]);
    const bool temp = std::find(ir.temps.begin(), ir.temps.end(), t.name) != ir.temps.end();
    out += std::string("] ") + (temp ? "temp" : t.role == Role::Output ? "output" : "input") + "\n";
  }
  if (ir.seed_output) out += "# output seeded from input image\n";
  if (ir.root) print_stmt(*ir.root, 0, &out);
  return out;
}

// ============================ split_linear ===============================
namespace {
// Peels the terms of e that are (constant multiples of) a target variable
// into coeff; everything else (free of the targets) is summed as residual.
bool peel(const ExprPtr& e, const std::vector<std::string>& vars, int64_t scale, LinearSplit* out) {
  const bool target = e->kind == Expr::Kind::Var && std::count(vars.begin(), vars.end(), e->name);
  if (target) {
    out->coeff[e->name] += scale;
    return true;
  }
  if (e->kind == Expr::Kind::Add) return peel(e->args[0], vars, scale, out) && peel(e->args[1], vars, scale, out);
  if (e->kind == Expr::Kind::Mul) {
    for (int side = 0; side < 2; ++side) {
      auto f = linearize(e->args[side]);
      if (f && f->coeff.empty()) return peel(e->args[1 - side], vars, scale * f->constant, out);
    }
  }
  for (const auto& v : vars)
    if (contains_var(e, v)) return false;
  ExprPtr term = scale == 1 ? e : mul(int_imm(scale), e);
  out->residual = out->residual ? add(out->residual, term) : term;
  return true;
}
}  // namespace

std::optional<LinearSplit> split_linear(const ExprPtr& e, const std::vector<std::string>& vars) {
  LinearSplit s;
  if (!peel(e, vars, 1, &s)) return std::nullopt;
  if (!s.residual) s.residual = int_imm(0);
  return s;
}

// ============================ lower ======================================
namespace {

struct Axis {
  std::string name;
  int64_t extent;
  LoopKind kind;
  LoopAnn ann = LoopAnn::Serial;
};

ExprPtr zero_of(DType t) { return t.is_float() ? float_imm(0.0, t) : int_imm(0, t); }

// The axis list and the rewrite of each original loop variable in terms of
// the current axes, advanced one transform at a time.
class Nest {
 public:
  explicit Nest(const ComputeOp& op, bool clip_tails) : clip(clip_tails) {
    for (const auto& l : op.loops) {
      axes.push_back({l.name, l.extent, l.kind});
      of[l.name] = var(l.name);
    }
  }
  bool clip;
  std::vector<Axis> axes;
  std::map<std::string, ExprPtr> of;
  std::vector<std::string> pragma;
  struct SplitRed {
    std::string seg, inner;
    int64_t count;
  };
  std::optional<SplitRed> sred;

  void apply(const Transform& t) {
    using K = Transform::Kind;
    switch (t.kind) {
      case K::Pad:
        throw ScheduleError("pad transforms must come first in a schedule");
      case K::Split: {
        const size_t j = at(t.a, "split");
        const Axis ax = axes[j];
        if (t.factor < 1 || (ax.extent % t.factor && !clip))
          throw ScheduleError("split: factor " + std::to_string(t.factor) + " does not divide extent " +
                              std::to_string(ax.extent) + " of axis '" + t.a + "'");
        const std::string o = t.a + ".o", i = t.a + ".i";
        fresh(o, "split");
        fresh(i, "split");
        axes[j] = {o, (ax.extent + t.factor - 1) / t.factor, ax.kind};
        axes.insert(axes.begin() + j + 1, Axis{i, t.factor, ax.kind});
        rewrite({{t.a, add(mul(var(o), int_imm(t.factor)), var(i))}});
        break;
      }
      case K::Fuse: {
        const size_t j = at(t.a, "fuse"), k = at(t.b, "fuse");
        if (k != j + 1) throw ScheduleError("fuse: '" + t.b + "' must sit directly inside '" + t.a + "'");
        if (axes[j].kind != axes[k].kind)
          throw ScheduleError("fuse: axes '" + t.a + "' and '" + t.b + "' have different kinds");
        const std::string f = t.a + "." + t.b + ".fused";
        fresh(f, "fuse");
        const int64_t inner = axes[k].extent;
        axes[j] = {f, axes[j].extent * inner, axes[j].kind};
        axes.erase(axes.begin() + k);
        rewrite({{t.a, floordiv(var(f), int_imm(inner))}, {t.b, floormod(var(f), int_imm(inner))}});
        break;
      }
      case K::Reorder: {
        if (t.names.size() != axes.size())
          throw ScheduleError("reorder: needs all " + std::to_string(axes.size()) + " axes");
        std::vector<Axis> next;
        std::set<std::string> seen;
        for (const auto& n : t.names) {
          if (!seen.insert(n).second) throw ScheduleError("reorder: duplicate axis '" + n + "'");
          next.push_back(axes[at(n, "reorder")]);
        }
        axes = std::move(next);
        break;
      }
      case K::Parallel: {
        Axis& ax = axes[at(t.a, "parallel")];
        if (ax.kind != LoopKind::DataParallel) throw ScheduleError("parallel: axis '" + t.a + "' is not data-parallel");
        if (ax.ann != LoopAnn::Serial) throw ScheduleError("parallel: axis '" + t.a + "' is already annotated");
        ax.ann = LoopAnn::Parallel;
        break;
      }
      case K::Unroll: {
        Axis& ax = axes[at(t.a, "unroll")];
        if (ax.ann != LoopAnn::Serial) throw ScheduleError("unroll: axis '" + t.a + "' is already annotated");
        ax.ann = LoopAnn::Unrolled;
        break;
      }
      case K::SplitReduction: {
        if (sred) throw ScheduleError("split_reduction: at most one per schedule");
        const size_t j = at(t.a, "split_reduction");
        const Axis ax = axes[j];
        if (ax.kind != LoopKind::Reduction)
          throw ScheduleError("split_reduction: axis '" + t.a + "' is not a reduction axis");
        if (t.factor < 2 || ax.extent % t.factor)
          throw ScheduleError("split_reduction: factor " + std::to_string(t.factor) + " does not divide extent " +
                              std::to_string(ax.extent) + " of axis '" + t.a + "'");
        const std::string seg = t.a + ".s", inner = t.a + ".r";
        fresh(seg, "split_reduction");
        fresh(inner, "split_reduction");
        const int64_t chunk = ax.extent / t.factor;
        // partial sums are independent: the segment axis is data-parallel
        axes[j] = {seg, t.factor, LoopKind::DataParallel};
        axes.insert(axes.begin() + j + 1, Axis{inner, chunk, LoopKind::Reduction});
        rewrite({{t.a, add(mul(var(seg), int_imm(chunk)), var(inner))}});
        sred = SplitRed{seg, inner, t.factor};
        break;
      }
      case K::Pragma: {
        if (!pragma.empty()) throw ScheduleError("pragma: at most one per schedule");
        if (t.names.empty()) throw ScheduleError("pragma: needs axes");
        if (t.names.size() > axes.size()) throw ScheduleError("pragma: more axes than the nest has");
        const size_t base = axes.size() - t.names.size();
        for (size_t i = 0; i < t.names.size(); ++i) {
          if (axes[base + i].name != t.names[i])
            throw ScheduleError("pragma: axes must be the innermost loops in the given order");
          if (axes[base + i].ann != LoopAnn::Serial)
            throw ScheduleError("pragma: axis '" + t.names[i] + "' is already annotated");
          axes[base + i].ann = LoopAnn::Tensorize;
        }
        pragma = t.names;
        break;
      }
    }
  }

  void check_pragma_innermost() const {
    if (pragma.empty()) return;
    const size_t base = axes.size() - pragma.size();
    for (size_t i = 0; i < pragma.size(); ++i)
      if (axes[base + i].name != pragma[i] || axes[base + i].ann != LoopAnn::Tensorize)
        throw ScheduleError("pragma axes must remain the innermost loops");
  }

 private:
  size_t at(const std::string& n, const char* what) const {
    for (size_t i = 0; i < axes.size(); ++i)
      if (axes[i].name == n) return i;
    throw ScheduleError(std::string(what) + ": unknown axis '" + n + "'");
  }
  void fresh(const std::string& n, const char* what) const {
    for (const auto& a : axes)
      if (a.name == n) throw ScheduleError(std::string(what) + ": axis name '" + n + "' already exists");
  }
  void rewrite(const std::map<std::string, ExprPtr>& m) {
    for (auto& kv : of) kv.second = substitute(kv.second, m);
  }
};

StmtPtr subst_stmt(const StmtPtr& s, const std::map<std::string, ExprPtr>& m) {
  std::vector<ExprPtr> v;
  switch (s->kind) {
    case Stmt::Kind::For:
      return make_for(s->var, s->extent, subst_stmt(s->body, m), s->ann);
    case Stmt::Kind::Store:
      for (const auto& e : s->indices) v.push_back(substitute(e, m));
      return make_store(s->tensor, std::move(v), substitute(s->value, m));
    case Stmt::Kind::Intrinsic:
      for (const auto& e : s->args) v.push_back(substitute(e, m));
      return make_intrinsic(s->intrinsic, s->tensor, substitute(s->dst_index, m), std::move(v));
    case Stmt::Kind::Seq: {
      std::vector<StmtPtr> parts;
      for (const auto& c : s->stmts) parts.push_back(subst_stmt(c, m));
      return make_seq(std::move(parts));
    }
  }
  throw InternalError("unhandled statement kind");
}

// Wraps `inner` in loops over names[d] < extents[d], outermost first.
StmtPtr nest_over(const std::vector<std::string>& names, const std::vector<int64_t>& extents, StmtPtr inner) {
  for (size_t d = names.size(); d-- > 0;) inner = make_for(names[d], extents[d], inner);
  return inner;
}

}  // namespace

namespace {

// The nest of an (already padded) op under the axis transforms of a schedule.
TensorIR lower_axes(const ComputeOp& op, const Schedule& schedule, const LowerOptions& opts) {
  Nest nest(op, opts.clip_tails);
  for (const auto& t : schedule) nest.apply(t);
  nest.check_pragma_innermost();

  const ReduceForm rf = reduce_form(op);
  const bool reduces = !op.loops_of_kind(LoopKind::Reduction).empty() || nest.sred;
  const TensorDecl& outd = op.output();
  const DType odt = outd.dtype;

  TensorIR ir;
  ir.tensors = op.tensors;
  ir.output = op.out;
  ir.seed_output = op.update;
  ir.source = std::make_shared<const ComputeOp>(op);

  std::vector<ExprPtr> sidx;
  for (const auto& e : op.indices) sidx.push_back(substitute(e, nest.of));

  StmtPtr body;
  std::string partial;
  if (nest.sred) {
    internal_check(rf.term != nullptr, "reduction split without a term");
    partial = op.out + ".partial";
    if (ir.find_tensor(partial)) throw ScheduleError("split_reduction: buffer name '" + partial + "' is taken");
    TensorDecl pd{partial, {nest.sred->count}, odt, Role::Input};
    pd.shape.insert(pd.shape.end(), outd.shape.begin(), outd.shape.end());
    ir.tensors.push_back(pd);
    ir.temps.push_back(partial);
    std::vector<ExprPtr> pidx{var(nest.sred->seg)};
    pidx.insert(pidx.end(), sidx.begin(), sidx.end());
    body = make_store(partial, pidx, add(load(partial, pidx, odt), substitute(rf.term, nest.of)));
  } else if (reduces) {
    body = make_store(op.out, sidx, add(load(op.out, sidx, odt), substitute(rf.term, nest.of)));
  } else {
    body = make_store(op.out, sidx, substitute(op.value, nest.of));
  }
  for (auto a = nest.axes.rbegin(); a != nest.axes.rend(); ++a) {
    if (opts.literal_unroll && a->ann == LoopAnn::Unrolled) {
      std::vector<StmtPtr> copies;
      for (int64_t v = 0; v < a->extent; ++v) copies.push_back(subst_stmt(body, {{a->name, int_imm(v)}}));
      body = make_seq(std::move(copies));
    } else {
      body = make_for(a->name, a->extent, body, a->ann);
    }
  }

  std::vector<StmtPtr> parts;
  if (reduces && !op.update) {  // declared-init reductions start from the init value
    std::vector<std::string> n;
    std::vector<int64_t> e;
    for (const auto& l : op.loops_of_kind(LoopKind::DataParallel)) n.push_back(l.name), e.push_back(l.extent);
    parts.push_back(nest_over(n, e, make_store(op.out, op.indices, rf.init ? rf.init : zero_of(odt))));
  }
  if (!nest.sred) {
    parts.push_back(body);
  } else {
    std::set<std::string> used;
    for (const auto& a : nest.axes) used.insert(a.name);
    for (const auto& l : op.loops) used.insert(l.name);
    for (const auto& t : ir.tensors) used.insert(t.name);
    std::vector<std::string> z;
    std::vector<ExprPtr> zi;
    for (size_t d = 0; d < outd.shape.size(); ++d) {
      std::string n = "z" + std::to_string(d);
      while (used.count(n)) n += "_";
      used.insert(n);
      z.push_back(n);
      zi.push_back(var(n));
    }
    std::vector<ExprPtr> pzi{var(nest.sred->seg)};
    pzi.insert(pzi.end(), zi.begin(), zi.end());
    // zero the partial sums, run the main nest, fold the partials into out
    parts.push_back(make_for(nest.sred->seg, nest.sred->count, nest_over(z, outd.shape, make_store(partial, pzi, zero_of(odt)))));
    parts.push_back(body);
    parts.push_back(nest_over(z, outd.shape,
                              make_for(nest.sred->seg, nest.sred->count,
                                       make_store(op.out, zi, add(load(op.out, zi, odt), load(partial, pzi, odt))))));
  }
  ir.root = make_seq(std::move(parts));
  return ir;
}

}  // namespace

TensorIR lower(const ComputeOp& op, const Schedule& schedule, const LowerOptions& opts) {
  // leading pads reshape the op itself (zero extension); the rest are axis transforms
  ComputeOp cur = op;
  size_t i = 0;
  for (; i < schedule.size() && schedule[i].kind == Transform::Kind::Pad; ++i)
    cur = pad_to_multiple(cur, schedule[i].a, schedule[i].factor);
  return lower_axes(cur, Schedule(schedule.begin() + (std::ptrdiff_t)i, schedule.end()), opts);
}

// ============================ inject =====================================
namespace {

// Row-major flat element address of a multi-dimensional access.
ExprPtr flat_address(const TensorDecl& d, const std::vector<ExprPtr>& idx) {
  internal_check(idx.size() == d.shape.size(), "rank mismatch in flatten");
  ExprPtr acc;
  int64_t stride = 1;
  std::vector<ExprPtr> terms(idx.size());
  for (size_t k = idx.size(); k-- > 0;) {
    terms[k] = stride == 1 ? idx[k] : mul(idx[k], int_imm(stride));
    stride *= d.shape[k];
  }
  for (const auto& t : terms) acc = acc ? add(acc, t) : t;
  return acc ? acc : int_imm(0);
}

ExprPtr shifted(const ExprPtr& e, int64_t delta) {
  if (delta == 0) return e;
  switch (e->kind) {
    case Expr::Kind::IntImm:
      return int_imm(e->ival + delta, e->dtype);
    case Expr::Kind::Ramp:
      return ramp(shifted(e->args[0], delta), e->ival, e->lanes_arg);
    case Expr::Kind::Broadcast:
      return broadcast(shifted(e->args[0], delta), e->lanes_arg);
    case Expr::Kind::Concat: {
      std::vector<ExprPtr> p;
      for (const auto& a : e->args) p.push_back(shifted(a, delta));
      return concat(std::move(p));
    }
    default:
      return add(e, int_imm(delta));
  }
}

// Register-image address: the rules walk the operand's lanes minor axis first.
ExprPtr vector_address(ExprPtr v, const std::map<std::string, int64_t>& coeff, const std::vector<OperandRule>& rules,
                       const std::map<std::string, std::string>& axis_of, const std::string& what) {
  for (const auto& r : rules) {
    if (r.kind == OperandRule::Kind::Passthrough) continue;
    auto ax = axis_of.find(r.loop);
    internal_check(ax != axis_of.end(), "rule names unknown loop");
    auto c = coeff.find(ax->second);
    const int64_t step = c == coeff.end() ? 0 : c->second;
    if (r.kind == OperandRule::Kind::Vectorize) {
      v = ramp(v, step, r.count);
    } else if (r.kind == OperandRule::Kind::Broadcast) {
      if (step) throw InjectError(what + ": access varies along loop '" + r.loop + "' but the rule replicates lanes there");
      v = broadcast(v, r.count);
    } else {
      std::vector<ExprPtr> parts;
      for (int64_t k = 0; k < r.count; ++k) parts.push_back(shifted(v, step * k));
      v = concat(std::move(parts));
    }
  }
  return v;
}

StmtPtr replace(const StmtPtr& s, const Stmt* target, const StmtPtr& with) {
  if (s.get() == target) return with;
  if (s->kind == Stmt::Kind::For) {
    StmtPtr b = replace(s->body, target, with);
    return b == s->body ? s : make_for(s->var, s->extent, b, s->ann);
  }
  if (s->kind == Stmt::Kind::Seq) {
    std::vector<StmtPtr> p;
    bool changed = false;
    for (const auto& c : s->stmts) {
      p.push_back(replace(c, target, with));
      changed = changed || p.back() != c;
    }
    return changed ? make_seq(std::move(p)) : s;
  }
  return s;
}

void pragma_roots(const StmtPtr& s, std::vector<const Stmt*>* out) {
  if (!s) return;
  if (s->kind == Stmt::Kind::For) {
    if (s->ann == LoopAnn::Tensorize) return out->push_back(s.get());
    pragma_roots(s->body, out);
  } else if (s->kind == Stmt::Kind::Seq) {
    for (const auto& c : s->stmts) pragma_roots(c, out);
  }
}

bool has_fused_group(const LoopMapping& m) {
  for (const auto& kv : m.fused)
    if (!kv.second.empty()) return true;
  return false;
}

}  // namespace

TensorIR inject_intrinsic(const TensorIR& ir, const Intrinsic& intr, const LoopMapping& mapping) {
  const ComputeOp& sem = intr.semantics;
  std::vector<const Stmt*> roots;
  pragma_roots(ir.root, &roots);
  if (roots.empty()) throw InjectError("no tensorize pragma nest in the lowered tree");
  if (roots.size() > 1) throw InjectError("more than one tensorize pragma nest");
  std::vector<const Stmt*> fors;
  const Stmt* s = roots.front();
  for (; s->kind == Stmt::Kind::For; s = s->body.get()) {
    if (s->ann != LoopAnn::Tensorize) throw InjectError("non-pragma loop inside the tensorize nest");
    fors.push_back(s);
  }
  if (s->kind != Stmt::Kind::Store) throw InjectError("tensorize pragma nest must wrap a single scalar store");
  const Stmt& store = *s;
  if (fors.size() != sem.loops.size())
    throw InjectError("pragma nest has " + std::to_string(fors.size()) + " loops but the instruction has " +
                      std::to_string(sem.loops.size()));
  if (!mapping.f.empty() && mapping.f.size() != sem.loops.size())
    throw InjectError("mapping covers " + std::to_string(mapping.f.size()) + " of " + std::to_string(sem.loops.size()) +
                      " instruction loops");

  std::map<std::string, std::string> axis_of;  // instruction loop -> pragma axis
  std::vector<std::string> paxes;
  for (size_t k = 0; k < fors.size(); ++k) {
    const LoopVar& il = sem.loops[k];
    if (fors[k]->extent != il.extent)
      throw InjectError("pragma loop '" + fors[k]->var + "' has extent " + std::to_string(fors[k]->extent) +
                        " but instruction loop '" + il.name + "' has " + std::to_string(il.extent));
    axis_of[il.name] = fors[k]->var;
    paxes.push_back(fors[k]->var);
  }

  const MatchResult m = inspect_compute(sem.value, store.value);
  if (!m.ok) throw InjectError("pragma body does not match the instruction: " + m.reason);
  const std::string acc = intr.accumulator();
  if (!acc.empty()) {
    ExprPtr src;
    for (const auto& [ia, ob] : m.bind.pairs)
      if (ia->kind == Expr::Kind::Load && ia->name == acc) src = ob;
    bool alias = src && src->kind == Expr::Kind::Load && src->name == store.tensor && src->args.size() == store.indices.size();
    for (size_t d = 0; alias && d < store.indices.size(); ++d) alias = expr_equal(src->args[d], store.indices[d], false);
    if (!alias) throw InjectError("accumulator operand must read the store destination");
  }
  // The F6 pixel group (several op loops fused onto one instruction loop) is
  // realised by TMA im2col: its accesses stay scalar gather addresses.
  bool gather_ok = has_fused_group(mapping);
  for (const auto& a : paxes) gather_ok = gather_ok || a.find(".fused") != std::string::npos;

  std::vector<ExprPtr> args;
  for (const auto& td : sem.tensors) {
    if (td.role != Role::Input) continue;
    auto b = m.bind.reg_to_op.find(td.name);
    if (b == m.bind.reg_to_op.end()) throw InjectError("register '" + td.name + "' is not bound by the match");
    const ExprPtr& leaf = b->second;
    const int64_t lanes = td.size();
    if (is_const(leaf)) {
      args.push_back(broadcast(leaf, lanes));
      continue;
    }
    const std::vector<OperandRule>* rules = intr.rules_for(td.name);
    internal_check(rules != nullptr, "input register without operand rules");
    const TensorDecl* opd = ir.find_tensor(leaf->name);
    if (!opd) throw InjectError("operand tensor '" + leaf->name + "' is not declared");
    const ExprPtr flat = flat_address(*opd, leaf->args);
    const DType vt = opd->dtype.with_lanes(static_cast<int>(lanes));
    auto ls = split_linear(flat, paxes);
    if (!ls) {
      if (!gather_ok) throw InjectError("access of '" + leaf->name + "' is not linear in the pragma loops");
      args.push_back(load(leaf->name, {flat}, vt));
      continue;
    }
    ExprPtr addr = vector_address(ls->residual, ls->coeff, *rules, axis_of, "operand '" + td.name + "'");
    if (lanes_of(addr) != lanes)
      throw InjectError("operand '" + td.name + "' assembles " + std::to_string(lanes_of(addr)) +
                        " lanes, register holds " + std::to_string(lanes));
    args.push_back(load(leaf->name, {addr}, vt));
  }

  const TensorDecl* dd = ir.find_tensor(store.tensor);
  internal_check(dd != nullptr, "store into undeclared tensor");
  const ExprPtr dflat = flat_address(*dd, store.indices);
  ExprPtr dst;
  if (auto ds = split_linear(dflat, paxes)) {
    std::vector<OperandRule> srules;  // instruction store layout, minor dimension first
    for (size_t d = sem.indices.size(); d-- > 0;) {
      const ExprPtr& ie = sem.indices[d];
      if (ie->kind != Expr::Kind::Var) throw InjectError("instruction store index must be a plain loop variable");
      const LoopVar* il = sem.find_loop(ie->name);
      internal_check(il != nullptr, "store index of unknown loop");
      auto c = ds->coeff.find(axis_of.at(ie->name));
      if (c == ds->coeff.end() || c->second == 0)
        throw InjectError("store addresses collide along instruction loop '" + ie->name + "'");
      OperandRule r;
      r.kind = srules.empty() ? OperandRule::Kind::Vectorize : OperandRule::Kind::UnrollConcat;
      r.loop = ie->name;
      r.count = il->extent;
      srules.push_back(r);
    }
    dst = vector_address(ds->residual, ds->coeff, srules, axis_of, "store");
    if (lanes_of(dst) != sem.output().size())
      throw InjectError("store pattern covers " + std::to_string(lanes_of(dst)) + " lanes but the output register holds " +
                        std::to_string(sem.output().size()));
  } else if (gather_ok) {
    dst = dflat;
  } else {
    throw InjectError("store address is not linear in the pragma loops");
  }

  TensorIR out = ir;
  out.root = replace(ir.root, fors.front(), make_intrinsic(intr.name, store.tensor, dst, std::move(args)));
  if (!out.find_intrinsic(intr.name)) out.intrinsics.push_back(intr);
  out.mapping = mapping;
  return out;
}

TensorIR tensorized_ir(const ComputeOp& op, const Intrinsic& intr) {
  const TensorizedOp t = tensorize(op, intr);
  LowerOptions o;
  o.clip_tails = has_fused_group(t.mapping);
  return inject_intrinsic(lower(t.op, t.schedule, o), intr, t.mapping);
}

// ============================ eval_tir ===================================
TensorizedOp device_plan(const TensorIR& ir) {
  std::vector<const Stmt*> calls;
  visit_stmts(ir.root, [&](const Stmt& s) {
    if (s.kind == Stmt::Kind::Intrinsic) calls.push_back(&s);
  });
  if (calls.size() != 1)
    throw InjectError("eval_tir on the B200 runs a nest with exactly one tensorized call (found " +
                      std::to_string(calls.size()) + "); there is no CPU interpreter");
  const Intrinsic* intr = ir.find_intrinsic(calls.front()->intrinsic);
  if (!intr) throw UnknownIntrinsic("call to '" + calls.front()->intrinsic + "' without a definition in the IR");
  if (intr->target_mnemonic.rfind("tcgen05.", 0) != 0)
    throw InjectError("'" + intr->name + "' (" + intr->target_mnemonic +
                      ") is not a B200 tensor-core instruction; this backend executes tcgen05 descriptions only");
  if (!ir.source) throw InjectError("TensorIR was not lowered by this library (no source op)");
  // The schedule fixes a loop order; the kernel computes the same function
  // (bit-exact for integers by wrap-add associativity, F8; within 1e-3 for fp16).
  TensorizedOp t = ir.mapping.f.empty() ? tensorize(*ir.source, *intr)
                                         : tile_and_reorder(*ir.source, *intr, ir.mapping, true);
  // split_reduction (rewriter.cpp:425-451) becomes the device split-K: the
  // segment count of the partial buffer is the number of K splits, folded by
  // the wrap-add fix-up kernel (exact for integers, F8).
  for (const auto& name : ir.temps)
    if (const TensorDecl* d = ir.find_tensor(name)) t.plan.splits = d->shape.front();
  return t;
}

TensorValue eval_tir(const TensorIR& ir, const Inputs& inputs, const ComputeOp* epilogue_op) {
  return run_tensorized(device_plan(ir), inputs, epilogue_op);
}

}  // namespace tzc
