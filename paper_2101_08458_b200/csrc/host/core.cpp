// tzc host library, part 1: scalar types, expressions, tensor ops, parser.
// Semantics follow the reference (/root/reference/proj): dtype rules
// dtype.cpp:40-101, expression IR expr.hpp:22-113, op validation and typing
// compute_op.cpp:85-243, reduce_form :245-282, grammar parser.hpp:12-26.
#include <algorithm>
#include <bit>
#include <cctype>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <set>

#include "tzc/tzc.hpp"

namespace tzc {

// ============================ scalar types ===============================
std::string dtype_name(const DType& t) {
  std::string b = t.kind == DType::Kind::Int ? "i" : t.kind == DType::Kind::UInt ? "u" : t.kind == DType::Kind::Float ? "fp" : "";
  std::string s = t.defined() ? b + std::to_string(t.bits) : "invalid";
  if (t.lanes != 1) s += "x" + std::to_string(t.lanes);
  return s;
}

DType dtype_from_name(const std::string& n) {
  static const std::pair<const char*, DType> table[] = {{"u8", kU8},   {"i8", kI8},   {"u16", kU16}, {"i16", kI16},
                                                        {"u32", kU32}, {"i32", kI32}, {"fp16", kF16}, {"fp32", kF32}};
  for (const auto& [k, v] : table)
    if (n == k) return v;
  throw SyntaxError("unknown dtype '" + n + "'");
}

int64_t wrap_int(int64_t v, const DType& t) {
  if (!t.is_int() || t.bits < 1 || t.bits > 64) throw InternalError("wrap_int on a non-integer dtype");
  if (t.bits == 64) return v;
  const uint64_t mask = (uint64_t{1} << t.bits) - 1;
  uint64_t u = static_cast<uint64_t>(v) & mask;
  if (t.is_signed() && (u >> (t.bits - 1)) & 1) u |= ~mask;
  return static_cast<int64_t>(u);
}

uint16_t f64_to_f16_bits(double x) {
  const uint16_t sign = std::signbit(x) ? 0x8000 : 0;
  if (std::isnan(x)) return sign | 0x7e00;
  const double a = std::fabs(x);
  if (std::isinf(a)) return sign | 0x7c00;
  if (a == 0.0) return sign;
  int e2;
  std::frexp(a, &e2);
  int msb = e2 - 1;
  if (msb > 15) return sign | 0x7c00;
  const int ulp = msb < -14 ? -24 : msb - 10;
  double q = std::nearbyint(std::ldexp(a, -ulp));  // exact scaling, RNE
  if (msb < -14) return sign | static_cast<uint16_t>(q);
  if (q >= 2048.0) {
    q = 1024.0;
    ++msb;
  }
  if (msb > 15) return sign | 0x7c00;
  return sign | static_cast<uint16_t>(((msb + 15) << 10) | (static_cast<int>(q) - 1024));
}

double f16_bits_to_f64(uint16_t b) {
  const double s = (b & 0x8000) ? -1.0 : 1.0;
  const int e = (b >> 10) & 0x1f, f = b & 0x3ff;
  if (e == 0x1f) return f ? std::nan("") : s * HUGE_VAL;
  if (e == 0) return s * std::ldexp(static_cast<double>(f), -24);
  return s * std::ldexp(static_cast<double>(f | 0x400), e - 25);
}

double round_f16(double x) { return f16_bits_to_f64(f64_to_f16_bits(x)); }

// ============================ expressions ================================
namespace {
ExprPtr make(Expr::Kind k, DType t, std::vector<ExprPtr> args = {}) {
  auto e = std::make_shared<Expr>();
  e->kind = k;
  e->dtype = t;
  e->args = std::move(args);
  return e;
}
}  // namespace

ExprPtr int_imm(int64_t v, DType t) {
  auto e = std::make_shared<Expr>();
  e->kind = Expr::Kind::IntImm;
  e->dtype = t;
  e->ival = v;
  return e;
}
ExprPtr float_imm(double v, DType t) {
  auto e = std::make_shared<Expr>();
  e->kind = Expr::Kind::FloatImm;
  e->dtype = t;
  e->fval = v;
  return e;
}
ExprPtr var(const std::string& n) {
  auto e = std::make_shared<Expr>();
  e->kind = Expr::Kind::Var;
  e->name = n;
  return e;
}
ExprPtr load(const std::string& tensor, std::vector<ExprPtr> idx, DType t) {
  auto e = std::make_shared<Expr>();
  e->kind = Expr::Kind::Load;
  e->name = tensor;
  e->args = std::move(idx);
  e->dtype = t;
  return e;
}
ExprPtr cast(DType t, ExprPtr s) { return make(Expr::Kind::Cast, t, {std::move(s)}); }
// Binary nodes take the left operand's type (untyped until infer_types for
// parsed ops; typed when lowering builds `out + term` from typed parts).
ExprPtr add(ExprPtr a, ExprPtr b) {
  const DType t = a->dtype;
  return make(Expr::Kind::Add, t, {std::move(a), std::move(b)});
}
ExprPtr mul(ExprPtr a, ExprPtr b) {
  const DType t = a->dtype;
  return make(Expr::Kind::Mul, t, {std::move(a), std::move(b)});
}
ExprPtr floordiv(ExprPtr a, ExprPtr b) { return make(Expr::Kind::FloorDiv, kI32, {std::move(a), std::move(b)}); }
ExprPtr floormod(ExprPtr a, ExprPtr b) { return make(Expr::Kind::FloorMod, kI32, {std::move(a), std::move(b)}); }
ExprPtr ramp(ExprPtr base, int64_t stride, int64_t lanes) {
  auto e = std::const_pointer_cast<Expr>(make(Expr::Kind::Ramp, kI32, {std::move(base)}));
  e->ival = stride;
  e->lanes_arg = lanes;
  return e;
}
ExprPtr broadcast(ExprPtr v, int64_t lanes) {
  const DType t = v->dtype;  // read before the move below (argument order is unspecified)
  auto e = std::const_pointer_cast<Expr>(make(Expr::Kind::Broadcast, t, {std::move(v)}));
  e->lanes_arg = lanes;
  return e;
}
ExprPtr concat(std::vector<ExprPtr> parts) { return make(Expr::Kind::Concat, kI32, std::move(parts)); }

int64_t lanes_of(const ExprPtr& e) {
  switch (e->kind) {
    case Expr::Kind::Ramp:
    case Expr::Kind::Broadcast:
      return lanes_of(e->args[0]) * e->lanes_arg;
    case Expr::Kind::Concat: {
      int64_t n = 0;
      for (const auto& a : e->args) n += lanes_of(a);
      return n;
    }
    case Expr::Kind::Load:
      return e->args.size() == 1 ? lanes_of(e->args[0]) : 1;
    default:
      return 1;
  }
}

bool expr_equal(const ExprPtr& a, const ExprPtr& b, bool cmp_dtype) {
  if (a.get() == b.get()) return true;
  if (!a || !b || a->kind != b->kind) return false;
  if (cmp_dtype && a->dtype != b->dtype) return false;
  if (a->ival != b->ival || a->lanes_arg != b->lanes_arg || a->name != b->name) return false;
  if (a->kind == Expr::Kind::FloatImm && !(a->fval == b->fval)) return false;
  if (a->kind == Expr::Kind::Cast && a->dtype != b->dtype) return false;  // the cast target is semantic
  if (a->args.size() != b->args.size()) return false;
  for (size_t i = 0; i < a->args.size(); ++i)
    if (!expr_equal(a->args[i], b->args[i], cmp_dtype)) return false;
  return true;
}

ExprPtr substitute(const ExprPtr& e, const std::map<std::string, ExprPtr>& s) {
  if (e->kind == Expr::Kind::Var) {
    auto it = s.find(e->name);
    return it == s.end() ? e : it->second;
  }
  if (e->args.empty()) return e;
  auto c = std::make_shared<Expr>(*e);
  for (auto& a : c->args) a = substitute(a, s);
  return c;
}

void collect_vars(const ExprPtr& e, std::vector<std::string>* out) {
  if (e->kind == Expr::Kind::Var) {
    if (std::find(out->begin(), out->end(), e->name) == out->end()) out->push_back(e->name);
    return;
  }
  for (const auto& a : e->args) collect_vars(a, out);
}

bool contains_var(const ExprPtr& e, const std::string& n) {
  if (e->kind == Expr::Kind::Var) return e->name == n;
  for (const auto& a : e->args)
    if (contains_var(a, n)) return true;
  return false;
}

std::optional<AffineForm> linearize(const ExprPtr& e) {
  switch (e->kind) {
    case Expr::Kind::IntImm:
      return AffineForm{{}, e->ival};
    case Expr::Kind::Var:
      return AffineForm{{{e->name, 1}}, 0};
    case Expr::Kind::Add: {
      auto a = linearize(e->args[0]), b = linearize(e->args[1]);
      if (!a || !b) return std::nullopt;
      for (const auto& [v, c] : b->coeff) a->coeff[v] += c;
      a->constant += b->constant;
      for (auto it = a->coeff.begin(); it != a->coeff.end();) it = it->second == 0 ? a->coeff.erase(it) : std::next(it);
      return a;
    }
    case Expr::Kind::Mul: {
      auto a = linearize(e->args[0]), b = linearize(e->args[1]);
      if (!a || !b) return std::nullopt;
      if (!a->coeff.empty() && !b->coeff.empty()) return std::nullopt;  // product of variables
      const AffineForm& lin = a->coeff.empty() ? *b : *a;
      const int64_t k = a->coeff.empty() ? a->constant : b->constant;
      AffineForm r;
      for (const auto& [v, c] : lin.coeff)
        if (c * k != 0) r.coeff[v] = c * k;
      r.constant = lin.constant * k;
      return r;
    }
    default:
      return std::nullopt;
  }
}

namespace {
std::string float_text(double v) {
  char buf[64];
  std::snprintf(buf, sizeof buf, "%.17g", v);
  std::string s(buf);
  if (s.find_first_of(".eEn") == std::string::npos) s += ".0";
  return s;
}
int prec(const ExprPtr& e) {
  switch (e->kind) {
    case Expr::Kind::Add:
      return 1;
    case Expr::Kind::Mul:
    case Expr::Kind::FloorDiv:
    case Expr::Kind::FloorMod:
      return 2;
    default:
      return 3;
  }
}
}  // namespace

std::string expr_to_string(const ExprPtr& e) {
  auto wrap = [](const ExprPtr& c, int p) {
    std::string s = expr_to_string(c);
    return prec(c) < p ? "(" + s + ")" : s;
  };
  auto list = [](const std::vector<ExprPtr>& v) {
    std::string s;
    for (size_t i = 0; i < v.size(); ++i) s += (i ? ", " : "") + expr_to_string(v[i]);
    return s;
  };
  switch (e->kind) {
    case Expr::Kind::IntImm:
      return std::to_string(e->ival);
    case Expr::Kind::FloatImm:
      return float_text(e->fval);
    case Expr::Kind::Var:
      return e->name;
    case Expr::Kind::Load:
      return e->name + "[" + list(e->args) + "]";
    case Expr::Kind::Cast:
      return "cast<" + dtype_name(e->dtype) + ">(" + expr_to_string(e->args[0]) + ")";
    case Expr::Kind::Add:
      return wrap(e->args[0], 1) + " + " + wrap(e->args[1], 2);
    case Expr::Kind::Mul:
      return wrap(e->args[0], 2) + " * " + wrap(e->args[1], 3);
    case Expr::Kind::FloorDiv:
      return wrap(e->args[0], 2) + " / " + wrap(e->args[1], 3);  // reference spelling (src/expr.cpp:342-347)
    case Expr::Kind::FloorMod:
      return wrap(e->args[0], 2) + " % " + wrap(e->args[1], 3);
    case Expr::Kind::Ramp:
      return "ramp(" + expr_to_string(e->args[0]) + ", " + std::to_string(e->ival) + ", " + std::to_string(e->lanes_arg) + ")";
    case Expr::Kind::Broadcast:
      return "broadcast(" + expr_to_string(e->args[0]) + ", " + std::to_string(e->lanes_arg) + ")";
    case Expr::Kind::Concat:
      return "concat(" + list(e->args) + ")";
  }
  return "?";
}

// ============================ tensor ops =================================
const TensorDecl* ComputeOp::find_tensor(const std::string& n) const {
  for (const auto& t : tensors)
    if (t.name == n) return &t;
  return nullptr;
}
const LoopVar* ComputeOp::find_loop(const std::string& n) const {
  for (const auto& l : loops)
    if (l.name == n) return &l;
  return nullptr;
}
const TensorDecl& ComputeOp::output() const {
  for (const auto& t : tensors)
    if (t.role == Role::Output) return t;
  throw ValidationError("compute op has no output tensor");
}
std::vector<LoopVar> ComputeOp::loops_of_kind(LoopKind k) const {
  std::vector<LoopVar> r;
  for (const auto& l : loops)
    if (l.kind == k) r.push_back(l);
  return r;
}

namespace {

bool load_at(const ExprPtr& e, const std::string& t, const std::vector<ExprPtr>& idx) {
  if (e->kind != Expr::Kind::Load || e->name != t || e->args.size() != idx.size()) return false;
  for (size_t i = 0; i < idx.size(); ++i)
    if (!expr_equal(e->args[i], idx[i], false)) return false;
  return true;
}

void check_refs(const ComputeOp& op, const ExprPtr& e) {
  switch (e->kind) {
    case Expr::Kind::Var:
      if (!op.find_loop(e->name)) throw ValidationError("reference to undeclared loop '" + e->name + "'");
      return;
    case Expr::Kind::Load: {
      const TensorDecl* t = op.find_tensor(e->name);
      if (!t) throw ValidationError("load from undeclared tensor '" + e->name + "'");
      if (e->args.size() != t->shape.size())
        throw ValidationError("tensor '" + e->name + "' has rank " + std::to_string(t->shape.size()) +
                              " but is indexed with " + std::to_string(e->args.size()) + " subscripts");
      for (const auto& i : e->args) {
        check_refs(op, i);
        if (!linearize(i))
          throw ValidationError("non-affine index expression '" + expr_to_string(i) + "' on tensor '" + e->name + "'");
      }
      return;
    }
    case Expr::Kind::Ramp:
    case Expr::Kind::Broadcast:
    case Expr::Kind::Concat:
    case Expr::Kind::FloorDiv:
    case Expr::Kind::FloorMod:
      throw ValidationError("vector/lowered expression node in surface op");
    default:
      for (const auto& a : e->args) check_refs(op, a);
  }
}

void collect_loads(const ExprPtr& e, std::vector<const Expr*>* out) {
  if (e->kind == Expr::Kind::Load) out->push_back(e.get());
  for (const auto& a : e->args) collect_loads(a, out);
}

}  // namespace

void validate(const ComputeOp& op) {
  std::set<std::string> names;
  for (const auto& t : op.tensors) {
    if (t.name.empty()) throw ValidationError("tensor with empty name");
    if (!names.insert(t.name).second) throw ValidationError("duplicate declaration of '" + t.name + "'");
    if (t.shape.empty()) throw ValidationError("tensor '" + t.name + "' has empty shape");
    for (int64_t d : t.shape)
      if (d <= 0) throw ValidationError("tensor '" + t.name + "' has non-positive extent");
    if (!t.dtype.defined() || !t.dtype.is_scalar()) throw ValidationError("tensor '" + t.name + "' needs a scalar dtype");
  }
  for (const auto& l : op.loops) {
    if (l.name.empty()) throw ValidationError("loop with empty name");
    if (!names.insert(l.name).second) throw ValidationError("duplicate declaration of '" + l.name + "'");
    if (l.extent <= 0) throw ValidationError("loop '" + l.name + "' has non-positive extent");
  }
  int outputs = 0;
  for (const auto& t : op.tensors) outputs += t.role == Role::Output;
  if (outputs != 1) throw ValidationError("expected exactly one output tensor, found " + std::to_string(outputs));
  const TensorDecl* out = op.find_tensor(op.out);
  if (!out || out->role != Role::Output) throw ValidationError("store target '" + op.out + "' is not the output tensor");
  if (op.indices.size() != out->shape.size()) throw ValidationError("store index count does not match output rank");
  if (!op.value) throw ValidationError("missing stored value");
  for (const auto& idx : op.indices) {
    check_refs(op, idx);
    if (!linearize(idx)) throw ValidationError("non-affine store index '" + expr_to_string(idx) + "'");
    std::vector<std::string> vs;
    collect_vars(idx, &vs);
    for (const auto& v : vs) {
      const LoopVar* l = op.find_loop(v);
      if (l && l->kind == LoopKind::Reduction) throw ValidationError("reduction loop '" + v + "' used in store index");
    }
  }
  check_refs(op, op.value);
  std::vector<const Expr*> loads;
  collect_loads(op.value, &loads);
  for (const auto& l : op.loops) {
    if (l.kind != LoopKind::Reduction) continue;
    bool used = false;
    for (const Expr* ld : loads)
      for (const auto& i : ld->args) used = used || contains_var(i, l.name);
    if (!used) throw ValidationError("reduction loop '" + l.name + "' does not appear in any load");
  }
  if (op.update) {
    const bool canon = op.value->kind == Expr::Kind::Add &&
                       (load_at(op.value->args[0], op.out, op.indices) || load_at(op.value->args[1], op.out, op.indices));
    if (!canon) throw ValidationError("accumulate-form value must be 'output-load + term' at the top level");
  } else {
    for (const Expr* ld : loads)
      if (ld->name == op.out) throw ValidationError("output '" + op.out + "' read without accumulate form");
  }
}

namespace {
ExprPtr type_expr(const ComputeOp& op, const ExprPtr& e) {
  switch (e->kind) {
    case Expr::Kind::IntImm:
    case Expr::Kind::FloatImm:
      return e;
    case Expr::Kind::Var: {
      auto c = std::make_shared<Expr>(*e);
      c->dtype = kI32;
      return c;
    }
    case Expr::Kind::Load: {
      const TensorDecl* t = op.find_tensor(e->name);
      internal_check(t != nullptr, "typing an unvalidated op");
      auto c = std::make_shared<Expr>(*e);
      for (auto& i : c->args) {
        i = type_expr(op, i);
        if (!i->dtype.is_int()) throw TypeError("non-integer index on tensor '" + e->name + "'");
      }
      c->dtype = t->dtype;
      return c;
    }
    case Expr::Kind::Cast: {
      auto c = std::make_shared<Expr>(*e);
      c->args[0] = type_expr(op, e->args[0]);
      if (!c->dtype.defined()) throw TypeError("cast without target dtype");
      return c;
    }
    case Expr::Kind::Add:
    case Expr::Kind::Mul: {
      auto c = std::make_shared<Expr>(*e);
      c->args[0] = type_expr(op, e->args[0]);
      c->args[1] = type_expr(op, e->args[1]);
      if (c->args[0]->dtype != c->args[1]->dtype)
        throw TypeError(std::string(e->kind == Expr::Kind::Add ? "add" : "mul") + " operands disagree: " +
                        dtype_name(c->args[0]->dtype) + " vs " + dtype_name(c->args[1]->dtype) + " in '" +
                        expr_to_string(e) + "' (insert explicit casts)");
      c->dtype = c->args[0]->dtype;
      return c;
    }
    default:
      throw TypeError("unexpected node in surface expression");
  }
}
}  // namespace

ComputeOp infer_types(const ComputeOp& op) {
  ComputeOp r = op;
  for (auto& i : r.indices) i = type_expr(op, i);
  r.value = type_expr(op, r.value);
  if (r.value->dtype != op.output().dtype)
    throw TypeError("stored value is " + dtype_name(r.value->dtype) + " but output '" + op.out + "' is " +
                    dtype_name(op.output().dtype) + " (no implicit conversion)");
  return r;
}

ReduceForm reduce_form(const ComputeOp& op) {
  ReduceForm rf;
  bool has_red = false;
  for (const auto& l : op.loops) has_red = has_red || l.kind == LoopKind::Reduction;
  auto mentions_red = [&](const ExprPtr& e) {
    for (const auto& l : op.loops)
      if (l.kind == LoopKind::Reduction && contains_var(e, l.name)) return true;
    return false;
  };
  if (op.update) {
    const ExprPtr& l = op.value->args[0];
    const bool l_acc = l->kind == Expr::Kind::Load && l->name == op.out;
    rf.term = has_red ? (l_acc ? op.value->args[1] : l) : nullptr;
    return rf;
  }
  if (!has_red) return rf;
  if (op.value->kind == Expr::Kind::Add) {
    const bool lr = mentions_red(op.value->args[0]), rr = mentions_red(op.value->args[1]);
    if (lr != rr) {
      rf.init = lr ? op.value->args[1] : op.value->args[0];
      rf.term = lr ? op.value->args[0] : op.value->args[1];
      return rf;
    }
  }
  rf.term = op.value;
  return rf;
}

bool op_equal(const ComputeOp& a, const ComputeOp& b, bool cmp) {
  if (a.tensors.size() != b.tensors.size() || a.loops.size() != b.loops.size()) return false;
  for (size_t i = 0; i < a.tensors.size(); ++i) {
    const auto &x = a.tensors[i], &y = b.tensors[i];
    if (x.name != y.name || x.shape != y.shape || x.dtype != y.dtype || x.role != y.role) return false;
  }
  for (size_t i = 0; i < a.loops.size(); ++i) {
    const auto &x = a.loops[i], &y = b.loops[i];
    if (x.name != y.name || x.extent != y.extent || x.kind != y.kind) return false;
  }
  if (a.out != b.out || a.update != b.update || a.indices.size() != b.indices.size()) return false;
  for (size_t i = 0; i < a.indices.size(); ++i)
    if (!expr_equal(a.indices[i], b.indices[i], cmp)) return false;
  return expr_equal(a.value, b.value, cmp);
}

std::string print_compute(const ComputeOp& op) {
  std::string s;
  for (const auto& t : op.tensors) {
    s += "tensor " + t.name + " : " + dtype_name(t.dtype) + " [";
    for (size_t i = 0; i < t.shape.size(); ++i) s += (i ? ", " : "") + std::to_string(t.shape[i]);
    s += t.role == Role::Output ? "] output\n" : "] input\n";
  }
  for (const auto& l : op.loops)
    s += "loop " + l.name + " : " + (l.kind == LoopKind::DataParallel ? "dp " : "red ") + std::to_string(l.extent) + "\n";
  s += op.out + "[";
  for (size_t i = 0; i < op.indices.size(); ++i) s += (i ? ", " : "") + expr_to_string(op.indices[i]);
  s += "]";
  if (op.update) {
    const ExprPtr& l = op.value->args[0];
    const bool l_acc = l->kind == Expr::Kind::Load && l->name == op.out;
    s += " += " + expr_to_string(l_acc ? op.value->args[1] : l);
  } else {
    s += " = " + expr_to_string(op.value);
  }
  return s + "\n";
}

// ============================ parser =====================================
namespace {

struct Tok {
  enum K { Ident, Int, Float, Punct, End } k = End;
  std::string text;
  int64_t ival = 0;
  double fval = 0;
  int line = 1;
};

class Lexer {
 public:
  explicit Lexer(const std::string& s) : s_(s) { next_tok(); }
  const Tok& peek() const { return t_; }
  Tok take() {
    Tok r = t_;
    next_tok();
    return r;
  }
  bool punct(const char* p) {
    if (t_.k == Tok::Punct && t_.text == p) {
      next_tok();
      return true;
    }
    return false;
  }
  void need(const char* p) {
    if (!punct(p)) fail(std::string("expected '") + p + "'");
  }
  std::string ident(const char* what) {
    if (t_.k != Tok::Ident) fail(std::string("expected ") + what);
    return take().text;
  }
  int64_t integer(const char* what) {
    if (t_.k != Tok::Int) fail(std::string("expected ") + what);
    return take().ival;
  }
  [[noreturn]] void fail(const std::string& m) const {
    throw SyntaxError("line " + std::to_string(t_.line) + ": " + m + ", got " +
                      (t_.k == Tok::End ? std::string("end of input") : "'" + t_.text + "'"));
  }

 private:
  void next_tok() {
    for (;;) {
      if (i_ >= s_.size()) break;
      const char c = s_[i_];
      if (c == '\n') {
        ++line_;
        ++i_;
      } else if (std::isspace(static_cast<unsigned char>(c))) {
        ++i_;
      } else if (c == '#') {
        while (i_ < s_.size() && s_[i_] != '\n') ++i_;
      } else {
        break;
      }
    }
    t_ = Tok{};
    t_.line = line_;
    if (i_ >= s_.size()) return;
    const char c = s_[i_];
    const size_t b = i_;
    if (std::isalpha(static_cast<unsigned char>(c)) || c == '_') {
      while (i_ < s_.size() && (std::isalnum(static_cast<unsigned char>(s_[i_])) || s_[i_] == '_' || s_[i_] == '.')) ++i_;
      t_.k = Tok::Ident;
      t_.text = s_.substr(b, i_ - b);
      return;
    }
    if (std::isdigit(static_cast<unsigned char>(c))) {
      bool fl = false;
      while (i_ < s_.size()) {
        const char d = s_[i_];
        if (std::isdigit(static_cast<unsigned char>(d))) {
          ++i_;
        } else if (d == '.' || d == 'e' || d == 'E') {
          fl = true;
          ++i_;
          if ((d == 'e' || d == 'E') && i_ < s_.size() && (s_[i_] == '+' || s_[i_] == '-')) ++i_;
        } else {
          break;
        }
      }
      t_.text = s_.substr(b, i_ - b);
      if (fl) {
        t_.k = Tok::Float;
        t_.fval = std::strtod(t_.text.c_str(), nullptr);
      } else {
        t_.k = Tok::Int;
        t_.ival = std::strtoll(t_.text.c_str(), nullptr, 10);
      }
      return;
    }
    if (c == '+' && i_ + 1 < s_.size() && s_[i_ + 1] == '=') {
      t_.k = Tok::Punct;
      t_.text = "+=";
      i_ += 2;
      return;
    }
    if (std::string(":[](),+*<>=").find(c) != std::string::npos) {
      t_.k = Tok::Punct;
      t_.text = std::string(1, c);
      ++i_;
      return;
    }
    throw SyntaxError("line " + std::to_string(line_) + ": unexpected character '" + std::string(1, c) + "'");
  }
  const std::string& s_;
  size_t i_ = 0;
  int line_ = 1;
  Tok t_;
};

class Parser {
 public:
  explicit Parser(const std::string& s) : lx_(s) {}
  ComputeOp run() {
    ComputeOp op;
    bool stored = false;
    while (lx_.peek().k != Tok::End) {
      if (stored) lx_.fail("store statement must be the last statement");
      const Tok& t = lx_.peek();
      if (t.k == Tok::Ident && t.text == "tensor")
        tensor(&op);
      else if (t.k == Tok::Ident && t.text == "loop")
        loop(&op);
      else {
        store(&op);
        stored = true;
      }
    }
    if (!stored) throw SyntaxError("missing store statement");
    validate(op);
    return op;
  }

 private:
  void tensor(ComputeOp* op) {
    lx_.take();
    TensorDecl t;
    t.name = lx_.ident("tensor name");
    lx_.need(":");
    t.dtype = dtype_from_name(lx_.ident("dtype"));
    lx_.need("[");
    t.shape.push_back(lx_.integer("extent"));
    while (lx_.punct(",")) t.shape.push_back(lx_.integer("extent"));
    lx_.need("]");
    const std::string role = lx_.ident("'input' or 'output'");
    if (role == "input")
      t.role = Role::Input;
    else if (role == "output")
      t.role = Role::Output;
    else
      lx_.fail("expected 'input' or 'output'");
    op->tensors.push_back(std::move(t));
  }
  void loop(ComputeOp* op) {
    lx_.take();
    LoopVar l;
    l.name = lx_.ident("loop name");
    lx_.need(":");
    const std::string k = lx_.ident("'dp' or 'red'");
    if (k == "dp")
      l.kind = LoopKind::DataParallel;
    else if (k == "red")
      l.kind = LoopKind::Reduction;
    else
      lx_.fail("expected 'dp' or 'red'");
    l.extent = lx_.integer("loop extent");
    op->loops.push_back(std::move(l));
  }
  void store(ComputeOp* op) {
    op->out = lx_.ident("store target");
    lx_.need("[");
    op->indices.push_back(expr());
    while (lx_.punct(",")) op->indices.push_back(expr());
    lx_.need("]");
    if (lx_.punct("+=")) {
      op->update = true;
      op->value = add(load(op->out, op->indices), expr());  // canonical: accumulator on the left
    } else {
      lx_.need("=");
      op->value = expr();
    }
  }
  ExprPtr expr() {
    ExprPtr e = term();
    while (lx_.punct("+")) e = add(e, term());
    return e;
  }
  ExprPtr term() {
    ExprPtr e = factor();
    while (lx_.punct("*")) e = mul(e, factor());
    return e;
  }
  ExprPtr factor() {
    const Tok& t = lx_.peek();
    if (t.k == Tok::Int) return int_imm(lx_.take().ival);
    if (t.k == Tok::Float) return float_imm(lx_.take().fval);
    if (lx_.punct("(")) {
      ExprPtr e = expr();
      lx_.need(")");
      return e;
    }
    if (t.k == Tok::Ident) {
      if (t.text == "cast") {
        lx_.take();
        lx_.need("<");
        const DType d = dtype_from_name(lx_.ident("dtype"));
        lx_.need(">");
        lx_.need("(");
        ExprPtr e = expr();
        lx_.need(")");
        return cast(d, e);
      }
      const std::string n = lx_.take().text;
      if (lx_.punct("[")) {
        std::vector<ExprPtr> idx{expr()};
        while (lx_.punct(",")) idx.push_back(expr());
        lx_.need("]");
        return load(n, std::move(idx));
      }
      return var(n);
    }
    lx_.fail("expected expression");
  }
  Lexer lx_;
};

}  // namespace

ComputeOp parse_compute(const std::string& text) { return Parser(text).run(); }

}  // namespace tzc
