// tzc host library, part 2: the instruction-semantics registry.
// Same contract as the reference (/root/reference/proj/src/intrinsics.cpp:
// Intrinsic::accumulator :35-57, validate_intrinsic :59-101, .intr grammar
// :185-272, resolve :287-296), with the sm_100a tcgen05 descriptions added as
// builtins.  The tcgen05 texts are ordinary .intr programs in the reference's
// own grammar (they pass the reference's parse/inspect/inject
// unmodified).
#include <cctype>
#include <fstream>
#include <map>
#include <set>
#include <sstream>

#include "tzc/tzc.hpp"

namespace tzc {

std::string OperandRule::kind_name(Kind k) {
  switch (k) {
    case Kind::Vectorize: return "vectorize";
    case Kind::Broadcast: return "broadcast";
    case Kind::UnrollConcat: return "unroll_concat";
    case Kind::Passthrough: return "passthrough";
  }
  return "?";
}

const std::vector<OperandRule>* Intrinsic::rules_for(const std::string& t) const {
  for (const auto& [n, r] : operand_rules)
    if (n == t) return &r;
  return nullptr;
}

namespace {
bool loads_at(const ExprPtr& e, const std::string& t, const std::vector<ExprPtr>& idx) {
  if (e->kind == Expr::Kind::Load && e->name == t && e->args.size() == idx.size()) {
    bool same = true;
    for (size_t i = 0; i < idx.size(); ++i) same = same && expr_equal(e->args[i], idx[i], false);
    if (same) return true;
  }
  for (const auto& a : e->args)
    if (loads_at(a, t, idx)) return true;
  return false;
}
}  // namespace

std::string Intrinsic::accumulator() const {
  if (semantics.update) return semantics.out;
  for (const auto& t : semantics.tensors)
    if (t.role == Role::Input && loads_at(semantics.value, t.name, semantics.indices)) return t.name;
  return "";
}

void validate_intrinsic(const Intrinsic& intr) {
  if (intr.name.empty()) throw RuleError("intrinsic without a name");
  validate(intr.semantics);
  if (intr.requires_inplace_acc != intr.semantics.update)
    throw RuleError("requires_inplace_acc must mirror accumulate-form semantics");
  std::set<std::string> seen;
  for (const auto& [tensor, rules] : intr.operand_rules) {
    const TensorDecl* t = intr.semantics.find_tensor(tensor);
    if (!t) throw RuleError("rule for unknown tensor '" + tensor + "'");
    if (t->role != Role::Input) throw RuleError("rule for non-input tensor '" + tensor + "'");
    if (!seen.insert(tensor).second) throw RuleError("duplicate rule for tensor '" + tensor + "'");
    if (rules.empty()) throw RuleError("empty rule list for tensor '" + tensor + "'");
    int64_t lanes = 1;
    for (const auto& r : rules) {
      if (r.kind == OperandRule::Kind::Passthrough) {
        if (!r.loop.empty()) throw RuleError("passthrough takes no loop argument");
        continue;
      }
      const LoopVar* l = intr.semantics.find_loop(r.loop);
      if (!l) throw RuleError("rule on tensor '" + tensor + "' references unknown loop '" + r.loop + "'");
      if (r.count != l->extent)
        throw RuleError("rule count " + std::to_string(r.count) + " on '" + tensor + "' must equal extent of loop '" +
                        r.loop + "' (" + std::to_string(l->extent) + ")");
      lanes *= r.count;
    }
    if (lanes != t->size())
      throw RuleError("rules on '" + tensor + "' cover " + std::to_string(lanes) + " lanes but the register holds " +
                      std::to_string(t->size()));
  }
  for (const auto& t : intr.semantics.tensors)
    if (t.role == Role::Input && !seen.count(t.name)) throw RuleError("input tensor '" + t.name + "' has no operand rule");
}

Intrinsic parse_intrinsic(const std::string& text, const std::string& name) {
  std::string sem;
  std::vector<std::string> rule_lines;
  std::string mnemonic;
  bool have_mnemonic = false;
  std::istringstream in(text);
  std::string line;
  while (std::getline(in, line)) {
    const size_t b = line.find_first_not_of(" \t");
    const std::string t = b == std::string::npos ? "" : line.substr(b);
    if (t.rfind("rule", 0) == 0) {
      rule_lines.push_back(t);
    } else if (t.rfind("mnemonic", 0) == 0) {
      const size_t q1 = t.find('"'), q2 = t.rfind('"');
      if (q1 == std::string::npos || q2 <= q1) throw SyntaxError("mnemonic line must carry a quoted string");
      mnemonic = t.substr(q1 + 1, q2 - q1 - 1);
      have_mnemonic = true;
    } else {
      sem += line + "\n";
    }
  }
  if (!have_mnemonic) throw SyntaxError("intrinsic description lacks a mnemonic");
  Intrinsic intr;
  intr.name = name;
  intr.semantics = infer_types(parse_compute(sem));
  intr.target_mnemonic = mnemonic;
  intr.requires_inplace_acc = intr.semantics.update;
  for (const auto& rl : rule_lines) {
    // rule <tensor>: kind(loop) kind(loop) ...
    std::string body = rl.substr(4);
    const size_t colon = body.find(':');
    if (colon == std::string::npos) throw SyntaxError("rule line without ':'");
    std::string tensor = body.substr(0, colon);
    tensor.erase(0, tensor.find_first_not_of(" \t"));
    tensor.erase(tensor.find_last_not_of(" \t") + 1);
    if (tensor.empty()) throw SyntaxError("rule line without tensor name");
    std::istringstream items(body.substr(colon + 1));
    std::vector<OperandRule> rules;
    std::string item;
    while (items >> item) {
      OperandRule r;
      const size_t p = item.find('(');
      const std::string kind = p == std::string::npos ? item : item.substr(0, p);
      if (kind == "vectorize")
        r.kind = OperandRule::Kind::Vectorize;
      else if (kind == "broadcast")
        r.kind = OperandRule::Kind::Broadcast;
      else if (kind == "unroll_concat")
        r.kind = OperandRule::Kind::UnrollConcat;
      else if (kind == "passthrough")
        r.kind = OperandRule::Kind::Passthrough;
      else
        throw SyntaxError("unknown rule kind '" + kind + "'");
      if (r.kind != OperandRule::Kind::Passthrough) {
        if (p == std::string::npos || item.back() != ')') throw SyntaxError("rule '" + kind + "' needs a loop argument");
        r.loop = item.substr(p + 1, item.size() - p - 2);
        const LoopVar* l = intr.semantics.find_loop(r.loop);
        r.count = l ? l->extent : 0;
      }
      rules.push_back(std::move(r));
    }
    intr.operand_rules.emplace_back(tensor, std::move(rules));
  }
  validate_intrinsic(intr);
  return intr;
}

namespace {

// The reference's three builtins (proj/src/intrinsics.cpp:113-156 define the
// same instruction semantics; texts written here in the .intr grammar).
const char* kVdot16x4 =
    "tensor a : u8 [64] input\ntensor b : i8 [64] input\ntensor c : i32 [16] input\ntensor d : i32 [16] output\n"
    "loop i : dp 16\nloop j : red 4\n"
    "d[i] = c[i] + cast<i32>(a[i * 4 + j]) * cast<i32>(b[i * 4 + j])\n"
    "rule a: vectorize(j) broadcast(i)\nrule b: vectorize(j) unroll_concat(i)\nrule c: vectorize(i)\n"
    "mnemonic \"llvm.x86.avx512.vpdpbusd.512\"\n";
const char* kVdot4x4 =
    "tensor a : u8 [16] input\ntensor b : i8 [16] input\ntensor c : i32 [4] input\ntensor d : i32 [4] output\n"
    "loop i : dp 4\nloop j : red 4\n"
    "d[i] = c[i] + cast<i32>(a[i * 4 + j]) * cast<i32>(b[i * 4 + j])\n"
    "rule a: vectorize(j) broadcast(i)\nrule b: vectorize(j) unroll_concat(i)\nrule c: vectorize(i)\n"
    "mnemonic \"llvm.aarch64.neon.usdot.v4i32.v16i8\"\n";
const char* kWmma16 =
    "tensor a : fp16 [16, 16] input\ntensor b : fp16 [16, 16] input\ntensor c : fp32 [16, 16] output\n"
    "loop x : dp 16\nloop y : dp 16\nloop k : red 16\n"
    "c[x, y] += cast<fp32>(a[x, k]) * cast<fp32>(b[k, y])\n"
    "rule a: vectorize(k) unroll_concat(x)\nrule b: vectorize(y) unroll_concat(k)\n"
    "mnemonic \"llvm.nvvm.wmma.m16n16k16.mma.row.row.f32.f32\"\n";

// tcgen05.mma (sm_100a): one CTA-wide MMA, D in TMEM (+= in place), A/B in
// shared memory.  kind::i8: u8 x s8 -> s32, K = 32 per instruction (256 bits).
// kind::f16: f16 x f16 -> f32, K = 16.  B K-major (b[n,k]) or MN-major (b[k,n]).
std::string tcgen05_text(bool f16, int n, bool mn_major) {
  const int k = f16 ? 16 : 32;
  const std::string da = f16 ? "fp16" : "u8", db = f16 ? "fp16" : "i8", dd = f16 ? "fp32" : "i32";
  const std::string bshape = mn_major ? "[" + std::to_string(k) + ", " + std::to_string(n) + "]"
                                      : "[" + std::to_string(n) + ", " + std::to_string(k) + "]";
  std::ostringstream os;
  os << "tensor a : " << da << " [128, " << k << "] input\n"
     << "tensor b : " << db << " " << bshape << " input\n"
     << "tensor d : " << dd << " [128, " << n << "] output\n"
     << "loop m : dp 128\nloop n : dp " << n << "\nloop k : red " << k << "\n"
     << "d[m, n] += cast<" << dd << ">(a[m, k]) * cast<" << dd << ">(" << (mn_major ? "b[k, n]" : "b[n, k]") << ")\n"
     << "rule a: vectorize(k) unroll_concat(m)\n"
     << (mn_major ? "rule b: vectorize(n) unroll_concat(k)\n" : "rule b: vectorize(k) unroll_concat(n)\n")
     << "mnemonic \"tcgen05.mma.cta_group::1.kind::" << (f16 ? "f16" : "i8") << " m128n" << n << "k" << k
     << (mn_major ? " b.mn_major" : "") << "\"\n";
  return os.str();
}

const std::map<std::string, Intrinsic>& table() {
  static const std::map<std::string, Intrinsic> t = [] {
    std::map<std::string, Intrinsic> m;
    m.emplace("vdot_16x4", parse_intrinsic(kVdot16x4, "vdot_16x4"));
    m.emplace("vdot_4x4", parse_intrinsic(kVdot4x4, "vdot_4x4"));
    m.emplace("wmma_16x16x16", parse_intrinsic(kWmma16, "wmma_16x16x16"));
    for (int n : {64, 128, 256}) {
      const std::string ns = std::to_string(n);
      m.emplace("tcgen05_i8_m128n" + ns + "k32", parse_intrinsic(tcgen05_text(false, n, false), "tcgen05_i8_m128n" + ns + "k32"));
      m.emplace("tcgen05_f16_m128n" + ns + "k16", parse_intrinsic(tcgen05_text(true, n, false), "tcgen05_f16_m128n" + ns + "k16"));
      m.emplace("tcgen05_f16_m128n" + ns + "k16_mn",
                parse_intrinsic(tcgen05_text(true, n, true), "tcgen05_f16_m128n" + ns + "k16_mn"));
    }
    return m;
  }();
  return t;
}

}  // namespace

const Intrinsic& builtin(const std::string& name) {
  auto it = table().find(name);
  if (it == table().end()) throw UnknownIntrinsic("no built-in intrinsic named '" + name + "'");
  return it->second;
}

std::vector<std::string> builtin_names() {
  std::vector<std::string> v;
  for (const auto& kv : table()) v.push_back(kv.first);
  return v;
}

Intrinsic load_intrinsic(const std::string& path) {
  std::ifstream f(path);
  if (!f) throw IoError("cannot open intrinsic file '" + path + "'");
  std::stringstream ss;
  ss << f.rdbuf();
  std::string stem = path.substr(path.find_last_of("/\\") == std::string::npos ? 0 : path.find_last_of("/\\") + 1);
  if (stem.rfind('.') != std::string::npos) stem = stem.substr(0, stem.rfind('.'));
  return parse_intrinsic(ss.str(), stem);
}

Intrinsic resolve_intrinsic(const std::string& ref) {
  if (ref.size() > 5 && ref.compare(ref.size() - 5, 5, ".intr") == 0) return load_intrinsic(ref);
  auto it = table().find(ref);
  if (it != table().end()) return it->second;
  std::ifstream probe(ref);
  if (probe) return load_intrinsic(ref);
  throw UnknownIntrinsic("'" + ref + "' is neither a built-in nor a readable file");
}

std::string print_intrinsic(const Intrinsic& intr) {
  std::string s = "# intrinsic " + intr.name + "\n" + print_compute(intr.semantics);
  for (const auto& [t, rules] : intr.operand_rules) {
    s += "rule " + t + ":";
    for (const auto& r : rules) {
      s += " " + OperandRule::kind_name(r.kind);
      if (r.kind != OperandRule::Kind::Passthrough) s += "(" + r.loop + ")";
    }
    s += "\n";
  }
  return s + "mnemonic \"" + intr.target_mnemonic + "\"\n";
}

}  // namespace tzc
