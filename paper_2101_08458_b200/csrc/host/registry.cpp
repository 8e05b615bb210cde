// tzc host library, part 2: the instruction-semantics registry.
//
// An instruction description (SPEC.md "Intrinsic definition file (.intr)") is
// three kinds of line: the semantics block in the .tdsl grammar (parsed by
// parse_compute), one "rule <register>: kind(loop) ..." line per input
// register saying how its lanes are filled from memory, and one
// `mnemonic "<text>"` line naming the target instruction.  Entry points
// replaced: /root/reference/proj/include/tzc/intrinsics.hpp:15-65 (same
// names, arguments and error kinds: SyntaxError for malformed lines,
// RuleError for rules inconsistent with the semantics, UnknownIntrinsic /
// IoError from resolve / load).
//
// Builtins: the reference's three CPU descriptions (restated below in the
// .intr grammar) plus the sm_100a tcgen05.mma descriptions this backend
// executes.  The tcgen05 texts are ordinary .intr programs (SURVEY.md F5:
// the reference's own parse / inspect / inject accept them unmodified).
#include <cctype>
#include <cstring>
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
// Does expression e load tensor t at exactly the index list idx anywhere?
bool loads_at(const ExprPtr& e, const std::string& t, const std::vector<ExprPtr>& idx) {
  if (e->kind == Expr::Kind::Load && e->name == t && e->args.size() == idx.size()) {
    size_t i = 0;
    while (i < idx.size() && expr_equal(e->args[i], idx[i], false)) ++i;
    if (i == idx.size()) return true;
  }
  for (const auto& a : e->args)
    if (loads_at(a, t, idx)) return true;
  return false;
}
}  // namespace

// The register the instruction accumulates into: the output for "+=" forms,
// else the input read at the store's own index (d[i] = c[i] + ...).
std::string Intrinsic::accumulator() const {
  if (semantics.update) return semantics.out;
  for (const auto& t : semantics.tensors)
    if (t.role == Role::Input && loads_at(semantics.value, t.name, semantics.indices)) return t.name;
  return "";
}

// Consistency of the operand rules with the semantics: every input register
// has exactly one non-empty rule list; each rule names a loop of the
// semantics and spans its whole extent; the lanes the rules enumerate are
// exactly the register's element count.
void validate_intrinsic(const Intrinsic& intr) {
  if (intr.name.empty()) throw RuleError("an intrinsic needs a name");
  validate(intr.semantics);
  if (intr.requires_inplace_acc != intr.semantics.update)
    throw RuleError("requires_inplace_acc must equal the semantics' update (+=) form");
  std::map<std::string, const TensorDecl*> pending;  // input registers still without rules
  for (const auto& t : intr.semantics.tensors)
    if (t.role == Role::Input) pending[t.name] = &t;
  std::set<std::string> ruled;
  for (const auto& [reg, rules] : intr.operand_rules) {
    const TensorDecl* t = intr.semantics.find_tensor(reg);
    const std::string where = "operand rules of '" + reg + "'";
    if (!t) throw RuleError(where + ": no such tensor in the semantics");
    if (t->role != Role::Input) throw RuleError(where + ": only input registers take rules");
    if (!ruled.insert(reg).second) throw RuleError(where + ": given twice");
    if (rules.empty()) throw RuleError(where + ": empty");
    pending.erase(reg);
    int64_t lanes = 1;
    for (const auto& r : rules) {
      if (r.kind == OperandRule::Kind::Passthrough) {
        if (!r.loop.empty()) throw RuleError(where + ": passthrough has no loop argument");
        continue;
      }
      const LoopVar* l = intr.semantics.find_loop(r.loop);
      if (!l) throw RuleError(where + ": loop '" + r.loop + "' is not a loop of the semantics");
      if (r.count != l->extent)
        throw RuleError(where + ": " + OperandRule::kind_name(r.kind) + "(" + r.loop + ") spans " +
                        std::to_string(r.count) + " lanes, the loop's extent is " + std::to_string(l->extent));
      lanes *= r.count;
    }
    if (lanes != t->size())
      throw RuleError(where + ": the rules enumerate " + std::to_string(lanes) + " lanes, the register has " +
                      std::to_string(t->size()) + " elements");
  }
  if (!pending.empty()) throw RuleError("input register '" + pending.begin()->first + "' has no operand rules");
}

namespace {

std::string strip(const std::string& s) {
  const size_t b = s.find_first_not_of(" \t\r");
  if (b == std::string::npos) return "";
  return s.substr(b, s.find_last_not_of(" \t\r") - b + 1);
}

bool starts_with(const std::string& s, const char* word) { return s.compare(0, std::strlen(word), word) == 0; }

// "rule <register>: kind(loop) kind(loop) ..." -> (register, rules); the
// lane counts are filled from the semantics' loop extents (0 for a loop the
// semantics lacks, which validate_intrinsic then reports).
std::pair<std::string, std::vector<OperandRule>> parse_rule_line(const std::string& line, const ComputeOp& sem) {
  const std::string body = line.substr(4);  // after "rule"
  const size_t colon = body.find(':');
  if (colon == std::string::npos) throw SyntaxError("rule line '" + line + "': expected 'rule <register>: ...'");
  const std::string reg = strip(body.substr(0, colon));
  if (reg.empty()) throw SyntaxError("rule line '" + line + "': missing register name");
  static const std::map<std::string, OperandRule::Kind> kinds = {
      {"vectorize", OperandRule::Kind::Vectorize},
      {"broadcast", OperandRule::Kind::Broadcast},
      {"unroll_concat", OperandRule::Kind::UnrollConcat},
      {"passthrough", OperandRule::Kind::Passthrough}};
  std::vector<OperandRule> rules;
  std::istringstream words(body.substr(colon + 1));
  for (std::string w; words >> w;) {
    const size_t open = w.find('(');
    const std::string kw = w.substr(0, open);
    auto k = kinds.find(kw);
    if (k == kinds.end()) throw SyntaxError("rule line '" + line + "': unknown rule kind '" + kw + "'");
    OperandRule r;
    r.kind = k->second;
    if (r.kind != OperandRule::Kind::Passthrough) {
      if (open == std::string::npos || w.back() != ')')
        throw SyntaxError("rule line '" + line + "': " + kw + " takes a loop, as " + kw + "(<loop>)");
      r.loop = w.substr(open + 1, w.size() - open - 2);
      const LoopVar* l = sem.find_loop(r.loop);
      r.count = l ? l->extent : 0;
    }
    rules.push_back(std::move(r));
  }
  return {reg, std::move(rules)};
}

}  // namespace

Intrinsic parse_intrinsic(const std::string& text, const std::string& name) {
  std::string semantics;
  std::vector<std::string> rule_lines;
  std::vector<std::string> mnemonics;
  std::istringstream in(text);
  for (std::string raw; std::getline(in, raw);) {
    const std::string t = strip(raw);
    if (starts_with(t, "rule"))
      rule_lines.push_back(t);
    else if (starts_with(t, "mnemonic"))
      mnemonics.push_back(t);
    else
      semantics += raw + "\n";  // everything else is the .tdsl block
  }
  if (mnemonics.empty()) throw SyntaxError("instruction description '" + name + "' has no mnemonic line");
  std::string mnemonic;
  for (const auto& m : mnemonics) {  // the last one wins
    const size_t first = m.find('"'), last = m.rfind('"');
    if (first == std::string::npos || last == first)
      throw SyntaxError("mnemonic line '" + m + "': expected mnemonic \"<text>\"");
    mnemonic = m.substr(first + 1, last - first - 1);
  }
  Intrinsic intr;
  intr.name = name;
  intr.semantics = infer_types(parse_compute(semantics));
  intr.target_mnemonic = mnemonic;
  intr.requires_inplace_acc = intr.semantics.update;
  for (const auto& rl : rule_lines) intr.operand_rules.push_back(parse_rule_line(rl, intr.semantics));
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
std::string tcgen05_text(bool f16, int n, bool mn_major, int m = 128) {
  const int k = f16 ? 16 : 32;
  const std::string da = f16 ? "fp16" : "u8", db = f16 ? "fp16" : "i8", dd = f16 ? "fp32" : "i32";
  const std::string bshape = mn_major ? "[" + std::to_string(k) + ", " + std::to_string(n) + "]"
                                      : "[" + std::to_string(n) + ", " + std::to_string(k) + "]";
  std::ostringstream os;
  os << "tensor a : " << da << " [" << m << ", " << k << "] input\n"
     << "tensor b : " << db << " " << bshape << " input\n"
     << "tensor d : " << dd << " [" << m << ", " << n << "] output\n"
     << "loop m : dp " << m << "\nloop n : dp " << n << "\nloop k : red " << k << "\n"
     << "d[m, n] += cast<" << dd << ">(a[m, k]) * cast<" << dd << ">(" << (mn_major ? "b[k, n]" : "b[n, k]") << ")\n"
     << "rule a: vectorize(k) unroll_concat(m)\n"
     << (mn_major ? "rule b: vectorize(n) unroll_concat(k)\n" : "rule b: vectorize(k) unroll_concat(n)\n")
     << "mnemonic \"tcgen05.mma.cta_group::" << (m == 256 ? 2 : 1) << ".kind::" << (f16 ? "f16" : "i8") << " m" << m
     << "n" << n << "k" << k
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
    // cta_group::2: one MMA over a CTA pair's 256 rows (conv_tc2.cuh; each
    // CTA loads its 128 A rows and half of B)
    for (int n : {128, 256}) {
      const std::string nm = "tcgen05_i8_m256n" + std::to_string(n) + "k32";
      m.emplace(nm, parse_intrinsic(tcgen05_text(false, n, false, 256), nm));
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
