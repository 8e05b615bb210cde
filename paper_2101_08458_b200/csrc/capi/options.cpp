// Plan options: the process defaults (tzc_b200_set_option) and the
// per-descriptor overrides installed by the measured tuner
// (tzc_b200_tune_* / tzc_b200_set_problem_options_*).
//
// A launch never reads shared mutable state while it plans: options_for()
// copies the defaults and applies the descriptor's overrides under one lock,
// and the resulting Options value is passed down through plan_problem /
// run_problem.  Options choose the kernel plan only, never the results.
#include <cstdio>
#include <cstdlib>
#include <map>
#include <cstring>
#include <fstream>
#include <mutex>
#include <sstream>
#include <string>
#include <utility>
#include <vector>

#include "../tzc_b200_internal.hpp"

namespace tzcb200 {
namespace {

// name -> field, legal range; an out-of-range value is rejected (the old
// behaviour silently clamped, which hid typos in tuning specs).
struct Knob {
  const char* name;
  int Options::*field;
  int64_t lo, hi;
  const int* allowed;  // optional explicit set (terminated by -1)
};
constexpr int kMtAllowed[] = {0, 1, 2, 4, -1};
constexpr int kBnAllowed[] = {0, 64, 128, 256, -1};
constexpr int kEgAllowed[] = {0, 1, 2, -1};
const Knob kKnobs[] = {
    {"splits", &Options::splits, 0, 1 << 16, nullptr},
    {"shifted_window", &Options::shifted_window, 0, 1, nullptr},
    {"ws_epi_groups", &Options::ws_epi_groups, 0, 2, kEgAllowed},
    {"tail_split", &Options::tail_split, 0, 1, nullptr},
    {"split_min_kb", &Options::split_min_kb, 0, 1 << 20, nullptr},
    {"splitk_inkernel", &Options::splitk_inkernel, 0, 1, nullptr},
    {"pingpong_kb", &Options::pingpong_kb, 0, 1 << 20, nullptr},
    {"ws_mt", &Options::ws_mt, 0, 4, kMtAllowed},
    {"ws_1x1_k", &Options::ws_1x1_k, 0, 1 << 20, nullptr},
    {"ws_1x1", &Options::ws_1x1, 0, 1, nullptr},
    {"bn", &Options::bn, 0, 256, kBnAllowed},
    {"tma_store_k", &Options::tma_store_k, 0, 1 << 20, nullptr},
    {"pair_min_kb", &Options::pair_min_kb, 0, 1 << 20, nullptr},
    {"pair_bn", &Options::pair_bn, 0, 256, nullptr},
    {"pair_min_round", &Options::pair_min_round, 0, 64, nullptr},
    {"s2d_one", &Options::s2d_one, 0, 1, nullptr},
    {"l2_a_max_out_mb", &Options::l2_a_max_out_mb, 0, 1 << 20, nullptr},
    {"producers", &Options::producers, 1, 2, nullptr},
    {"pair", &Options::pair, 0, 1, nullptr},
    {"st256", &Options::st256, 0, 1, nullptr},
    {"l2_hints", &Options::l2_hints, 0, 3, nullptr},
    {"tma_store", &Options::tma_store, 0, 2, nullptr},
    {"b_res", &Options::b_res, 0, 2, nullptr},
    {"stem_fused", &Options::stem_fused, 0, 1, nullptr},
};

std::mutex g_mu;
Options g_defaults = [] {
  Options o;
  if (std::getenv("TZC_B200_NO_WS")) o.shifted_window = 0;
  return o;
}();
// descriptor key -> validated overrides, applied on the defaults at each call
std::map<std::string, std::vector<std::pair<std::string, int64_t>>> g_problem;

}  // namespace

bool apply_option(Options* o, const std::string& name, int64_t value, std::string* err) {
  for (const Knob& k : kKnobs) {
    if (name != k.name) continue;
    bool ok = value >= k.lo && value <= k.hi;
    if (ok && k.allowed) {
      ok = false;
      for (const int* a = k.allowed; *a >= 0; ++a) ok = ok || value == *a;
    }
    if (!ok) {
      if (err) *err = "option '" + name + "': illegal value " + std::to_string(value);
      return false;
    }
    o->*k.field = (int)value;
    return true;
  }
  if (err) *err = "unknown option '" + name + "'";
  return false;
}

const char* const* option_names() {
  static const std::vector<const char*> names = [] {
    std::vector<const char*> v;
    for (const Knob& k : kKnobs) v.push_back(k.name);
    v.push_back(nullptr);
    return v;
  }();
  return names.data();
}

Status load_problem_options(const std::string& path, int* count);
namespace {
std::once_flag g_cache_once;
// TZC_B200_PLAN_CACHE=<file>: install a saved plan cache before the first launch
void autoload_plan_cache() {
  std::call_once(g_cache_once, [] {
    const char* path = std::getenv("TZC_B200_PLAN_CACHE");
    if (!path || !*path) return;
    int n = 0;
    Status st = load_problem_options(path, &n);
    if (!st.ok()) std::fprintf(stderr, "tzc_b200: TZC_B200_PLAN_CACHE not loaded: %s\n", st.msg.c_str());
  });
}
}  // namespace

Options options_for(const std::string& key) {
  autoload_plan_cache();
  std::lock_guard<std::mutex> lk(g_mu);
  Options o = g_defaults;
  if (!key.empty()) {
    auto it = g_problem.find(key);
    if (it != g_problem.end())
      for (const auto& [n, v] : it->second) apply_option(&o, n, v, nullptr);
  }
  return o;
}

// "name=value;name=value" applied on top of *out; the items in *items.
Status parse_option_spec(const std::string& spec, Options* out,
                         std::vector<std::pair<std::string, int64_t>>* items) {
  Options o = *out;
  std::vector<std::pair<std::string, int64_t>> it;
  size_t i = 0;
  while (i < spec.size()) {
    size_t j = spec.find(';', i);
    if (j == std::string::npos) j = spec.size();
    const std::string kv = spec.substr(i, j - i);
    i = j + 1;
    if (kv.empty()) continue;
    const size_t eq = kv.find('=');
    if (eq == std::string::npos) return Status(TZC_E_VALIDATION, "option spec item '" + kv + "' has no '='");
    int64_t v = 0;
    try {
      v = std::stoll(kv.substr(eq + 1));
    } catch (...) {
      return Status(TZC_E_VALIDATION, "option spec item '" + kv + "': not an integer");
    }
    std::string err;
    if (!apply_option(&o, kv.substr(0, eq), v, &err)) return Status(TZC_E_VALIDATION, err);
    it.emplace_back(kv.substr(0, eq), v);
  }
  *out = o;
  if (items) *items = std::move(it);
  return Status();
}

Status set_default_option(const std::string& name, int64_t value) {
  std::lock_guard<std::mutex> lk(g_mu);
  std::string err;
  if (!apply_option(&g_defaults, name, value, &err)) return Status(TZC_E_VALIDATION, err);
  return Status();
}

// Installs the overrides `spec` for descriptor `key`; an empty spec removes them.
Status set_problem_options(const std::string& key, const std::string& spec) {
  Options o;
  std::vector<std::pair<std::string, int64_t>> items;
  Status st = parse_option_spec(spec, &o, &items);
  if (!st.ok()) return st;
  std::lock_guard<std::mutex> lk(g_mu);
  if (items.empty()) g_problem.erase(key);
  else g_problem[key] = std::move(items);
  return Status();
}

void clear_problem_options() {
  std::lock_guard<std::mutex> lk(g_mu);
  g_problem.clear();
}

// ---- the plan cache on disk ----------------------------------------------------
// One installed problem per line: "<kind><hex descriptor bytes> <spec>" where
// kind is 'c' (tzc_conv_desc) or 'g' (tzc_gemm_desc), followed by a readable
// "# ..." summary of the descriptor; '#' lines are comments.  The SURVEY's
// text plan cache: a tuned suite is saved once and every later process (or
// the CLI) loads it instead of searching again.
namespace {
std::string hex_of(const std::string& raw) {
  static const char* h = "0123456789abcdef";
  std::string s;
  for (unsigned char c : raw) {
    s += h[c >> 4];
    s += h[c & 15];
  }
  return s;
}
bool unhex(const std::string& s, std::string* out) {
  if (s.size() % 2) return false;
  auto v = [](char c) { return c >= '0' && c <= '9' ? c - '0' : c >= 'a' && c <= 'f' ? c - 'a' + 10 : -1; };
  out->clear();
  for (size_t i = 0; i < s.size(); i += 2) {
    const int a = v(s[i]), b = v(s[i + 1]);
    if (a < 0 || b < 0) return false;
    out->push_back((char)(a * 16 + b));
  }
  return true;
}
std::string summary_of(const std::string& key) {
  std::ostringstream os;
  if (key[0] == 'c' && key.size() == 1 + sizeof(tzc_conv_desc)) {
    tzc_conv_desc c;
    std::memcpy(&c, key.data() + 1, sizeof(c));
    os << "conv " << (c.profile == TZC_PROFILE_F16 ? "f16" : "u8i8") << " n=" << c.n << " hp=" << c.hp << " wp=" << c.wp
       << " c=" << c.c << " k=" << c.k << " r=" << c.r << " s=" << c.s << " stride=" << c.stride;
  } else if (key[0] == 'g' && key.size() == 1 + sizeof(tzc_gemm_desc)) {
    tzc_gemm_desc g;
    std::memcpy(&g, key.data() + 1, sizeof(g));
    os << "gemm " << (g.profile == TZC_PROFILE_F16 ? "f16" : "u8i8") << " m=" << g.m << " n=" << g.n << " k=" << g.k;
  }
  return os.str();
}
}  // namespace

Status save_problem_options(const std::string& path, int* count) {
  std::lock_guard<std::mutex> lk(g_mu);
  std::ofstream f(path);
  if (!f) return Status(TZC_E_IO, "cannot write plan cache '" + path + "'");
  f << "# tzc_b200 plan cache v1: <kind+descriptor hex> <options>  # descriptor\n";
  int n = 0;
  for (const auto& [key, items] : g_problem) {
    std::string spec;
    for (const auto& [name, v] : items) spec += (spec.empty() ? "" : ";") + name + "=" + std::to_string(v);
    f << key[0] << hex_of(key.substr(1)) << " " << spec << "  # " << summary_of(key) << "\n";
    ++n;
  }
  if (!f) return Status(TZC_E_IO, "writing plan cache '" + path + "' failed");
  if (count) *count = n;
  return Status();
}

Status load_problem_options(const std::string& path, int* count) {
  std::ifstream f(path);
  if (!f) return Status(TZC_E_IO, "cannot read plan cache '" + path + "'");
  std::string line;
  int n = 0, lineno = 0;
  std::vector<std::pair<std::string, std::string>> entries;
  while (std::getline(f, line)) {
    ++lineno;
    const size_t hash = line.find('#');
    if (hash != std::string::npos) line = line.substr(0, hash);
    std::istringstream is(line);
    std::string k, spec;
    if (!(is >> k)) continue;
    is >> spec;
    std::string raw;
    const size_t want = k[0] == 'c' ? sizeof(tzc_conv_desc) : k[0] == 'g' ? sizeof(tzc_gemm_desc) : 0;
    if (!want || !unhex(k.substr(1), &raw) || raw.size() != want)
      return Status(TZC_E_VALIDATION, path + ":" + std::to_string(lineno) + ": bad descriptor key");
    Options probe;
    Status st = parse_option_spec(spec, &probe, nullptr);
    if (!st.ok()) return Status(TZC_E_VALIDATION, path + ":" + std::to_string(lineno) + ": " + st.msg);
    entries.emplace_back(std::string(1, k[0]) + raw, spec);
  }
  for (const auto& [key, spec] : entries) {  // all lines valid: install them
    Status st = set_problem_options(key, spec);
    if (!st.ok()) return st;
    ++n;
  }
  if (count) *count = n;
  return Status();
}

}  // namespace tzcb200
