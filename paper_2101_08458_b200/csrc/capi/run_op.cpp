// Level-2 C entry: op text + instruction + HOST buffers (the reference-facing
// plugin).  Parses and inspects with the tzc host library, lowers to a kernel
// plan and runs it (tzc::run_tensorized_packed).  Exceptions map onto the
// reference's error kinds (proj/include/tzc/errors.hpp:26-38).
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <unordered_map>

#include "../tzc_b200_internal.hpp"
#include "tzc/tzc.hpp"

namespace {

int code_of(const std::string& kind) {
  static const std::unordered_map<std::string, int> m = {
      {"SyntaxError", TZC_E_SYNTAX},           {"ValidationError", TZC_E_VALIDATION},
      {"TypeError", TZC_E_TYPE},               {"RuleError", TZC_E_RULE},
      {"UnknownIntrinsic", TZC_E_UNKNOWN_INTR}, {"ScheduleError", TZC_E_SCHEDULE},
      {"DivisibilityError", TZC_E_DIVISIBILITY}, {"PadUnsupported", TZC_E_PAD},
      {"InjectError", TZC_E_INJECT},           {"ShapeError", TZC_E_SHAPE},
      {"MissingInput", TZC_E_MISSING_INPUT},   {"NoFeasibleMapping", TZC_E_NO_MAPPING},
      {"IoError", TZC_E_IO},                   {"DeviceError", TZC_E_DEVICE}};
  auto it = m.find(kind);
  return it == m.end() ? TZC_E_INTERNAL : it->second;
}

// Parsed op + tensorization, cached by (op text, intrinsic): planning is
// microseconds but an e2e serving loop calls the same op repeatedly.
struct Cached {
  tzc::TensorizedOp t;
};
std::mutex g_mu;
std::map<std::pair<std::string, std::string>, Cached> g_cache;

// std::map nodes are stable: the pointer stays valid for the process lifetime
const tzc::TensorizedOp* tensorized(const std::string& op_text, const std::string& intr_ref) {
  std::lock_guard<std::mutex> lk(g_mu);
  auto key = std::make_pair(op_text, intr_ref);
  auto it = g_cache.find(key);
  if (it != g_cache.end()) return &it->second.t;
  tzc::ComputeOp op = tzc::infer_types(tzc::parse_compute(op_text));
  tzc::Intrinsic intr = tzc::resolve_intrinsic(intr_ref);
  Cached c{tzc::tensorize(op, intr)};
  return &g_cache.emplace(key, std::move(c)).first->second.t;
}

}  // namespace

extern "C" TZC_API int tzc_b200_run_op(const char* op_tdsl, const char* intrinsic, const char* requant_tdsl,
                                       int32_t n_inputs, const char* const* names, const void* const* host_inputs,
                                       void* host_out, int64_t out_bytes) {
  try {
    if (!op_tdsl || !intrinsic || !host_out || (n_inputs > 0 && (!names || !host_inputs)))
      throw tzc::MissingInput("NULL argument");
    const tzc::TensorizedOp& t = *tensorized(op_tdsl, intrinsic);
    std::map<std::string, const void*> in;
    for (int32_t i = 0; i < n_inputs; ++i) in[names[i]] = host_inputs[i];
    if (requant_tdsl) {
      const tzc::ComputeOp ep = tzc::parse_compute(requant_tdsl);
      tzc::run_tensorized_packed(t, in, host_out, out_bytes, &ep);
    } else {
      tzc::run_tensorized_packed(t, in, host_out, out_bytes, nullptr);
    }
    return TZC_OK;
  } catch (const tzc::Error& e) {
    tzcb200::set_last_error(e.what());
    return code_of(e.kind());
  } catch (const std::exception& e) {
    tzcb200::set_last_error(e.what());
    return TZC_E_INTERNAL;
  }
}

namespace {

int put(const std::string& s, char* buf, int64_t n) {
  if (!buf || (int64_t)s.size() + 1 > n) throw tzc::ShapeError("text buffer too small: need " + std::to_string(s.size() + 1));
  std::memcpy(buf, s.c_str(), s.size() + 1);
  return TZC_OK;
}

template <typename F>
int guarded(F f) {
  try {
    return f();
  } catch (const tzc::Error& e) {
    tzcb200::set_last_error(e.what());
    return code_of(e.kind());
  } catch (const std::exception& e) {
    tzcb200::set_last_error(e.what());
    return TZC_E_INTERNAL;
  }
}

}  // namespace

extern "C" TZC_API int tzc_b200_parse(const char* op_tdsl, char* buf, int64_t n) {
  return guarded([&] { return put(tzc::print_compute(tzc::infer_types(tzc::parse_compute(op_tdsl))), buf, n); });
}

extern "C" TZC_API int tzc_b200_inspect(const char* op_tdsl, const char* intrinsic, int32_t grouped, char* buf,
                                        int64_t n) {
  return guarded([&] {
    const tzc::ComputeOp op = tzc::infer_types(tzc::parse_compute(op_tdsl));
    const tzc::Intrinsic intr = tzc::resolve_intrinsic(intrinsic);
    const tzc::MatchResult mr = tzc::match_operation(op, intr);
    std::string s;
    if (mr.ok) {
      const auto ms = grouped ? tzc::enumerate_group_mappings(op, intr, mr.bind) : tzc::enumerate_mappings(op, intr, mr.bind);
      for (const auto& m : ms) s += m.to_string() + "\n";
    }
    return put(s, buf, n);
  });
}

extern "C" TZC_API int tzc_b200_describe(const char* op_tdsl, const char* intrinsic, char* buf, int64_t n) {
  return guarded([&] {
    const tzc::TensorizedOp& t = *tensorized(op_tdsl, intrinsic);
    std::string s = "mapping " + t.mapping.to_string() + "\nplan " + t.plan.describe() + "\n";
    s += tzc::print_schedule(t.schedule);
    return put(s, buf, n);
  });
}

extern "C" TZC_API int tzc_b200_builtins(char* buf, int64_t n) {
  return guarded([&] {
    std::string s;
    for (const auto& b : tzc::builtin_names()) s += b + "\n";
    return put(s, buf, n);
  });
}

extern "C" TZC_API int tzc_b200_print_intrinsic(const char* intrinsic, char* buf, int64_t n) {
  return guarded([&] { return put(tzc::print_intrinsic(tzc::resolve_intrinsic(intrinsic)), buf, n); });
}

// ---- the reference's lowering chain (lower -> inject_intrinsic -> eval_tir) ----
namespace {

tzc::TensorIR lowered(const char* op_tdsl, const char* schedule, const char* intrinsic) {
  const tzc::ComputeOp op = tzc::infer_types(tzc::parse_compute(op_tdsl));
  if (!schedule) {
    if (!intrinsic) throw tzc::MissingInput("NULL schedule needs an intrinsic");
    return tzc::tensorized_ir(op, tzc::resolve_intrinsic(intrinsic));
  }
  tzc::TensorIR ir = tzc::lower(op, tzc::parse_schedule(schedule));
  if (intrinsic) ir = tzc::inject_intrinsic(ir, tzc::resolve_intrinsic(intrinsic), tzc::LoopMapping{});
  return ir;
}

}  // namespace

extern "C" TZC_API int tzc_b200_lower(const char* op_tdsl, const char* schedule, const char* intrinsic, char* buf,
                                      int64_t n) {
  return guarded([&] {
    if (!op_tdsl) throw tzc::MissingInput("NULL op");
    return put(tzc::print_tensor_ir(lowered(op_tdsl, schedule, intrinsic)), buf, n);
  });
}

extern "C" TZC_API int tzc_b200_eval_tir(const char* op_tdsl, const char* schedule, const char* intrinsic,
                                         const char* requant_tdsl, int32_t n_inputs, const char* const* names,
                                         const void* const* host_inputs, void* host_out, int64_t out_bytes) {
  return guarded([&] {
    if (!op_tdsl || !intrinsic || !host_out || (n_inputs > 0 && (!names || !host_inputs)))
      throw tzc::MissingInput("NULL argument");
    const tzc::TensorizedOp t = tzc::device_plan(lowered(op_tdsl, schedule, intrinsic));
    std::map<std::string, const void*> in;
    for (int32_t i = 0; i < n_inputs; ++i) in[names[i]] = host_inputs[i];
    if (requant_tdsl) {
      const tzc::ComputeOp ep = tzc::parse_compute(requant_tdsl);
      tzc::run_tensorized_packed(t, in, host_out, out_bytes, &ep);
    } else {
      tzc::run_tensorized_packed(t, in, host_out, out_bytes, nullptr);
    }
    return TZC_OK;
  });
}

extern "C" TZC_API int tzc_b200_tensor_text(const char* path, int64_t max_elems, char* buf, int64_t n) {
  return guarded([&] {
    if (!path) throw tzc::MissingInput("NULL path");
    return put(tzc::tensor_to_text(tzc::load_tensor(path), max_elems), buf, n);
  });
}

extern "C" TZC_API int tzc_b200_tensor_roundtrip(const char* src, const char* dst) {
  return guarded([&] {
    if (!src || !dst) throw tzc::MissingInput("NULL path");
    tzc::save_tensor(dst, tzc::load_tensor(src));
    return TZC_OK;
  });
}
