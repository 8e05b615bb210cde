// tzc-b200: the reference CLI's device-facing subcommands (proj/src/cli.cpp:
// inspect :440-470, tensorize, run :379-434, verify :227-283) over the B200
// backend.  `run` executes the tensorized op on the GPU through
// lower -> inject_intrinsic -> eval_tir; `verify` cross-checks that result
// against a tensor saved in the reference's TNSR container (e.g. by the
// reference's own `tzc run --output`), with the reference's compare() metric.
// Exit codes follow the reference (cli.cpp:41-47): 0 ok, 1 domain failure
// (no mapping / divisibility / pad / inject / device, or verify FAIL),
// 2 usage or parse error.
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <iostream>
#include <map>
#include <sstream>
#include <string>
#include <vector>

#include "tzc/tzc.hpp"

namespace {

const char* kUsage =
    "usage: tzc-b200 <command> [args]\n"
    "  builtins\n"
    "  inspect   OP.tdsl --intrinsic X [--format text|structured]\n"
    "  tensorize OP.tdsl --intrinsic X [--schedule-out PATH]\n"
    "  run       OP.tdsl --intrinsic X [--schedule PATH] [--input name=PATH]... [--seed N]\n"
    "            [--epilogue OP.tdsl] [--output PATH] [--format text|structured]\n"
    "  tune      OP.tdsl --intrinsic X [--reps N] [--input name=PATH]... [--seed N]\n"
    "  verify    OP.tdsl --intrinsic X --expect PATH [--input name=PATH]... [--seed N]\n"
    "            [--epilogue OP.tdsl] [--rtol R] [--format text|structured]\n";

struct Usage : std::runtime_error {
  using std::runtime_error::runtime_error;
};

struct Args {
  std::string cmd, op_path, intrinsic, schedule, schedule_out, output, expect, epilogue, format = "text";
  std::vector<std::string> inputs;
  uint64_t seed = 0;
  double rtol = 0.0;
  bool rtol_set = false;
  int reps = 10;
};

Args parse_args(int argc, char** argv) {
  if (argc < 2) throw Usage("missing command");
  Args a;
  a.cmd = argv[1];
  for (int i = 2; i < argc; ++i) {
    const std::string k = argv[i];
    auto val = [&]() -> std::string {
      if (i + 1 >= argc) throw Usage(k + " needs a value");
      return argv[++i];
    };
    if (k == "--intrinsic") a.intrinsic = val();
    else if (k == "--schedule") a.schedule = val();
    else if (k == "--schedule-out") a.schedule_out = val();
    else if (k == "--input") a.inputs.push_back(val());
    else if (k == "--output") a.output = val();
    else if (k == "--expect") a.expect = val();
    else if (k == "--epilogue") a.epilogue = val();
    else if (k == "--format") a.format = val();
    else if (k == "--seed") a.seed = std::strtoull(val().c_str(), nullptr, 10);
    else if (k == "--rtol") a.rtol = std::atof(val().c_str()), a.rtol_set = true;
    else if (k == "--reps") a.reps = std::atoi(val().c_str());
    else if (!k.empty() && k[0] == '-') throw Usage("unknown option " + k);
    else if (a.op_path.empty()) a.op_path = k;
    else throw Usage("unexpected argument " + k);
  }
  if (a.format != "text" && a.format != "structured") throw Usage("--format must be text or structured");
  return a;
}

std::string read_file(const std::string& path) {
  std::ifstream f(path);
  if (!f) throw tzc::IoError("cannot open '" + path + "'");
  std::stringstream ss;
  ss << f.rdbuf();
  return ss.str();
}

tzc::ComputeOp load_op(const Args& a) {
  if (a.op_path.empty()) throw Usage("missing OP.tdsl");
  return tzc::infer_types(tzc::parse_compute(read_file(a.op_path)));
}

tzc::Intrinsic need_intrinsic(const Args& a) {
  if (a.intrinsic.empty()) throw Usage("--intrinsic is required");
  return tzc::resolve_intrinsic(a.intrinsic);
}

std::string json_str(const std::string& s) {
  std::string o = "\"";
  for (char c : s) {
    if (c == '"' || c == '\\') o += '\\', o += c;
    else if (c == '\n') o += "\\n";
    else o += c;
  }
  return o + "\"";
}

// Given inputs (name=path TNSR files) plus seeded random images for the rest,
// exactly as the reference's `run` fills them (seed + declaration index).
tzc::Inputs gather_inputs(const Args& a, const tzc::ComputeOp& op) {
  tzc::Inputs in;
  for (const auto& spec : a.inputs) {
    const auto eq = spec.find('=');
    if (eq == std::string::npos) throw tzc::ValidationError("--input expects name=path, got '" + spec + "'");
    in.emplace(spec.substr(0, eq), tzc::load_tensor(spec.substr(eq + 1)));
  }
  uint64_t k = 0;
  for (const auto& td : op.tensors) {
    const bool needed = td.role == tzc::Role::Input || (td.name == op.out && op.update);
    if (needed && !in.count(td.name)) in.emplace(td.name, tzc::random_tensor(td, a.seed + k));
    ++k;
  }
  return in;
}

tzc::TensorValue execute(const Args& a, const tzc::ComputeOp& op) {
  const tzc::Intrinsic intr = need_intrinsic(a);
  tzc::TensorIR ir;
  if (a.schedule.empty()) {
    ir = tzc::tensorized_ir(op, intr);
  } else {
    ir = tzc::inject_intrinsic(tzc::lower(op, tzc::load_schedule(a.schedule)), intr, tzc::LoopMapping{});
  }
  const tzc::Inputs in = gather_inputs(a, op);
  if (a.epilogue.empty()) return tzc::eval_tir(ir, in);
  const tzc::ComputeOp ep = tzc::parse_compute(read_file(a.epilogue));
  return tzc::eval_tir(ir, in, &ep);
}

int cmd_inspect(const Args& a, std::ostream& out) {
  const tzc::ComputeOp op = load_op(a);
  const tzc::Intrinsic intr = need_intrinsic(a);
  const tzc::MatchResult m = tzc::match_operation(op, intr);
  std::vector<tzc::LoopMapping> maps;
  if (m.ok) maps = tzc::enumerate_group_mappings(op, intr, m.bind);
  if (a.format == "structured") {
    out << "{\n  \"match\": " << (m.ok ? "true" : "false") << ",\n";
    if (!m.ok) out << "  \"reason\": " << json_str(m.reason) << ",\n";
    out << "  \"mappings\": [";
    for (size_t i = 0; i < maps.size(); ++i)
      out << (i ? ", " : "") << "{\"assignment\": " << json_str(maps[i].to_string())
          << ", \"needs_padding\": " << (maps[i].needs_padding ? "true" : "false") << "}";
    out << "]\n}\n";
  } else if (!m.ok) {
    out << "no match: " << m.reason << "\n";
  } else {
    for (size_t i = 0; i < maps.size(); ++i)
      out << "mapping " << i << ": " << maps[i].to_string() << "\n";
  }
  if (!m.ok || maps.empty()) return 1;
  return 0;
}

int cmd_tensorize(const Args& a, std::ostream& out) {
  const tzc::ComputeOp op = load_op(a);
  const tzc::Intrinsic intr = need_intrinsic(a);
  const tzc::TensorizedOp t = tzc::tensorize(op, intr);
  out << tzc::print_tensor_ir(tzc::tensorized_ir(op, intr));
  if (!a.schedule_out.empty()) {
    std::ofstream f(a.schedule_out);
    if (!f) throw tzc::IoError("cannot open '" + a.schedule_out + "' for writing");
    f << tzc::print_schedule(t.schedule);
  }
  return 0;
}

int cmd_run(const Args& a, std::ostream& out) {
  const tzc::ComputeOp op = load_op(a);
  const tzc::TensorValue r = execute(a, op);
  if (!a.output.empty()) tzc::save_tensor(a.output, r);
  if (a.format == "structured") {
    out << "{\n  \"output\": " << json_str(tzc::tensor_to_text(r));
    if (!a.output.empty()) out << ",\n  \"saved\": " << json_str(a.output);
    out << "\n}\n";
  } else {
    out << tzc::tensor_to_text(r) << "\n";
    if (!a.output.empty()) out << "saved: " << a.output << "\n";
  }
  return 0;
}

int cmd_verify(const Args& a, std::ostream& out) {
  const tzc::ComputeOp op = load_op(a);
  if (a.expect.empty()) throw Usage("--expect PATH is required (a TNSR tensor saved by the reference)");
  const tzc::TensorValue want = tzc::load_tensor(a.expect);
  if (want.is_float() && !a.rtol_set)
    throw tzc::ValidationError("floating-point outputs accumulate in a different order once tensorized; pass an explicit --rtol");
  const tzc::TensorValue got = execute(a, op);
  if (got.dtype != want.dtype || got.shape != want.shape)
    throw tzc::ShapeError("device result " + tzc::tensor_to_text(got, 0) + " vs expected " + tzc::tensor_to_text(want, 0));
  const tzc::Deviation d = tzc::compare(want, got, a.rtol);
  std::string first;
  for (int64_t k = 0; k < want.size() && d.mismatches; ++k) {
    const double rv = want.is_float() ? want.fdata[k] : double(want.idata[k]);
    const double gv = got.is_float() ? got.fdata[k] : double(got.idata[k]);
    if (std::abs(rv - gv) / std::max(std::abs(rv), 1.0) > a.rtol) {
      std::ostringstream ss;
      ss << "flat index " << k << ": expected " << rv << " vs device " << gv;
      first = ss.str();
      break;
    }
  }
  const bool pass = d.mismatches == 0;
  if (a.format == "structured") {
    out << "{\n  \"max_rel\": " << d.max_rel << ",\n  \"mismatches\": " << d.mismatches
        << ",\n  \"bitexact\": " << (d.bitexact ? "true" : "false") << ",\n  \"pass\": " << (pass ? "true" : "false");
    if (!first.empty()) out << ",\n  \"first_mismatch\": " << json_str(first);
    out << "\n}\n";
  } else {
    out << "max rel deviation: " << d.max_rel << "\n";
    out << "bitexact: " << (d.bitexact ? "yes" : "no") << "\n";
    if (!first.empty()) out << "first mismatch: " << first << "\n";
    out << (pass ? "PASS" : "FAIL") << "\n";
  }
  return pass ? 0 : 1;
}

// The device analogue of `tzc tune --target gpu` (proj/src/cli.cpp tune
// subcommand): candidate plans timed with CUDA events, the log printed.
int cmd_tune(const Args& a, std::ostream& out) {
  const tzc::ComputeOp op = load_op(a);
  const tzc::TensorizedOp t = tzc::tensorize(op, need_intrinsic(a));
  out << "plan " << t.plan.describe() << "\n" << tzc::tune_tensorized(t, gather_inputs(a, op), a.reps);
  return 0;
}

bool domain_failure(const std::string& kind) {
  return kind == "NoFeasibleMapping" || kind == "DivisibilityError" || kind == "PadUnsupported" ||
         kind == "InjectError" || kind == "DeviceError";
}

}  // namespace

int main(int argc, char** argv) {
  try {
    const Args a = parse_args(argc, argv);
    if (a.cmd == "builtins") {
      for (const auto& n : tzc::builtin_names()) std::cout << n << "\n";
      return 0;
    }
    if (a.cmd == "inspect") return cmd_inspect(a, std::cout);
    if (a.cmd == "tensorize") return cmd_tensorize(a, std::cout);
    if (a.cmd == "run") return cmd_run(a, std::cout);
    if (a.cmd == "verify") return cmd_verify(a, std::cout);
    if (a.cmd == "tune") return cmd_tune(a, std::cout);
    throw Usage("unknown command '" + a.cmd + "'");
  } catch (const Usage& e) {
    std::cerr << "error: " << e.what() << "\n" << kUsage;
    return 2;
  } catch (const tzc::Error& e) {
    std::cerr << "error: " << e.what() << "\n";
    return domain_failure(e.kind()) ? 1 : 2;
  } catch (const std::exception& e) {
    std::cerr << "internal error: " << e.what() << "\n";
    return 2;
  }
}
