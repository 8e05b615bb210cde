// A reference-style C++ caller: reference header paths, reference names, the
// lowering chain lower -> inject_intrinsic -> print_tensor_ir (proj/tests/
// acceptance.cpp criterion 2 shape), compiled against libtzc_b200.so.
// tests/test_cli.py builds and runs it on CPU (no device needed).
#include <iostream>
#include <sstream>

#include "tzc/compute_op.hpp"
#include "tzc/inspector.hpp"
#include "tzc/intrinsics.hpp"
#include "tzc/parser.hpp"
#include "tzc/rewriter.hpp"
#include "tzc/tensor_ir.hpp"

int main(int argc, char** argv) {
  if (argc < 3) return 2;
  std::stringstream text;
  text << std::cin.rdbuf();
  try {
    tzc::ComputeOp op = tzc::infer_types(tzc::parse_compute(text.str()));
    const tzc::Intrinsic& intr = tzc::builtin(argv[1]);
    tzc::InspectionReport rep = tzc::inspect(op, intr);
    if (!rep.match.ok || rep.mappings.empty()) return 1;
    tzc::TensorIR ir = tzc::inject_intrinsic(tzc::lower(op, tzc::parse_schedule(argv[2])), intr, tzc::LoopMapping{});
    std::cout << tzc::print_tensor_ir(ir);
  } catch (const tzc::Error& e) {
    std::cerr << e.kind() << ": " << e.what() << "\n";
    return 1;
  }
  return 0;
}
