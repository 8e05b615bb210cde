// Prints the C++ workload generators' texts (tzc/workloads.hpp, the
// reference's proj/include/tzc/workloads.hpp:13-64 API) so
// tests/test_reference_api.py can compare them with the reference's own
// generators, and exercises pad_to_multiple / embed / slice from C++.
#include <iostream>

#include "tzc/rewriter.hpp"
#include "tzc/vm.hpp"
#include "tzc/workloads.hpp"

int main() {
  using namespace tzc;
  std::cout << "@matmul_i8\n" << matmul_tdsl(48, 32, 96);
  std::cout << "@matmul_f16\n" << matmul_tdsl(16, 32, 48, fp16_profile());
  for (const auto& e : bank_by_name("table1")) std::cout << "@table1 " << e.shape.name << "\n" << e.tdsl;
  for (const auto& e : bank_by_name("resnet18_3d")) std::cout << "@resnet18_3d " << e.shape.name << "\n" << e.tdsl;
  std::cout << "@conv2d_f16\n" << conv2d_tdsl({"x", 32, 10, 16, 3, 2}, 16, 16, fp16_profile());
  // embed / slice round trip
  TensorValue v = TensorValue::zeros(kI32, {2, 3});
  for (int i = 0; i < 6; ++i) v.idata[i] = i + 1;
  TensorValue big = embed(v, {4, 5});
  TensorValue back = slice(big, {2, 3});
  std::cout << "@embed " << (back.idata == v.idata ? "ok" : "bad") << " " << big.idata[5] << " " << big.idata[4]
            << "\n";
  return 0;
}
