// TEST INFRASTRUCTURE — NOT PRODUCT CODE.
//
// Plain C ABI over the reference implementation (`tzc`, compiled unmodified
// from /root/reference/proj/src with -Dtzc=tzc_ref, see oracle/Makefile), so
// the Python test harness (tests/, bench.py's cpu_baseline / --impl
// reference arm, __graft_entry__.smoke) can drive the reference's own
// parser, seeded input generator, interpreter (eval_reference, the oracle)
// and tensorized-body executor (eval_tir, the reference's hot path) through
// ctypes.  Nothing in paper_2101_08458_b200/ links or loads this.
//
// Reference entry points wrapped here (all under /root/reference/proj):
//   parse_compute / infer_types   include/tzc/parser.hpp:28, compute_op.hpp:61
//   random_inputs                 src/vm.cpp:59-68
//   eval_reference                src/vm.cpp:444-508
//   inspect/tile_and_reorder/lower/inject_intrinsic/eval_tir
//                                 src/inspector.cpp:218, src/rewriter.cpp:245,509,789,
//                                 src/vm.cpp:510-516
//   matmul_tdsl / conv2d_tdsl     src/workloads.cpp:41-92
//   f64_to_f16_bits / wrap_int    src/dtype.cpp:40-101
//
// Tensors cross the boundary packed at their declared width (u8/i8: 1 byte,
// i16/u16: 2, i32/u32: 4, fp16: binary16 bits, fp32: float), row-major.

#include <cstdint>
#include <cstring>
#include <exception>
#include <sstream>
#include <string>
#include <vector>

#include "tzc/dtype.hpp"
#include "tzc/errors.hpp"
#include "tzc/inspector.hpp"
#include "tzc/intrinsics.hpp"
#include "tzc/parser.hpp"
#include "tzc/rewriter.hpp"
#include "tzc/vm.hpp"
#include "tzc/workloads.hpp"

using namespace tzc;

namespace {

thread_local std::string g_err;

int fail(const std::string& msg) {
  g_err = msg;
  return -1;
}

int64_t elem_bytes(const DType& t) { return t.bits / 8; }

ComputeOp op_from(const char* text) { return infer_types(parse_compute(text)); }

void pack(const TensorValue& v, void* out) {
  int64_t n = v.size();
  if (v.dtype == kF16) {
    auto* p = static_cast<uint16_t*>(out);
    for (int64_t i = 0; i < n; ++i) p[i] = f64_to_f16_bits(v.fdata[i]);
  } else if (v.dtype == kF32) {
    auto* p = static_cast<float*>(out);
    for (int64_t i = 0; i < n; ++i) p[i] = static_cast<float>(v.fdata[i]);
  } else {
    int64_t b = elem_bytes(v.dtype);
    auto* p = static_cast<uint8_t*>(out);
    for (int64_t i = 0; i < n; ++i) {
      uint64_t u = static_cast<uint64_t>(v.idata[i]);
      std::memcpy(p + i * b, &u, b);  // little-endian low bytes
    }
  }
}

TensorValue unpack(const TensorDecl& td, const void* in) {
  TensorValue v = TensorValue::zeros(td.dtype, td.shape);
  int64_t n = v.size();
  if (td.dtype == kF16) {
    auto* p = static_cast<const uint16_t*>(in);
    for (int64_t i = 0; i < n; ++i) v.fdata[i] = f16_bits_to_f64(p[i]);
  } else if (td.dtype == kF32) {
    auto* p = static_cast<const float*>(in);
    for (int64_t i = 0; i < n; ++i) v.fdata[i] = static_cast<double>(p[i]);
  } else {
    int64_t b = elem_bytes(td.dtype);
    auto* p = static_cast<const uint8_t*>(in);
    for (int64_t i = 0; i < n; ++i) {
      uint64_t u = 0;
      std::memcpy(&u, p + i * b, b);
      v.idata[i] = wrap_int(static_cast<int64_t>(u), td.dtype);
    }
  }
  return v;
}

Inputs gather(const ComputeOp& op, int n, const char* const* names,
              const void* const* bufs) {
  Inputs in;
  for (int i = 0; i < n; ++i) {
    const TensorDecl* td = op.find_tensor(names[i]);
    if (!td) throw MissingInput(std::string("no tensor named '") + names[i] + "'");
    in.emplace(td->name, unpack(*td, bufs[i]));
  }
  return in;
}

int put_text(const std::string& s, char* buf, int64_t buflen) {
  if (static_cast<int64_t>(s.size()) + 1 > buflen)
    return fail("buffer too small: need " + std::to_string(s.size() + 1));
  std::memcpy(buf, s.c_str(), s.size() + 1);
  return 0;
}

int check_bytes(const TensorValue& v, int64_t nbytes) {
  int64_t want = v.size() * elem_bytes(v.dtype);
  if (nbytes != want)
    return fail("output buffer holds " + std::to_string(nbytes) + " bytes, need " +
                std::to_string(want));
  return 0;
}

TensorIR tensorized_ir(const ComputeOp& op, const Intrinsic& intr) {
  InspectionReport rep = inspect(op, intr);
  if (!rep.match.ok) throw InjectError("no structural match: " + rep.match.reason);
  const LoopMapping* pick = nullptr;
  for (const auto& m : rep.mappings)
    if (!m.needs_padding) {
      pick = &m;
      break;
    }
  if (!pick) throw NoFeasibleMapping("no dividing mapping");
  TensorizedOp t = tile_and_reorder(op, intr, *pick);
  return inject_intrinsic(lower(t.op, t.schedule), intr, t.mapping);
}

}  // namespace

#define TZCREF_TRY try {
#define TZCREF_CATCH                         \
  }                                          \
  catch (const std::exception& e) {          \
    return fail(e.what());                   \
  }

extern "C" {

const char* tzcref_last_error(void) { return g_err.c_str(); }

// "tensor <name> <dtype> <in|out> <rank> d0 ..\n" per tensor, "loop <name>
// <dp|red> <extent>\n" per loop, then "update <0|1>\n".
int tzcref_op_info(const char* op_text, char* buf, int64_t buflen) {
  TZCREF_TRY
  ComputeOp op = op_from(op_text);
  std::ostringstream os;
  for (const auto& t : op.tensors) {
    os << "tensor " << t.name << " " << dtype_name(t.dtype) << " "
       << (t.role == Role::Input ? "in" : "out") << " " << t.shape.size();
    for (int64_t d : t.shape) os << " " << d;
    os << "\n";
  }
  for (const auto& l : op.loops)
    os << "loop " << l.name << " "
       << (l.kind == LoopKind::DataParallel ? "dp" : "red") << " " << l.extent << "\n";
  os << "update " << (op.update ? 1 : 0) << "\n";
  return put_text(os.str(), buf, buflen);
  TZCREF_CATCH
}

// random_inputs(op, seed)[tensor], packed. The output image of an
// accumulate-form op is included (it is an input to such ops).
int tzcref_random_tensor(const char* op_text, const char* tensor, uint64_t seed,
                         void* out, int64_t nbytes) {
  TZCREF_TRY
  ComputeOp op = op_from(op_text);
  Inputs in = random_inputs(op, seed);
  auto it = in.find(tensor);
  if (it == in.end()) return fail(std::string("no random input named '") + tensor + "'");
  if (check_bytes(it->second, nbytes)) return -1;
  pack(it->second, out);
  return 0;
  TZCREF_CATCH
}

int tzcref_eval_reference(const char* op_text, int n, const char* const* names,
                          const void* const* bufs, void* out, int64_t nbytes) {
  TZCREF_TRY
  ComputeOp op = op_from(op_text);
  TensorValue r = eval_reference(op, gather(op, n, names, bufs));
  if (check_bytes(r, nbytes)) return -1;
  pack(r, out);
  return 0;
  TZCREF_CATCH
}

// The reference's hot path: inspect -> tile_and_reorder -> lower ->
// inject_intrinsic -> eval_tir with the named builtin (or .intr path).
int tzcref_eval_tir(const char* op_text, const char* intrinsic, int n,
                    const char* const* names, const void* const* bufs, void* out,
                    int64_t nbytes) {
  TZCREF_TRY
  ComputeOp op = op_from(op_text);
  Intrinsic intr = resolve_intrinsic(intrinsic);
  TensorIR ir = tensorized_ir(op, intr);
  TensorValue r = eval_tir(ir, gather(op, n, names, bufs));
  if (check_bytes(r, nbytes)) return -1;
  pack(r, out);
  return 0;
  TZCREF_CATCH
}

int tzcref_tensorize(const char* op_text, const char* intrinsic, char* buf,
                     int64_t buflen) {
  TZCREF_TRY
  ComputeOp op = op_from(op_text);
  Intrinsic intr = resolve_intrinsic(intrinsic);
  return put_text(print_tensor_ir(tensorized_ir(op, intr)), buf, buflen);
  TZCREF_CATCH
}

// print_tensor_ir(lower(op, parse_schedule(schedule))), injected with
// `intrinsic` when non-NULL (empty mapping: inject only checks its size).
int tzcref_lower(const char* op_text, const char* schedule, const char* intrinsic,
                 char* buf, int64_t buflen) {
  TZCREF_TRY
  ComputeOp op = op_from(op_text);
  TensorIR ir = lower(op, parse_schedule(schedule));
  if (intrinsic) ir = inject_intrinsic(ir, resolve_intrinsic(intrinsic), LoopMapping{});
  return put_text(print_tensor_ir(ir), buf, buflen);
  TZCREF_CATCH
}

// Writes random_inputs(op, seed) (the tensors an eval needs) as
// <dir>/<name>.tnsr and eval_reference's output as <dir>/expect.tnsr, with
// the reference's own save_tensor: fixtures for the device CLI's verify.
int tzcref_save_case(const char* op_text, uint64_t seed, const char* dir) {
  TZCREF_TRY
  ComputeOp op = op_from(op_text);
  Inputs in = random_inputs(op, seed);
  for (const auto& [name, v] : in) save_tensor(std::string(dir) + "/" + name + ".tnsr", v);
  save_tensor(std::string(dir) + "/expect.tnsr", eval_reference(op, in));
  return 0;
  TZCREF_CATCH
}

// tensor_to_text(load_tensor(path), max_elems) as the reference renders it.
int tzcref_tensor_text(const char* path, int64_t max_elems, char* buf, int64_t buflen) {
  TZCREF_TRY
  return put_text(tensor_to_text(load_tensor(path), max_elems), buf, buflen);
  TZCREF_CATCH
}

// "<assignment> <needs_padding>\n" per mapping; empty when no match.
int tzcref_inspect(const char* op_text, const char* intrinsic, char* buf,
                   int64_t buflen) {
  TZCREF_TRY
  ComputeOp op = op_from(op_text);
  Intrinsic intr = resolve_intrinsic(intrinsic);
  InspectionReport rep = inspect(op, intr);
  std::ostringstream os;
  if (rep.match.ok)
    for (const auto& m : rep.mappings)
      os << m.to_string() << " " << (m.needs_padding ? 1 : 0) << "\n";
  return put_text(os.str(), buf, buflen);
  TZCREF_CATCH
}

int tzcref_matmul_tdsl(int64_t m, int64_t n, int64_t k, int fp16, char* buf,
                       int64_t buflen) {
  TZCREF_TRY
  return put_text(matmul_tdsl(m, n, k, fp16 ? fp16_profile() : int8_profile()), buf,
                  buflen);
  TZCREF_CATCH
}

int tzcref_conv2d_tdsl(int64_t in_c, int64_t in_hw, int64_t out_c, int64_t kernel,
                       int64_t stride, int64_t lane_block, int64_t red_block,
                       int fp16, char* buf, int64_t buflen) {
  TZCREF_TRY
  ConvShape c{"conv", in_c, in_hw, out_c, kernel, stride};
  return put_text(
      conv2d_tdsl(c, lane_block, red_block, fp16 ? fp16_profile() : int8_profile()),
      buf, buflen);
  TZCREF_CATCH
}

int tzcref_conv3d_tdsl(int64_t in_c, int64_t in_hw, int64_t out_c, int64_t kernel,
                       int64_t stride, int64_t lane_block, int64_t red_block,
                       int fp16, char* buf, int64_t buflen) {
  TZCREF_TRY
  ConvShape c{"conv3d", in_c, in_hw, out_c, kernel, stride};
  return put_text(
      conv3d_tdsl(c, lane_block, red_block, fp16 ? fp16_profile() : int8_profile()),
      buf, buflen);
  TZCREF_CATCH
}

uint16_t tzcref_f64_to_f16_bits(double x) { return f64_to_f16_bits(x); }
double tzcref_f16_bits_to_f64(uint16_t b) { return f16_bits_to_f64(b); }

}  // extern "C"
