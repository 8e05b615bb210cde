// Tensor container I/O in the reference's "TNSR" format
// (proj/src/vm.cpp:686-822), so device outputs can be cross-checked against
// tensors the reference saved (`tzc run --output`) and vice versa.
#include <algorithm>
#include <cstring>
#include <fstream>
#include <iomanip>
#include <sstream>

#include "tzc/tzc.hpp"

namespace tzc {

namespace {

const DType kCodes[] = {kU8, kI8, kU16, kI16, kU32, kI32, kF16, kF32};

uint8_t code_of(const DType& t) {
  for (uint8_t c = 0; c < 8; ++c)
    if (kCodes[c] == t) return c;
  throw IoError("tensor container does not support dtype " + dtype_name(t));
}

void put_le(std::ostream& os, uint64_t v, int bytes) {
  char b[8];
  for (int i = 0; i < bytes; ++i) b[i] = static_cast<char>(v >> (8 * i));
  os.write(b, bytes);
}

uint64_t get_le(std::istream& is, int bytes) {
  unsigned char b[8] = {};
  is.read(reinterpret_cast<char*>(b), bytes);
  if (!is) throw IoError("truncated tensor container");
  uint64_t v = 0;
  for (int i = bytes; i-- > 0;) v = (v << 8) | b[i];
  return v;
}

}  // namespace

void write_tensor(std::ostream& os, const TensorValue& v) {
  os.write("TNSR", 4);
  os.put(1);
  os.put(static_cast<char>(code_of(v.dtype)));
  os.put(static_cast<char>(v.shape.size()));
  for (int64_t d : v.shape) put_le(os, static_cast<uint64_t>(d), 8);
  const int w = v.dtype.bits / 8;
  for (int64_t i = 0; i < v.size(); ++i) {
    if (v.dtype == kF16) {
      put_le(os, f64_to_f16_bits(v.fdata[i]), 2);
    } else if (v.dtype == kF32) {
      const float f = static_cast<float>(v.fdata[i]);
      uint32_t u;
      std::memcpy(&u, &f, 4);
      put_le(os, u, 4);
    } else {
      put_le(os, static_cast<uint64_t>(wrap_int(v.idata[i], v.dtype)), w);
    }
  }
  if (!os) throw IoError("failed to write tensor container");
}

TensorValue read_tensor(std::istream& is) {
  char magic[4];
  is.read(magic, 4);
  if (!is || std::memcmp(magic, "TNSR", 4) != 0) throw IoError("not a tensor container (bad magic)");
  const int version = is.get();
  if (version != 1) throw IoError("unsupported tensor container version " + std::to_string(version));
  const int code = is.get();
  if (code < 0 || code > 7) throw IoError("unknown dtype code " + std::to_string(code));
  const DType t = kCodes[code];
  const int rank = is.get();
  if (rank < 0 || !is) throw IoError("truncated tensor container");
  std::vector<int64_t> shape;
  for (int d = 0; d < rank; ++d) shape.push_back(static_cast<int64_t>(get_le(is, 8)));
  TensorValue v = TensorValue::zeros(t, shape);
  const int w = t.bits / 8;
  for (int64_t i = 0; i < v.size(); ++i) {
    if (t == kF16) {
      v.fdata[i] = f16_bits_to_f64(static_cast<uint16_t>(get_le(is, 2)));
    } else if (t == kF32) {
      const uint32_t u = static_cast<uint32_t>(get_le(is, 4));
      float f;
      std::memcpy(&f, &u, 4);
      v.fdata[i] = f;
    } else {
      v.idata[i] = wrap_int(static_cast<int64_t>(get_le(is, w)), t);
    }
  }
  return v;
}

void save_tensor(const std::string& path, const TensorValue& v) {
  std::ofstream f(path, std::ios::binary);
  if (!f) throw IoError("cannot open '" + path + "' for writing");
  write_tensor(f, v);
}

TensorValue load_tensor(const std::string& path) {
  std::ifstream f(path, std::ios::binary);
  if (!f) throw IoError("cannot open '" + path + "'");
  return read_tensor(f);
}

std::string tensor_to_text(const TensorValue& v, int64_t max_elems) {
  std::ostringstream os;
  os << dtype_name(v.dtype) << " [";
  for (size_t d = 0; d < v.shape.size(); ++d) os << (d ? ", " : "") << v.shape[d];
  os << "] =" << std::setprecision(9);
  const int64_t n = std::min<int64_t>(v.size(), max_elems);
  for (int64_t k = 0; k < n; ++k) {
    if (v.is_float()) os << " " << v.fdata[k];
    else os << " " << v.idata[k];
  }
  if (n < v.size()) os << " ... (" << v.size() << " total)";
  return os.str();
}

}  // namespace tzc
