// Level-2 entry (op text + host buffers).  Filled in by the tzc host library.
#include "../tzc_b200_internal.hpp"

extern "C" TZC_API int tzc_b200_run_op(const char*, const char*, const char*, int32_t, const char* const*,
                               const void* const*, void*, int64_t) {
  return TZC_E_INTERNAL;
}
