"""ctypes mirror of include/tzc_b200.h (the C ABI of libtzc_b200.so).

This module only loads and declares; it never computes.  If the in-tree
library is missing the import of :func:`lib` raises — there is no fallback.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libtzc_b200.so")
# TZC_B200_CHECKS=1 loads the instrumented build (libtzc_b200_checks.so:
# mbarrier watchdogs and output-bounds asserts that trap; `make checks`)
if os.environ.get("TZC_B200_CHECKS") == "1":
    LIB_PATH = os.path.join(_HERE, "libtzc_b200_checks.so")

TZC_OK = 0
PROFILE_U8I8, PROFILE_F16 = 0, 1
EP_I32, EP_REQUANT_I8, EP_F32, EP_CAST_F16 = 0, 1, 2, 3

ERROR_KINDS = {
    -1: "SyntaxError", -2: "ValidationError", -3: "TypeError", -4: "RuleError",
    -5: "UnknownIntrinsic", -6: "ScheduleError", -7: "DivisibilityError", -8: "PadUnsupported",
    -9: "InjectError", -10: "ShapeError", -11: "MissingInput", -12: "NoFeasibleMapping",
    -13: "IoError", -20: "DeviceError", -30: "InternalError",
}

# Every exported symbol the header declares (checked by tests/test_capi.py).
EXPORTS = (
    "tzc_b200_conv2d_i8", "tzc_b200_conv2d_f16", "tzc_b200_gemm_i8", "tzc_b200_gemm_f16",
    "tzc_b200_plan_conv", "tzc_b200_plan_gemm", "tzc_b200_set_splits", "tzc_b200_set_option",
    "tzc_b200_unblock_data", "tzc_b200_unblock_kernel", "tzc_b200_run_op", "tzc_b200_eval_tir", "tzc_b200_lower",
    "tzc_b200_tensor_text", "tzc_b200_tensor_roundtrip",
    "tzc_b200_tune_conv", "tzc_b200_tune_gemm", "tzc_b200_clear_tuning",
    "tzc_b200_set_problem_options_conv", "tzc_b200_set_problem_options_gemm", "tzc_b200_tune_candidates",
    "tzc_b200_save_tuning", "tzc_b200_load_tuning",
    "tzc_b200_parse", "tzc_b200_inspect", "tzc_b200_describe", "tzc_b200_builtins",
    "tzc_b200_print_intrinsic",
    "tzc_b200_last_error", "tzc_b200_launch_count", "tzc_b200_last_launch", "tzc_b200_device_ok", "tzc_b200_version",
)


class TzcError(RuntimeError):
    """A non-zero status from the C ABI; ``kind`` mirrors tzc::Error::kind()."""

    def __init__(self, code: int, msg: str):
        self.code = code
        self.kind = ERROR_KINDS.get(code, "Error")
        super().__init__(f"{self.kind}: {msg}")


class OutLayout(C.Structure):
    _fields_ = [("nb", C.c_int32), ("pad_", C.c_int32), ("stride_m", C.c_int64),
                ("stride_blk", C.c_int64)]


class ConvDesc(C.Structure):
    _fields_ = [("profile", C.c_int32), ("n", C.c_int32), ("hp", C.c_int32), ("wp", C.c_int32),
                ("c", C.c_int32), ("k", C.c_int32), ("r", C.c_int32), ("s", C.c_int32),
                ("stride", C.c_int32), ("pad_", C.c_int32), ("w_stride_k", C.c_int64),
                ("w_stride_tap", C.c_int64), ("out", OutLayout)]


class GemmDesc(C.Structure):
    _fields_ = [("profile", C.c_int32), ("m", C.c_int32), ("n", C.c_int32), ("k", C.c_int32),
                ("b_kn", C.c_int32), ("pad_", C.c_int32), ("out", OutLayout)]


class Epilogue(C.Structure):
    _fields_ = [("kind", C.c_int32), ("scale", C.c_float)]


class LaunchInfo(C.Structure):
    _fields_ = [("kernel", C.c_int32), ("cta_group", C.c_int32), ("bm", C.c_int32), ("bn", C.c_int32),
                ("bk_bytes", C.c_int32), ("a_mode", C.c_int32), ("grid", C.c_int32), ("splits", C.c_int32)]


class Plan(C.Structure):
    _fields_ = [("bm", C.c_int32), ("bn", C.c_int32), ("bk_bytes", C.c_int32), ("stages", C.c_int32),
                ("a_mode", C.c_int32), ("splits", C.c_int32), ("grid", C.c_int32),
                ("smem_bytes", C.c_int32), ("tiles_m", C.c_int32), ("tiles_n", C.c_int32),
                ("workspace_bytes", C.c_int64)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


_lock = threading.Lock()
_lib = None


def lib():
    """Load libtzc_b200.so (in-tree).  Raises if it was not built."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise RuntimeError(
                    f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
                    " (or make -C paper_2101_08458_b200); there is no CPU fallback")
            L = C.CDLL(LIB_PATH)
            P = C.c_void_p
            for fn, desc in (("tzc_b200_conv2d_i8", ConvDesc), ("tzc_b200_conv2d_f16", ConvDesc),
                             ("tzc_b200_gemm_i8", GemmDesc), ("tzc_b200_gemm_f16", GemmDesc)):
                f = getattr(L, fn)
                f.argtypes = [C.POINTER(desc), P, P, P, P, C.POINTER(Epilogue), P]
                f.restype = C.c_int
            for fn, desc in (("tzc_b200_tune_conv", ConvDesc), ("tzc_b200_tune_gemm", GemmDesc)):
                getattr(L, fn).argtypes = [C.POINTER(desc), P, P, P, P, C.POINTER(Epilogue), C.c_int32, C.c_int32,
                                           C.c_char_p, C.c_int64, P]
            L.tzc_b200_set_problem_options_conv.argtypes = [C.POINTER(ConvDesc), C.c_char_p]
            L.tzc_b200_set_problem_options_gemm.argtypes = [C.POINTER(GemmDesc), C.c_char_p]
            L.tzc_b200_tune_candidates.argtypes = [C.c_char_p, C.c_int64]
            L.tzc_b200_plan_conv.argtypes = [C.POINTER(ConvDesc), C.POINTER(Plan)]
            L.tzc_b200_plan_gemm.argtypes = [C.POINTER(GemmDesc), C.POINTER(Plan)]
            L.tzc_b200_set_splits.argtypes = [C.c_int32]
            L.tzc_b200_set_option.argtypes = [C.c_char_p, C.c_int64]
            L.tzc_b200_unblock_data.argtypes = [P, P] + [C.c_int32] * 5 + [P]
            L.tzc_b200_unblock_kernel.argtypes = [P, P] + [C.c_int32] * 7 + [P]
            L.tzc_b200_run_op.argtypes = [C.c_char_p, C.c_char_p, C.c_char_p, C.c_int32,
                                          C.POINTER(C.c_char_p), C.POINTER(P), P, C.c_int64]
            L.tzc_b200_eval_tir.argtypes = [C.c_char_p, C.c_char_p, C.c_char_p, C.c_char_p, C.c_int32,
                                            C.POINTER(C.c_char_p), C.POINTER(P), P, C.c_int64]
            L.tzc_b200_lower.argtypes = [C.c_char_p, C.c_char_p, C.c_char_p, C.c_char_p, C.c_int64]
            L.tzc_b200_tensor_text.argtypes = [C.c_char_p, C.c_int64, C.c_char_p, C.c_int64]
            L.tzc_b200_tensor_roundtrip.argtypes = [C.c_char_p, C.c_char_p]
            L.tzc_b200_parse.argtypes = [C.c_char_p, C.c_char_p, C.c_int64]
            L.tzc_b200_inspect.argtypes = [C.c_char_p, C.c_char_p, C.c_int32, C.c_char_p, C.c_int64]
            L.tzc_b200_describe.argtypes = [C.c_char_p, C.c_char_p, C.c_char_p, C.c_int64]
            L.tzc_b200_builtins.argtypes = [C.c_char_p, C.c_int64]
            L.tzc_b200_print_intrinsic.argtypes = [C.c_char_p, C.c_char_p, C.c_int64]
            L.tzc_b200_last_error.restype = C.c_char_p
            L.tzc_b200_launch_count.restype = C.c_uint64
            L.tzc_b200_device_ok.restype = C.c_int
            L.tzc_b200_version.restype = C.c_char_p
            _lib = L
        return _lib


def check(rc: int):
    if rc != TZC_OK:
        raise TzcError(rc, lib().tzc_b200_last_error().decode())
