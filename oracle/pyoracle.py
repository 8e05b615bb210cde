"""TEST INFRASTRUCTURE — NOT PRODUCT CODE.

ctypes front for the two checkers (see oracle/Makefile):

* ``Ref``  — the reference implementation itself (``oracle/_ref/libtzc_ref.so``,
  compiled unmodified from /root/reference/proj/src with ``-Dtzc=tzc_ref``)
  behind ``oracle/ref_bridge.cpp``: parse, ``random_inputs``,
  ``eval_reference`` (the oracle, proj/src/vm.cpp:444-508) and ``eval_tir``
  (the reference's hot path, proj/src/vm.cpp:510-516).
* ``Orc``  — our C restatement (``oracle/_build/liboracle.so``), pinned to
  ``Ref`` and to the reference's golden vectors in tests/test_oracle.py.

Only tests/, bench.py's cpu_baseline / ``--impl reference`` legs and
``__graft_entry__.smoke()`` import this module.
"""
from __future__ import annotations

import ctypes as C
import os
import threading
from concurrent.futures import ThreadPoolExecutor

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libtzc_ref.so")
ORC_SO = os.path.join(HERE, "_build", "liboracle.so")

NP_DTYPE = {"u8": np.uint8, "i8": np.int8, "u16": np.uint16, "i16": np.int16,
            "u32": np.uint32, "i32": np.int32, "fp16": np.uint16, "fp32": np.float32}
ORC_CODE = {"u8": 0, "i8": 1, "u16": 2, "i16": 3, "u32": 4, "i32": 5, "fp16": 6, "fp32": 7}

_P = C.c_void_p
_I64 = C.c_int64


def _ptr(a):
    return None if a is None else C.c_void_p(a.ctypes.data)


class OpInfo:
    """Tensor/loop declarations of a parsed op (as the reference sees it)."""

    def __init__(self, text: str):
        self.tensors = {}   # name -> (dtype, role, shape)
        self.order = []
        self.loops = []     # (name, kind, extent)
        self.update = False
        for line in text.splitlines():
            f = line.split()
            if not f:
                continue
            if f[0] == "tensor":
                rank = int(f[4])
                self.tensors[f[1]] = (f[2], f[3], tuple(int(x) for x in f[5:5 + rank]))
                self.order.append(f[1])
            elif f[0] == "loop":
                self.loops.append((f[1], f[2], int(f[3])))
            elif f[0] == "update":
                self.update = f[1] == "1"

    @property
    def output(self):
        return next(n for n in self.order if self.tensors[n][1] == "out")

    def np_dtype(self, name):
        return NP_DTYPE[self.tensors[name][0]]

    def shape(self, name):
        return self.tensors[name][2]


class Ref:
    """The reference implementation (compiled from /root/reference)."""

    _lock = threading.Lock()
    _lib = None

    @classmethod
    def available(cls) -> bool:
        return os.path.exists(REF_SO)

    @classmethod
    def lib(cls):
        with cls._lock:
            if cls._lib is None:
                if not os.path.exists(REF_SO):
                    raise RuntimeError(f"reference oracle not built: {REF_SO} (run make -C oracle)")
                L = C.CDLL(REF_SO)
                L.tzcref_last_error.restype = C.c_char_p
                for fn in ("tzcref_op_info",):
                    getattr(L, fn).argtypes = [C.c_char_p, C.c_char_p, _I64]
                L.tzcref_random_tensor.argtypes = [C.c_char_p, C.c_char_p, C.c_uint64, _P, _I64]
                L.tzcref_eval_reference.argtypes = [C.c_char_p, C.c_int, C.POINTER(C.c_char_p),
                                                    C.POINTER(_P), _P, _I64]
                L.tzcref_eval_tir.argtypes = [C.c_char_p, C.c_char_p, C.c_int, C.POINTER(C.c_char_p),
                                              C.POINTER(_P), _P, _I64]
                L.tzcref_tensorize.argtypes = [C.c_char_p, C.c_char_p, C.c_char_p, _I64]
                L.tzcref_inspect.argtypes = [C.c_char_p, C.c_char_p, C.c_char_p, _I64]
                L.tzcref_lower.argtypes = [C.c_char_p, C.c_char_p, C.c_char_p, C.c_char_p, _I64]
                L.tzcref_save_case.argtypes = [C.c_char_p, C.c_uint64, C.c_char_p]
                L.tzcref_tensor_text.argtypes = [C.c_char_p, _I64, C.c_char_p, _I64]
                L.tzcref_matmul_tdsl.argtypes = [_I64, _I64, _I64, C.c_int, C.c_char_p, _I64]
                L.tzcref_conv2d_tdsl.argtypes = [_I64] * 7 + [C.c_int, C.c_char_p, _I64]
                L.tzcref_conv3d_tdsl.argtypes = [_I64] * 7 + [C.c_int, C.c_char_p, _I64]
                L.tzcref_f64_to_f16_bits.argtypes = [C.c_double]
                L.tzcref_f64_to_f16_bits.restype = C.c_uint16
                L.tzcref_f16_bits_to_f64.argtypes = [C.c_uint16]
                L.tzcref_f16_bits_to_f64.restype = C.c_double
                cls._lib = L
            return cls._lib

    @classmethod
    def _check(cls, rc):
        if rc != 0:
            raise RuntimeError(cls.lib().tzcref_last_error().decode())

    @classmethod
    def _text(cls, fn, *args, cap=1 << 20):
        buf = C.create_string_buffer(cap)
        cls._check(fn(*args, buf, cap))
        return buf.value.decode()

    @classmethod
    def op_info(cls, op_text: str) -> OpInfo:
        return OpInfo(cls._text(cls.lib().tzcref_op_info, op_text.encode()))

    @classmethod
    def matmul_tdsl(cls, m, n, k, fp16=False) -> str:
        return cls._text(cls.lib().tzcref_matmul_tdsl, m, n, k, int(fp16))

    @classmethod
    def conv2d_tdsl(cls, in_c, in_hw, out_c, kernel, stride=1, lane_block=16, red_block=4,
                    fp16=False) -> str:
        return cls._text(cls.lib().tzcref_conv2d_tdsl, in_c, in_hw, out_c, kernel, stride,
                         lane_block, red_block, int(fp16))

    @classmethod
    def conv3d_tdsl(cls, in_c, in_hw, out_c, kernel, stride=1, lane_block=16, red_block=4,
                    fp16=False) -> str:
        return cls._text(cls.lib().tzcref_conv3d_tdsl, in_c, in_hw, out_c, kernel, stride,
                         lane_block, red_block, int(fp16))

    @classmethod
    def tensorize(cls, op_text, intrinsic) -> str:
        return cls._text(cls.lib().tzcref_tensorize, op_text.encode(), intrinsic.encode())

    @classmethod
    def save_case(cls, op_text, seed, directory):
        cls._check(cls.lib().tzcref_save_case(op_text.encode(), seed, directory.encode()))

    @classmethod
    def tensor_text(cls, path, max_elems=1 << 30) -> str:
        return cls._text(cls.lib().tzcref_tensor_text, path.encode(), max_elems, cap=1 << 26)

    @classmethod
    def lower(cls, op_text, schedule, intrinsic=None) -> str:
        return cls._text(cls.lib().tzcref_lower, op_text.encode(), schedule.encode(),
                         None if intrinsic is None else intrinsic.encode())

    @classmethod
    def inspect(cls, op_text, intrinsic) -> list:
        t = cls._text(cls.lib().tzcref_inspect, op_text.encode(), intrinsic.encode())
        return [ln.rsplit(" ", 1) for ln in t.splitlines() if ln]

    @classmethod
    def random_inputs(cls, op_text: str, seed: int) -> dict:
        """random_inputs(op, seed) (proj/src/vm.cpp:59-68), packed."""
        info = cls.op_info(op_text)
        out = {}
        for name in info.order:
            role = info.tensors[name][1]
            if role == "in" or (role == "out" and info.update):
                a = np.empty(info.shape(name), dtype=info.np_dtype(name))
                cls._check(cls.lib().tzcref_random_tensor(op_text.encode(), name.encode(), seed,
                                                          _ptr(a), a.nbytes))
                out[name] = a
        return out

    @classmethod
    def _eval(cls, fn, pre, op_text, inputs):
        info = cls.op_info(op_text)
        names = list(inputs)
        arrs = [np.ascontiguousarray(inputs[n], dtype=info.np_dtype(n)) for n in names]
        out = np.empty(info.shape(info.output), dtype=info.np_dtype(info.output))
        cn = (C.c_char_p * len(names))(*[n.encode() for n in names])
        cp = (_P * len(names))(*[a.ctypes.data for a in arrs])
        cls._check(fn(op_text.encode(), *pre, len(names), cn, cp, _ptr(out), out.nbytes))
        return out

    @classmethod
    def eval_reference(cls, op_text: str, inputs: dict) -> np.ndarray:
        return cls._eval(cls.lib().tzcref_eval_reference, (), op_text, inputs)

    @classmethod
    def eval_tir(cls, op_text: str, intrinsic: str, inputs: dict) -> np.ndarray:
        return cls._eval(cls.lib().tzcref_eval_tir, (intrinsic.encode(),), op_text, inputs)

    @classmethod
    def f64_to_f16_bits(cls, x: float) -> int:
        return cls.lib().tzcref_f64_to_f16_bits(x)


class Orc:
    """Our C restatement of the reference arithmetic (oracle/oracle.c)."""

    _lib = None
    _lock = threading.Lock()

    @classmethod
    def lib(cls):
        with cls._lock:
            if cls._lib is None:
                if not os.path.exists(ORC_SO):
                    raise RuntimeError(f"oracle restatement not built: {ORC_SO} (run make -C oracle)")
                L = C.CDLL(ORC_SO)
                L.orc_random_fill.argtypes = [C.c_int, C.c_uint64, _I64, _P]
                L.orc_f64_to_f16_bits.argtypes = [C.c_double]
                L.orc_f64_to_f16_bits.restype = C.c_uint16
                L.orc_f16_bits_to_f64.argtypes = [C.c_uint16]
                L.orc_f16_bits_to_f64.restype = C.c_double
                L.orc_wrap_int.argtypes = [_I64, C.c_int, C.c_int]
                L.orc_wrap_int.restype = _I64
                L.orc_matmul_u8i8.argtypes = [_I64] * 3 + [_P] * 4 + [_I64] * 2
                L.orc_matmul_f16.argtypes = [_I64] * 3 + [_P] * 4 + [_I64] * 2
                L.orc_conv2d_nhwc_u8i8.argtypes = [_I64] * 8 + [_P] * 4 + [_I64] * 2
                L.orc_conv2d_nhwc_f16.argtypes = [_I64] * 8 + [_P] * 4 + [_I64] * 2
                L.orc_conv2d_blocked_u8i8.argtypes = [_I64] * 7 + [_P] * 4 + [_I64] * 2
                L.orc_conv2d_blocked_f16.argtypes = [_I64] * 7 + [_P] * 4 + [_I64] * 2
                L.orc_requant_i8.argtypes = [_I64, _P, C.c_float, _P]
                L.orc_cast_f16.argtypes = [_I64, _P, _P]
                cls._lib = L
            return cls._lib

    # ---- inputs ------------------------------------------------------------
    @classmethod
    def random_tensor(cls, dtype: str, shape, seed: int) -> np.ndarray:
        a = np.empty(shape, dtype=NP_DTYPE[dtype])
        cls.lib().orc_random_fill(ORC_CODE[dtype], seed, a.size, _ptr(a))
        return a

    @classmethod
    def random_inputs(cls, decls, seed: int, update=True) -> dict:
        """decls: ordered [(name, dtype, role, shape)] as declared in the op;
        mirrors random_inputs' seed + declaration-index rule (vm.cpp:59-68)."""
        out = {}
        for k, (name, dt, role, shape) in enumerate(decls):
            if role == "in" or (role == "out" and update):
                out[name] = cls.random_tensor(dt, shape, seed + k)
        return out

    # ---- arithmetic ----------------------------------------------------------
    @staticmethod
    def _par(fn, lo, hi, threads):
        threads = max(1, min(threads, hi - lo))
        if threads == 1:
            fn(lo, hi)
            return
        step = (hi - lo + threads - 1) // threads
        with ThreadPoolExecutor(threads) as ex:
            list(ex.map(lambda a: fn(a, min(hi, a + step)), range(lo, hi, step)))

    @classmethod
    def matmul(cls, A, B, seed=None, fp16=False, threads=os.cpu_count()):
        M, K = A.shape
        N = B.shape[1] if fp16 else B.shape[0]
        out = np.zeros((M, N), dtype=np.float32 if fp16 else np.int32)
        fn = cls.lib().orc_matmul_f16 if fp16 else cls.lib().orc_matmul_u8i8
        A, B = np.ascontiguousarray(A), np.ascontiguousarray(B)
        s = None if seed is None else np.ascontiguousarray(seed)
        cls._par(lambda a, b: fn(M, N, K, _ptr(A), _ptr(B), _ptr(s), _ptr(out), a, b), 0, M, threads)
        return out

    @classmethod
    def conv2d_nhwc(cls, x, w, stride, seed=None, fp16=False, threads=os.cpu_count()):
        N, Hp, Wp, Cin = x.shape
        K, R, S, _ = w.shape
        OH, OW = (Hp - R) // stride + 1, (Wp - S) // stride + 1
        out = np.zeros((N, OH, OW, K), dtype=np.float32 if fp16 else np.int32)
        fn = cls.lib().orc_conv2d_nhwc_f16 if fp16 else cls.lib().orc_conv2d_nhwc_u8i8
        x, w = np.ascontiguousarray(x), np.ascontiguousarray(w)
        s = None if seed is None else np.ascontiguousarray(seed)
        cls._par(lambda a, b: fn(N, Hp, Wp, Cin, K, R, S, stride, _ptr(x), _ptr(w), _ptr(s),
                                 _ptr(out), a, b), 0, N, threads)
        return out

    @classmethod
    def conv2d_blocked(cls, data, kernel, stride, seed=None, fp16=False, threads=os.cpu_count()):
        CO, H, W, cb = data.shape
        KO, _, R, _, kb, _ = kernel.shape
        OH = (H - R) // stride + 1
        out = np.zeros((KO, OH, OH, kb), dtype=np.float32 if fp16 else np.int32)
        fn = cls.lib().orc_conv2d_blocked_f16 if fp16 else cls.lib().orc_conv2d_blocked_u8i8
        data, kernel = np.ascontiguousarray(data), np.ascontiguousarray(kernel)
        s = None if seed is None else np.ascontiguousarray(seed)
        cls._par(lambda a, b: fn(CO * cb, H, KO * kb, R, stride, cb, kb, _ptr(data), _ptr(kernel),
                                 _ptr(s), _ptr(out), a, b), 0, OH, threads)
        return out

    @classmethod
    def requant_i8(cls, c, scale: float):
        c = np.ascontiguousarray(c, dtype=np.int32)
        q = np.empty(c.shape, dtype=np.int8)
        cls.lib().orc_requant_i8(c.size, _ptr(c), C.c_float(scale), _ptr(q))
        return q

    @classmethod
    def cast_f16(cls, c):
        c = np.ascontiguousarray(c, dtype=np.float32)
        h = np.empty(c.shape, dtype=np.uint16)
        cls.lib().orc_cast_f16(c.size, _ptr(c), _ptr(h))
        return h

    @classmethod
    def f64_to_f16_bits(cls, x: float) -> int:
        return cls.lib().orc_f64_to_f16_bits(x)
