"""Op-level API (the reference-facing entry point): a .tdsl op text plus an
instruction (builtin name or .intr path) and HOST numpy buffers, exactly the
inputs ``tzc verify op.tdsl --intrinsic X`` works from
(/root/reference/proj/src/cli.cpp:227-283).  Parsing, inspection, tiling and
the kernel plan are done by the C++ tzc host library inside libtzc_b200.so;
the tensorized body runs on the B200.  No CPU fallback exists.
"""
from __future__ import annotations

import ctypes as C
import re

import numpy as np

from ._capi import check, lib

NP = {"u8": np.uint8, "i8": np.int8, "u16": np.uint16, "i16": np.int16, "u32": np.uint32, "i32": np.int32,
      "fp16": np.uint16, "fp32": np.float32}


def _text(fn, *args, cap=1 << 16):
    while True:
        buf = C.create_string_buffer(cap)
        rc = fn(*args, buf, cap)
        if rc == 0:
            return buf.value.decode()
        if "buffer too small" in lib().tzc_b200_last_error().decode() and cap < (1 << 26):
            cap *= 16
            continue
        check(rc)


def parse(op_text: str) -> str:
    """parse_compute + infer_types, printed back (print_compute)."""
    return _text(lib().tzc_b200_parse, op_text.encode())


def builtin_names() -> list:
    return _text(lib().tzc_b200_builtins).split()


def print_intrinsic(intrinsic: str) -> str:
    """The instruction description in the reference's .intr grammar."""
    return _text(lib().tzc_b200_print_intrinsic, intrinsic.encode())


def inspect(op_text: str, intrinsic: str, grouped: bool = False) -> list:
    """Feasible loop mappings, reference order ("{y->i, k->j}" strings)."""
    return [ln for ln in _text(lib().tzc_b200_inspect, op_text.encode(), intrinsic.encode(), int(grouped)).splitlines()
            if ln]


def describe(op_text: str, intrinsic: str) -> str:
    return _text(lib().tzc_b200_describe, op_text.encode(), intrinsic.encode())


def declarations(op_text: str):
    """[(name, dtype, role, shape)] in declaration order."""
    out = []
    for m in re.finditer(r"tensor (\w+) : (\w+) \[([\d, ]+)\] (input|output)", op_text):
        out.append((m.group(1), m.group(2), m.group(4), tuple(int(v) for v in m.group(3).split(","))))
    return out


def _enc(s):
    return None if s is None else s.encode()


def lower(op_text: str, schedule: str | None = None, intrinsic: str | None = None) -> str:
    """print_tensor_ir(lower(op, schedule)) (+ inject_intrinsic when ``intrinsic``
    is given); ``schedule=None`` uses tile_and_reorder's schedule of the first
    device-realisable mapping (proj/include/tzc/rewriter.hpp:85-95)."""
    return _text(lib().tzc_b200_lower, op_text.encode(), _enc(schedule), _enc(intrinsic))


def tensor_text(path: str, max_elems: int = 64) -> str:
    """tensor_to_text(load_tensor(path)) — the reference's TNSR container."""
    return _text(lib().tzc_b200_tensor_text, path.encode(), max_elems)


def tensor_roundtrip(src: str, dst: str) -> None:
    check(lib().tzc_b200_tensor_roundtrip(src.encode(), dst.encode()))


def eval_tir(op_text: str, intrinsic: str, inputs: dict, schedule: str | None = None, epilogue: str | None = None,
             out: np.ndarray | None = None):
    """The reference chain lower -> inject_intrinsic -> eval_tir, executed on the
    B200 (tcgen05 instructions only).  Buffers as for :func:`run_op`."""
    return run_op(op_text, intrinsic, inputs, epilogue, out, _schedule=schedule, _via_ir=True)


def run_op(op_text: str, intrinsic: str, inputs: dict, epilogue: str | None = None, out: np.ndarray | None = None,
           _schedule: str | None = None, _via_ir: bool = False):
    """Execute the tensorized op on the GPU from host buffers.

    ``inputs`` maps tensor names to arrays at the declared element width
    (fp16 as uint16 bit patterns); accumulate-form ops take the output's
    initial image under the output's name.  ``epilogue`` is the optional
    requantize / cast op over the output (fused)."""
    decl = declarations(op_text)
    out_decl = next(d for d in decl if d[2] == "output")
    odt = out_decl[1]
    if epilogue is not None:
        odt = next(d for d in declarations(epilogue) if d[2] == "output")[1]
    if out is None:
        out = np.empty(out_decl[3], dtype=NP[odt])
    names = list(inputs)
    arrs = [np.ascontiguousarray(inputs[n]) for n in names]
    cn = (C.c_char_p * len(names))(*[n.encode() for n in names])
    cp = (C.c_void_p * len(names))(*[a.ctypes.data for a in arrs])
    if _via_ir:
        rc = lib().tzc_b200_eval_tir(op_text.encode(), _enc(_schedule), intrinsic.encode(), _enc(epilogue),
                                     len(names), cn, cp, C.c_void_p(out.ctypes.data), out.nbytes)
    else:
        rc = lib().tzc_b200_run_op(op_text.encode(), intrinsic.encode(), _enc(epilogue), len(names), cn, cp,
                                   C.c_void_p(out.ctypes.data), out.nbytes)
    check(rc)
    return out
