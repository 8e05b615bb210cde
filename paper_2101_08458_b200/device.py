"""Device-level wrappers over the C ABI for torch CUDA tensors.

torch supplies device memory and streams only; every byte of arithmetic is
done by the sm_100a kernels in libtzc_b200.so (tcgen05 kind::i8 / kind::f16).
"""
from __future__ import annotations

import ctypes as C

import torch

from ._capi import (EP_CAST_F16, EP_F32, EP_I32, EP_REQUANT_I8, PROFILE_F16, PROFILE_U8I8,
                    ConvDesc, Epilogue, GemmDesc, OutLayout, Plan, check, lib)

EPILOGUES = {"i32": EP_I32, "requant_i8": EP_REQUANT_I8, "f32": EP_F32, "f16": EP_CAST_F16}
_OUT_DTYPE = {EP_I32: torch.int32, EP_REQUANT_I8: torch.int8, EP_F32: torch.float32,
              EP_CAST_F16: torch.float16}


def _ptr(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def _stream(stream):
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def nhwc_layout(n_channels: int) -> OutLayout:
    return OutLayout(nb=n_channels, stride_m=n_channels, stride_blk=0)


def blocked_layout(n_channels: int, m: int, kb: int) -> OutLayout:
    """conv2d_tdsl output [K/kb, OH, OW, kb] (proj/src/workloads.cpp:85-86)."""
    return OutLayout(nb=kb, stride_m=kb, stride_blk=m * kb)


def conv_desc(x_shape, w_shape, stride, f16=False, w_layout="krsc", out_layout=None) -> ConvDesc:
    n, hp, wp, c = x_shape
    if w_layout == "krsc":
        k, r, s, c2 = w_shape
        wsk, wst = r * s * c, c
    elif w_layout == "rskc":
        r, s, k, c2 = w_shape
        wsk, wst = c, k * c
    else:
        raise ValueError(w_layout)
    assert c == c2, "channel mismatch"
    oh, ow = (hp - r) // stride + 1, (wp - s) // stride + 1
    d = ConvDesc(profile=PROFILE_F16 if f16 else PROFILE_U8I8, n=n, hp=hp, wp=wp, c=c, k=k, r=r, s=s,
                 stride=stride, w_stride_k=wsk, w_stride_tap=wst)
    d.out = out_layout if out_layout is not None else nhwc_layout(k)
    return d, (n, oh, ow, k)


def plan_conv(d: ConvDesc) -> dict:
    p = Plan()
    check(lib().tzc_b200_plan_conv(C.byref(d), C.byref(p)))
    return p.as_dict()


def plan_gemm(d: GemmDesc) -> dict:
    p = Plan()
    check(lib().tzc_b200_plan_gemm(C.byref(d), C.byref(p)))
    return p.as_dict()


def conv2d(x, w, stride=1, seed=None, epilogue="i32", scale=1.0, out=None, w_layout="krsc",
           out_layout=None, out_shape=None, stream=None):
    """Valid conv over pre-padded NHWC ``x`` ([N,Hp,Wp,C] uint8 / float16) with
    weights ``w`` ([K,R,S,C] int8 / float16, or [R,S,K,C] with w_layout='rskc')."""
    f16 = x.dtype == torch.float16
    d, shape = conv_desc(tuple(x.shape), tuple(w.shape), stride, f16, w_layout, out_layout)
    kind = EPILOGUES[epilogue]
    if out is None:
        out = torch.empty(out_shape or shape, dtype=_OUT_DTYPE[kind], device=x.device)
    ep = Epilogue(kind=kind, scale=scale)
    fn = lib().tzc_b200_conv2d_f16 if f16 else lib().tzc_b200_conv2d_i8
    check(fn(C.byref(d), _ptr(x), _ptr(w), _ptr(seed), _ptr(out), C.byref(ep), _stream(stream)))
    return out


def gemm(a, b, seed=None, epilogue="i32", scale=1.0, out=None, b_kn=False, out_layout=None, stream=None):
    """C = seed + A @ B^T (B [N,K]) or A @ B (b_kn, B [K,N]), tcgen05 on sm_100a."""
    f16 = a.dtype == torch.float16
    m, k = a.shape
    n = b.shape[1] if b_kn else b.shape[0]
    d = GemmDesc(profile=PROFILE_F16 if f16 else PROFILE_U8I8, m=m, n=n, k=k, b_kn=int(b_kn))
    d.out = out_layout if out_layout is not None else nhwc_layout(n)
    kind = EPILOGUES[epilogue]
    if out is None:
        out = torch.empty((m, n), dtype=_OUT_DTYPE[kind], device=a.device)
    ep = Epilogue(kind=kind, scale=scale)
    fn = lib().tzc_b200_gemm_f16 if f16 else lib().tzc_b200_gemm_i8
    check(fn(C.byref(d), _ptr(a), _ptr(b), _ptr(seed), _ptr(out), C.byref(ep), _stream(stream)))
    return out


def tune_conv2d(x, w, stride=1, seed=None, epilogue="i32", scale=1.0, out=None, w_layout="krsc",
                out_layout=None, out_shape=None, stream=None, reps=10, apply=True):
    """Measured-time plan search for this conv (tzc_b200_tune_conv): returns
    (best candidate index, log text); with ``apply`` later launches of the same
    descriptor use the winner."""
    f16 = x.dtype == torch.float16
    d, shape = conv_desc(tuple(x.shape), tuple(w.shape), stride, f16, w_layout, out_layout)
    kind = EPILOGUES[epilogue]
    if out is None:
        out = torch.empty(out_shape or shape, dtype=_OUT_DTYPE[kind], device=x.device)
    ep = Epilogue(kind=kind, scale=scale)
    log = C.create_string_buffer(1 << 14)
    best = lib().tzc_b200_tune_conv(C.byref(d), _ptr(x), _ptr(w), _ptr(seed), _ptr(out), C.byref(ep), int(reps),
                                    int(apply), log, len(log), _stream(stream))
    if best < 0:
        check(best)
    return best, log.value.decode()


def tune_gemm(a, b, seed=None, epilogue="i32", scale=1.0, out=None, b_kn=False, out_layout=None, stream=None,
              reps=10, apply=True):
    """As :func:`tune_conv2d` for a matmul (tzc_b200_tune_gemm)."""
    f16 = a.dtype == torch.float16
    m, k = a.shape
    n = b.shape[1] if b_kn else b.shape[0]
    d = GemmDesc(profile=PROFILE_F16 if f16 else PROFILE_U8I8, m=m, n=n, k=k, b_kn=int(b_kn))
    d.out = out_layout if out_layout is not None else nhwc_layout(n)
    kind = EPILOGUES[epilogue]
    if out is None:
        out = torch.empty((m, n), dtype=_OUT_DTYPE[kind], device=a.device)
    ep = Epilogue(kind=kind, scale=scale)
    log = C.create_string_buffer(1 << 14)
    best = lib().tzc_b200_tune_gemm(C.byref(d), _ptr(a), _ptr(b), _ptr(seed), _ptr(out), C.byref(ep), int(reps),
                                    int(apply), log, len(log), _stream(stream))
    if best < 0:
        check(best)
    return best, log.value.decode()


def tune_candidates() -> list:
    buf = C.create_string_buffer(1 << 12)
    check(lib().tzc_b200_tune_candidates(buf, len(buf)))
    return buf.value.decode().split("\n")[:-1]


def set_conv_plan(x_shape, w_shape, stride=1, f16=False, w_layout="krsc", out_layout=None, spec=""):
    """Install (or clear, spec="") per-descriptor plan options for this conv."""
    d, _ = conv_desc(tuple(x_shape), tuple(w_shape), stride, f16, w_layout, out_layout)
    check(lib().tzc_b200_set_problem_options_conv(C.byref(d), spec.encode()))


def clear_tuning():
    check(lib().tzc_b200_clear_tuning())


def save_tuning(path: str) -> int:
    """Write every installed per-descriptor plan to the plan-cache file `path`."""
    n = C.c_int32(0)
    check(lib().tzc_b200_save_tuning(str(path).encode(), C.byref(n)))
    return n.value


def load_tuning(path: str) -> int:
    """Install the plans a saved plan-cache file holds; returns how many."""
    n = C.c_int32(0)
    check(lib().tzc_b200_load_tuning(str(path).encode(), C.byref(n)))
    return n.value


def unblock_data(src, c, h, w, cb, stream=None):
    dst = torch.empty((1, h, w, c), dtype=src.dtype, device=src.device)
    check(lib().tzc_b200_unblock_data(_ptr(src), _ptr(dst), c, h, w, cb, src.element_size(), _stream(stream)))
    return dst


def unblock_kernel(src, k, c, r, s, kb, cb, stream=None):
    dst = torch.empty((k, r, s, c), dtype=src.dtype, device=src.device)
    check(lib().tzc_b200_unblock_kernel(_ptr(src), _ptr(dst), k, c, r, s, kb, cb, src.element_size(),
                                        _stream(stream)))
    return dst


def set_splits(n: int):
    check(lib().tzc_b200_set_splits(n))


def set_option(name: str, value: int):
    check(lib().tzc_b200_set_option(name.encode(), int(value)))


def launch_count() -> int:
    return int(lib().tzc_b200_launch_count())


LAUNCH_KERNELS = {0: "general", 1: "shifted_window", 2: "s2d_stem", 3: "cta_pair", 4: "k7_gemm", 5: "stem_fused"}


def last_launch() -> dict:
    """The executed tile of this thread's most recent conv / GEMM launch
    (tzc_b200_last_launch): kernel family, cta_group, bm, bn, bk_bytes, ..."""
    from ._capi import LaunchInfo
    info = LaunchInfo()
    check(lib().tzc_b200_last_launch(C.byref(info)))
    out = {f: getattr(info, f) for f, _ in LaunchInfo._fields_}
    out["kernel"] = LAUNCH_KERNELS.get(out["kernel"], str(out["kernel"]))
    return out
