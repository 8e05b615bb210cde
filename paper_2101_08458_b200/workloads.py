"""Workload op-text generators and the ResNet-50 conv bank.

* ``matmul_tdsl`` / ``conv2d_tdsl`` emit exactly the reference's texts
  (/root/reference/proj/src/workloads.cpp:41-92): int8 matmul keeps B as
  [N,K], fp16 matmul as [K,N]; conv is channel-blocked and valid.
* ``conv2d_nhwc_tdsl`` is the batched generator this backend adds
  (SURVEY.md §2.1 row 10): NHWC data with a leading batch dim over a
  spatially pre-padded input, [K,R,S,C] weights, [N,OH,OW,K] output.  It is
  ordinary surface DSL, so the reference parser/interpreter accept it
  unchanged (that is how parity is checked).
* ``requant_tdsl`` / ``cast_f16_tdsl`` are the reference-expressible
  epilogue ops.
* ``RESNET50_V15`` is SURVEY.md Appendix A (23 distinct conv shapes).
"""
from __future__ import annotations

from dataclasses import dataclass


def _dt(fp16: bool):
    return ("fp16", "fp16", "fp32") if fp16 else ("u8", "i8", "i32")


def matmul_tdsl(m: int, n: int, k: int, fp16: bool = False) -> str:
    d, w, a = _dt(fp16)
    b_decl = f"[{k}, {n}]" if fp16 else f"[{n}, {k}]"
    b_idx = "B[k, y]" if fp16 else "B[y, k]"
    return (f"tensor A : {d} [{m}, {k}] input\n"
            f"tensor B : {w} {b_decl} input\n"
            f"tensor C : {a} [{m}, {n}] output\n"
            f"loop x : dp {m}\nloop y : dp {n}\nloop k : red {k}\n"
            f"C[x, y] += cast<{a}>(A[x, k]) * cast<{a}>({b_idx})\n")


def _strided(o: str, st: int, i: str) -> str:
    return f"{o} + {i}" if st == 1 else f"{o} * {st} + {i}"


def conv2d_tdsl(in_c, in_hw, out_c, kernel, stride=1, lane_block=16, red_block=4, fp16=False) -> str:
    d, w, a = _dt(fp16)
    co, ko = in_c // red_block, out_c // lane_block
    ohw = (in_hw - kernel) // stride + 1
    data = f"data[co, {_strided('oh', stride, 'r')}, {_strided('ow', stride, 's')}, ci]"
    return (f"tensor data : {d} [{co}, {in_hw}, {in_hw}, {red_block}] input\n"
            f"tensor kernel : {w} [{ko}, {co}, {kernel}, {kernel}, {lane_block}, {red_block}] input\n"
            f"tensor out : {a} [{ko}, {ohw}, {ohw}, {lane_block}] output\n"
            f"loop ko : dp {ko}\nloop oh : dp {ohw}\nloop ow : dp {ohw}\nloop ki : dp {lane_block}\n"
            f"loop co : red {co}\nloop r : red {kernel}\nloop s : red {kernel}\nloop ci : red {red_block}\n"
            f"out[ko, oh, ow, ki] += cast<{a}>({data}) * cast<{a}>(kernel[ko, co, r, s, ki, ci])\n")


def conv3d_tdsl(in_c, in_hw, out_c, kernel, stride=1, lane_block=16, red_block=4, fp16=False) -> str:
    """The reference's conv3d_tdsl (proj/src/workloads.cpp:94-121): channel-blocked
    valid 3-D conv, data [C/rb, D, H, W, rb], kernel [K/lb, C/rb, kd, kh, kw, lb, rb]."""
    d, w, a = _dt(fp16)
    co, ko = in_c // red_block, out_c // lane_block
    o = (in_hw - kernel) // stride + 1
    x = (f"data[co, {_strided('od', stride, 'rd')}, {_strided('oh', stride, 'rh')}, "
         f"{_strided('ow', stride, 'rw')}, ci]")
    return (f"tensor data : {d} [{co}, {in_hw}, {in_hw}, {in_hw}, {red_block}] input\n"
            f"tensor kernel : {w} [{ko}, {co}, {kernel}, {kernel}, {kernel}, {lane_block}, {red_block}] input\n"
            f"tensor out : {a} [{ko}, {o}, {o}, {o}, {lane_block}] output\n"
            f"loop ko : dp {ko}\nloop od : dp {o}\nloop oh : dp {o}\nloop ow : dp {o}\nloop ki : dp {lane_block}\n"
            f"loop co : red {co}\nloop rd : red {kernel}\nloop rh : red {kernel}\nloop rw : red {kernel}\n"
            f"loop ci : red {red_block}\n"
            f"out[ko, od, oh, ow, ki] += cast<{a}>({x}) * cast<{a}>(kernel[ko, co, rd, rh, rw, ki, ci])\n")


def conv2d_nhwc_tdsl(n, hp, wp, c, k, r, s, stride=1, fp16=False) -> str:
    d, w, a = _dt(fp16)
    oh, ow = (hp - r) // stride + 1, (wp - s) // stride + 1
    x = f"data[n, {_strided('oh', stride, 'r')}, {_strided('ow', stride, 's')}, c]"
    return (f"tensor data : {d} [{n}, {hp}, {wp}, {c}] input\n"
            f"tensor kernel : {w} [{k}, {r}, {s}, {c}] input\n"
            f"tensor out : {a} [{n}, {oh}, {ow}, {k}] output\n"
            f"loop n : dp {n}\nloop oh : dp {oh}\nloop ow : dp {ow}\nloop k : dp {k}\n"
            f"loop r : red {r}\nloop s : red {s}\nloop c : red {c}\n"
            f"out[n, oh, ow, k] += cast<{a}>({x}) * cast<{a}>(kernel[k, r, s, c])\n")


def _shape_str(shape):
    return "[" + ", ".join(str(x) for x in shape) + "]"


def _idx(shape):
    names = [f"i{j}" for j in range(len(shape))]
    loops = "".join(f"loop {nm} : dp {e}\n" for nm, e in zip(names, shape))
    return names, loops


def requant_tdsl(shape, scale: float, src="C", dst="Q") -> str:
    """Q = cast<i8>(cast<fp32>(C) * s) over an i32 tensor of ``shape``."""
    names, loops = _idx(shape)
    ix = ", ".join(names)
    return (f"tensor {src} : i32 {_shape_str(shape)} input\n"
            f"tensor {dst} : i8 {_shape_str(shape)} output\n{loops}"
            f"{dst}[{ix}] = cast<i8>(cast<fp32>({src}[{ix}]) * {float_literal(scale)})\n")


def cast_f16_tdsl(shape, src="C", dst="H") -> str:
    names, loops = _idx(shape)
    ix = ", ".join(names)
    return (f"tensor {src} : fp32 {_shape_str(shape)} input\n"
            f"tensor {dst} : fp16 {_shape_str(shape)} output\n{loops}"
            f"{dst}[{ix}] = cast<fp16>({src}[{ix}])\n")


def float_literal(x: float) -> str:
    """Decimal literal the reference lexer reads back exactly (strtod)."""
    s = repr(float(x))
    if "e" in s or "E" in s:
        s = "%.17e" % x
    if "." not in s and "e" not in s:
        s += ".0"
    return s


# ---- ResNet-50 v1.5 distinct conv shapes ------------
@dataclass(frozen=True)
class ConvLayer:
    name: str
    c: int       # input channels
    h: int       # input spatial extent, pad materialised (H + 2*pad)
    k: int       # output channels
    r: int       # square filter
    stride: int
    occ: int     # occurrences in the network

    def out_hw(self) -> int:
        return (self.h - self.r) // self.stride + 1

    def macs(self, batch: int) -> int:
        o = self.out_hw()
        return batch * o * o * self.k * self.c * self.r * self.r

    def ops(self, batch: int) -> int:
        return 2 * self.macs(batch)

    def algo_bytes(self, batch: int, e_in: int = 1, e_out: int = 1) -> int:
        o = self.out_hw()
        return (batch * self.h * self.h * self.c * e_in + self.k * self.r * self.r * self.c * e_in
                + batch * o * o * self.k * e_out)


RESNET50_V15 = [
    ConvLayer("stem7x7", 3, 230, 64, 7, 2, 1),
    ConvLayer("c2_1x1_64_64", 64, 56, 64, 1, 1, 1),
    ConvLayer("c2_3x3_64", 64, 58, 64, 3, 1, 3),
    ConvLayer("c2_1x1_64_256", 64, 56, 256, 1, 1, 4),
    ConvLayer("c2_1x1_256_64", 256, 56, 64, 1, 1, 2),
    ConvLayer("c3_1x1_256_128", 256, 56, 128, 1, 1, 1),
    ConvLayer("c3_3x3s2_128", 128, 58, 128, 3, 2, 1),
    ConvLayer("c3_1x1_128_512", 128, 28, 512, 1, 1, 4),
    ConvLayer("c3_1x1s2_256_512", 256, 56, 512, 1, 2, 1),
    ConvLayer("c3_1x1_512_128", 512, 28, 128, 1, 1, 3),
    ConvLayer("c3_3x3_128", 128, 30, 128, 3, 1, 3),
    ConvLayer("c4_1x1_512_256", 512, 28, 256, 1, 1, 1),
    ConvLayer("c4_3x3s2_256", 256, 30, 256, 3, 2, 1),
    ConvLayer("c4_1x1_256_1024", 256, 14, 1024, 1, 1, 6),
    ConvLayer("c4_1x1s2_512_1024", 512, 28, 1024, 1, 2, 1),
    ConvLayer("c4_1x1_1024_256", 1024, 14, 256, 1, 1, 5),
    ConvLayer("c4_3x3_256", 256, 16, 256, 3, 1, 5),
    ConvLayer("c5_1x1_1024_512", 1024, 14, 512, 1, 1, 1),
    ConvLayer("c5_3x3s2_512", 512, 16, 512, 3, 2, 1),
    ConvLayer("c5_1x1_512_2048", 512, 7, 2048, 1, 1, 3),
    ConvLayer("c5_1x1s2_1024_2048", 1024, 14, 2048, 1, 2, 1),
    ConvLayer("c5_1x1_2048_512", 2048, 7, 512, 1, 1, 2),
    ConvLayer("c5_3x3_512", 512, 9, 512, 3, 1, 2),
]


def requant_scale(kg: int) -> float:
    """Power-of-two scale mapping ~3 sigma of a u8 x i8 sum over kg terms onto
    the int8 range (most outputs in range, tails wrap as the reference does)."""
    import math
    sigma = 10880.0 * math.sqrt(kg)
    return 2.0 ** -round(math.log2(3 * sigma / 127.0))


# The paper's Table-1 convolution bank (proj/src/workloads.cpp:123-142, table1_bank):
# (name, in_c, in_hw, out_c, kernel, stride), lowered by conv2d_tdsl with the
# reference's (lane_block, red_block) = (16, 4) channel blocking.
TABLE1_BANK = [
    ("conv01", 288, 35, 384, 3, 2), ("conv02", 160, 9, 224, 3, 1), ("conv03", 1056, 7, 192, 1, 1),
    ("conv04", 80, 73, 192, 3, 1), ("conv05", 128, 16, 128, 3, 1), ("conv06", 192, 16, 192, 3, 1),
    ("conv07", 256, 16, 256, 3, 1), ("conv08", 1024, 14, 512, 1, 1), ("conv09", 128, 16, 160, 3, 1),
    ("conv10", 576, 14, 192, 1, 1), ("conv11", 96, 16, 128, 3, 1), ("conv12", 1024, 14, 256, 1, 1),
    ("conv13", 576, 14, 128, 1, 1), ("conv14", 64, 29, 96, 3, 1), ("conv15", 64, 56, 128, 1, 2),
    ("conv16", 608, 14, 192, 1, 1),
]

# The resnet18-3d bank (proj/src/workloads.cpp:149-162, resnet18_3d_bank), lowered
# by conv3d_tdsl with (16, 4) blocking: (name, in_c, in_hw, out_c, kernel, stride).
RESNET18_3D_BANK = [
    ("block2_conv", 64, 56, 64, 3, 1), ("block3_down", 64, 56, 128, 3, 2), ("block3_conv", 128, 28, 128, 3, 1),
    ("block3_skip", 64, 56, 128, 1, 2), ("block4_down", 128, 28, 256, 3, 2), ("block4_conv", 256, 14, 256, 3, 1),
    ("block4_skip", 128, 28, 256, 1, 2), ("block5_down", 256, 14, 512, 3, 2), ("block5_conv", 512, 7, 512, 3, 1),
    ("block5_skip", 256, 14, 512, 1, 2),
]
