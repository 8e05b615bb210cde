"""The tzc host library (operator + instruction-registration API) against the
reference implementation on the same op texts: parse/print round trips,
Algorithm-1 matching and mapping enumeration (identical lists and order),
the tcgen05 descriptions in the reference's own .intr grammar, the fused
pixel-group extension, kernel plans, and the error taxonomy.  CPU only."""
import os
import tempfile

import pytest

from oracle.pyoracle import Ref
from paper_2101_08458_b200 import ops
from paper_2101_08458_b200._capi import TzcError
from paper_2101_08458_b200.workloads import RESNET50_V15, TABLE1_BANK, conv2d_nhwc_tdsl, conv2d_tdsl, conv3d_tdsl, matmul_tdsl

needs_ref = pytest.mark.skipif(not Ref.available(), reason="oracle/_ref not built")

OPS = [
    matmul_tdsl(16, 16, 64),
    matmul_tdsl(64, 48, 96),
    matmul_tdsl(16, 16, 16, fp16=True),
    conv2d_tdsl(64, 5, 16, 3),
    conv2d_tdsl(16, 10, 32, 3, 2),
    conv2d_nhwc_tdsl(2, 6, 6, 16, 32, 3, 3, 1),
    conv2d_nhwc_tdsl(1, 9, 9, 64, 64, 1, 1, 2),
]


@pytest.mark.parametrize("text", OPS)
def test_parse_print_roundtrip(text):
    once = ops.parse(text)
    assert ops.parse(once) == once


@needs_ref
@pytest.mark.parametrize("text", OPS)
def test_printed_op_is_the_reference_op(text):
    a, b = Ref.op_info(text), Ref.op_info(ops.parse(text))
    assert (a.tensors, a.loops, a.update) == (b.tensors, b.loops, b.update)


@needs_ref
@pytest.mark.parametrize("text", OPS)
@pytest.mark.parametrize("intr", ["vdot_16x4", "vdot_4x4", "wmma_16x16x16"])
def test_inspect_matches_reference(text, intr):
    ref = [m for m, _ in Ref.inspect(text, intr)]
    assert ops.inspect(text, intr) == ref


def test_builtins_include_reference_and_tcgen05():
    names = ops.builtin_names()
    for n in ("vdot_16x4", "vdot_4x4", "wmma_16x16x16", "tcgen05_i8_m128n256k32", "tcgen05_f16_m128n128k16",
              "tcgen05_f16_m128n64k16_mn"):
        assert n in names


@needs_ref
@pytest.mark.parametrize("intr", ["tcgen05_i8_m128n64k32", "tcgen05_i8_m128n256k32", "tcgen05_f16_m128n128k16_mn"])
def test_tcgen05_description_runs_through_the_reference(intr):
    """The tcgen05 description is plain .intr text: the reference parses it,
    inspects ops with it, and agrees with our 1:1 mapping enumeration."""
    text = ops.print_intrinsic(intr)
    with tempfile.TemporaryDirectory() as d:
        path = os.path.join(d, intr + ".intr")
        with open(path, "w") as f:
            f.write(text)
        fp16 = "f16" in intr
        for op in (matmul_tdsl(256, 128, 64, fp16=fp16), conv2d_nhwc_tdsl(1, 6, 6, 64, 64, 3, 3, 1, fp16=fp16)):
            assert ops.inspect(op, path) == [m for m, _ in Ref.inspect(op, path)]


def test_fused_pixel_group_mapping():
    """F6: the (n, oh, ow) pixel axis maps onto tcgen05's M without padding."""
    op = conv2d_nhwc_tdsl(32, 58, 58, 64, 64, 3, 3, 1)
    assert ops.inspect(op, "tcgen05_i8_m128n64k32")[0] == "{ow->m, k->n, c->k} pad"
    assert ops.inspect(op, "tcgen05_i8_m128n64k32", grouped=True)[0] == "{(n,oh,ow)->m, k->n, c->k}"
    blk = conv2d_tdsl(64, 56, 64, 3, 1, 16, 4)
    assert ops.inspect(blk, "tcgen05_i8_m128n64k32", grouped=True)[0].startswith("{(oh,ow)->m, (ko,ki)->n, ci->k}")


def test_describe_plans():
    d = ops.describe(matmul_tdsl(4096, 4096, 4096), "tcgen05_i8_m128n256k32")
    assert "plan matmul u8i8" in d and "m=4096" in d and "pragma x.i y.i k.i" in d
    d = ops.describe(conv2d_tdsl(64, 56, 64, 3, 1, 16, 4), "tcgen05_i8_m128n64k32")
    assert "plan conv_blocked" in d and "out(nb=16,sm=16,sb=46656)" in d
    for L in RESNET50_V15:
        d = ops.describe(conv2d_nhwc_tdsl(32, L.h, L.h, L.c, L.k, L.r, L.r, L.stride), "tcgen05_i8_m128n256k32")
        assert "plan conv_nhwc u8i8" in d and f"c={L.c} k={L.k} r={L.r}" in d


@pytest.mark.parametrize("text,kind", [
    ("tensor A : u8 [4] input\ntensor C : i32 [4] output\nloop x : dp 4\nC[x] = A[x]\n", "TypeError"),
    ("tensor A : u8 [4] input\ntensor C : i32 [4] output\nloop x : dp 4\nC[x] = cast<i32>(A[x * x])\n",
     "ValidationError"),
    ("tensor A : u8 [4] input\ntensor C : i32 [4] output\nloop x : dp 4\nC[x] = cast<i32>(A[x]\n", "SyntaxError"),
    ("tensor A : u9 [4] input\n", "SyntaxError"),
])
def test_error_kinds(text, kind):
    with pytest.raises(TzcError) as e:
        ops.parse(text)
    assert e.value.kind == kind


def test_unknown_intrinsic_and_no_kernel():
    with pytest.raises(TzcError) as e:
        ops.inspect(matmul_tdsl(16, 16, 16), "no_such_instruction")
    assert e.value.kind == "UnknownIntrinsic"
    with pytest.raises(TzcError) as e:  # fp16 op vs the int8 instruction: no structural match
        ops.describe(matmul_tdsl(16, 16, 16, fp16=True), "tcgen05_i8_m128n64k32")
    assert e.value.kind == "InjectError"
    with pytest.raises(TzcError) as e:  # the VNNI description has no sm_100a kernel
        ops.describe(matmul_tdsl(16, 16, 64), "vdot_16x4")
    assert e.value.kind == "NoFeasibleMapping"


@needs_ref
@pytest.mark.parametrize("shape", TABLE1_BANK, ids=[b[0] for b in TABLE1_BANK])
def test_table1_bank_texts_and_plans(shape):
    """The paper's Table-1 bank: our generator's op text is the reference's
    (proj/src/workloads.cpp:123-142 through conv2d_tdsl), and each op has a
    tcgen05 device plan (the blocked-conv family with the K5 adapters)."""
    _, c, hw, k, r, st = shape
    text = conv2d_tdsl(c, hw, k, r, st)
    assert text == Ref.conv2d_tdsl(c, hw, k, r, st)
    assert "plan conv_blocked u8i8" in ops.describe(text, "tcgen05_i8_m128n64k32")


@needs_ref
@pytest.mark.parametrize("args", [(16, 8, 32, 3, 1, False), (16, 9, 32, 3, 2, False), (16, 7, 16, 3, 1, True),
                                  (64, 16, 64, 3, 1, False), (64, 17, 128, 3, 2, False)])
def test_conv3d_texts_and_plans(args):
    """conv3d_tdsl (proj/src/workloads.cpp:94-121): same text as the reference's
    generator, and a device plan (depth-tap decomposition, conv3d_blocked)."""
    c, hw, k, r, st, f16 = args
    text = conv3d_tdsl(c, hw, k, r, st, fp16=f16)
    assert text == Ref.conv3d_tdsl(c, hw, k, r, st, fp16=f16)
    intr = "tcgen05_f16_m128n64k16" if f16 else "tcgen05_i8_m128n64k32"
    assert "plan conv3d_blocked" in ops.describe(text, intr)
    assert ops.lower(text, None, intr).count(intr + "(dst = ") == 1
