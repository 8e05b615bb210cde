"""The reference's lowering chain in the tzc host library — schedule text,
lower(), inject_intrinsic(), print_tensor_ir() and eval_tir()'s dispatch —
against the reference on the same ops and schedules (CPU only):

* the golden conv IR snapshot of the reference's acceptance test
  (proj/tests/acceptance.cpp:181-203, fixture tests/golden/conv_ir_c2_vdot_16x4.txt);
* seeded random schedules (split / fuse / reorder / parallel / unroll /
  split_reduction / pragma) lowered by both libraries: identical text, or both
  reject the schedule;
* injection of the reference's CPU instructions and of the tcgen05 descriptions;
* the backend's fused pixel group (F6), which the reference cannot inject, and
  the error kinds (pad in-kernel, no CPU interpreter behind eval_tir)."""
import os
import random
import tempfile

import numpy as np
import pytest

from oracle.pyoracle import Ref
from paper_2101_08458_b200 import ops
from paper_2101_08458_b200._capi import TzcError
from paper_2101_08458_b200.workloads import conv2d_nhwc_tdsl, conv2d_tdsl, matmul_tdsl

needs_ref = pytest.mark.skipif(not Ref.available(), reason="oracle/_ref not built")
GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")

C2_OP = conv2d_tdsl(4, 6, 16, 3)  # acceptance criterion 2: conv2d_tdsl({"c2", 4, 6, 16, 3, 1}, 16, 4)
C2_SCHED = "split ki 16\nsplit ci 4\nreorder ko oh ow ki.o co r s ci.o ki.i ci.i\npragma ki.i ci.i\n"


def test_golden_conv_ir_snapshot():
    want = open(os.path.join(GOLD, "conv_ir_c2_vdot_16x4.txt")).read()
    assert ops.lower(C2_OP, C2_SCHED, "vdot_16x4") == want


@needs_ref
def test_golden_schedule_is_the_references():
    assert Ref.lower(C2_OP, C2_SCHED, "vdot_16x4") == Ref.tensorize(C2_OP, "vdot_16x4")


def random_schedule(text, rng):
    """A random valid-or-invalid transform sequence over the op's loops."""
    axes = [[n, e, k == "red"] for n, k, e in Ref.op_info(text).loops]
    lines = []
    sred = False
    for _ in range(rng.randint(0, 5)):
        kind = rng.choice(["split", "split", "fuse", "reorder", "parallel", "unroll", "split_reduction"])
        j = rng.randrange(len(axes))
        name, ext, red = axes[j]
        if kind == "split":
            divs = [d for d in range(1, ext + 1) if ext % d == 0]
            f = rng.choice(divs)
            lines.append(f"split {name} {f}")
            axes[j:j + 1] = [[name + ".o", ext // f, red], [name + ".i", f, red]]
        elif kind == "fuse" and j + 1 < len(axes) and axes[j + 1][2] == red:
            b = axes[j + 1]
            lines.append(f"fuse {name} {b[0]}")
            axes[j:j + 2] = [[f"{name}.{b[0]}.fused", ext * b[1], red]]
        elif kind == "reorder":
            perm = axes[:]
            rng.shuffle(perm)
            lines.append("reorder " + " ".join(a[0] for a in perm))
            axes = perm
        elif kind in ("parallel", "unroll"):
            lines.append(f"{kind} {name}")
        elif kind == "split_reduction" and red and not sred and ext % 2 == 0:
            lines.append(f"split_reduction {name} 2")
            axes[j:j + 1] = [[name + ".s", 2, False], [name + ".r", ext // 2, True]]
            sred = True
    if rng.random() < 0.5:
        lines.append("pragma " + axes[-1][0])
    return "\n".join(lines) + "\n"


SCHED_OPS = [
    matmul_tdsl(8, 4, 6),
    matmul_tdsl(4, 4, 4, fp16=True),
    conv2d_tdsl(8, 5, 16, 3),
    conv2d_tdsl(4, 7, 16, 3, 2),
    conv2d_nhwc_tdsl(1, 4, 4, 2, 2, 3, 3, 1),
    "tensor A : u8 [4, 6] input\ntensor O : i32 [4] output\nloop x : dp 4\nloop k : red 6\n"
    "O[x] = 7 + cast<i32>(A[x, k])\n",
    "tensor A : i32 [3, 5] input\ntensor O : i32 [3, 5] output\nloop x : dp 3\nloop y : dp 5\nO[x, y] = A[x, y] * 2\n",
]


def _both(fn_ours, fn_ref):
    try:
        ours = fn_ours()
    except TzcError as e:
        ours = ("error", e)
    try:
        ref = fn_ref()
    except RuntimeError as e:
        ref = ("error", e)
    return ours, ref


@needs_ref
@pytest.mark.parametrize("op_i", range(len(SCHED_OPS)))
def test_random_schedules_lower_like_the_reference(op_i):
    text = SCHED_OPS[op_i]
    rng = random.Random(1000 + op_i)
    agreed = 0
    for trial in range(40):
        sched = random_schedule(text, rng)
        if trial == 0:
            sched = ""  # the unscheduled nest
        ours, ref = _both(lambda: ops.lower(text, sched), lambda: Ref.lower(text, sched))
        if isinstance(ref, tuple):
            assert isinstance(ours, tuple), f"reference rejects, we accept:\n{sched}\n{ref[1]}"
            kind = str(ref[1]).split(":")[0]
            assert str(ours[1]).split(":")[0] == kind or kind not in ("ScheduleError", "SyntaxError"), (sched, ref, ours)
        else:
            assert ours == ref, sched
            agreed += 1
    assert agreed >= 10


# (op, schedule, instruction): the reference's CPU instructions and tcgen05 on linear (unfused) mappings
INJECT_CASES = [
    (matmul_tdsl(32, 32, 8), "split y 16\nsplit k 4\nreorder x y.o k.o y.i k.i\npragma y.i k.i\n", "vdot_16x4"),
    (matmul_tdsl(16, 8, 8), "split y 4\nsplit k 4\nreorder x y.o k.o y.i k.i\npragma y.i k.i\n", "vdot_4x4"),
    (matmul_tdsl(32, 32, 32, fp16=True),
     "split x 16\nsplit y 16\nsplit k 16\nreorder x.o y.o k.o x.i y.i k.i\npragma x.i y.i k.i\n", "wmma_16x16x16"),
    (C2_OP, C2_SCHED, "vdot_16x4"),
    (matmul_tdsl(256, 128, 64),
     "split x 128\nsplit y 64\nsplit k 32\nreorder x.o y.o k.o x.i y.i k.i\npragma x.i y.i k.i\n",
     "tcgen05_i8_m128n64k32"),
    (matmul_tdsl(128, 256, 32),
     "split x 128\nsplit y 256\nsplit k 32\nreorder x.o y.o k.o x.i y.i k.i\npragma x.i y.i k.i\n",
     "tcgen05_i8_m128n256k32"),
]


@needs_ref
@pytest.mark.parametrize("case", range(len(INJECT_CASES)))
def test_inject_matches_reference(case):
    text, sched, intr = INJECT_CASES[case]
    if intr.startswith("tcgen05"):
        # the reference resolves builtins by name; hand it the same .intr text
        path = os.path.join(tempfile.mkdtemp(), f"{intr}.intr")  # the reference names it by the file stem
        with open(path, "w") as f:
            f.write(ops.print_intrinsic(intr))
        ref_intr = path
    else:
        ref_intr = intr
    ref = Ref.lower(text, sched, ref_intr)
    ours = ops.lower(text, sched, intr)
    assert ours == ref
    assert ours.count(intr + "(dst = ") == 1


def test_tile_and_reorder_schedule_lowers_to_one_tcgen05_call():
    """Our own tile_and_reorder schedule for the tcgen05 matmul: one call, no pragma loops left."""
    ir = ops.lower(matmul_tdsl(256, 256, 64), None, "tcgen05_i8_m128n256k32")
    assert ir.count("tcgen05_i8_m128n256k32(dst = ") == 1
    assert "tensorize" not in ir
    assert "for x.o : 2 {" in ir and "for k.o : 2 {" in ir


def test_fused_pixel_group_injects_as_gather():
    """F6: (n, oh, ow) fused onto tcgen05's M — the reference cannot inject this
    (non-affine in the pragma loops); here the operands stay gather addresses."""
    text = conv2d_nhwc_tdsl(2, 10, 10, 64, 64, 3, 3, 1)
    ir = ops.lower(text, None, "tcgen05_i8_m128n64k32")
    assert ir.count("tcgen05_i8_m128n64k32(dst = ") == 1
    assert ".fused" in ir and " / " in ir and " % " in ir
    sched = ops.describe(text, "tcgen05_i8_m128n64k32")
    assert "fuse oh ow" in sched and "fuse n oh.ow.fused" in sched
    # a pixel count that is not a multiple of 128: the tail tile is clipped on
    # the device, so the outer loop takes ceil(100 / 128) = 1 iteration
    ir = ops.lower(conv2d_tdsl(64, 12, 64, 3), None, "tcgen05_i8_m128n64k32")
    assert "for oh.ow.fused.o : 1 {" in ir and ir.count("tcgen05_i8_m128n64k32(dst = ") == 1
    with pytest.raises(TzcError, match="ScheduleError"):  # a user schedule stays strict
        ops.lower(conv2d_tdsl(64, 12, 64, 3), "fuse oh ow\nsplit oh.ow.fused 128\n")


def test_lowering_errors():
    text = matmul_tdsl(16, 16, 16)
    with pytest.raises(TzcError, match="ScheduleError"):
        ops.lower(text, "split x 5\n")
    with pytest.raises(TzcError, match="ScheduleError"):
        ops.lower(text, "split x 4\nfuse x.o y\n")
    with pytest.raises(TzcError, match="SyntaxError"):
        ops.lower(text, "tile x 4\n")
    with pytest.raises(TzcError, match="InjectError"):
        ops.lower(text, "split y 16\n", "vdot_16x4")  # no pragma nest


def test_eval_tir_has_no_cpu_interpreter():
    """eval_tir refuses CPU instructions before touching the device."""
    text = matmul_tdsl(32, 32, 8)
    sched, intr = INJECT_CASES[0][1], INJECT_CASES[0][2]
    ins = {"A": np.zeros((32, 8), np.uint8), "B": np.zeros((32, 8), np.int8), "C": np.zeros((32, 32), np.int32)}
    with pytest.raises(TzcError, match="InjectError"):
        ops.eval_tir(text, intr, ins, schedule=sched)


def random_tcgen05_schedule(rng, n=128):
    """Split onto tcgen05's (m, n, k) = (128, n, 32) pragma nest; the outer axes
    are shuffled and annotated at random (split_reduction on k.o included)."""
    outer = ["x.o", "y.o", "k.o"]
    lines = ["split x 128", f"split y {n}", "split k 32"]
    if rng.random() < 0.4:
        lines.append("split_reduction k.o 2")
        outer = ["x.o", "y.o", "k.o.s", "k.o.r"]
    rng.shuffle(outer)
    lines.append("reorder " + " ".join(outer + ["x.i", "y.i", "k.i"]))
    for a in outer:
        r = rng.random()
        if r < 0.25 and not a.startswith("k.o.r") and a != "k.o":
            lines.append(f"parallel {a}")
        elif r < 0.45:
            lines.append(f"unroll {a}")
    lines.append("pragma x.i y.i k.i")
    return "\n".join(lines) + "\n"


@needs_ref
def test_random_tcgen05_schedules_inject_like_the_reference():
    text = matmul_tdsl(256, 256, 128)
    intr = "tcgen05_i8_m128n128k32"
    path = os.path.join(tempfile.mkdtemp(), f"{intr}.intr")
    with open(path, "w") as f:
        f.write(ops.print_intrinsic(intr))
    rng = random.Random(7)
    for _ in range(12):
        sched = random_tcgen05_schedule(rng)
        ours, ref = _both(lambda: ops.lower(text, sched, intr), lambda: Ref.lower(text, sched, path))
        assert not isinstance(ref, tuple), (sched, ref)
        assert ours == ref, sched
