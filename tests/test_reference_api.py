"""The reference's C++ API as a drop-in boundary.

* The reference's own acceptance program (proj/tests/acceptance.cpp) is
  compiled UNCHANGED against include/ + libtzc_b200.so and run.  The
  criteria that need only the host API pass: C2 (golden conv x vdot_16x4
  rewrite snapshot), C3 (exhaustive mapping oracle), C4 (work conservation
  ledger incl. the padded kernel), C8 (negative paths).  The criteria that
  execute vdot / wmma nests on the reference's CPU interpreter (C1, C5, C7)
  fail with InjectError — this backend has no CPU VM by design — and C6
  (the CPU threading / unroll sketch tuner) fails as out of scope.
* pad_to_multiple (via lower's leading pad transforms) prints the same
  padded nests as the reference and refuses the same reduction pads.
* The C++ workload generators emit the reference's texts byte for byte.
"""
import os
import subprocess

import pytest

from oracle.pyoracle import Ref
from paper_2101_08458_b200 import ops
from paper_2101_08458_b200._capi import TzcError
from paper_2101_08458_b200.workloads import matmul_tdsl

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_2101_08458_b200")
ACC = "/root/reference/proj/tests/acceptance.cpp"
needs_ref = pytest.mark.skipif(not Ref.available(), reason="oracle/_ref not built")


def _build(src, out):
    subprocess.run(["g++", "-std=c++20", "-O1", "-I", os.path.join(ROOT, "include"), src, "-o", out, "-L", LIBDIR,
                    "-ltzc_b200", f"-Wl,-rpath,{LIBDIR}"], check=True, capture_output=True, text=True)


@pytest.mark.skipif(not os.path.exists(ACC), reason="the reference's acceptance.cpp is not present")
def test_reference_acceptance_compiles_and_host_criteria_pass(tmp_path):
    exe = str(tmp_path / "acceptance")
    _build(ACC, exe)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    lines = {int(ln.split()[1].rstrip(":")): ln for ln in r.stdout.splitlines() if ln.startswith("criterion")}
    assert sorted(lines) == list(range(1, 9)), r.stdout
    for c in (2, 3, 4, 8):
        assert "PASS" in lines[c], lines[c]
    for c in (1, 5, 7):  # need the reference's CPU interpreter
        assert "FAIL" in lines[c] and "InjectError" in lines[c] and "no CPU interpreter" in lines[c], lines[c]
    assert "FAIL" in lines[6] and "out of scope" in lines[6], lines[6]


@needs_ref
def test_cpp_workload_generators_are_the_references(tmp_path):
    exe = str(tmp_path / "workloads")
    _build(os.path.join(ROOT, "tests", "cpp", "workloads.cpp"), exe)
    out = subprocess.run([exe], capture_output=True, text=True, check=True).stdout
    parts = {}
    key = None
    for ln in out.splitlines(keepends=True):
        if ln.startswith("@"):
            key = ln[1:].strip()
            parts[key] = ""
        else:
            parts[key] += ln
    assert parts["matmul_i8"] == Ref.matmul_tdsl(48, 32, 96)
    assert parts["matmul_f16"] == Ref.matmul_tdsl(16, 32, 48, fp16=True)
    assert parts["conv2d_f16"] == Ref.conv2d_tdsl(32, 10, 16, 3, 2, 16, 16, fp16=True)
    from paper_2101_08458_b200.workloads import RESNET18_3D_BANK, TABLE1_BANK
    for name, c, hw, k, r, st in TABLE1_BANK:
        assert parts[f"table1 {name}"] == Ref.conv2d_tdsl(c, hw, k, r, st, 16, 4), name
    for name, c, hw, k, r, st in RESNET18_3D_BANK:
        assert parts[f"resnet18_3d {name}"] == Ref.conv3d_tdsl(c, hw, k, r, st, 16, 4), name
    assert [k for k in parts if k.startswith("embed")] == ["embed ok 4 0"]  # big[1][0] = v[1][0] = 4, big[0][4] is the zero extension


PAD_CASES = [
    (matmul_tdsl(8, 8, 6), "pad k 4\npad x 16\nsplit x 16\n"),
    (matmul_tdsl(10, 12, 20), "pad y 16\npad k 32\nsplit k 8\n"),
    (matmul_tdsl(16, 16, 16), "pad x 16\n"),  # already a multiple: identity
]


@needs_ref
@pytest.mark.parametrize("text,sched", PAD_CASES)
def test_pad_to_multiple_lowers_like_the_reference(text, sched):
    assert ops.lower(text, sched) == Ref.lower(text, sched)


@needs_ref
def test_pad_legality_matches_the_reference():
    # the reduction term has an additive tail: extra iterations would not add zeros
    text = ("tensor A : i32 [6] input\ntensor C : i32 [1] output\nloop i : dp 1\nloop k : red 6\n"
            "C[i] += A[k] + 1\n")
    with pytest.raises(RuntimeError, match="PadUnsupported"):
        Ref.lower(text, "pad k 4\n")
    with pytest.raises(TzcError) as e:
        ops.lower(text, "pad k 4\n")
    assert e.value.kind == "PadUnsupported"
    # a data-parallel pad is always legal (grows the output)
    assert ops.lower(text, "pad i 4\n") == Ref.lower(text, "pad i 4\n")
