"""The device CLI end to end on the B200: `tzc-b200 verify` runs the op
(lower -> inject_intrinsic -> eval_tir) on inputs the REFERENCE saved and
compares with the output the reference computed (tests/golden/make_tnsr.py):
int8 bit-exact, fp16 within 1e-3; a corrupted expectation FAILs with exit 1."""
import os
import subprocess

import numpy as np
import pytest

from paper_2101_08458_b200 import ops
from tests.golden.make_tnsr import CASES

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "paper_2101_08458_b200", "tzc-b200")


def case_args(name):
    d = os.path.join(ROOT, "tests", "golden", "tnsr", name)
    _, _, intr, rtol = CASES[name]
    ins = [a for f in sorted(os.listdir(d)) if f.endswith(".tnsr") and f != "expect.tnsr"
           for a in ("--input", f"{f[:-5]}={os.path.join(d, f)}")]
    extra = ["--rtol", str(rtol)] if rtol else []
    return d, [os.path.join(d, "op.tdsl"), "--intrinsic", intr, *ins, *extra]


def cli(*args):
    p = subprocess.run([CLI, *args], capture_output=True, text=True, timeout=300)
    return p.returncode, p.stdout, p.stderr


@pytest.mark.parametrize("name", sorted(CASES))
def test_cli_verify_against_reference_tensors(cuda, name):
    d, args = case_args(name)
    rc, out, err = cli("verify", *args, "--expect", os.path.join(d, "expect.tnsr"))
    assert rc == 0, out + err
    assert out.strip().endswith("PASS")
    if CASES[name][3] is None:
        assert "bitexact: yes" in out


@pytest.mark.parametrize("name", ["mm_i8", "conv_blocked_i8"])
def test_cli_run_output_and_failing_verify(cuda, name, tmp_path):
    d, args = case_args(name)
    out_path = str(tmp_path / "got.tnsr")
    rc, out, err = cli("run", *args, "--output", out_path)
    assert rc == 0, err
    assert open(out_path, "rb").read() == open(os.path.join(d, "expect.tnsr"), "rb").read()
    raw = bytearray(open(os.path.join(d, "expect.tnsr"), "rb").read())
    raw[-1] ^= 0x40  # flip one output element
    bad = tmp_path / "bad.tnsr"
    bad.write_bytes(bytes(raw))
    rc, out, _ = cli("verify", *args, "--expect", str(bad), "--format", "structured")
    assert rc == 1 and '"pass": false' in out and '"mismatches": 1' in out


@pytest.mark.parametrize("name", ["mm_i8", "conv_nhwc_i8"])
def test_cli_tune(cuda, name):
    """`tzc-b200 tune`: 20 candidate plans timed on the device, the winner reported."""
    d, args = case_args(name)
    rc, out, err = cli("tune", *args[:3], "--reps", "3")
    assert rc == 0, err
    lines = out.strip().splitlines()
    assert lines[0].startswith("plan ")
    assert sum(ln.startswith("candidate ") for ln in lines) == 20
    assert lines[-1].startswith("best ")
