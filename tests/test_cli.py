"""The device CLI (paper_2101_08458_b200/tzc-b200) and the TNSR tensor
container on CPU: files written by the reference's save_tensor read back to the
reference's own tensor_to_text and re-save byte-identically; inspect /
tensorize / error exit codes follow the reference CLI (proj/src/cli.cpp:41-47)."""
import glob
import os
import shutil
import subprocess
import tempfile

import pytest

from oracle.pyoracle import Ref
from paper_2101_08458_b200 import ops

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "paper_2101_08458_b200", "tzc-b200")
TNSR = sorted(glob.glob(os.path.join(ROOT, "tests", "golden", "tnsr", "*", "*.tnsr")))
needs_ref = pytest.mark.skipif(not Ref.available(), reason="oracle/_ref not built")
needs_cli = pytest.mark.skipif(not os.path.exists(CLI), reason="tzc-b200 not built")


def cli(*args):
    p = subprocess.run([CLI, *args], capture_output=True, text=True, timeout=120)
    return p.returncode, p.stdout, p.stderr


def test_fixtures_present():
    assert len(TNSR) >= 16


@pytest.mark.parametrize("path", TNSR, ids=lambda p: "/".join(p.split("/")[-2:]))
def test_container_roundtrip_is_byte_identical(path):
    out = os.path.join(tempfile.mkdtemp(), "copy.tnsr")
    ops.tensor_roundtrip(path, out)
    assert open(out, "rb").read() == open(path, "rb").read()


@needs_ref
@pytest.mark.parametrize("path", TNSR, ids=lambda p: "/".join(p.split("/")[-2:]))
def test_container_reads_like_the_reference(path):
    assert ops.tensor_text(path, 1 << 30) == Ref.tensor_text(path)
    assert ops.tensor_text(path) == Ref.tensor_text(path, 64)


def test_container_errors(tmp_path):
    bad = tmp_path / "bad.tnsr"
    bad.write_bytes(b"NOPE\x01\x05\x01" + b"\x00" * 8)
    with pytest.raises(Exception, match="IoError"):
        ops.tensor_text(str(bad))
    src = open(TNSR[0], "rb").read()
    (tmp_path / "short.tnsr").write_bytes(src[:-1])
    with pytest.raises(Exception, match="IoError"):
        ops.tensor_text(str(tmp_path / "short.tnsr"), 1 << 30)


@needs_cli
def test_cli_inspect_and_tensorize():
    d = os.path.join(ROOT, "tests", "golden", "tnsr", "conv_nhwc_i8")
    op = os.path.join(d, "op.tdsl")
    rc, out, _ = cli("inspect", op, "--intrinsic", "tcgen05_i8_m128n64k32")
    assert rc == 0 and out.splitlines()[0] == "mapping 0: {(n,oh,ow)->m, k->n, c->k}"
    sched = os.path.join(tempfile.mkdtemp(), "s.txt")
    rc, out, _ = cli("tensorize", op, "--intrinsic", "tcgen05_i8_m128n64k32", "--schedule-out", sched)
    assert rc == 0
    assert out == ops.lower(open(op).read(), None, "tcgen05_i8_m128n64k32")
    assert ops.lower(open(op).read(), open(sched).read(), "tcgen05_i8_m128n64k32").count("tcgen05_i8_m128n64k32(") == 1
    rc, out, _ = cli("builtins")
    assert rc == 0 and "tcgen05_i8_m128n256k32" in out.split()


@needs_cli
def test_cli_exit_codes(tmp_path):
    d = os.path.join(ROOT, "tests", "golden", "tnsr", "mm_f16")
    op = os.path.join(d, "op.tdsl")
    assert cli("frobnicate")[0] == 2
    assert cli("run", op)[0] == 2  # --intrinsic missing
    (tmp_path / "bad.tdsl").write_text("tensor A : u8 [4] input\nnonsense\n")
    assert cli("inspect", str(tmp_path / "bad.tdsl"), "--intrinsic", "vdot_16x4")[0] == 2
    # float outputs need an explicit --rtol, as in the reference's verify
    rc, _, err = cli("verify", op, "--intrinsic", "tcgen05_f16_m128n128k16_mn", "--expect", os.path.join(d, "expect.tnsr"))
    assert rc == 2 and "rtol" in err
    # a CPU instruction never executes (no CPU interpreter): domain failure
    mm = os.path.join(ROOT, "tests", "golden", "tnsr", "mm_i8", "op.tdsl")
    shutil.copy(mm, tmp_path / "mm.tdsl")
    rc, _, err = cli("run", str(tmp_path / "mm.tdsl"), "--intrinsic", "vdot_16x4")
    assert rc == 1 and ("InjectError" in err or "NoFeasibleMapping" in err) and "sm_100a kernel" in err


@needs_cli
def test_cli_tune_without_device_is_a_domain_failure():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a device is present (tests/test_gpu_cli.py covers tune)")
    op = os.path.join(ROOT, "tests", "golden", "tnsr", "mm_i8", "op.tdsl")
    rc, out, err = cli("tune", op, "--intrinsic", "tcgen05_i8_m128n128k32")
    assert rc == 1 and out.startswith("plan matmul u8i8") and "DeviceError" in err


def test_reference_style_cpp_caller(tmp_path):
    """C++ drop-in: a caller written against the reference's header paths and names
    builds against libtzc_b200.so and prints acceptance criterion 2's golden IR."""
    from tests.test_tensor_ir import C2_OP, C2_SCHED
    exe = str(tmp_path / "chain")
    lib_dir = os.path.join(ROOT, "paper_2101_08458_b200")
    subprocess.run(["g++", "-std=c++17", "-O1", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "chain.cpp"), "-o", exe, "-L", lib_dir, "-ltzc_b200",
                    f"-Wl,-rpath,{lib_dir}"], check=True, timeout=300)
    p = subprocess.run([exe, "vdot_16x4", C2_SCHED], input=C2_OP, capture_output=True, text=True, timeout=60)
    assert p.returncode == 0, p.stderr
    assert p.stdout == open(os.path.join(ROOT, "tests", "golden", "conv_ir_c2_vdot_16x4.txt")).read()
