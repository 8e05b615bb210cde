"""The reference-facing entry (tzc_b200_run_op): op text + instruction +
HOST buffers, parsed/inspected/planned by the C++ host library and run on the
B200 — against the reference's own outputs (golden fixtures) and the oracle."""
import hashlib
import os

import numpy as np
import pytest

from oracle.pyoracle import Orc
from paper_2101_08458_b200 import ops
from paper_2101_08458_b200.workloads import conv2d_nhwc_tdsl, matmul_tdsl, requant_tdsl
from tests.gpu_helpers import rel_dev
from tests.test_oracle import SEEDED, SEEDED_NAMES, decls

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def instr_for(text, n=64):
    if "fp16" in text:
        mn = "_mn" if "B[k, y]" in text else ""
        return f"tcgen05_f16_m128n{n}k16{mn}"
    return f"tcgen05_i8_m128n{n}k32"


@pytest.mark.parametrize("name", [n for n in SEEDED_NAMES if n.startswith(("mm_", "conv_"))])
def test_run_op_reference_fixtures(cuda, name):
    text = str(SEEDED[name + "__text"])
    ins = Orc.random_inputs(decls(text), int(SEEDED[name + "__seed"]), update=True)
    got = ops.run_op(text, instr_for(text), ins)
    want = SEEDED[name + "__out"]
    if "f16" in name:
        assert rel_dev(want, got) <= 1e-3
    else:
        assert np.array_equal(got, want)


def test_run_op_c1_with_fused_requant(cuda):
    """configs[0] through the op-level API: the reference's exact op text,
    blocked layouts, accumulate-form seed, fused requant epilogue op."""
    g = np.load(os.path.join(GOLD, "c1.npz"))
    text = str(g["text"])
    ins = Orc.random_inputs(decls(text), int(g["seed"]))
    out = ops.run_op(text, "tcgen05_i8_m128n64k32", ins)
    assert hashlib.sha256(out.tobytes()).hexdigest() == str(g["sha_i32"])
    q = ops.run_op(text, "tcgen05_i8_m128n64k32", ins, epilogue=requant_tdsl(out.shape, 2.0 ** -12, src="out"))
    assert q.dtype == np.int8
    assert hashlib.sha256(q.tobytes()).hexdigest() == str(g["sha_i8"])


def test_run_op_matmul_requant_and_no_seed(cuda):
    text = matmul_tdsl(512, 256, 384)
    ins = Orc.random_inputs(decls(text), 77)
    ref = Orc.matmul(ins["A"], ins["B"], ins["C"])
    q = ops.run_op(text, "tcgen05_i8_m128n256k32", ins, epilogue=requant_tdsl((512, 256), 0.0123))
    assert np.array_equal(q, Orc.requant_i8(ref, np.float32(0.0123)))
    no_seed = {k: v for k, v in ins.items() if k != "C"}
    assert np.array_equal(ops.run_op(text, "tcgen05_i8_m128n256k32", no_seed), Orc.matmul(ins["A"], ins["B"]))


@pytest.mark.parametrize("n,h,c,k,r,st", [(2, 12, 64, 128, 3, 1), (2, 21, 3, 64, 7, 2), (1, 14, 256, 512, 1, 2),
                                           (11, 10, 64, 64, 3, 1), (9, 29, 3, 64, 7, 2)])
def test_run_op_conv_nhwc(cuda, n, h, c, k, r, st):
    """Batched ops run as image chunks over three streams (H2D / kernel / D2H
    overlapped): uneven chunk counts, seeds and the fused requant stay exact."""
    text = conv2d_nhwc_tdsl(n, h, h, c, k, r, r, st)
    ins = Orc.random_inputs(decls(text), 5)
    ref = Orc.conv2d_nhwc(ins["data"], ins["kernel"], st, ins["out"])
    assert np.array_equal(ops.run_op(text, "tcgen05_i8_m128n64k32", ins), ref)
    q = ops.run_op(text, "tcgen05_i8_m128n64k32", ins, epilogue=requant_tdsl(ref.shape, 2.0 ** -11, src="out"))
    assert np.array_equal(q, Orc.requant_i8(ref, 2.0 ** -11))


def test_run_op_matmul_chunked_uneven(cuda):
    text = matmul_tdsl(1000, 128, 96)
    ins = Orc.random_inputs(decls(text), 78)
    ref = Orc.matmul(ins["A"], ins["B"], ins["C"])
    assert np.array_equal(ops.run_op(text, "tcgen05_i8_m128n128k32", ins), ref)


def test_run_op_errors(cuda):
    from paper_2101_08458_b200._capi import TzcError
    text = matmul_tdsl(128, 64, 64)
    ins = Orc.random_inputs(decls(text), 1)
    with pytest.raises(TzcError) as e:
        ops.run_op(text, "tcgen05_i8_m128n64k32", {"A": ins["A"]})
    assert e.value.kind == "MissingInput"
    with pytest.raises(TzcError) as e:
        ops.run_op(text, "tcgen05_i8_m128n64k32", ins, epilogue="tensor Z : i32 [2] input\ntensor Q : i8 [2] output\n"
                   "loop i : dp 2\nQ[i] = cast<i8>(Z[i])\n")
    assert e.value.kind == "InjectError"


def test_run_op_concurrent_threads(cuda):
    """Independent ops from several host threads (per-thread device buffers
    and streams in the library) stay exact."""
    from concurrent.futures import ThreadPoolExecutor
    cases = []
    for i, (n, h, c, k, r, st) in enumerate([(3, 12, 64, 64, 3, 1), (2, 21, 3, 64, 7, 2), (4, 9, 128, 256, 1, 1),
                                              (5, 10, 64, 128, 3, 2)]):
        text = conv2d_nhwc_tdsl(n, h, h, c, k, r, r, st)
        ins = Orc.random_inputs(decls(text), 40 + i)
        cases.append((text, ins, Orc.conv2d_nhwc(ins["data"], ins["kernel"], st, ins["out"])))

    def run(case):
        text, ins, _ = case
        return [ops.run_op(text, "tcgen05_i8_m128n64k32", ins) for _ in range(3)]

    with ThreadPoolExecutor(4) as ex:
        results = list(ex.map(run, cases))
    for (text, ins, ref), outs in zip(cases, results):
        for got in outs:
            assert np.array_equal(got, ref)


# ---- the reference chain lower -> inject_intrinsic -> eval_tir on the device ----
MM_SCHED = "split x 128\nsplit y {n}\nsplit k 32\nreorder x.o y.o k.o x.i y.i k.i\npragma x.i y.i k.i\n"


@pytest.mark.parametrize("n", [64, 256])
def test_eval_tir_matmul_reference_schedule(cuda, n):
    """An explicit reference-grammar schedule, injected with tcgen05 and executed
    by eval_tir: bit-exact vs the oracle, with and without the fused requant."""
    text = matmul_tdsl(256, 512, 192)
    ins = Orc.random_inputs(decls(text), 31)
    ref = Orc.matmul(ins["A"], ins["B"], ins["C"])
    intr = f"tcgen05_i8_m128n{n}k32"
    assert np.array_equal(ops.eval_tir(text, intr, ins, schedule=MM_SCHED.format(n=n)), ref)
    q = ops.eval_tir(text, intr, ins, schedule=MM_SCHED.format(n=n), epilogue=requant_tdsl((256, 512), 2.0 ** -13))
    assert np.array_equal(q, Orc.requant_i8(ref, 2.0 ** -13))


def test_eval_tir_conv_fused_pixel_group(cuda):
    """The tile_and_reorder schedule (fused n.oh.ow onto M), lowered, injected, run."""
    text = conv2d_nhwc_tdsl(2, 12, 12, 64, 128, 3, 3, 1)
    ins = Orc.random_inputs(decls(text), 8)
    ref = Orc.conv2d_nhwc(ins["data"], ins["kernel"], 1, ins["out"])
    assert np.array_equal(ops.eval_tir(text, "tcgen05_i8_m128n64k32", ins), ref)


def test_eval_tir_blocked_c1_matches_reference_sha(cuda):
    """configs[0] exactly as the reference lowers it, through eval_tir: the
    sha256 of the reference's own output (tests/golden/c1.npz)."""
    g = np.load(os.path.join(GOLD, "c1.npz"))
    text = str(g["text"])
    ins = Orc.random_inputs(decls(text), int(g["seed"]))
    out = ops.eval_tir(text, "tcgen05_i8_m128n64k32", ins)
    assert hashlib.sha256(out.tobytes()).hexdigest() == str(g["sha_i32"])


# ---- measured-time tuner (tzc_b200_tune_conv / _gemm) ----
def test_tuner_installs_a_plan_and_results_stay_exact(cuda):
    import torch

    from paper_2101_08458_b200 import device as D
    dev = torch.device("cuda:0")
    x = torch.from_numpy(Orc.random_tensor("u8", (4, 16, 16, 64), 3)).to(dev)
    w = torch.from_numpy(Orc.random_tensor("i8", (128, 3, 3, 64), 4)).to(dev)
    ref = Orc.conv2d_nhwc(x.cpu().numpy(), w.cpu().numpy(), 1)
    try:
        best, log = D.tune_conv2d(x, w, 1, epilogue="requant_i8", scale=2.0 ** -12, reps=3)
        lines = log.strip().splitlines()
        assert sum(ln.startswith("candidate ") for ln in lines) == 20 and lines[-1].startswith(f"best {best} ")
        assert 0 <= best < len(D.tune_candidates())
        q = D.conv2d(x, w, 1, epilogue="requant_i8", scale=2.0 ** -12).cpu().numpy()
        assert np.array_equal(q, Orc.requant_i8(ref, 2.0 ** -12))
        a = torch.from_numpy(Orc.random_tensor("u8", (384, 256), 5)).to(dev)
        b = torch.from_numpy(Orc.random_tensor("i8", (512, 256), 6)).to(dev)
        best, _ = D.tune_gemm(a, b, reps=3)
        assert np.array_equal(D.gemm(a, b).cpu().numpy(), Orc.matmul(a.cpu().numpy(), b.cpu().numpy()))
    finally:
        D.clear_tuning()


def test_eval_tir_random_reference_schedules(cuda):
    """Seeded random tcgen05 schedules (reordered / annotated outer loops,
    split_reduction) lowered, injected and executed: bit-exact every time."""
    import random

    from tests.test_tensor_ir import random_tcgen05_schedule
    text = matmul_tdsl(256, 256, 128)
    ins = Orc.random_inputs(decls(text), 19)
    ref = Orc.matmul(ins["A"], ins["B"], ins["C"])
    rng = random.Random(7)
    for _ in range(6):
        sched = random_tcgen05_schedule(rng)
        assert np.array_equal(ops.eval_tir(text, "tcgen05_i8_m128n128k32", ins, schedule=sched), ref), sched


def test_eval_tir_split_reduction_becomes_device_split_k(cuda):
    """A schedule's split_reduction (rewriter.cpp:425-451) runs as the device
    split-K (partials + wrap-add fix-up launch), bit-exact."""
    from paper_2101_08458_b200 import device as D
    text = matmul_tdsl(256, 256, 1024)
    ins = Orc.random_inputs(decls(text), 23)
    ref = Orc.matmul(ins["A"], ins["B"], ins["C"])
    plain = "split x 128\nsplit y 128\nsplit k 32\nreorder x.o y.o k.o x.i y.i k.i\npragma x.i y.i k.i\n"
    split = ("split x 128\nsplit y 128\nsplit k 32\nsplit_reduction k.o 4\n"
             "reorder x.o y.o k.o.s k.o.r x.i y.i k.i\npragma x.i y.i k.i\n")
    # the in-kernel fix-up (default): one launch per op, bit-exact
    assert np.array_equal(ops.eval_tir(text, "tcgen05_i8_m128n128k32", ins, schedule=split), ref)
    # with the separate fix-up kernel (and no automatic split) the fold launch is visible
    D.set_option("splitk_inkernel", 0)
    D.set_option("split_min_kb", 1 << 20)
    try:
        n0 = D.launch_count()
        assert np.array_equal(ops.eval_tir(text, "tcgen05_i8_m128n128k32", ins, schedule=plain), ref)
        n1 = D.launch_count()
        assert np.array_equal(ops.eval_tir(text, "tcgen05_i8_m128n128k32", ins, schedule=split), ref)
        n2 = D.launch_count()
    finally:
        D.set_option("splitk_inkernel", 1)
        D.set_option("split_min_kb", 0)
    assert n2 - n1 > n1 - n0  # the fix-up (fold) kernel launched
    assert "C.partial" in ops.lower(text, split, "tcgen05_i8_m128n128k32")


@pytest.mark.parametrize("shape", __import__("paper_2101_08458_b200.workloads", fromlist=["x"]).TABLE1_BANK,
                         ids=lambda b: b[0])
def test_table1_bank_on_device(cuda, shape):
    """The paper's Table-1 bank (proj/src/workloads.cpp:123-142), exactly as the
    reference lowers it (blocked layouts, accumulate-form seed), through
    tzc_b200_run_op with tcgen05: bit-exact vs the oracle, and the fused requant."""
    from paper_2101_08458_b200.workloads import conv2d_tdsl
    _, c, hw, k, r, st = shape
    text = conv2d_tdsl(c, hw, k, r, st)
    ins = Orc.random_inputs(decls(text), 1000 + c)
    ref = Orc.conv2d_blocked(ins["data"], ins["kernel"], st, ins["out"])
    assert np.array_equal(ops.run_op(text, "tcgen05_i8_m128n64k32", ins), ref)
    q = ops.run_op(text, "tcgen05_i8_m128n64k32", ins, epilogue=requant_tdsl(ref.shape, 2.0 ** -14, src="out"))
    assert np.array_equal(q, Orc.requant_i8(ref, 2.0 ** -14))


@pytest.mark.parametrize("name", ["conv3d_i8", "conv3d_s2_i8"])
def test_conv3d_run_op_with_requant(cuda, name):
    """conv3d_tdsl through tzc_b200_run_op (depth-tap decomposition chained through
    the int32 C-seed): the reference's own output (saved by make_tnsr.py) bit for
    bit, and the fused requant on the last tap."""
    from tests.gpu_helpers import read_tnsr
    d = os.path.join(GOLD, "tnsr", name)
    text = open(os.path.join(d, "op.tdsl")).read()
    ins = {n: read_tnsr(os.path.join(d, n + ".tnsr")) for n in ("data", "kernel", "out")}
    want = read_tnsr(os.path.join(d, "expect.tnsr"))
    assert np.array_equal(ops.run_op(text, "tcgen05_i8_m128n64k32", ins), want)
    q = ops.run_op(text, "tcgen05_i8_m128n64k32", ins, epilogue=requant_tdsl(want.shape, 2.0 ** -13, src="out"))
    assert np.array_equal(q, Orc.requant_i8(want, 2.0 ** -13))


@pytest.mark.parametrize("shape", __import__("paper_2101_08458_b200.workloads", fromlist=["x"]).RESNET18_3D_BANK,
                         ids=lambda b: b[0])
def test_resnet18_3d_bank_on_device(cuda, shape):
    """The resnet18-3d bank at full size through tzc_b200_run_op; 64 sampled
    output elements recomputed exactly (int64 sums wrapped to int32) — the full
    op is hours of reference-VM time."""
    from paper_2101_08458_b200.workloads import conv3d_tdsl
    _, c, hw, k, r, st = shape
    text = conv3d_tdsl(c, hw, k, r, st)
    dec = decls(text)
    data = Orc.random_tensor("u8", dec[0][3], 100 + c)
    kern = Orc.random_tensor("i8", dec[1][3], 200 + k)
    out = ops.run_op(text, "tcgen05_i8_m128n64k32", {"data": data, "kernel": kern})
    rng = np.random.default_rng(c * k)
    ko_n, o = out.shape[0], out.shape[1]
    for _ in range(64):
        ko, od, oh, ow, ki = (int(rng.integers(0, n)) for n in (ko_n, o, o, o, 16))
        x = data[:, od * st:od * st + r, oh * st:oh * st + r, ow * st:ow * st + r, :].astype(np.int64)
        w = kern[ko, :, :, :, :, ki, :].astype(np.int64)
        want = np.int64((x * w).sum()).astype(np.int32)
        assert out[ko, od, oh, ow, ki] == want, (ko, od, oh, ow, ki)


@pytest.mark.parametrize("n", [64, 128, 256])
@pytest.mark.parametrize("form", ["matmul", "conv3x3", "conv1x1"])
def test_instruction_n_is_the_executed_tile(cuda, n, form):
    """The selected tcgen05 description's N is the N tile the launch runs
    (it used to be advisory), for the general and the
    shifted-window kernels alike; results stay bit-exact."""
    from paper_2101_08458_b200 import device as D
    if form == "matmul":
        text = matmul_tdsl(384, 256, 192)
        ins = Orc.random_inputs(decls(text), 90)
        ref = Orc.matmul(ins["A"], ins["B"], ins["C"])
    else:
        r = 3 if form == "conv3x3" else 1
        text = conv2d_nhwc_tdsl(2, 14, 14, 64, 256, r, r, 1)
        ins = Orc.random_inputs(decls(text), 91)
        ref = Orc.conv2d_nhwc(ins["data"], ins["kernel"], 1, ins["out"])
    got = ops.run_op(text, f"tcgen05_i8_m128n{n}k32", ins)
    info = D.last_launch()
    assert info["bn"] == n and info["cta_group"] == 1, info
    assert np.array_equal(got, ref)


@pytest.mark.parametrize("n", [128, 256])
@pytest.mark.parametrize("form", ["matmul", "conv3x3"])
def test_m256_instruction_runs_the_cta_pair_kernel(cuda, n, form):
    """tcgen05_i8_m256n{N}k32 (cta_group::2): the fused-requant op runs on the
    CTA-pair kernel (256 rows per MMA, each CTA loads half of B), bit-exact."""
    from paper_2101_08458_b200 import device as D
    if form == "matmul":
        text = matmul_tdsl(768, 256, 512)
        ins = Orc.random_inputs(decls(text), 92)
        ref = Orc.matmul(ins["A"], ins["B"], ins["C"])
        shape = (768, 256)
        epi = requant_tdsl(shape, 2.0 ** -14)
    else:
        text = conv2d_nhwc_tdsl(2, 16, 16, 128, 256, 3, 3, 1)
        ins = Orc.random_inputs(decls(text), 93)
        ref = Orc.conv2d_nhwc(ins["data"], ins["kernel"], 1, ins["out"])
        epi = requant_tdsl(ref.shape, 2.0 ** -14, src="out")
    q = ops.run_op(text, f"tcgen05_i8_m256n{n}k32", ins, epilogue=epi)
    info = D.last_launch()
    assert info["kernel"] == "cta_pair" and info["cta_group"] == 2 and info["bm"] == 256 and info["bn"] == n, info
    assert np.array_equal(q, Orc.requant_i8(ref, 2.0 ** -14))
