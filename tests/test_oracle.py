"""Pins the oracle (oracle/oracle.c, our C restatement of the reference's
arithmetic) to the reference: golden vectors frozen from the reference's own
tests and from the reference implementation itself (tests/golden/, made by
tests/golden/make_golden.py), plus live cross-checks against
oracle/_ref/libtzc_ref.so when it is present.  CPU only."""
import hashlib
import os
import re

import numpy as np
import pytest

from oracle.pyoracle import Orc, Ref

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    return np.load(os.path.join(GOLD, name), allow_pickle=False)


def decls(text):
    """[(name, dtype, role, shape)] in declaration order."""
    out = []
    for m in re.finditer(r"tensor (\w+) : (\w+) \[([\d, ]+)\] (input|output)", text):
        shape = tuple(int(v) for v in m.group(3).split(","))
        out.append((m.group(1), m.group(2), "in" if m.group(4) == "input" else "out", shape))
    return out


def scale_of(text):
    m = re.search(r"\* ([0-9.eE+-]+)\)", text)
    return float(m.group(1))


def orc_eval(name, text, seed):
    """Evaluate a golden op with the restatement, from regenerated inputs."""
    d = decls(text)
    update = "+=" in text
    ins = Orc.random_inputs(d, seed, update=update)
    if name.startswith("mm_"):
        return Orc.matmul(ins["A"], ins["B"], ins["C"], fp16="f16" in name)
    if name.startswith("conv_blk"):
        st = 2 if "s2" in name.split("_")[-1] else 1
        return Orc.conv2d_blocked(ins["data"], ins["kernel"], st, ins["out"], fp16="f16" in name)
    if name.startswith("conv_nhwc"):
        st = 2 if re.search(r"r\ds2$", name) else 1
        return Orc.conv2d_nhwc(ins["data"], ins["kernel"], st, ins["out"], fp16="f16" in name)
    if name.startswith("requant"):
        return Orc.requant_i8(ins["C"], np.float32(scale_of(text)))
    if name.startswith("cast_f16"):
        return Orc.cast_f16(ins["C"])
    raise KeyError(name)


# ---- binary16 rounding (proj/tests/test_dtype.cpp:74-155) ------------------
def test_f16_vectors_match_reference_and_numpy():
    g = load("f16_vectors.npz")
    mine = np.array([Orc.f64_to_f16_bits(x) for x in g["inputs"]], np.uint16)
    assert np.array_equal(mine, g["bits"])
    # the reference's own frozen expectations (test_dtype.cpp:79-103)
    expect = [0x0000, 0x8000, 0x3c00, 0xbc00, 0x4000, 0x7bff, 0x7c00, 0x7bff, 0xfc00, 0x2e66, 0x3555,
              0x6800, 0x6800, 0x6801, 0x0001, 0x0000, 0x0001, 0x0400, 0x03ff, 0x0000, 0x8000, 0x3e00,
              0x3801, 0x4200, 0x6400, 0x7c00, 0xfc00]
    assert list(g["bits"]) == expect
    # an independent IEEE-754 implementation
    fin = np.isfinite(g["inputs"])
    assert np.array_equal(np.array(g["inputs"][fin], np.float64).astype(np.float16).view(np.uint16), mine[fin])
    prod = np.array([Orc.f64_to_f16_bits(a * b) for a, b in zip(g["mul_a"], g["mul_b"])], np.uint16)
    assert list(prod) == list(g["mul_bits"]) == [0x3c02, 0x251e, 0x3cf0, 0x7c00, 0xc820]


def test_f16_roundtrip_exhaustive():
    """Every finite binary16 value decodes and re-encodes to itself."""
    L = Orc.lib()
    for b in range(0, 0x10000, 7):
        e = (b >> 10) & 0x1F
        if e == 0x1F:
            continue
        assert L.orc_f64_to_f16_bits(L.orc_f16_bits_to_f64(b)) == b


# ---- hand-checked answers (proj/tests/test_vm.cpp:49-137, test_smoke.py:31-40)
def test_known_answers():
    g = load("known_answers.npz")
    assert g["mm2_zero_seed"].tolist() == [[19, 22], [43, 50]]
    assert g["mm2_seeded"].tolist() == [[119, 222], [343, 450]]
    assert g["i32_wrap"].tolist() == [-589934592]
    assert g["f2i_trunc"].tolist() == [2, -2, 0, 0]
    want = g["smoke_c0"].astype(np.int64) + g["smoke_a"].astype(np.int64) @ g["smoke_b"].astype(np.int64).T
    assert np.array_equal(g["smoke_out"], want)
    # the restatement on the same cases
    A = np.array([[1, 2], [3, 4]], np.uint8)
    Bt = np.array([[5, 7], [6, 8]], np.int8)  # B[k, y] of the 2x2 op, as [y, k]
    assert Orc.matmul(A, Bt).tolist() == [[19, 22], [43, 50]]
    assert Orc.matmul(A, Bt, np.array([[100, 200], [300, 400]], np.int32)).tolist() == [[119, 222], [343, 450]]
    got = Orc.matmul(g["smoke_a"], g["smoke_b"], g["smoke_c0"])
    assert np.array_equal(got, g["smoke_out"])


def test_requant_semantics_vectors():
    """SURVEY.md Appendix B probe 6: cast<i8>(cast<fp32>(C) * 2^-7)."""
    c = np.array([0, 127, 128, 255, -129, 16383, -16385, 2147483647], np.int32)
    assert Orc.requant_i8(c, np.float32(0.0078125)).tolist() == [0, 0, 1, 1, -1, 127, -128, 0]


# ---- seeded ops evaluated by the reference ---------------------------------
SEEDED = load("seeded.npz")
SEEDED_NAMES = sorted({k.split("__")[0] for k in SEEDED.files})


@pytest.mark.parametrize("name", SEEDED_NAMES)
def test_restatement_matches_reference_golden(name):
    text = str(SEEDED[name + "__text"])
    seed = int(SEEDED[name + "__seed"])
    want = SEEDED[name + "__out"]
    got = orc_eval(name, text, seed)
    assert got.dtype == want.dtype and got.shape == want.shape
    assert np.array_equal(got.view(np.uint8), want.view(np.uint8)), f"{name}: bit mismatch"


def test_c1_full_size_hash():
    """BASELINE config 1 at full size (conv2d_tdsl({64,56,64,3,1},16,4)): the
    restatement reproduces the reference's int32 and requantized outputs."""
    g = load("c1.npz")
    text = str(g["text"])
    ins = Orc.random_inputs(decls(text), int(g["seed"]))
    out = Orc.conv2d_blocked(ins["data"], ins["kernel"], 1, ins["out"])
    assert hashlib.sha256(out.tobytes()).hexdigest() == str(g["sha_i32"])
    q = Orc.requant_i8(out, np.float32(2.0 ** -12))
    assert hashlib.sha256(q.tobytes()).hexdigest() == str(g["sha_i8"])


# ---- live cross-checks against the compiled reference ----------------------
needs_ref = pytest.mark.skipif(not Ref.available(), reason="oracle/_ref not built (no /root/reference)")


@needs_ref
@pytest.mark.parametrize("seed", [0, 1, 1000])
def test_rng_matches_reference(seed):
    for text in (Ref.matmul_tdsl(9, 7, 33), Ref.matmul_tdsl(5, 6, 7, fp16=True),
                 Ref.conv2d_tdsl(16, 6, 16, 3, 1, 16, 4)):
        info = Ref.op_info(text)
        d = [(n, *info.tensors[n]) for n in info.order]
        mine = Orc.random_inputs(d, seed, update=info.update)
        ref = Ref.random_inputs(text, seed)
        assert mine.keys() == ref.keys()
        for k in ref:
            assert np.array_equal(mine[k].view(np.uint8), ref[k].view(np.uint8)), k


@needs_ref
def test_eval_tir_equals_eval_reference():
    """The reference's hot path (eval_tir with vdot_16x4) is bit-exact to its
    oracle on a batched NHWC conv — the op form the B200 path executes."""
    from paper_2101_08458_b200.workloads import conv2d_nhwc_tdsl
    t = conv2d_nhwc_tdsl(1, 5, 5, 16, 32, 3, 3, 1)
    ins = Ref.random_inputs(t, 3)
    assert np.array_equal(Ref.eval_tir(t, "vdot_16x4", ins), Ref.eval_reference(t, ins))


@needs_ref
def test_live_restatement_random_ops():
    rng = np.random.default_rng(1)
    from paper_2101_08458_b200.workloads import conv2d_nhwc_tdsl
    for _ in range(4):
        n, h, c, k, r = 1, int(rng.integers(3, 7)), int(rng.choice([4, 8, 16])), 16, int(rng.choice([1, 3]))
        st = int(rng.choice([1, 2]))
        if h < r:
            continue
        t = conv2d_nhwc_tdsl(n, h, h, c, k, r, r, st)
        seed = int(rng.integers(0, 1 << 30))
        ref = Ref.eval_reference(t, Ref.random_inputs(t, seed))
        ins = Orc.random_inputs(decls(t), seed)
        got = Orc.conv2d_nhwc(ins["data"], ins["kernel"], st, ins["out"])
        assert np.array_equal(ref, got)
