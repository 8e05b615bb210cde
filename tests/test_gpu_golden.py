"""GPU path vs fixtures produced by the REFERENCE implementation itself
(tests/golden/, see make_golden.py): the seeded reference evaluations, and
BASELINE config 1 exactly as the reference lowers it (channel-blocked
conv2d_tdsl layouts: K5 adapters in, blocked epilogue layout out)."""
import hashlib
import os

import numpy as np
import pytest
import torch

from oracle.pyoracle import Orc
from paper_2101_08458_b200 import device as D
from tests.gpu_helpers import rel_dev, to_dev
from tests.test_oracle import SEEDED, SEEDED_NAMES, decls

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _run_fixture(cuda, name):
    text = str(SEEDED[name + "__text"])
    seed = int(SEEDED[name + "__seed"])
    f16 = "f16" in name
    ins = Orc.random_inputs(decls(text), seed, update=True)
    dev = lambda a, h=False: to_dev(a, cuda, h)  # noqa: E731
    if name.startswith("mm_"):
        return D.gemm(dev(ins["A"], f16), dev(ins["B"], f16), dev(ins["C"]), epilogue="f32" if f16 else "i32",
                      b_kn=f16).cpu().numpy()
    if name.startswith("conv_nhwc"):
        st = 2 if name.endswith("s2") else 1
        return D.conv2d(dev(ins["data"], f16), dev(ins["kernel"], f16), st, dev(ins["out"]),
                        epilogue="f32" if f16 else "i32").cpu().numpy()
    if name.startswith("conv_blk"):
        data, kern, seedimg = ins["data"], ins["kernel"], ins["out"]
        co, h, _, cb = data.shape
        ko, _, r, _, kb, _ = kern.shape
        st = 2 if name.endswith("s2") else 1
        c, k = co * cb, ko * kb
        x = D.unblock_data(dev(data, f16), c, h, h, cb)
        w = D.unblock_kernel(dev(kern, f16), k, c, r, r, kb, cb)
        oh = (h - r) // st + 1
        lay = D.blocked_layout(k, oh * oh, kb)
        out = torch.empty(seedimg.shape, dtype=torch.float32 if f16 else torch.int32, device=cuda)
        D.conv2d(x, w, st, dev(seedimg), epilogue="f32" if f16 else "i32", out=out, out_layout=lay)
        return out.cpu().numpy()
    pytest.skip("epilogue-only fixture (covered by the fused-epilogue tests)")


@pytest.mark.parametrize("name", [n for n in SEEDED_NAMES if not n.startswith(("requant", "cast"))])
def test_seeded_reference_fixtures(cuda, name):
    want = SEEDED[name + "__out"]
    got = _run_fixture(cuda, name)
    assert got.shape == want.shape
    if "f16" in name:
        assert rel_dev(want, got) <= 1e-3
    else:
        assert np.array_equal(got, want), f"{(got != want).sum()} mismatches"


def test_c1_exact_reference_lowering(cuda):
    """configs[0]: conv2d_tdsl({64,56,64,3,1},16,4), seed 1000, against the
    reference's own full-size output (sha256 of all 186 624 int32 values and of
    the requantized int8 image)."""
    g = np.load(os.path.join(GOLD, "c1.npz"))
    ins = Orc.random_inputs(decls(str(g["text"])), int(g["seed"]))
    dev = lambda a: to_dev(a, cuda)  # noqa: E731
    x = D.unblock_data(dev(ins["data"]), 64, 56, 56, 4)
    w = D.unblock_kernel(dev(ins["kernel"]), 64, 64, 3, 3, 16, 4)
    lay = D.blocked_layout(64, 54 * 54, 16)
    out = torch.empty((4, 54, 54, 16), dtype=torch.int32, device=cuda)
    D.conv2d(x, w, 1, dev(ins["out"]), out=out, out_layout=lay)
    got = out.cpu().numpy()
    assert hashlib.sha256(got.tobytes()).hexdigest() == str(g["sha_i32"])
    assert np.array_equal(got.ravel()[g["sample_idx"]], g["sample_i32"])
    q = torch.empty((4, 54, 54, 16), dtype=torch.int8, device=cuda)
    D.conv2d(x, w, 1, dev(ins["out"]), epilogue="requant_i8", scale=2.0 ** -12, out=q, out_layout=lay)
    assert hashlib.sha256(q.cpu().numpy().tobytes()).hexdigest() == str(g["sha_i8"])


@pytest.mark.parametrize("m,n,k", [(200, 24, 48), (77, 40, 96), (130, 200, 144)])
def test_ragged_gemm_i8(cuda, m, n, k):
    """Channel / K extents that are not tile multiples: TMA zero fill on the
    K tail, masked element stores on the N tail."""
    A = Orc.random_tensor("u8", (m, k), 31)
    B = Orc.random_tensor("i8", (n, k), 32)
    C0 = Orc.random_tensor("i32", (m, n), 33)
    ref = Orc.matmul(A, B, C0)
    got = D.gemm(to_dev(A, cuda), to_dev(B, cuda), to_dev(C0, cuda)).cpu().numpy()
    assert np.array_equal(ref, got)
    q = D.gemm(to_dev(A, cuda), to_dev(B, cuda), to_dev(C0, cuda), epilogue="requant_i8", scale=2.0 ** -9)
    assert np.array_equal(Orc.requant_i8(ref, 2.0 ** -9), q.cpu().numpy())


def test_ragged_conv_i8_c48(cuda):
    n, hp, c, k, r = 2, 9, 48, 80, 3
    x = Orc.random_tensor("u8", (n, hp, hp, c), 41)
    w = Orc.random_tensor("i8", (k, r, r, c), 42)
    ref = Orc.conv2d_nhwc(x, w, 1)
    got = D.conv2d(to_dev(x, cuda), to_dev(w, cuda), 1).cpu().numpy()
    assert np.array_equal(ref, got)
