"""GPU parity: the sm_100a kernels (through the C ABI) vs the CPU oracle on
the reference's seeded inputs.  int8 paths must be bit-exact (int32
accumulators and requantized int8); fp16 paths within 1e-3 relative under
the reference's compare() metric (proj/src/vm.cpp:626-639; tolerance from
proj/tests/acceptance.cpp:152-155)."""
import numpy as np
import pytest
import torch

from oracle.pyoracle import Orc
from paper_2101_08458_b200 import device as D
from tests.gpu_helpers import out_seed, rel_dev, to_dev

pytestmark = pytest.mark.gpu
F16_TOL = 1e-3


def _gemm_case(cuda, m, n, k, seed=1000, with_seed=True, epilogue="i32", scale=2.0 ** -14, splits=0):
    A = Orc.random_tensor("u8", (m, k), seed)
    B = Orc.random_tensor("i8", (n, k), seed + 1)
    C0 = Orc.random_tensor("i32", (m, n), seed + 2) if with_seed else None
    ref = Orc.matmul(A, B, C0)
    D.set_splits(splits)
    try:
        got = D.gemm(to_dev(A, cuda), to_dev(B, cuda), None if C0 is None else to_dev(C0, cuda),
                     epilogue=epilogue, scale=scale)
        torch.cuda.synchronize()
    finally:
        D.set_splits(0)
    got = got.cpu().numpy()
    if epilogue == "requant_i8":
        ref = Orc.requant_i8(ref, scale)
    return ref, got


@pytest.mark.parametrize("m,n,k", [(128, 256, 128), (256, 256, 512), (200, 96, 256), (384, 128, 64),
                                   (129, 64, 1024), (1000, 512, 320)])
def test_gemm_i8_int32_bitexact(cuda, m, n, k):
    ref, got = _gemm_case(cuda, m, n, k)
    assert np.array_equal(ref, got), f"mismatches: {(ref != got).sum()}"


def test_gemm_i8_no_seed(cuda):
    ref, got = _gemm_case(cuda, 256, 128, 256, with_seed=False)
    assert np.array_equal(ref, got)


@pytest.mark.parametrize("scale", [2.0 ** -14, 2.0 ** -7, 1.0, 2.0 ** -40, 0.0123, -0.37, 3.0e30, 1e-40])
def test_gemm_i8_requant_bitexact(cuda, scale):
    ref, got = _gemm_case(cuda, 256, 256, 512, epilogue="requant_i8", scale=scale)
    assert np.array_equal(ref, got), f"mismatches: {(ref != got).sum()}"


@pytest.mark.parametrize("splits", [2, 3, 7])
def test_gemm_i8_splitk_bitexact(cuda, splits):
    ref, got = _gemm_case(cuda, 256, 256, 1024, splits=splits)
    assert np.array_equal(ref, got)
    ref, got = _gemm_case(cuda, 256, 256, 1024, splits=splits, epilogue="requant_i8")
    assert np.array_equal(ref, got)


CONV_CASES = [
    # n, hp, wp, c, k, r, stride
    (2, 10, 10, 64, 64, 3, 1),
    (1, 12, 12, 128, 128, 3, 2),
    (2, 9, 9, 256, 64, 1, 1),
    (1, 14, 14, 256, 512, 1, 2),
    (3, 16, 16, 512, 256, 3, 1),
    (1, 58, 58, 64, 64, 3, 1),
    (2, 21, 21, 3, 64, 7, 2),     # C=3 stem: K7 im2col path
    (1, 15, 15, 3, 64, 7, 2),
]


@pytest.mark.parametrize("n,hp,wp,c,k,r,stride", CONV_CASES)
def test_conv_i8_bitexact(cuda, n, hp, wp, c, k, r, stride):
    x = Orc.random_tensor("u8", (n, hp, wp, c), 1000)
    w = Orc.random_tensor("i8", (k, r, r, c), 1001)
    oh, ow = (hp - r) // stride + 1, (wp - r) // stride + 1
    s0 = Orc.random_tensor("i32", (n, oh, ow, k), 1002)
    ref = Orc.conv2d_nhwc(x, w, stride, s0)
    got = D.conv2d(to_dev(x, cuda), to_dev(w, cuda), stride, to_dev(s0, cuda)).cpu().numpy()
    assert np.array_equal(ref, got), f"mismatches: {(ref != got).sum()} / {ref.size}"
    scale = 2.0 ** -13
    q = D.conv2d(to_dev(x, cuda), to_dev(w, cuda), stride, to_dev(s0, cuda), epilogue="requant_i8",
                 scale=scale).cpu().numpy()
    assert np.array_equal(Orc.requant_i8(ref, scale), q)


def test_conv_i8_rskc_weights(cuda):
    """conv2d_tdsl with (lane_block, red_block) = (K, C) puts weights as [R,S,K,C]."""
    n, hp, c, k, r = 1, 10, 64, 128, 3
    x = Orc.random_tensor("u8", (n, hp, hp, c), 7)
    w = Orc.random_tensor("i8", (k, r, r, c), 8)
    ref = Orc.conv2d_nhwc(x, w, 1)
    w_rskc = np.ascontiguousarray(w.transpose(1, 2, 0, 3))
    got = D.conv2d(to_dev(x, cuda), to_dev(w_rskc, cuda), 1, w_layout="rskc").cpu().numpy()
    assert np.array_equal(ref, got)


def test_gemm_f16(cuda):
    m, n, k = 256, 128, 512
    A = Orc.random_tensor("fp16", (m, k), 3)
    B = Orc.random_tensor("fp16", (k, n), 4)
    C0 = Orc.random_tensor("fp32", (m, n), 5)
    ref = Orc.matmul(A, B, C0, fp16=True)
    got = D.gemm(to_dev(A, cuda, True), to_dev(B, cuda, True), to_dev(C0, cuda), epilogue="f32",
                 b_kn=True).cpu().numpy()
    assert rel_dev(ref, got) <= F16_TOL


def test_conv_f16(cuda):
    n, hp, c, k, r = 2, 12, 64, 128, 3
    x = Orc.random_tensor("fp16", (n, hp, hp, c), 11)
    w = Orc.random_tensor("fp16", (k, r, r, c), 12)
    ref = Orc.conv2d_nhwc(x, w, 1, fp16=True)
    got = D.conv2d(to_dev(x, cuda, True), to_dev(w, cuda, True), 1, epilogue="f32").cpu().numpy()
    assert rel_dev(ref, got) <= F16_TOL
    h = D.conv2d(to_dev(x, cuda, True), to_dev(w, cuda, True), 1, epilogue="f16").cpu()
    h = h.view(torch.int16).numpy().view(np.uint16)
    # the cast is RNE of the fp32 accumulator; compare in value space
    hv = h.view(np.float16).astype(np.float64)
    assert rel_dev(ref, hv) <= 1e-3 + 2 ** -11


EDGE_I32 = [0, 1, -1, 127, 128, 255, 256, -128, -129, 2**24 - 1, 2**24, 2**24 + 1, 2**24 + 3,
            -(2**24) - 1, 2**25 + 2, 2**30 + 2**6, 2**31 - 1, -(2**31), -(2**31) + 1, 16383, -16385,
            2147483647 - 64, 33554431, -33554431]


@pytest.mark.parametrize("scale", [2.0 ** -7, 2.0 ** -14, 1.0, 2.0 ** -31, 2.0 ** -32, 0.0078125, 0.3,
                                   -1.5, 7.0e20, 9.3e18, -9.3e18, 1e-45, float("inf")])
def test_requant_edges_bitexact(cuda, scale):
    """A = 0, so C == C-seed: drives the fused requant over int32 edge values
    (RNE boundaries at 2^24, INT_MIN/INT_MAX, saturation at 2^63, denormals)."""
    rng = np.random.default_rng(5)
    vals = np.array(EDGE_I32 + list(rng.integers(-(2**31), 2**31, size=4096 - len(EDGE_I32))), dtype=np.int64)
    m, n, k = 128, 32, 64
    seed = vals[: m * n].astype(np.int32).reshape(m, n)
    A = np.zeros((m, k), np.uint8)
    B = Orc.random_tensor("i8", (n, k), 9)
    got = D.gemm(to_dev(A, cuda), to_dev(B, cuda), to_dev(seed, cuda), epilogue="requant_i8",
                 scale=scale).cpu().numpy()
    assert np.array_equal(Orc.requant_i8(seed, scale), got)
