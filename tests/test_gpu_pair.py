"""CTA-pair kernel (conv_tc2_kernel, tcgen05.mma.cta_group::2, M=256 tiles,
B split across the pair) vs the oracle: bit-exact for tiled GEMM / 1x1 and
TMA-im2col convs, odd M-tile counts (the last pair's second tile is empty),
BN 128 / 256, and the same results as the single-CTA kernel."""
import numpy as np
import pytest
import torch

from oracle.pyoracle import Orc
from paper_2101_08458_b200 import device as D
from tests.gpu_helpers import to_dev

pytestmark = pytest.mark.gpu
PAIR_DEFAULT = 0  # the library defaults (conv_tc.cu g_pair, g_pair_min_kb)
PAIR_MIN_KB = 16


def with_pair(on, fn):
    """The pair kernel runs the TMA-store epilogue: force it for every tile."""
    D.set_option("pair", on)
    D.set_option("pair_min_kb", 1)
    D.set_option("tma_store", 1)
    try:
        return fn()
    finally:
        D.set_option("pair", PAIR_DEFAULT)
        D.set_option("pair_min_kb", PAIR_MIN_KB)
        D.set_option("tma_store", 0)


@pytest.mark.parametrize("m,n,k", [(1000, 256, 512), (777, 128, 384), (4096, 256, 1024), (300, 512, 256 + 128),
                                   (128, 256, 384), (129, 128, 640)])
def test_pair_gemm_requant(cuda, m, n, k):
    a = Orc.random_tensor("u8", (m, k), 500)
    b = Orc.random_tensor("i8", (n, k), 501)
    want = Orc.requant_i8(Orc.matmul(a, b), 2.0 ** -12)
    run = lambda: D.gemm(to_dev(a, cuda), to_dev(b, cuda), epilogue="requant_i8", scale=2.0 ** -12).cpu().numpy()
    assert np.array_equal(with_pair(1, run), want)
    assert np.array_equal(with_pair(0, run), want)


@pytest.mark.parametrize("n,hp,c,k,r,stride", [(2, 17, 128, 256, 3, 2), (3, 30, 256, 128, 1, 2), (1, 16, 512, 256, 1, 1),
                                               (2, 9, 256, 512, 3, 1), (1, 31, 128, 128, 3, 2)])
def test_pair_conv_requant(cuda, n, hp, c, k, r, stride):
    x = Orc.random_tensor("u8", (n, hp, hp, c), 510)
    w = Orc.random_tensor("i8", (k, r, r, c), 511)
    scale = 2.0 ** -13
    want = Orc.requant_i8(Orc.conv2d_nhwc(x, w, stride), scale)
    run = lambda: D.conv2d(to_dev(x, cuda), to_dev(w, cuda), stride, epilogue="requant_i8", scale=scale).cpu().numpy()
    assert np.array_equal(with_pair(1, run), want)


def test_pair_general_requant_scale(cuda):
    """A non-power-of-two scale (general requant path) through the pair kernel."""
    m, n, k = 640, 256, 768
    a = Orc.random_tensor("u8", (m, k), 520)
    b = Orc.random_tensor("i8", (n, k), 521)
    want = Orc.requant_i8(Orc.matmul(a, b), 0.00037)
    got = with_pair(1, lambda: D.gemm(to_dev(a, cuda), to_dev(b, cuda), epilogue="requant_i8",
                                      scale=0.00037).cpu().numpy())
    assert np.array_equal(got, want)


@pytest.mark.parametrize("m,n,k", [(1000, 256, 512), (129, 128, 640)])
def test_pair_direct_store_epilogue(cuda, m, n, k):
    """The pair kernel with the direct (256-bit row store) epilogue."""
    a = Orc.random_tensor("u8", (m, k), 530)
    b = Orc.random_tensor("i8", (n, k), 531)
    want = Orc.requant_i8(Orc.matmul(a, b), 2.0 ** -12)
    D.set_option("pair", 1)
    D.set_option("pair_min_kb", 1)
    try:
        got = D.gemm(to_dev(a, cuda), to_dev(b, cuda), epilogue="requant_i8", scale=2.0 ** -12).cpu().numpy()
    finally:
        D.set_option("pair", PAIR_DEFAULT)
        D.set_option("pair_min_kb", PAIR_MIN_KB)
    assert np.array_equal(got, want)
