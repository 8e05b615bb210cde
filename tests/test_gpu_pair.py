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
# the library defaults (tzc_b200_internal.hpp Options): pairs for BN = 256
# layers with >= 8 K blocks whose pair tiles fill a round of SM pairs
DEFAULTS = {"pair": 1, "pair_min_kb": 8, "pair_bn": 256, "pair_min_round": 1, "tma_store": 0, "pingpong_kb": 0}
FORCE = {"pair_min_kb": 1, "pair_bn": 0, "pair_min_round": 0, "pingpong_kb": 0}  # (pairs need one epilogue group)


def set_opts(opts):
    for k, v in opts.items():
        D.set_option(k, v)


def with_pair(on, fn, tma_store=1):
    """Force the pair kernel (on=1) for every eligible tile, or the single-CTA
    kernel (on=0); checks that the intended kernel ran."""
    set_opts({"pair": on, **FORCE, "tma_store": tma_store})
    try:
        out = fn()
        ran = D.last_launch()
        assert ran["kernel"] == ("cta_pair" if on else "general"), ran
        return out
    finally:
        set_opts(DEFAULTS)


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
    got = with_pair(1, lambda: D.gemm(to_dev(a, cuda), to_dev(b, cuda), epilogue="requant_i8",
                                      scale=2.0 ** -12).cpu().numpy(), tma_store=0)
    assert np.array_equal(got, want)
