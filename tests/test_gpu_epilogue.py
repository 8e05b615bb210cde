"""The TMA-store int8 epilogue (SMEM staging in the output map's swizzle,
one cp.async.bulk.tensor store per lane quarter and 128-byte column box) vs
the oracle and vs the direct-store epilogue: bit-exact, including ragged M
(rows clipped by the map), every BN (64/128/256 -> SWIZZLE_64B/128B, one or
two boxes), seeds (general requant path) and the simple 2^-k path."""
import numpy as np
import pytest
import torch

from oracle.pyoracle import Orc
from paper_2101_08458_b200 import device as D
from tests.gpu_helpers import to_dev

pytestmark = pytest.mark.gpu


def gemm_q(cuda, a, b, scale, seed=None, tma=True):
    D.set_option("tma_store", 1 if tma else 0)
    try:
        return D.gemm(to_dev(a, cuda), to_dev(b, cuda), None if seed is None else to_dev(seed, cuda),
                      epilogue="requant_i8", scale=scale).cpu().numpy()
    finally:
        D.set_option("tma_store", 0)


@pytest.mark.parametrize("m,n,k", [(1000, 64, 64), (777, 128, 128), (1283, 256, 64), (300, 512, 256),
                                   (128, 64, 32), (4096, 256, 128)])
@pytest.mark.parametrize("scale", [2.0 ** -12, 0.0003])
def test_tma_store_gemm_requant(cuda, m, n, k, scale):
    a = Orc.random_tensor("u8", (m, k), 400)
    b = Orc.random_tensor("i8", (n, k), 401)
    want = Orc.requant_i8(Orc.matmul(a, b), scale)
    assert np.array_equal(gemm_q(cuda, a, b, scale), want)
    assert np.array_equal(gemm_q(cuda, a, b, scale, tma=False), want)


def test_tma_store_with_seed(cuda):
    m, n, k = 515, 128, 96
    a = Orc.random_tensor("u8", (m, k), 410)
    b = Orc.random_tensor("i8", (n, k), 411)
    s0 = Orc.random_tensor("i32", (m, n), 412)
    want = Orc.requant_i8(Orc.matmul(a, b, s0), 2.0 ** -10)
    assert np.array_equal(gemm_q(cuda, a, b, 2.0 ** -10, seed=s0), want)


@pytest.mark.parametrize("n,hp,c,k,r,stride", [(2, 30, 64, 256, 1, 1), (3, 17, 128, 64, 3, 2), (1, 58, 64, 128, 1, 2)])
def test_tma_store_conv_requant(cuda, n, hp, c, k, r, stride):
    x = Orc.random_tensor("u8", (n, hp, hp, c), 420)
    w = Orc.random_tensor("i8", (k, r, r, c), 421)
    scale = 2.0 ** -13
    want = Orc.requant_i8(Orc.conv2d_nhwc(x, w, stride), scale)
    for tma in (1, 0):
        D.set_option("tma_store", tma)
        try:
            got = D.conv2d(to_dev(x, cuda), to_dev(w, cuda), stride, epilogue="requant_i8", scale=scale).cpu().numpy()
        finally:
            D.set_option("tma_store", 0)
        assert np.array_equal(got, want), tma


def test_tma_store_output_untouched_outside(cuda):
    """Clipping: a 1000-row output inside a larger buffer; rows past M keep their bytes."""
    m, n, k = 1000, 256, 64
    a = Orc.random_tensor("u8", (m, k), 430)
    b = Orc.random_tensor("i8", (n, k), 431)
    for tma in (1, 0):
        big = torch.full((m + 200, n), 77, dtype=torch.int8, device=cuda)
        D.set_option("tma_store", tma)
        try:
            D.gemm(to_dev(a, cuda), to_dev(b, cuda), epilogue="requant_i8", scale=2.0 ** -12, out=big[:m])
        finally:
            D.set_option("tma_store", 0)
        got = big.cpu().numpy()
        assert np.array_equal(got[:m], Orc.requant_i8(Orc.matmul(a, b), 2.0 ** -12))
        assert (got[m:] == 77).all()


@pytest.mark.parametrize("n", [48, 80, 208, 96])
@pytest.mark.parametrize("st256", [1, 0])
def test_simple_requant_ragged_n_strided(cuda, n, st256):
    """The 2^-k fast path (256-bit or 128-bit row stores) with N not a multiple
    of the tile: columns past N inside a wider row buffer keep their bytes."""
    m, k = 700, 64
    a = Orc.random_tensor("u8", (m, k), 440)
    b = Orc.random_tensor("i8", (n, k), 441)
    big = torch.full((m, n + 112), 77, dtype=torch.int8, device=cuda)
    D.set_option("st256", st256)
    try:
        D.gemm(to_dev(a, cuda), to_dev(b, cuda), epilogue="requant_i8", scale=2.0 ** -9, out=big,
               out_layout=D.OutLayout(nb=n, stride_m=n + 112, stride_blk=0))
    finally:
        D.set_option("st256", 1)
    got = big.cpu().numpy()
    assert np.array_equal(got[:, :n], Orc.requant_i8(Orc.matmul(a, b), 2.0 ** -9))
    assert (got[:, n:] == 77).all()


@pytest.mark.parametrize("st256", [1, 0])
def test_simple_requant_ws_conv_256bit(cuda, st256):
    """Shifted-window conv (stride 1, 3x3) through the 256-bit store path."""
    x = Orc.random_tensor("u8", (2, 20, 20, 64), 450)
    w = Orc.random_tensor("i8", (64, 3, 3, 64), 451)
    want = Orc.requant_i8(Orc.conv2d_nhwc(x, w, 1), 2.0 ** -12)
    D.set_option("st256", st256)
    try:
        got = D.conv2d(to_dev(x, cuda), to_dev(w, cuda), 1, epilogue="requant_i8", scale=2.0 ** -12).cpu().numpy()
    finally:
        D.set_option("st256", 1)
    assert np.array_equal(got, want)


@pytest.mark.parametrize("st256", [1, 0])
def test_wide_stores_f16_and_raw_outputs(cuda, st256):
    """fp16-cast and raw int32 outputs through the 256-bit (st256=1) and the
    128-bit store paths: identical bytes."""
    from tests.gpu_helpers import rel_dev
    x = Orc.random_tensor("fp16", (2, 12, 12, 64), 460)
    w = Orc.random_tensor("fp16", (128, 3, 3, 64), 461)
    a = Orc.random_tensor("u8", (300, 256), 462)
    b = Orc.random_tensor("i8", (192, 256), 463)
    D.set_option("st256", st256)
    try:
        h = D.conv2d(to_dev(x, cuda, True), to_dev(w, cuda, True), 1, epilogue="f16").cpu()
        i32 = D.gemm(to_dev(a, cuda), to_dev(b, cuda)).cpu().numpy()
    finally:
        D.set_option("st256", 1)
    hv = h.view(torch.int16).numpy().view(np.uint16).view(np.float16).astype(np.float64)
    assert rel_dev(Orc.conv2d_nhwc(x, w, 1, fp16=True), hv) <= 1e-3 + 2 ** -11
    assert np.array_equal(i32, Orc.matmul(a, b))


def extreme_operands(shape_x, shape_w, seed):
    """Random u8 / i8 operands where the first half of the output channels see
    all-255 inputs against all -128 / +127 weights somewhere, so accumulators
    reach |c| >= 2^24 (the fp32 cast rounds: the checked 2^-k path must take
    its exact RNE24 fallback) next to ordinary ones."""
    x = Orc.random_tensor("u8", shape_x, seed)
    w = Orc.random_tensor("i8", shape_w, seed + 1)
    x = x.copy()
    w = w.copy()
    x.reshape(-1, shape_x[-1])[: x.reshape(-1, shape_x[-1]).shape[0] // 3] = 255
    k = shape_w[0]
    w[: k // 4] = -128
    w[k // 4: k // 2] = 127
    return x, w


@pytest.mark.parametrize("c,r,hp", [(1024, 1, 20), (128, 3, 22), (2048, 1, 9)])
@pytest.mark.parametrize("scale", [2.0 ** -12, 2.0 ** -6])
def test_simple_requant_checked_large_k(cuda, c, r, hp, scale):
    """K * 255 * 128 >= 2^24: the 2^-k fast path with its per-chunk |c| check
    (r = 3, C = 128 runs on the shifted-window kernel, the 1x1 layers on the
    general one), bit-exact to cast<i8>(cast<fp32>(C) * 2^-k) including the
    |c| >= 2^24 elements where the fp32 cast rounds."""
    n, k = 3, 256
    x, w = extreme_operands((n, hp, hp, c), (k, r, r, c), 700 + c + r)
    ref = Orc.conv2d_nhwc(x, w, 1)
    assert np.abs(ref.astype(np.int64)).max() >= (1 << 24)  # the fallback is exercised
    got = D.conv2d(to_dev(x, cuda), to_dev(w, cuda), 1, epilogue="requant_i8", scale=scale).cpu().numpy()
    assert np.array_equal(got, Orc.requant_i8(ref, scale))
