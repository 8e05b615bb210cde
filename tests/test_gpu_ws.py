"""The weight-stationary shifted-window kernel (conv_ws.cuh) and the
space-to-depth stem path vs the oracle and vs the TMA-im2col kernel on the
same inputs: bit-exact int32 / requant, fp16 within 1e-3."""
import numpy as np
import pytest
import torch

from oracle.pyoracle import Orc
from paper_2101_08458_b200 import device as D
from tests.gpu_helpers import rel_dev, to_dev

pytestmark = pytest.mark.gpu

WS_CASES = [
    # n, hp, c, k, r  (stride 1, eligible for the shifted window)
    (3, 58, 64, 64, 3),
    (2, 30, 128, 128, 3),
    (2, 30, 64, 256, 3),
    (1, 16, 128, 64, 3),     # waste 1.31
    (2, 58, 128, 64, 3),     # SR 246 rows, two channel blocks... (c=128: one 128-B block)
    (1, 34, 256, 64, 5),     # 5x5, c_blocks 2
]


def run(cuda, x, w, stride, seed=None, ws=True, **kw):
    D.set_option("shifted_window", 1 if ws else 0)
    try:
        return D.conv2d(to_dev(x, cuda, x.dtype == np.uint16), to_dev(w, cuda, w.dtype == np.uint16), stride,
                        None if seed is None else to_dev(seed, cuda), **kw).cpu().numpy()
    finally:
        D.set_option("shifted_window", 1)


@pytest.mark.parametrize("n,hp,c,k,r", WS_CASES)
def test_ws_conv_bitexact(cuda, n, hp, c, k, r):
    x = Orc.random_tensor("u8", (n, hp, hp, c), 300)
    w = Orc.random_tensor("i8", (k, r, r, c), 301)
    o = hp - r + 1
    s0 = Orc.random_tensor("i32", (n, o, o, k), 302)
    ref = Orc.conv2d_nhwc(x, w, 1, s0)
    assert np.array_equal(run(cuda, x, w, 1, s0), ref)
    assert np.array_equal(run(cuda, x, w, 1, s0, ws=False), ref)
    scale = 2.0 ** -12
    q = run(cuda, x, w, 1, None, epilogue="requant_i8", scale=scale)
    assert np.array_equal(q, Orc.requant_i8(Orc.conv2d_nhwc(x, w, 1), scale))


@pytest.mark.parametrize("fused", [0, 1])
@pytest.mark.parametrize("n,hp,k", [(2, 230, 64), (1, 62, 64), (3, 62, 128), (2, 61, 64), (5, 230, 256)])
def test_s2d_stem_bitexact(cuda, n, hp, k, fused):
    """7x7 stride-2 over C=3: space-to-depth to 16-byte pixels + the pair-mode
    kernel; fused=1: the space-to-depth done inside the kernel (stem_ws.cuh:
    raw 1-D TMA staging -> transform warps), incl. odd extents (61)."""
    x = Orc.random_tensor("u8", (n, hp, hp, 3), 310)
    w = Orc.random_tensor("i8", (k, 7, 7, 3), 311)
    ref = Orc.conv2d_nhwc(x, w, 2)
    D.set_option("stem_fused", fused)
    try:
        assert np.array_equal(run(cuda, x, w, 2), ref)
        o = (hp - 7) // 2 + 1
        s0 = Orc.random_tensor("i32", (n, o, o, k), 312)
        assert np.array_equal(run(cuda, x, w, 2, s0), Orc.conv2d_nhwc(x, w, 2, s0))
        scale = 2.0 ** -11
        q = run(cuda, x, w, 2, None, epilogue="requant_i8", scale=scale)
        assert np.array_equal(q, Orc.requant_i8(ref, scale))
    finally:
        D.set_option("stem_fused", 0)


def test_ws_blocked_output_layout(cuda):
    """conv2d_tdsl's channel-blocked output written by the shifted-window epilogue."""
    n, hp, c, k, r = 1, 30, 64, 64, 3
    x = Orc.random_tensor("u8", (n, hp, hp, c), 320)
    w = Orc.random_tensor("i8", (k, r, r, c), 321)
    o = hp - r + 1
    ref = Orc.conv2d_nhwc(x, w, 1)  # [1, o, o, 64]
    lay = D.blocked_layout(k, o * o, 16)
    out = torch.empty((k // 16, o, o, 16), dtype=torch.int32, device=cuda)
    D.conv2d(to_dev(x, cuda), to_dev(w, cuda), 1, out=out, out_layout=lay)
    got = out.cpu().numpy()
    want = ref[0].reshape(o, o, k // 16, 16).transpose(2, 0, 1, 3)
    assert np.array_equal(got, want)


def test_ws_f16(cuda):
    n, hp, c, k, r = 2, 30, 64, 128, 3
    x = Orc.random_tensor("fp16", (n, hp, hp, c), 330)
    w = Orc.random_tensor("fp16", (k, r, r, c), 331)
    ref = Orc.conv2d_nhwc(x, w, 1, fp16=True)
    assert rel_dev(ref, run(cuda, x, w, 1, epilogue="f32")) <= 1e-3


@pytest.mark.parametrize("n,hp,c,k,r", WS_CASES + [(2, 9, 512, 64, 3), (5, 7, 64, 128, 3)])
def test_ws_requant_tiny_images(cuda, n, hp, c, k, r):
    """Requant of the padded grid, incl. tiny images (Wp < 32: one lane
    quarter's 32-pixel run spans several image rows and images), general
    (seeded) and 2^-k paths, with the tma_store option on and off (it must
    never change a result)."""
    x = Orc.random_tensor("u8", (n, hp, hp, c), 340)
    w = Orc.random_tensor("i8", (k, r, r, c), 341)
    o = hp - r + 1
    s0 = Orc.random_tensor("i32", (n, o, o, k), 342)
    for scale, seed in ((2.0 ** -13, None), (0.00071, s0)):
        want = Orc.requant_i8(Orc.conv2d_nhwc(x, w, 1, seed), scale)
        for tma in (1, 0):
            D.set_option("tma_store", tma)
            try:
                got = run(cuda, x, w, 1, seed, epilogue="requant_i8", scale=scale)
            finally:
                D.set_option("tma_store", 0)
            assert np.array_equal(got, want), (scale, tma)


@pytest.mark.parametrize("n,hp,k", [(2, 230, 64), (3, 62, 128), (2, 62, 256)])
def test_s2d_stem_f16(cuda, n, hp, k):
    """fp16 7x7 stride-2 stem over C=3: space-to-depth to 32-byte pixels and
    the shifted-window kernel with one K=16 MMA per tap (SWIZZLE_32B)."""
    x = Orc.random_tensor("fp16", (n, hp, hp, 3), 340)
    w = Orc.random_tensor("fp16", (k, 7, 7, 3), 341)
    d, _ = D.conv_desc((n, hp, hp, 3), (k, 7, 7, 3), 2, f16=True)
    assert D.plan_conv(d)["a_mode"] == 3
    ref = Orc.conv2d_nhwc(x, w, 2, fp16=True)
    assert rel_dev(ref, run(cuda, x, w, 2, epilogue="f32")) <= 1e-3
    o = (hp - 7) // 2 + 1
    s0 = Orc.random_tensor("fp32", (n, o, o, k), 342)
    assert rel_dev(Orc.conv2d_nhwc(x, w, 2, s0, fp16=True), run(cuda, x, w, 2, s0, epilogue="f32")) <= 1e-3


@pytest.mark.parametrize("n,hp,wp", [(2, 228, 228), (3, 64, 60), (2, 30, 36), (4, 12, 8), (1, 10, 14), (2, 22, 18)])
def test_s2d_stem_row_widths(cuda, n, hp, wp):
    """The one-launch S2D (rows from 32-bit loads + the weight rearrangement):
    Wp % 4 == 0 (row 2*h4+1 word-aligned) and == 2 (funnel-shifted), an even
    and an odd number of S2D pixels per row (the last pixel / pair on 16-bit
    loads), rectangular images; int32 and fused requant bit-exact."""
    x = Orc.random_tensor("u8", (n, hp, wp, 3), 320 + wp)
    w = Orc.random_tensor("i8", (64, 7, 7, 3), 321)
    ref = Orc.conv2d_nhwc(x, w, 2)
    xd, wd = to_dev(x, cuda), to_dev(w, cuda)
    assert np.array_equal(D.conv2d(xd, wd, 2).cpu().numpy(), ref)
    q = D.conv2d(xd, wd, 2, epilogue="requant_i8", scale=2.0 ** -10).cpu().numpy()
    assert np.array_equal(q, Orc.requant_i8(ref, 2.0 ** -10))
