"""The shifted-window kernel's multi-tile work units (conv_ws.cuh, MT = 2 / 4
consecutive 128-row tiles per unit) — the plans the batch-256 headline bench
times for stem7x7, c2_3x3_64 and c2_1x1_64_64.

* At batch 256 the DEFAULT plans are checked (plan bm == 512, i.e. MT = 4),
  exactly as bench.py runs them: sampled whole images (first, last, and
  images whose padded-grid rows straddle work-unit boundaries) against the
  oracle, the all-element checksum (linearity), and the fused requant image
  against the oracle's requant of the int32 image.
* At small batches MT = 2 / 4 is FORCED ("ws_mt") with one or two epilogue
  groups ("ws_epi_groups": NACC = 2, TPW = MT / W tiles per warp) and with a
  seed + a general (non power-of-two) scale, so the t = 1..3 A-shift, the
  accumulator ring and the TPW / G epilogue split all run under test.

Semantics: eval_reference, /root/reference/proj/src/vm.cpp:444-508; requant
as the reference-expressible op cast<i8>(cast<fp32>(C) * s).
"""
import numpy as np
import pytest
import torch

from oracle.pyoracle import Orc
from paper_2101_08458_b200 import device as D
from paper_2101_08458_b200.workloads import RESNET50_V15, requant_scale
from tests.gpu_helpers import to_dev

pytestmark = pytest.mark.gpu

MT_LAYERS = ["stem7x7", "c2_3x3_64", "c2_1x1_64_64"]


def wrap32(v):
    return int(np.int64(v & 0xFFFFFFFF).astype(np.uint32).view(np.int32))


def layer(name):
    return next(x for x in RESNET50_V15 if x.name == name)


def checksum(xn, wn, L):
    """sum over every output element, from input window sums x weight sums."""
    o = L.out_hw()
    wsum = wn.astype(np.int64).sum(0)  # [R,S,C]
    tot = 0
    for r in range(L.r):
        for s in range(L.r):
            win = xn[:, r:r + L.stride * (o - 1) + 1:L.stride, s:s + L.stride * (o - 1) + 1:L.stride, :]
            tot += int(win.astype(np.int64).sum((0, 1, 2)) @ wsum[r, s])
    return wrap32(tot)


def straddling_images(L, nb, mt):
    """Images whose padded-grid rows cross a work-unit boundary at several
    tile offsets t (the unit is mt*128 rows of the padded grid)."""
    hp = L.h if L.name != "stem7x7" else (L.h + 1) // 2  # stem: space-to-depth grid
    hw = hp * hp
    unit = mt * 128
    picks = set()
    for u in (1, 7, 123, 1001):
        q = u * unit + 3 * 128 // 2  # inside the unit's third/fourth tile
        img = q // hw
        if img < nb:
            picks.add(img)
    return sorted(picks)


@pytest.mark.parametrize("name", MT_LAYERS)
def test_default_plan_b256_mt4(cuda, name):
    L = layer(name)
    nb = 256
    g = torch.Generator(device=cuda)
    g.manual_seed(41)
    x = torch.randint(0, 256, (nb, L.h, L.h, L.c), dtype=torch.uint8, device=cuda, generator=g)
    w = torch.randint(-128, 128, (L.k, L.r, L.r, L.c), dtype=torch.int8, device=cuda, generator=g)
    d, _ = D.conv_desc(tuple(x.shape), tuple(w.shape), L.stride)
    plan = D.plan_conv(d)
    assert plan["bm"] == 512 and plan["a_mode"] in (2, 3), plan  # MT = 4 shifted-window units
    out = D.conv2d(x, w, L.stride).cpu().numpy()
    s = requant_scale(L.c * L.r * L.r)
    q = D.conv2d(x, w, L.stride, epilogue="requant_i8", scale=s).cpu().numpy()
    xn, wn = x.cpu().numpy(), w.cpu().numpy()
    imgs = sorted({0, nb - 1, *straddling_images(L, nb, 4)})
    assert len(imgs) >= 4
    for img in imgs:
        ref = Orc.conv2d_nhwc(xn[img:img + 1], wn, L.stride)
        assert np.array_equal(out[img:img + 1], ref), f"image {img}"
        assert np.array_equal(q[img:img + 1], Orc.requant_i8(ref, s)), f"image {img} (requant)"
    assert wrap32(int(out.astype(np.int64).sum())) == checksum(xn, wn, L)
    assert np.array_equal(Orc.requant_i8(out, s), q)


FORCED = [
    # name, nb, hp, c, k, r, stride (stride-2 C=3 7x7 = the space-to-depth stem)
    ("stem7x7", 6, 230, 3, 64, 7, 2),
    ("c2_3x3_64", 5, 58, 64, 64, 3, 1),
    ("c2_1x1_64_64", 7, 56, 64, 64, 1, 1),
    ("3x3_64_128", 4, 30, 64, 128, 3, 1),   # BN = 128: MT <= 2 (2 * MT * BN <= 512 TMEM columns)
    ("3x3_64_64_small", 11, 16, 64, 64, 3, 1),  # Wp < 32: a lane quarter's 32 rows span image rows
]


@pytest.mark.parametrize("name,nb,hp,c,k,r,st", FORCED, ids=[f[0] for f in FORCED])
@pytest.mark.parametrize("mt", [2, 4])
@pytest.mark.parametrize("eg", [1, 2])
def test_forced_mt(cuda, name, nb, hp, c, k, r, st, mt, eg):
    if 2 * mt * k > 512:
        pytest.skip("MT*BN exceeds TMEM")
    x = Orc.random_tensor("u8", (nb, hp, hp, c), 500 + mt)
    w = Orc.random_tensor("i8", (k, r, r, c), 510 + eg)
    o = (hp - r) // st + 1
    s0 = Orc.random_tensor("i32", (nb, o, o, k), 520)
    D.set_option("ws_mt", mt)
    D.set_option("ws_epi_groups", eg)
    try:
        d, _ = D.conv_desc(x.shape, w.shape, st)
        plan = D.plan_conv(d)
        assert plan["bm"] == 128 * mt and plan["a_mode"] in (2, 3), plan
        xd, wd = to_dev(x, cuda), to_dev(w, cuda)
        got = D.conv2d(xd, wd, st, to_dev(s0, cuda)).cpu().numpy()
        s = requant_scale(c * r * r)
        q = D.conv2d(xd, wd, st, epilogue="requant_i8", scale=s).cpu().numpy()  # 2^-k, simple path
        qg = D.conv2d(xd, wd, st, to_dev(s0, cuda), epilogue="requant_i8",
                      scale=0.000731).cpu().numpy()  # general scale + seed
    finally:
        D.set_option("ws_mt", 0)
        D.set_option("ws_epi_groups", 0)
    ref = Orc.conv2d_nhwc(x, w, st, s0)
    assert np.array_equal(got, ref)
    assert np.array_equal(q, Orc.requant_i8(Orc.conv2d_nhwc(x, w, st), s))
    assert np.array_equal(qg, Orc.requant_i8(ref, 0.000731))


@pytest.mark.parametrize("inkernel", [1, 0])
def test_forced_split_on_ws_layer_runs_split_k(cuda, inkernel):
    """A forced split-K on a stride-1 3x3 conv (eligible for the shifted
    window) must plan AND run on the general kernel as split-K (the
    ws branch used to ignore it and report a plan it did not run): one launch
    with the in-kernel fix-up, two with the separate fix-up kernel."""
    n, hp, c, k, r = 2, 16, 256, 128, 3
    x = Orc.random_tensor("u8", (n, hp, hp, c), 530)
    w = Orc.random_tensor("i8", (k, r, r, c), 531)
    D.set_splits(3)
    D.set_option("splitk_inkernel", inkernel)
    try:
        d, _ = D.conv_desc(x.shape, w.shape, 1)
        plan = D.plan_conv(d)
        assert plan["splits"] == 3 and plan["a_mode"] == 1, plan
        c0 = D.launch_count()
        got = D.conv2d(to_dev(x, cuda), to_dev(w, cuda), 1).cpu().numpy()
        assert D.launch_count() - c0 == (1 if inkernel else 2)
    finally:
        D.set_splits(0)
        D.set_option("splitk_inkernel", 1)
    assert np.array_equal(got, Orc.conv2d_nhwc(x, w, 1))
