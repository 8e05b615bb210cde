"""Parity at BASELINE.json's full sizes, through size-independent properties
the oracle can afford: sampled rows / images recomputed by the CPU oracle,
and a checksum-of-checksums (linearity: the wrapping sum of every output
element equals sum(seed) + sum_k colsum(A)[k] * colsum(B)[k] mod 2^32)."""
import numpy as np
import pytest
import torch

from oracle.pyoracle import Orc
from paper_2101_08458_b200 import device as D
from paper_2101_08458_b200.workloads import RESNET50_V15, requant_scale
from tests.gpu_helpers import to_dev

pytestmark = pytest.mark.gpu


def wrap32(v):
    return np.int64(np.uint64(v & 0xFFFFFFFF).astype(np.uint32).view(np.int32))


def test_c2_matmul_4096_full(cuda):
    """configs[1]: int8 matmul 4096^3, int32 accumulation (random full-range
    C-seed, wraps) and fused requant to int8."""
    m = n = k = 4096
    g = torch.Generator(device=cuda)
    g.manual_seed(2)
    A = torch.randint(0, 256, (m, k), dtype=torch.uint8, device=cuda, generator=g)
    B = torch.randint(-128, 128, (n, k), dtype=torch.int8, device=cuda, generator=g)
    C0 = torch.randint(-(2 ** 31), 2 ** 31, (m, n), dtype=torch.int32, device=cuda, generator=g)
    out = D.gemm(A, B, C0).cpu().numpy()
    q = D.gemm(A, B, C0, epilogue="requant_i8", scale=2.0 ** -14).cpu().numpy()
    An, Bn, Cn = A.cpu().numpy(), B.cpu().numpy(), C0.cpu().numpy()
    rows = np.random.default_rng(0).choice(m, 64, replace=False)
    ref = Orc.matmul(An[rows], Bn, Cn[rows])
    assert np.array_equal(out[rows], ref)
    assert np.array_equal(q[rows], Orc.requant_i8(ref, 2.0 ** -14))
    # requant of the whole int32 image == fused int8 image
    assert np.array_equal(Orc.requant_i8(out, 2.0 ** -14), q)
    total = int(Cn.astype(np.int64).sum()) + int(An.astype(np.int64).sum(0) @ Bn.astype(np.int64).sum(0))
    assert wrap32(int(out.astype(np.int64).sum())) == wrap32(total)


@pytest.mark.parametrize("layer", [L.name for L in RESNET50_V15])
def test_resnet50_layer_b32(cuda, layer):
    """configs[2] shapes at batch 32: two whole images recomputed by the
    oracle, the requant image checked against the oracle's requant of the
    GPU int32 image, and the all-element checksum."""
    L = next(x for x in RESNET50_V15 if x.name == layer)
    nb = 32
    g = torch.Generator(device=cuda)
    g.manual_seed(5)
    x = torch.randint(0, 256, (nb, L.h, L.h, L.c), dtype=torch.uint8, device=cuda, generator=g)
    w = torch.randint(-128, 128, (L.k, L.r, L.r, L.c), dtype=torch.int8, device=cuda, generator=g)
    out = D.conv2d(x, w, L.stride).cpu().numpy()
    s = requant_scale(L.c * L.r * L.r)
    q = D.conv2d(x, w, L.stride, epilogue="requant_i8", scale=s).cpu().numpy()
    xn, wn = x.cpu().numpy(), w.cpu().numpy()
    for img in (0, nb - 1):
        ref = Orc.conv2d_nhwc(xn[img:img + 1], wn, L.stride)
        assert np.array_equal(out[img:img + 1], ref), f"image {img}"
    assert np.array_equal(Orc.requant_i8(out, s), q)
    # checksum: sum over outputs = sum_{r,s,c} (sum of x over the tap's strided window) * (sum_k w)
    o = L.out_hw()
    wsum = wn.astype(np.int64).sum(0)  # [R,S,C]
    tot = 0
    for r in range(L.r):
        for c_ in range(L.r):
            win = xn[:, r:r + L.stride * (o - 1) + 1:L.stride, c_:c_ + L.stride * (o - 1) + 1:L.stride, :]
            tot += int(win.astype(np.int64).sum((0, 1, 2)) @ wsum[r, c_])
    assert wrap32(int(out.astype(np.int64).sum())) == wrap32(tot)


@pytest.mark.parametrize("layer", [L.name for L in RESNET50_V15])
def test_resnet50_layer_f16_b64(cuda, layer):
    """configs[3]: the fp16 suite at batch 64 with fp32 accumulation (kind::f16
    MMAs, fp32 TMEM accumulators): the first and last images against the
    oracle's fp16 conv (per-op fp32 rounding in declared order) within the
    reference's compare() tolerance 1e-3; fp16-cast outputs on the same run."""
    from tests.gpu_helpers import rel_dev
    L = next(x for x in RESNET50_V15 if x.name == layer)
    nb = 64
    x = Orc.random_tensor("fp16", (nb, L.h, L.h, L.c), 900)
    w = Orc.random_tensor("fp16", (L.k, L.r, L.r, L.c), 901)
    xd, wd = to_dev(x, cuda, True), to_dev(w, cuda, True)
    out = D.conv2d(xd, wd, L.stride, epilogue="f32").cpu().numpy()
    h16 = D.conv2d(xd, wd, L.stride, epilogue="f16").cpu().numpy().astype(np.float32)
    for img in (0, nb - 1):
        ref = Orc.conv2d_nhwc(x[img:img + 1], w, L.stride, fp16=True)
        assert rel_dev(ref, out[img:img + 1]) <= 1e-3, f"image {img}"
        assert rel_dev(ref, h16[img:img + 1]) <= 1e-3, f"image {img} (fp16 cast)"
    assert np.isfinite(out).all()


@pytest.mark.parametrize("layer", ["c5_3x3_512", "c5_1x1_2048_512"])
def test_tail_split_b256(cuda, layer):
    """196 tiles on 148 SMs: the last round's tiles are split along K (int32
    partials + fix-up) while whole tiles keep the fused epilogue.  Images from
    the whole-tile region and from the split tail, int32 and requant."""
    L = next(x for x in RESNET50_V15 if x.name == layer)
    nb = 256
    g = torch.Generator(device=cuda)
    g.manual_seed(11)
    x = torch.randint(0, 256, (nb, L.h, L.h, L.c), dtype=torch.uint8, device=cuda, generator=g)
    w = torch.randint(-128, 128, (L.k, L.r, L.r, L.c), dtype=torch.int8, device=cuda, generator=g)
    D.set_option("tail_split", 1)
    try:
        d, _ = D.conv_desc(tuple(x.shape), tuple(w.shape), L.stride)
        plan = D.plan_conv(d)
        assert plan["splits"] > 1 and plan["grid"] == 148, plan
        out = D.conv2d(x, w, L.stride).cpu().numpy()
        s = requant_scale(L.c * L.r * L.r)
        q = D.conv2d(x, w, L.stride, epilogue="requant_i8", scale=s).cpu().numpy()
    finally:
        D.set_option("tail_split", 0)
    xn, wn = x.cpu().numpy(), w.cpu().numpy()
    for img in (0, 150, 200, nb - 1):  # rows 7350.. (whole tiles) and >= 9472 (split tail)
        ref = Orc.conv2d_nhwc(xn[img:img + 1], wn, L.stride)
        assert np.array_equal(out[img:img + 1], ref), f"image {img}"
        assert np.array_equal(q[img:img + 1], Orc.requant_i8(ref, s)), f"image {img} (requant)"
