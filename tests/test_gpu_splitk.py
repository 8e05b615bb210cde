"""Split-K with the in-kernel fix-up (conv_tc.cuh: every split stores its
int32 / fp32 partial slice, the last split to arrive at a (tile, epilogue
warp) arrival counter adds them and runs the real epilogue; the counters are
left at zero for the next launch).  This is the device form of the
reference's split_reduction (/root/reference/proj/src/rewriter.cpp:425-451):
integer partials wrap-add, associative, so bit-exact for any split order (F8).

* automatic split for under-filled grids (the small-M c4 / c5 layers at
  small batch), with a C-seed and the general requant scale;
* repeated CUDA-graph replays of one captured split launch (the counters
  must reset every time);
* fp16 split-K within the compare() tolerance;
* equality with the separate fix-up kernel's result."""
import numpy as np
import pytest
import torch

from oracle.pyoracle import Orc
from paper_2101_08458_b200 import device as D
from paper_2101_08458_b200.workloads import RESNET50_V15, requant_scale
from tests.gpu_helpers import rel_dev, to_dev

pytestmark = pytest.mark.gpu


def layer(name):
    return next(x for x in RESNET50_V15 if x.name == name)


@pytest.mark.parametrize("name,nb", [("c5_3x3_512", 4), ("c5_1x1_2048_512", 8), ("c4_3x3_256", 2),
                                     ("c5_1x1s2_1024_2048", 3)])
def test_auto_split_small_batch(cuda, name, nb):
    L = layer(name)
    x = Orc.random_tensor("u8", (nb, L.h, L.h, L.c), 600)
    w = Orc.random_tensor("i8", (L.k, L.r, L.r, L.c), 601)
    o = L.out_hw()
    s0 = Orc.random_tensor("i32", (nb, o, o, L.k), 602)
    D.set_option("shifted_window", 0)
    D.set_option("split_min_kb", 4)  # automatic split for under-filled grids (off by default)
    try:
        d, _ = D.conv_desc(x.shape, w.shape, L.stride)
        plan = D.plan_conv(d)
        assert plan["splits"] > 1, plan  # under-filled grid: split automatically
        xd, wd, sd = to_dev(x, cuda), to_dev(w, cuda), to_dev(s0, cuda)
        c0 = D.launch_count()
        got = D.conv2d(xd, wd, L.stride, sd).cpu().numpy()
        assert D.launch_count() - c0 == 1  # the fix-up is inside the kernel
        s = requant_scale(L.c * L.r * L.r)
        q = D.conv2d(xd, wd, L.stride, epilogue="requant_i8", scale=s).cpu().numpy()
        qg = D.conv2d(xd, wd, L.stride, sd, epilogue="requant_i8", scale=0.000613).cpu().numpy()
    finally:
        D.set_option("shifted_window", 1)
        D.set_option("split_min_kb", 0)
    ref = Orc.conv2d_nhwc(x, w, L.stride, s0)
    assert np.array_equal(got, ref)
    assert np.array_equal(q, Orc.requant_i8(Orc.conv2d_nhwc(x, w, L.stride), s))
    assert np.array_equal(qg, Orc.requant_i8(ref, 0.000613))


def test_split_graph_replays_reset_counters(cuda):
    L = layer("c5_3x3_512")
    nb = 4
    x = Orc.random_tensor("u8", (nb, L.h, L.h, L.c), 610)
    w = Orc.random_tensor("i8", (L.k, L.r, L.r, L.c), 611)
    xd, wd = to_dev(x, cuda), to_dev(w, cuda)
    s = requant_scale(L.c * L.r * L.r)
    out = torch.empty((nb, L.out_hw(), L.out_hw(), L.k), dtype=torch.int8, device=cuda)
    st = torch.cuda.Stream()
    D.set_option("shifted_window", 0)
    D.set_splits(3)
    try:
        with torch.cuda.stream(st):
            D.conv2d(xd, wd, L.stride, epilogue="requant_i8", scale=s, out=out, stream=st)  # eager: workspace
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            D.conv2d(xd, wd, L.stride, epilogue="requant_i8", scale=s, out=out, stream=st)
        want = Orc.requant_i8(Orc.conv2d_nhwc(x, w, L.stride), s)
        for _ in range(4):
            out.zero_()
            torch.cuda.synchronize()
            with torch.cuda.stream(st):
                g.replay()
            torch.cuda.synchronize()
            assert np.array_equal(out.cpu().numpy(), want)
    finally:
        D.set_option("shifted_window", 1)
        D.set_splits(0)


def test_split_inkernel_equals_fixup_kernel(cuda):
    A = Orc.random_tensor("u8", (384, 2048), 620)
    B = Orc.random_tensor("i8", (512, 2048), 621)
    C0 = Orc.random_tensor("i32", (384, 512), 622)
    res = {}
    for ink in (1, 0):
        D.set_option("splitk_inkernel", ink)
        D.set_splits(5)
        try:
            res[ink] = D.gemm(to_dev(A, cuda), to_dev(B, cuda), to_dev(C0, cuda)).cpu().numpy()
        finally:
            D.set_splits(0)
            D.set_option("splitk_inkernel", 1)
    assert np.array_equal(res[1], res[0])
    assert np.array_equal(res[1], Orc.matmul(A, B, C0))


def test_split_f16(cuda):
    A = Orc.random_tensor("fp16", (256, 1024), 630)
    B = Orc.random_tensor("fp16", (1024, 256), 631)  # matmul_tdsl's fp16 layout: B [K, N]
    D.set_splits(4)
    try:
        got = D.gemm(to_dev(A, cuda, True), to_dev(B, cuda, True), epilogue="f32", b_kn=True).cpu().numpy()
    finally:
        D.set_splits(0)
    assert rel_dev(Orc.matmul(A, B, fp16=True), got) <= 1e-3


@pytest.mark.parametrize("opts,n,hp", [({"b_res": 1}, 4, 100), ({"producers": 1}, 2, 20),
                                       ({"b_res": 1, "producers": 1}, 4, 100), ({"pingpong_kb": 16}, 3, 20)])
def test_general_kernel_pipeline_options(cuda, opts, n, hp):
    """The general kernel's operand-pipeline variants (resident B tile loaded
    once per CTA; one or two TMA producer warps) plan the same tiles and stay
    bit-exact, int32 and fused requant."""
    from paper_2101_08458_b200 import device as D
    c, k, r = 128, 128, 3
    x = Orc.random_tensor("u8", (n, hp, hp, c), 540)
    w = Orc.random_tensor("i8", (k, r, r, c), 541)
    D.set_option("shifted_window", 0)
    for kk, v in opts.items():
        D.set_option(kk, v)
    try:
        xd, wd = to_dev(x, cuda), to_dev(w, cuda)
        got = D.conv2d(xd, wd, 1).cpu().numpy()
        assert D.last_launch()["kernel"] == "general"
        q = D.conv2d(xd, wd, 1, epilogue="requant_i8", scale=2.0 ** -13).cpu().numpy()
    finally:
        D.set_option("shifted_window", 1)
        D.set_option("b_res", 2)
        D.set_option("producers", 2)
        D.set_option("pingpong_kb", 0)
    ref = Orc.conv2d_nhwc(x, w, 1)
    assert np.array_equal(got, ref)
    assert np.array_equal(q, Orc.requant_i8(ref, 2.0 ** -13))
