"""Small launches of every kernel family for compute-sanitizer
(memcheck / racecheck / synccheck): tools/sanitize.sh runs this under each
tool and profiles/r02_sanitizer.md summarises the logs.  Each case is also
checked against the oracle so a sanitizer-clean run is a correct run."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from oracle.pyoracle import Orc  # noqa: E402
from paper_2101_08458_b200 import device as D  # noqa: E402

dev = torch.device("cuda:0")


def t(a, f16=False):
    x = torch.from_numpy(np.ascontiguousarray(a)).to(dev)
    return x.view(torch.float16) if f16 else x


def conv(n, hp, c, k, r, st, opts=(), seed=True, scale=None, label=""):
    for kk, v in opts:
        D.set_option(kk, v)
    try:
        x = Orc.random_tensor("u8", (n, hp, hp, c), 1)
        w = Orc.random_tensor("i8", (k, r, r, c), 2)
        o = (hp - r) // st + 1
        s0 = Orc.random_tensor("i32", (n, o, o, k), 3) if seed else None
        d, _ = D.conv_desc(x.shape, w.shape, st)
        plan = D.plan_conv(d)
        if scale is None:
            got = D.conv2d(t(x), t(w), st, None if s0 is None else t(s0)).cpu().numpy()
            ok = np.array_equal(got, Orc.conv2d_nhwc(x, w, st, s0))
        else:
            got = D.conv2d(t(x), t(w), st, None if s0 is None else t(s0), epilogue="requant_i8",
                           scale=scale).cpu().numpy()
            ok = np.array_equal(got, Orc.requant_i8(Orc.conv2d_nhwc(x, w, st, s0), scale))
    finally:
        for kk, _ in opts:
            D.set_option(kk, {"ws_mt": 0, "ws_epi_groups": 0, "splits": 0, "pair": 1, "pair_min_kb": 8,
                              "pair_bn": 256, "pair_min_round": 1, "shifted_window": 1, "tma_store": 0, "tail_split": 0, "stem_fused": 0,
                              "splitk_inkernel": 1, "b_res": 2, "producers": 2, "s2d_one": 1, "pingpong_kb": 0}[kk])  # library defaults
    ran = D.last_launch()
    print(f"{label:34s} plan a_mode={plan['a_mode']} bm={plan['bm']} bn={plan['bn']} splits={plan['splits']} "
          f"ran {ran['kernel']} cta_group={ran['cta_group']} bm={ran['bm']} bn={ran['bn']} "
          f"{'OK' if ok else 'MISMATCH'}", flush=True)
    return ok


def main():
    ok = True
    ok &= conv(2, 10, 64, 128, 3, 1, opts=[("shifted_window", 0)], label="conv_tc im2col BN128")
    ok &= conv(1, 9, 256, 256, 1, 1, opts=[("shifted_window", 0)], seed=False, scale=2.0 ** -12,
               label="conv_tc tiled BN256 requant")
    ok &= conv(2, 12, 64, 64, 3, 2, label="conv_tc im2col s2 BN64")
    ok &= conv(2, 18, 64, 64, 3, 1, label="conv_ws MT1")
    ok &= conv(3, 18, 64, 64, 3, 1, opts=[("ws_mt", 2)], seed=False, scale=2.0 ** -12, label="conv_ws MT2 requant")
    ok &= conv(3, 18, 64, 64, 3, 1, opts=[("ws_mt", 4), ("ws_epi_groups", 2)], label="conv_ws MT4 EG2")
    ok &= conv(2, 62, 3, 64, 7, 2, seed=False, scale=2.0 ** -11, label="s2d stem pair MT auto")
    ok &= conv(2, 62, 3, 64, 7, 2, opts=[("ws_mt", 4)], label="s2d stem pair MT4")
    ok &= conv(2, 62, 3, 64, 7, 2, opts=[("stem_fused", 1)], label="fused stem (stem_ws)")
    ok &= conv(3, 61, 3, 128, 7, 2, opts=[("stem_fused", 1)], seed=False, scale=2.0 ** -11,
               label="fused stem odd extent requant")
    ok &= conv(2, 10, 256, 128, 3, 1, opts=[("splits", 3), ("splitk_inkernel", 0)], label="split-K + fix-up kernel")
    ok &= conv(2, 10, 256, 128, 3, 1, opts=[("splits", 3)], label="split-K, in-kernel fix-up")
    ok &= conv(2, 10, 256, 256, 3, 1, opts=[("shifted_window", 0), ("pair", 1), ("pair_min_kb", 1), ("pair_min_round", 0)],
               seed=False, scale=2.0 ** -13, label="conv_tc2 CTA pair")
    ok &= conv(2, 10, 64, 256, 1, 1, opts=[("shifted_window", 0), ("tma_store", 1)], seed=False,
               scale=2.0 ** -12, label="conv_tc TMA-store epilogue")
    ok &= conv(3, 10, 128, 128, 3, 1, opts=[("shifted_window", 0), ("pair", 1), ("pair_min_kb", 1), ("pair_bn", 0), ("pair_min_round", 0)],
               seed=False, scale=2.0 ** -13, label="conv_tc2 CTA pair BN128")
    ok &= conv(4, 100, 128, 128, 3, 1, opts=[("shifted_window", 0), ("b_res", 1)], seed=False, scale=2.0 ** -13,
               label="conv_tc resident B (301 tiles)")
    ok &= conv(2, 10, 64, 128, 3, 1, opts=[("shifted_window", 0), ("producers", 1)], label="conv_tc one producer")
    ok &= conv(2, 10, 64, 256, 1, 1, opts=[("shifted_window", 0), ("pingpong_kb", 16)], seed=False,
               scale=2.0 ** -12, label="conv_tc ping-pong epilogue groups")
    ok &= conv(2, 62, 3, 64, 7, 2, opts=[("s2d_one", 0)], seed=False, scale=2.0 ** -11,
               label="s2d stem two-launch S2D")
    # fp16
    x = Orc.random_tensor("fp16", (2, 10, 10, 64), 5)
    w = Orc.random_tensor("fp16", (128, 3, 3, 64), 6)
    got = D.conv2d(t(x, True), t(w, True), 1, epilogue="f32").cpu().numpy()
    ref = Orc.conv2d_nhwc(x, w, 1, fp16=True)
    rel = float(np.max(np.abs(got - ref) / np.maximum(np.abs(ref), 1.0)))
    print(f"{'conv f16 (ws)':34s} max rel {rel:.2e} {'OK' if rel <= 1e-3 else 'MISMATCH'}", flush=True)
    ok &= rel <= 1e-3
    A = Orc.random_tensor("u8", (200, 256), 7)
    B = Orc.random_tensor("i8", (192, 256), 8)
    g = D.gemm(t(A), t(B)).cpu().numpy()
    good = np.array_equal(g, Orc.matmul(A, B))
    print(f"{'gemm ragged M/N':34s} {'OK' if good else 'MISMATCH'}", flush=True)
    ok &= good
    print("ALL OK" if ok else "SOME MISMATCH")
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
