"""Generates tests/golden/*.npz from the REFERENCE implementation itself
(oracle/_ref/libtzc_ref.so, compiled unmodified from /root/reference).

Run in the build container (needs /root/reference to have built oracle/_ref):
    python tests/golden/make_golden.py
The fixtures are committed; the GPU box never needs the reference.

Contents
  f16_vectors.npz    binary16 RNE known answers: the input values frozen in
                     proj/tests/test_dtype.cpp:78-104 (numpy-derived) and the
                     fp16 products of :138-155, with the reference's outputs.
  known_answers.npz  hand-checked cases of proj/tests/test_vm.cpp:49-137 and
                     proj/python/tests/test_smoke.py:31-40, evaluated by the
                     reference (eval_reference).
  seeded.npz         eval_reference outputs of small seeded ops (matmul_tdsl,
                     conv2d_tdsl, batched NHWC conv, fp16 twins, requant and
                     cast ops); inputs are regenerated from (op text, seed)
                     by random_inputs, so only outputs are stored.
  c1.npz             BASELINE config 1 exactly as the reference lowers it
                     (conv2d_tdsl({64,56,64,3,1},16,4), seed 1000): sha256 +
                     sampled values of the full int32 output and of its
                     requantized int8 image (s = 2^-12).
"""
import hashlib
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle.pyoracle import Ref  # noqa: E402
from paper_2101_08458_b200.workloads import (cast_f16_tdsl, conv2d_nhwc_tdsl,  # noqa: E402
                                             requant_tdsl)

# proj/tests/test_dtype.cpp:78-104 (inputs only; expected bits come from the reference)
F16_INPUTS = [0.0, -0.0, 1.0, -1.0, 2.0, 65504.0, 65520.0, 65519.999, -65520.0, 0.1, 1.0 / 3.0,
              2048.5, 2049.0, 2050.0, 5.960464477539063e-08, 2.9802322387695312e-08,
              2.980232238769532e-08, 6.103515625e-05, 6.097555160522461e-05, 1e-10, -1e-10, 1.5,
              0.5005, 3.0000000001, 1024.03125, float("inf"), float("-inf")]
# proj/tests/test_dtype.cpp:138-155 operand pairs
F16_MUL = [(1.0009765625, 1.0009765625), (0.0999755859375, 0.199951171875),
           (123.375, 0.01000213623046875), (300.0, 300.0), (-2.5, 3.30078125)]


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def f16_vectors():
    L = Ref.lib()
    bits = np.array([L.tzcref_f64_to_f16_bits(x) for x in F16_INPUTS], np.uint16)
    prod = np.array([L.tzcref_f64_to_f16_bits(a * b) for a, b in F16_MUL], np.uint16)
    np.savez(os.path.join(HERE, "f16_vectors.npz"), inputs=np.array(F16_INPUTS), bits=bits,
             mul_a=np.array([a for a, _ in F16_MUL]), mul_b=np.array([b for _, b in F16_MUL]), mul_bits=prod)


def known_answers():
    out = {}
    mm2 = ("tensor A : i8 [2, 2] input\ntensor B : i8 [2, 2] input\ntensor C : i32 [2, 2] output\n"
           "loop x : dp 2\nloop y : dp 2\nloop k : red 2\nC[x, y] += cast<i32>(A[x, k]) * cast<i32>(B[k, y])\n")
    A = np.array([[1, 2], [3, 4]], np.int8)
    B = np.array([[5, 6], [7, 8]], np.int8)
    out["mm2_zero_seed"] = Ref.eval_reference(mm2, {"A": A, "B": B, "C": np.zeros((2, 2), np.int32)})
    out["mm2_seeded"] = Ref.eval_reference(mm2, {"A": A, "B": B,
                                                 "C": np.array([[100, 200], [300, 400]], np.int32)})
    wrap = ("tensor A : i32 [1, 2] input\ntensor C : i32 [1] output\nloop i : dp 1\nloop k : red 2\n"
            "C[i] += A[i, k] * 2000000000\n")
    out["i32_wrap"] = Ref.eval_reference(wrap, {"A": np.array([[2, 2]], np.int32), "C": np.zeros(1, np.int32)})
    trunc = ("tensor A : fp32 [4] input\ntensor C : i32 [4] output\nloop i : dp 4\n"
             "C[i] = cast<i32>(A[i] * 1.0)\n")
    out["f2i_trunc"] = Ref.eval_reference(trunc, {"A": np.array([2.9, -2.9, 0.4, -0.4], np.float32)})
    # test_smoke.py:31-40: c0 + a @ b.T for the int8 matmul layout
    rng = np.random.default_rng(7)
    a = rng.integers(0, 256, size=(8, 12)).astype(np.uint8)
    b = rng.integers(-128, 128, size=(5, 12)).astype(np.int8)
    c0 = rng.integers(-1000, 1000, size=(8, 5)).astype(np.int32)
    out["smoke_a"], out["smoke_b"], out["smoke_c0"] = a, b, c0
    out["smoke_out"] = Ref.eval_reference(Ref.matmul_tdsl(8, 5, 12), {"A": a, "B": b, "C": c0})
    np.savez(os.path.join(HERE, "known_answers.npz"), **out)


SEEDED = [
    ("mm_i8_64x48x96", lambda: Ref.matmul_tdsl(64, 48, 96), 1000),
    ("mm_i8_128x64x256", lambda: Ref.matmul_tdsl(128, 64, 256), 1001),
    ("mm_f16_16x24x40", lambda: Ref.matmul_tdsl(16, 24, 40, fp16=True), 3),
    ("mm_f16_32x64x48", lambda: Ref.matmul_tdsl(32, 64, 48, fp16=True), 4),
    ("conv_blk_i8_16x10x32_r3", lambda: Ref.conv2d_tdsl(16, 10, 32, 3, 1, 16, 4), 7),
    ("conv_blk_i8_64x12x64_r3s2", lambda: Ref.conv2d_tdsl(64, 12, 64, 3, 2, 16, 4), 8),
    ("conv_blk_i8_kc_64x8x128_r3", lambda: Ref.conv2d_tdsl(64, 8, 128, 3, 1, 128, 64), 9),
    ("conv_blk_f16_16x8x16_r3s2", lambda: Ref.conv2d_tdsl(16, 8, 16, 3, 2, 16, 4, fp16=True), 5),
    ("conv_nhwc_i8_n2_h8_c64_k64_r3", lambda: conv2d_nhwc_tdsl(2, 8, 8, 64, 64, 3, 3, 1), 11),
    ("conv_nhwc_i8_n1_h9_c128_k64_r3s2", lambda: conv2d_nhwc_tdsl(1, 9, 9, 128, 64, 3, 3, 2), 12),
    ("conv_nhwc_i8_n2_h6_c256_k128_r1", lambda: conv2d_nhwc_tdsl(2, 6, 6, 256, 128, 1, 1, 1), 13),
    ("conv_nhwc_i8_n1_h13_c3_k64_r7s2", lambda: conv2d_nhwc_tdsl(1, 13, 13, 3, 64, 7, 7, 2), 14),
    ("conv_nhwc_f16_n2_h6_c64_k32_r3", lambda: conv2d_nhwc_tdsl(2, 6, 6, 64, 32, 3, 3, 1, fp16=True), 15),
    ("requant_i8_4096_s2m12", lambda: requant_tdsl((64, 64), 2.0 ** -12), 21),
    ("requant_i8_4096_s0p0123", lambda: requant_tdsl((64, 64), 0.0123), 22),
    ("requant_i8_4096_s1", lambda: requant_tdsl((64, 64), 1.0), 23),
    ("cast_f16_4096", lambda: cast_f16_tdsl((64, 64)), 24),
]


def seeded():
    out = {}
    for name, mk, seed in SEEDED:
        t = mk()
        ins = Ref.random_inputs(t, seed)
        out[name + "__text"] = np.array(t)
        out[name + "__seed"] = np.array(seed)
        out[name + "__out"] = Ref.eval_reference(t, ins)
        print(name, out[name + "__out"].shape, flush=True)
    np.savez_compressed(os.path.join(HERE, "seeded.npz"), **out)


def c1():
    t = Ref.conv2d_tdsl(64, 56, 64, 3, 1, 16, 4)
    ins = Ref.random_inputs(t, 1000)
    t0 = time.time()
    out = Ref.eval_reference(t, ins)
    dt = time.time() - t0
    q = Ref.eval_reference(requant_tdsl(out.shape, 2.0 ** -12, src="C", dst="Q"), {"C": out})
    idx = np.random.default_rng(0).integers(0, out.size, size=4096)
    np.savez(os.path.join(HERE, "c1.npz"), text=np.array(t), seed=np.array(1000), sha_i32=np.array(sha(out)),
             sha_i8=np.array(sha(q)), sample_idx=idx, sample_i32=out.ravel()[idx], sample_i8=q.ravel()[idx],
             ref_seconds=np.array(dt))
    print("c1", out.shape, f"{dt:.1f}s")


if __name__ == "__main__":
    assert Ref.available(), "build oracle/_ref first (make -C oracle ref)"
    f16_vectors()
    known_answers()
    seeded()
    if "--no-c1" not in sys.argv:
        c1()
