"""Generate the TNSR fixtures for the device CLI's `verify` (tests/test_gpu_cli.py).

Runs the REFERENCE (oracle/_ref/libtzc_ref.so, built from /root/reference) in
this container: random_inputs(op, seed) and eval_reference(op) are written with
the reference's own save_tensor (proj/src/vm.cpp:808-818) under
tests/golden/tnsr/<case>/ as <tensor>.tnsr + expect.tnsr, next to op.tdsl.

    python tests/golden/make_tnsr.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle.pyoracle import Ref  # noqa: E402
from paper_2101_08458_b200.workloads import conv2d_nhwc_tdsl, conv2d_tdsl, conv3d_tdsl, matmul_tdsl  # noqa: E402

# case -> (op text, seed, instruction, rtol or None)
CASES = {
    "mm_i8": (matmul_tdsl(256, 128, 64), 11, "tcgen05_i8_m128n128k32", None),
    "conv_nhwc_i8": (conv2d_nhwc_tdsl(2, 10, 10, 64, 64, 3, 3, 1), 12, "tcgen05_i8_m128n64k32", None),
    "conv_blocked_i8": (conv2d_tdsl(64, 12, 64, 3), 14, "tcgen05_i8_m128n64k32", None),
    "mm_f16": (matmul_tdsl(128, 128, 64, fp16=True), 13, "tcgen05_f16_m128n128k16_mn", 1e-3),
    # conv3d_tdsl (proj/src/workloads.cpp:94-121), the resnet18-3d bank's op form
    "conv3d_i8": (conv3d_tdsl(16, 8, 32, 3), 15, "tcgen05_i8_m128n64k32", None),
    "conv3d_s2_i8": (conv3d_tdsl(16, 9, 32, 3, 2), 16, "tcgen05_i8_m128n64k32", None),
    "conv3d_f16": (conv3d_tdsl(16, 7, 16, 3, fp16=True), 17, "tcgen05_f16_m128n64k16", 1e-3),
}


def main():
    for name, (text, seed, _, _) in CASES.items():
        d = os.path.join(ROOT, "tests", "golden", "tnsr", name)
        os.makedirs(d, exist_ok=True)
        with open(os.path.join(d, "op.tdsl"), "w") as f:
            f.write(text)
        Ref.save_case(text, seed, d)
        print(name, sorted(os.listdir(d)))


if __name__ == "__main__":
    main()
