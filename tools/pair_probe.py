"""Per-kernel tensor-pipe probe: single-wave and multi-wave GEMMs and deep-K
convs with the 1-SM (BN=256) and CTA-pair (cta_group::2, 256 x BN) kernels.
Run under ncu --metrics (tools/pair_probe.sh)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2101_08458_b200 import device as D  # noqa: E402
from paper_2101_08458_b200.workloads import RESNET50_V15, requant_scale  # noqa: E402

dev = torch.device("cuda:0")
g = torch.Generator(device=dev)
g.manual_seed(0)
for pair in (0, 1):
    D.set_option("pair", pair)
    D.set_option("pair_min_kb", 1 if pair else 16)
    for (m, n, k) in [(148 * 128, 256, 4096), (4096, 4096, 4096), (148 * 128, 256, 512)]:
        A = torch.randint(0, 256, (m, k), dtype=torch.uint8, device=dev, generator=g)
        B = torch.randint(-128, 128, (n, k), dtype=torch.int8, device=dev, generator=g)
        for _ in range(2):
            D.gemm(A, B, epilogue="requant_i8", scale=2.0 ** -14)
        torch.cuda.synchronize()
        print("pair", pair, "gemm", m, n, k, flush=True)
    for name in ("c4_3x3_256", "c5_3x3_512", "c3_3x3s2_128", "c4_1x1s2_512_1024"):
        L = next(x for x in RESNET50_V15 if x.name == name)
        x = torch.randint(0, 256, (256, L.h, L.h, L.c), dtype=torch.uint8, device=dev, generator=g)
        w = torch.randint(-128, 128, (L.k, L.r, L.r, L.c), dtype=torch.int8, device=dev, generator=g)
        D.set_option("shifted_window", 0)
        for _ in range(2):
            D.conv2d(x, w, L.stride, epilogue="requant_i8", scale=requant_scale(L.c * L.r * L.r))
        torch.cuda.synchronize()
        D.set_option("shifted_window", 1)
        print("pair", pair, name, flush=True)
