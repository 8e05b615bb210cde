"""Run selected ResNet-50 suite layers eagerly a few times (for ncu captures).
Usage: python tools/run_layer.py c5_3x3_512 [c2_1x1_64_256 ...] [--iters 3] [--batch 32]"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2101_08458_b200 import device as D  # noqa: E402
from paper_2101_08458_b200.workloads import RESNET50_V15, requant_scale  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("layers", nargs="+")
ap.add_argument("--iters", type=int, default=3)
ap.add_argument("--batch", type=int, default=32)
ap.add_argument("--splits", type=int, default=0)
a = ap.parse_args()
dev = torch.device("cuda:0")
D.set_splits(a.splits)
g = torch.Generator(device=dev)
g.manual_seed(0)
for name in a.layers:
    L = next(x for x in RESNET50_V15 if x.name == name)
    x = torch.randint(0, 256, (a.batch, L.h, L.h, L.c), dtype=torch.uint8, device=dev, generator=g)
    w = torch.randint(-128, 128, (L.k, L.r, L.r, L.c), dtype=torch.int8, device=dev, generator=g)
    d, _ = D.conv_desc(tuple(x.shape), tuple(w.shape), L.stride)
    print(name, D.plan_conv(d) if L.c % 64 == 0 else "k7")
    for _ in range(a.iters):
        D.conv2d(x, w, L.stride, epilogue="requant_i8", scale=requant_scale(L.c * L.r * L.r))
    torch.cuda.synchronize()
print("ok")
