"""One launch (after one warm-up) of every kernel family the benchmarks time,
for an ncu --set full capture (tools/ncu_families.sh): the batch-256 int8
suite's representative layers, the 4096^3 int8 GEMM (configs[1]) and fp16
layers (configs[3]).  Prints the plan of each."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2101_08458_b200 import device as D  # noqa: E402
from paper_2101_08458_b200.workloads import RESNET50_V15, requant_scale  # noqa: E402

I8 = ["stem7x7", "c2_1x1_64_64", "c2_3x3_64", "c2_1x1_64_256", "c2_1x1_256_64", "c3_1x1_256_128", "c3_3x3s2_128",
      "c3_3x3_128", "c4_3x3_256", "c5_1x1_512_2048", "c4_1x1s2_512_1024"]
F16 = ["stem7x7", "c4_3x3_256", "c2_1x1_64_256"]
dev = torch.device("cuda:0")
g = torch.Generator(device=dev)
g.manual_seed(0)
sel = sys.argv[1:] or ["all"]


def run(name, f16, batch):
    L = next(x for x in RESNET50_V15 if x.name == name)
    if f16:
        x = torch.rand((batch, L.h, L.h, L.c), device=dev, generator=g).half()
        w = torch.rand((L.k, L.r, L.r, L.c), device=dev, generator=g).half()
        kw = dict(epilogue="f16")
    else:
        x = torch.randint(0, 256, (batch, L.h, L.h, L.c), dtype=torch.uint8, device=dev, generator=g)
        w = torch.randint(-128, 128, (L.k, L.r, L.r, L.c), dtype=torch.int8, device=dev, generator=g)
        kw = dict(epilogue="requant_i8", scale=requant_scale(L.c * L.r * L.r))
    d, _ = D.conv_desc(tuple(x.shape), tuple(w.shape), L.stride, f16=f16)
    print(("f16 " if f16 else "i8  ") + name, D.plan_conv(d), flush=True)
    for _ in range(2):
        D.conv2d(x, w, L.stride, **kw)
    torch.cuda.synchronize()


for n in sel:  # explicit layer names
    if any(L.name == n for L in RESNET50_V15):
        run(n, False, 256)
if "suite" in sel:  # all 23 layers of the timed step, in suite order
    for L in RESNET50_V15:
        run(L.name, False, 256)
if "all" in sel or "i8" in sel:
    for n in I8:
        run(n, False, 256)
if "all" in sel or "gemm" in sel:
    A = torch.randint(0, 256, (4096, 4096), dtype=torch.uint8, device=dev, generator=g)
    B = torch.randint(-128, 128, (4096, 4096), dtype=torch.int8, device=dev, generator=g)
    for _ in range(2):
        D.gemm(A, B, epilogue="requant_i8", scale=2.0 ** -14)
    torch.cuda.synchronize()
    print("gemm4096 done", flush=True)
if "all" in sel or "f16" in sel:
    for n in F16:
        run(n, True, 64)
print("ok")
