"""Time the tcgen05 GEMM path over a shape sweep (eager, CUDA events).
Usage: python tools/gemm_sweep.py [MxNxK ...]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2101_08458_b200 import device as D  # noqa: E402
from paper_2101_08458_b200._capi import GemmDesc  # noqa: E402

dev = torch.device("cuda:0")
shapes = [(128, 256, 128), (128, 256, 4096), (148 * 128, 256, 128), (148 * 128, 256, 1024),
          (4096, 4096, 4096), (8192, 8192, 8192), (100352, 256, 64), (100352, 64, 64)]
if len(sys.argv) > 1:
    shapes = [tuple(int(v) for v in s.split("x")) for s in sys.argv[1:]]
for (m, n, k) in shapes:
    a = torch.randint(0, 256, (m, k), dtype=torch.uint8, device=dev)
    b = torch.randint(-128, 128, (n, k), dtype=torch.int8, device=dev)
    out = torch.empty((m, n), dtype=torch.int8, device=dev)
    for _ in range(3):
        D.gemm(a, b, epilogue="requant_i8", scale=2.0 ** -14, out=out)
    torch.cuda.synchronize()
    reps = 20
    # capture the repetitions in a CUDA graph so host launch cost is excluded
    st = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        for _ in range(reps):
            D.gemm(a, b, epilogue="requant_i8", scale=2.0 ** -14, out=out, stream=st)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = __import__("time").perf_counter()
    e0.record()
    for _ in range(reps):
        D.gemm(a, b, epilogue="requant_i8", scale=2.0 ** -14, out=out)
    e1.record()
    host_us = (__import__("time").perf_counter() - t0) / reps * 1e6
    torch.cuda.synchronize()
    eager_ms = e0.elapsed_time(e1) / reps
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(f"   eager {eager_ms*1e3:.1f} us/launch (host {host_us:.1f} us/call)")
    tops = 2 * m * n * k / (ms * 1e-3) / 1e12
    gbs = (m * k + n * k + m * n) / (ms * 1e-3) / 1e9
    d = GemmDesc(profile=0, m=m, n=n, k=k, b_kn=0)
    d.out = D.nhwc_layout(n)
    print(f"{m}x{n}x{k}: {ms*1e3:9.1f} us {tops:8.1f} TOPS {gbs:8.1f} GB/s plan={D.plan_gemm(d)}", flush=True)
