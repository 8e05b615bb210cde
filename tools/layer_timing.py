"""How much of a per-layer event time is the kernel?  For one layer at batch B:
(a) eager launch between events, (b) graph of 1 launch with external events
inside (bench graph B style), (c) graph of R launches timed from outside
(per-launch = total / R, back-to-back PDL launches), each after an L2 flush.
Usage: python tools/layer_timing.py c4_3x3_256 [--batch 256] [--reps 8]"""
import argparse
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2101_08458_b200 import device as D  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("layers", nargs="+")
ap.add_argument("--batch", type=int, default=256)
ap.add_argument("--reps", type=int, default=8)
ap.add_argument("--opt", action="append", default=[], help="name=value for tzc_b200_set_option")
a = ap.parse_args()
for o in a.opt:
    k, v = o.split("=")
    D.set_option(k, int(v))
dev = torch.device("cuda:0")
gen = torch.Generator(device=dev)
gen.manual_seed(0)
layers, bufs = bench.build_suite(torch, dev, a.batch, a.layers, gen)
stream = torch.cuda.Stream()
flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
rt = bench.Cudart()
for b in bufs:
    L = b["layer"]

    def launch():
        D.conv2d(b["x"], b["w"], L.stride, epilogue="requant_i8", scale=b["scale"], out=b["out"], stream=stream)

    with torch.cuda.stream(stream):
        launch()
    torch.cuda.synchronize()
    e0, e1 = rt.event(), rt.event()
    gB = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gB, stream=stream):
        rt.record(e0, stream)
        launch()
        rt.record(e1, stream)
    gC = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gC, stream=stream):
        for _ in range(a.reps):
            launch()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    res = {"eager": [], "graph_events": [], "graph_rep": []}
    for _ in range(10):
        flush.zero_()
        torch.cuda.synchronize()
        with torch.cuda.stream(stream):
            t0.record(stream)
            launch()
            t1.record(stream)
        torch.cuda.synchronize()
        res["eager"].append(t0.elapsed_time(t1))
        flush.zero_()
        torch.cuda.synchronize()
        with torch.cuda.stream(stream):
            gB.replay()
        torch.cuda.synchronize()
        res["graph_events"].append(rt.ms(e0, e1))
        flush.zero_()
        torch.cuda.synchronize()
        with torch.cuda.stream(stream):
            t0.record(stream)
            gC.replay()
            t1.record(stream)
        torch.cuda.synchronize()
        res["graph_rep"].append(t0.elapsed_time(t1) / a.reps)
    print(L.name, {k: round(1000 * statistics.median(v), 1) for k, v in res.items()}, "us")
