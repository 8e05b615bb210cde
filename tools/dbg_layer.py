import sys, numpy as np, torch
sys.path.insert(0, '.')
from oracle.pyoracle import Orc
from paper_2101_08458_b200 import device as D
from paper_2101_08458_b200.workloads import RESNET50_V15, requant_scale
dev = torch.device("cuda:0")
names = sys.argv[1].split(",")
for name in names:
    L = next(x for x in RESNET50_V15 if x.name == name)
    for nb in (32, 64, 128, 256):
        for opts in ({}, {"ws_epi_groups": 2}, {"shifted_window": 0}):
            for k, v in opts.items(): D.set_option(k, v)
            g = torch.Generator(device=dev); g.manual_seed(7)
            x = torch.randint(0, 256, (nb, L.h, L.h, L.c), dtype=torch.uint8, device=dev, generator=g)
            w = torch.randint(-128, 128, (L.k, L.r, L.r, L.c), dtype=torch.int8, device=dev, generator=g)
            d, _ = D.conv_desc(tuple(x.shape), tuple(w.shape), L.stride)
            plan = D.plan_conv(d)
            out = D.conv2d(x, w, L.stride).cpu().numpy()
            s = requant_scale(L.c * L.r * L.r)
            q = D.conv2d(x, w, L.stride, epilogue="requant_i8", scale=s).cpu().numpy()
            xn, wn = x.cpu().numpy(), w.cpu().numpy()
            res = []
            for img in (0, nb // 2, nb - 1):
                ref = Orc.conv2d_nhwc(xn[img:img+1], wn, L.stride)
                res.append((img, int((out[img:img+1] != ref).sum()), int((q[img:img+1] != Orc.requant_i8(ref, s)).sum())))
            print(name, nb, opts, plan["bm"], plan["a_mode"], plan["grid"], res, flush=True)
            for k in opts: D.set_option(k, {"ws_epi_groups": 0, "shifted_window": 1}[k])
