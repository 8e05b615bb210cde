import os, sys
sys.path.insert(0, ".")
import numpy as np, torch
from oracle.pyoracle import Orc
from paper_2101_08458_b200 import device as D
dev = torch.device("cuda:0")
n, hp, k = int(sys.argv[1]), int(sys.argv[2]), 64
x = Orc.random_tensor("u8", (n, hp, hp, 3), 1)
w = Orc.random_tensor("i8", (k, 7, 7, 3), 2)
got = D.conv2d(torch.from_numpy(x).to(dev), torch.from_numpy(w).to(dev), 2).cpu().numpy()
ref = Orc.conv2d_nhwc(x, w, 2)
print("flags", os.environ.get("TZC_STEM_DEBUG"), "mismatches", int((got != ref).sum()), "of", ref.size, flush=True)
