import sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
from oracle.pyoracle import Orc
from paper_2101_08458_b200 import device as D
from tests.gpu_helpers import to_dev
cuda = torch.device('cuda:0')
mode = sys.argv[1]
n, hp, c, k, r = 3, 58, 64, 64, 3
x = Orc.random_tensor("u8", (n, hp, hp, c), 300)
w = Orc.random_tensor("i8", (k, r, r, c), 301)
if mode == 'raw':
    out = D.conv2d(to_dev(x, cuda), to_dev(w, cuda), 1)
else:
    out = D.conv2d(to_dev(x, cuda), to_dev(w, cuda), 1, epilogue="requant_i8", scale=2.0**-12)
torch.cuda.synchronize()
print(mode, 'ok', D.plan_conv(D.conv_desc(tuple(x.shape), tuple(w.shape), 1)[0]))
