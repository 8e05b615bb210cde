import numpy as np, torch, sys
sys.path.insert(0, '.')
from oracle.pyoracle import Orc
from paper_2101_08458_b200 import device as D
cuda = torch.device('cuda:0')
D.set_option("pair", 1)
m, n, k = 1000, 256, 512
a = Orc.random_tensor("u8", (m, k), 500); b = Orc.random_tensor("i8", (n, k), 501)
want = Orc.requant_i8(Orc.matmul(a, b), 2.0 ** -12)
got = D.gemm(torch.from_numpy(a).to(cuda), torch.from_numpy(b).to(cuda), epilogue="requant_i8", scale=2.0 ** -12).cpu().numpy()
print("pair gemm ok", np.array_equal(got, want), (got != want).mean())
