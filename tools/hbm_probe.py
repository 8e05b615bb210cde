"""HBM bandwidth by direction on this GPU: write-only (fill), read-only
(reduction), copy.  Used to model write-heavy layers' rooflines."""
import torch

n = 1 << 30
x = torch.empty(n, dtype=torch.uint8, device="cuda")
y = torch.empty(n, dtype=torch.uint8, device="cuda")
x32 = x.view(torch.int32)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)


def t(f, reps=10):
    f()
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        f()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e-3


w = t(lambda: x.fill_(1))
r = t(lambda: x32.sum())
c = t(lambda: y.copy_(x))
print(f"write-only {n / w / 1e9:.0f} GB/s, read-only {n / r / 1e9:.0f} GB/s, copy {2 * n / c / 1e9:.0f} GB/s (r+w)")
