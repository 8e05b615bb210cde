"""Pinned host<->device copy bandwidth on this box: H2D alone, D2H alone, and
both directions concurrently (the e2e leg's ceiling)."""
import torch


def bw(fn, nbytes, it=10):
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(it):
        fn()
    e.record()
    torch.cuda.synchronize()
    return nbytes * it / (s.elapsed_time(e) * 1e-3) / 1e9


def main():
    n = 1 << 30
    h1 = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    h2 = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    d1 = torch.empty(n, dtype=torch.uint8, device="cuda")
    d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    print("h2d GB/s", round(bw(lambda: d1.copy_(h1, non_blocking=True), n), 1))
    print("d2h GB/s", round(bw(lambda: h2.copy_(d2, non_blocking=True), n), 1))

    def both():
        cur = torch.cuda.current_stream()
        s1.wait_stream(cur)
        s2.wait_stream(cur)
        with torch.cuda.stream(s1):
            d1.copy_(h1, non_blocking=True)
        with torch.cuda.stream(s2):
            h2.copy_(d2, non_blocking=True)
        cur.wait_stream(s1)
        cur.wait_stream(s2)
    print("bidir GB/s per direction", round(bw(both, n), 1))
    for mb in (4, 16, 64):
        m = mb << 20
        print(f"h2d {mb} MiB chunks GB/s", round(bw(lambda: d1[:m].copy_(h1[:m], non_blocking=True), m, 100), 1))


if __name__ == "__main__":
    main()
