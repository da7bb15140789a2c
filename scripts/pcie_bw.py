"""PCIe copy rates of the box (development aid): pinned 1 GB H2D alone, D2H
alone, and both at once on two streams (GB/s per direction)."""
import time

import torch

n = 256 * 1024 * 1024  # 1 GiB of fp32
h1 = torch.empty(n, pin_memory=True)
h2 = torch.empty(n, pin_memory=True)
d1 = torch.empty(n, device="cuda")
d2 = torch.empty(n, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def t(fn, k=5):
    fn()
    torch.cuda.synchronize()
    a = time.perf_counter()
    for _ in range(k):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - a) / k


def both():
    with torch.cuda.stream(s1):
        d1.copy_(h1, non_blocking=True)
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)


gb = n * 4 / 1e9
h2d = t(lambda: d1.copy_(h1, non_blocking=True))
d2h = t(lambda: h2.copy_(d2, non_blocking=True))
bo = t(both)
print(f"H2D {gb / h2d:.1f} GB/s, D2H {gb / d2h:.1f} GB/s, concurrent {gb / bo:.1f} GB/s each "
      f"({2 * gb / bo:.1f} aggregate)")
