"""Host link: 25 MB pinned H2D alone, D2H alone, and both at once on two streams (is the
link full duplex for the e2e l_product pipeline?)."""
import time
import torch

n = 256 * 256 * 96
h1 = torch.empty(n, dtype=torch.float32, pin_memory=True)
h2 = torch.empty(n, dtype=torch.float32, pin_memory=True)
d1 = torch.empty(n, dtype=torch.float32, device="cuda")
d2 = torch.empty(n, dtype=torch.float32, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def run(kind):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(10):
        if kind in ("h2d", "both"):
            with torch.cuda.stream(s1):
                d1.copy_(h1, non_blocking=True)
        if kind in ("d2h", "both"):
            with torch.cuda.stream(s2):
                h2.copy_(d2, non_blocking=True)
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / 10


for k in ("h2d", "d2h", "both", "h2d", "d2h", "both"):
    print(f"{k:5s}: {run(k) * 1e6:7.1f} us per 25 MB (each direction)")
