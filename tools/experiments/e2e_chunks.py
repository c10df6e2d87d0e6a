"""End-to-end l_product (pinned host buffers) vs the number of pipelined row chunks; raw link rates."""
import sys
import time
from pathlib import Path
import numpy as np
import torch
ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import paper_2202_02870_b200 as L  # noqa: E402
from paper_2202_02870_b200 import _native as nat  # noqa: E402

rng = np.random.default_rng(0)
a = torch.empty((256, 128, 3, 32), dtype=torch.float32, pin_memory=True).numpy()
b = torch.empty((128, 256, 3, 32), dtype=torch.float32, pin_memory=True).numpy()
c = torch.empty((256, 256, 3, 32), dtype=torch.float32, pin_memory=True).numpy()
a[...] = rng.standard_normal(a.shape)
b[...] = rng.standard_normal(b.shape)
spec = L.make_spec("dct", (256, 256, 3, 32))
d = torch.empty(c.size, dtype=torch.float32, device="cuda")
for name, fn in (("h2d 25MB", lambda: d.copy_(torch.from_numpy(c.reshape(-1)), non_blocking=True)),
                 ("d2h 25MB", lambda: torch.from_numpy(c.reshape(-1)).copy_(d, non_blocking=True))):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(10):
        fn()
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / 10
    print(f"{name}: {dt * 1e6:7.1f} us  {c.nbytes / dt / 1e9:6.1f} GB/s")
for ch in (1, 2, 4, 8, 16):
    nat.lib().ltb_debug_set_lprod_chunks(ch)
    ts = []
    for i in range(15):
        t0 = time.perf_counter()
        L.l_product(a, b, spec, out=c)
        ts.append(time.perf_counter() - t0)
    print(f"chunks {ch:2d}: {np.median(ts[3:]) * 1e6:8.1f} us  ({2491416576 / np.median(ts[3:]) / 1e9:7.1f} GFLOP/s)")
nat.lib().ltb_debug_set_lprod_chunks(8)
