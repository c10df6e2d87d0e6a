"""CUPTI timeline (torch.profiler) of one end-to-end l_product call from pinned host buffers:
start / end of every copy and kernel relative to the first, per stream."""
import sys
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
import time
for ch in [8]:
    ts = []
    for _ in range(10):
        t0 = time.perf_counter(); L.l_product(a, b, spec, out=c); ts.append(time.perf_counter() - t0)
    print(f"host wall per call: median {np.median(ts) * 1e6:.1f} us, min {min(ts) * 1e6:.1f} us")
    for _ in range(3):
        L.l_product(a, b, spec, out=c)
    with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
        L.l_product(a, b, spec, out=c)
    ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
    t0 = min(e.time_range.start for e in ev)
    print(f"--- {ch} row chunks: span {(max(e.time_range.end for e in ev) - t0):.1f} us")
    for e in sorted(ev, key=lambda e: e.time_range.start):
        print(f"  {e.time_range.start - t0:8.1f} {e.time_range.end - t0:8.1f}  {e.name[:60]}")
