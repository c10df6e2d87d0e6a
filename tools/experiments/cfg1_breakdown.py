"""Warm per-kernel device time (CUPTI) of config-1 PGA iterations (64x64x16 float64, DCT)."""
import sys
import time
from collections import defaultdict
from pathlib import Path
import numpy as np
import torch
ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
import paper_2202_02870_b200 as L  # noqa: E402
from paper_2202_02870_b200 import _native as nat  # noqa: E402
from paper_2202_02870_b200.completion import PGASolver, pga_schedule  # noqa: E402

m, mask = bench._cfg1_data() if hasattr(bench, "_cfg1_data") else (None, None)
if m is None:
    rng = np.random.default_rng(0)
    a = rng.standard_normal((64, 5, 16)); b = rng.standard_normal((5, 64, 16))
    spec0 = L.make_spec("dct", (64, 64, 16))
    m = L.l_product(a, b, spec0)
    mask = rng.random(m.shape) < 0.5
spec = L.make_spec("dct", m.shape)
cfg = L.CompletionConfig(spec=spec, mu0=0.01, mu_bar_ratio=1.0, tol=1e-300, max_iters=100)
mus, ts, betas = pga_schedule(cfg, 0.01)
s = PGASolver(np.asarray(m, dtype=np.float64), mask, spec, "fp64")
s.run(1, betas[:50], mus[:50], cfg.tol)
nat.sync()
nat.jacobi_stats(reset=True)
t0 = time.perf_counter()
s.run(51, betas[50:60], mus[50:60], cfg.tol)
nat.sync()
print(f"10 iterations: {(time.perf_counter() - t0) * 1e3:.2f} ms; sweeps/slice", nat.jacobi_stats(reset=True))
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    s.run(61, betas[60:70], mus[60:70], cfg.tol)
    nat.sync()
tot, cnt = defaultdict(float), defaultdict(int)
for e in prof.events():
    if e.device_type == torch.autograd.DeviceType.CUDA:
        tot[e.name] += e.device_time_total
        cnt[e.name] += 1
for k, t in sorted(tot.items(), key=lambda x: -x[1])[:8]:
    print(f"   {t / 10:8.1f} us/it x{cnt[k] // 10:<3d} {k[:100]}")
