"""Warm per-kernel device time of late config-3 PGA iterations (CUPTI via torch.profiler):
run K iterations, then profile W more and print each kernel's total / per-iteration time."""
import sys
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

K = int(sys.argv[1]) if len(sys.argv) > 1 else 120
W = int(sys.argv[2]) if len(sys.argv) > 2 else 5
PREC = sys.argv[3] if len(sys.argv) > 3 else "fp32"  # "fp64": the reference's precision
m, mask = bench._cfg3_data_host()
spec = L.make_spec("dct", bench.CFG3["shape"])
cfg = L.CompletionConfig(spec=spec, tol=1e-300, max_iters=K + W)
mu0 = cfg.nu * L.fro_norm(np.asarray(m, dtype=np.float64))
mus, ts, betas = pga_schedule(cfg, mu0)
s = PGASolver(np.asarray(m, dtype=np.float64), mask, spec, PREC)
s.run(1, betas[:K], mus[:K], cfg.tol)
nat.sync()
nat.jacobi_stats(reset=True)
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    s.run(K + 1, betas[K:K + W], mus[K:K + W], cfg.tol)
    nat.sync()
s.close()
tot = defaultdict(float)
cnt = defaultdict(int)
for e in prof.events():
    if e.device_type == torch.autograd.DeviceType.CUDA:
        tot[e.name] += e.device_time_total if hasattr(e, "device_time_total") else e.cuda_time_total
        cnt[e.name] += 1
allt = sum(tot.values())
print(f"{W} {PREC} iterations from {K + 1}: kernel time {allt / W:.1f} us per iteration; Jacobi (slices, sweeps[, max]) {nat.jacobi_stats(reset=True, with_max=True)}")
for name, t in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"{t / W:9.1f} us/it {100 * t / allt:5.1f}%  x{cnt[name] // W:<3d} {name[:110]}")
