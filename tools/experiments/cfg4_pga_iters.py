"""Config-4 PGA (1024x1024x3x64, Q (x) DFT64, complex64 transform domain): wall time and blocked-Jacobi
sweeps of each of the 50 iterations (carried complex SVT), then the per-kernel device time (CUPTI)
of the `W` iterations that follow (argv[3] == "ncu": those iterations between cudaProfilerStart / Stop
instead, for `ncu --profile-from-start off`)."""
import sys
import time
from collections import defaultdict
from pathlib import Path
import numpy as np
import torch
ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import paper_2202_02870_b200 as L  # noqa: E402
from paper_2202_02870_b200 import _native as nat  # noqa: E402
from paper_2202_02870_b200.completion import PGASolver, pga_schedule  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 50
W = int(sys.argv[2]) if len(sys.argv) > 2 else 2
rng = np.random.default_rng(0)
q, _ = np.linalg.qr(rng.standard_normal((3, 3)))
a4 = rng.standard_normal((1024, 20, 3, 64), dtype=np.float32)
b4 = rng.standard_normal((20, 1024, 3, 64), dtype=np.float32)
spec = L.make_spec("explicit", (1024, 1024, 3, 64), matrices={3: q, 4: L.build_fourier_matrix(64)})
m = L.l_product(a4, b4, spec)
mask = rng.random(m.shape) < 0.3
cfg = L.CompletionConfig(spec=spec, tol=1e-300, max_iters=N + W)
mu0 = cfg.nu * L.fro_norm(np.asarray(m, dtype=np.float64))
mus, ts, betas = pga_schedule(cfg, mu0)
s = PGASolver(np.asarray(m, dtype=np.float64), mask, spec, "fp32")
total = 0.0
for k in range(1, N + 1):
    nat.jacobi_stats(reset=True)
    t0 = time.perf_counter()
    s.run(k, betas[k - 1:k], mus[k - 1:k], cfg.tol)
    nat.sync()
    dt = time.perf_counter() - t0
    total += dt
    sl, sw = nat.jacobi_stats(reset=True)
    print(f"iteration {k:3d}: {dt * 1e3:8.1f} ms  slices {sl} sweeps {sw} ({sw / max(sl, 1):.2f} per slice)  mu {mus[k - 1]:.4g}",
          flush=True)
print(f"{N} iterations: {total:.2f} s = {N / total:.3f} it/s", flush=True)
if len(sys.argv) > 3 and sys.argv[3] == "ncu":
    # under `ncu --profile-from-start off`: only the last W iterations are visible to the profiler
    torch.cuda.profiler.start()
    s.run(N + 1, betas[N:N + W], mus[N:N + W], cfg.tol)
    nat.sync()
    torch.cuda.profiler.stop()
    s.close()
    sys.exit(0)
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    s.run(N + 1, betas[N:N + W], mus[N:N + W], cfg.tol)
    nat.sync()
s.close()
tot, cnt = defaultdict(float), defaultdict(int)
for e in prof.events():
    if e.device_type == torch.autograd.DeviceType.CUDA:
        tot[e.name] += e.device_time_total
        cnt[e.name] += 1
allt = sum(tot.values())
for name, t in sorted(tot.items(), key=lambda x: -x[1])[:16]:
    print(f"{t / W / 1e3:9.1f} ms/it {100 * t / allt:5.1f}%  x{cnt[name] // W:<4d} {name[:110]}")
