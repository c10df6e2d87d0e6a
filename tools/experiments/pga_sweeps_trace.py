"""Per-iteration Jacobi sweeps of the config-3 PGA (carried right bases vs cold), from iteration k0."""
import sys
import time
from pathlib import Path
import numpy as np
ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
import paper_2202_02870_b200 as L  # noqa: E402
from paper_2202_02870_b200 import _native as nat  # noqa: E402
from paper_2202_02870_b200.completion import PGASolver, pga_schedule  # noqa: E402

k0 = int(sys.argv[1]) if len(sys.argv) > 1 else 1
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 12
m, mask = bench._cfg3_data_host()
spec = L.make_spec("dct", bench.CFG3["shape"])
cfg = L.CompletionConfig(spec=spec, tol=1e-300, max_iters=200)
mu0 = cfg.nu * L.fro_norm(np.asarray(m, dtype=np.float64))
mus, ts, betas = pga_schedule(cfg, mu0)
for carry in (1, 0):
    nat.lib().ltb_debug_set_pga_carry(carry)
    s = PGASolver(np.asarray(m, dtype=np.float64), mask, spec, "fp32")
    out, ms = [], []
    for k in range(1, iters + 1):
        nat.jacobi_stats(reset=True)
        nat.sync()
        t0 = time.perf_counter()
        s.run(k, betas[k0 + k - 2:k0 + k - 1], mus[k0 + k - 2:k0 + k - 1], cfg.tol)
        nat.sync()
        ms.append(round((time.perf_counter() - t0) * 1e3, 2))
        sl, sw, mx = nat.jacobi_stats(reset=True, with_max=True)
        out.append((round(sw / max(sl, 1), 2), mx))
    s.close()
    print("carry", carry, "sweeps", out[:8], "...", out[-8:])
    seg = [(1, 14), (15, 49), (50, 60), (61, 120), (121, iters)]
    print("carry", carry, "ms per iteration by range", [(a, b, round(float(np.mean(ms[a - 1:b])), 2)) for a, b in seg if b <= iters],
          "total", round(sum(ms), 1))
nat.lib().ltb_debug_set_pga_carry(1)
