"""Config-3 PGA (200 iterations, chunks of 50): tensor-core transforms inside PGA on / off."""
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

m, mask = bench._cfg3_data_host()
spec = L.make_spec("dct", bench.CFG3["shape"])
cfg = L.CompletionConfig(spec=spec, tol=1e-300, max_iters=200)
mu0 = cfg.nu * L.fro_norm(np.asarray(m, dtype=np.float64))
mus, ts, betas = pga_schedule(cfg, mu0)
xs = {}
for tc in (0, 1, 0, 1):
    nat.lib().ltb_debug_set_pga_tc(tc)
    s = PGASolver(np.asarray(m, dtype=np.float64), mask, spec, "fp32")
    nat.sync()
    t0 = time.perf_counter()
    k = 1
    while k <= 200:
        recs, _ = s.run(k, betas[k - 1:k + 49], mus[k - 1:k + 49], cfg.tol)
        k += len(recs)
    nat.sync()
    dt = time.perf_counter() - t0
    xs[tc] = s.fetch(False)
    s.close()
    print(f"pga_tc={tc}: {200 / dt:7.1f} it/s")
print("rel diff", np.linalg.norm(xs[0] - xs[1]) / np.linalg.norm(xs[0]))
nat.lib().ltb_debug_set_pga_tc(1)
