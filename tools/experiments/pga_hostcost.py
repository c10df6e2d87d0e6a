import sys, time
from pathlib import Path
import numpy as np, torch
ROOT = Path('/root/repo'); sys.path.insert(0, str(ROOT))
import bench
import paper_2202_02870_b200 as L
from paper_2202_02870_b200 import _native as nat
from paper_2202_02870_b200.completion import PGASolver, pga_schedule
m, mask = bench._cfg3_data_host()
spec = L.make_spec("dct", bench.CFG3["shape"])
cfg = L.CompletionConfig(spec=spec, tol=1e-300, max_iters=200)
mu0 = cfg.nu * L.fro_norm(np.asarray(m, dtype=np.float64))
mus, ts, betas = pga_schedule(cfg, mu0)
for carry in (1, 0):
    nat.lib().ltb_debug_set_pga_carry(carry)
    s = PGASolver(np.asarray(m, dtype=np.float64), mask, spec, "fp32")
    k = 1
    for chunk in (1, 1, 10, 10):
        nat.sync(); t0 = time.perf_counter()
        recs, _ = s.run(k, betas[k - 1:k - 1 + chunk], mus[k - 1:k - 1 + chunk], cfg.tol)
        t1 = time.perf_counter()
        k += chunk
        print(f"carry {carry} chunk {chunk}: {1e3*(t1-t0)/chunk:.3f} ms/it")
    s.close()
