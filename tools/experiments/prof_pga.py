"""Small profiling driver: a few PGA iterations of BASELINE config 3 (f32) through the
device solver, for ncu captures of the fused transform / Jacobi SVT kernels."""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402
import paper_2202_02870_b200 as L  # noqa: E402
from paper_2202_02870_b200.completion import PGASolver, pga_schedule  # noqa: E402

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 3
k0 = int(sys.argv[2]) if len(sys.argv) > 2 else 1  # take mu from iteration k0 on (late-iteration thresholds)
m, mask = bench._cfg3_data_host()
spec = L.make_spec("dct", bench.CFG3["shape"])
cfg = L.CompletionConfig(spec=spec, tol=1e-300, max_iters=iters + k0 - 1)
mu0 = cfg.nu * L.fro_norm(np.asarray(m, dtype=np.float64))
mus, ts, betas = pga_schedule(cfg, mu0)
s = PGASolver(np.asarray(m, dtype=np.float64), mask, spec, "fp32")
recs, _ = s.run(1, betas[k0 - 1:], mus[k0 - 1:], cfg.tol)
print("iterations", len(recs), "rel", recs[-1][0] ** 0.5 / max(recs[-1][1], 1e-300) ** 0.5)
s.close()
