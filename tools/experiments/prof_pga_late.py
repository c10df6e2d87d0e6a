"""Config-3 PGA: run the first K iterations, then a profiled window of W iterations
(cudaProfilerStart/Stop; use ncu --profile-from-start off)."""
import sys
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
Wn = int(sys.argv[2]) if len(sys.argv) > 2 else 3
m, mask = bench._cfg3_data_host()
spec = L.make_spec("dct", bench.CFG3["shape"])
cfg = L.CompletionConfig(spec=spec, tol=1e-300, max_iters=K + Wn)
mu0 = cfg.nu * L.fro_norm(np.asarray(m, dtype=np.float64))
mus, ts, betas = pga_schedule(cfg, mu0)
s = PGASolver(np.asarray(m, dtype=np.float64), mask, spec, "fp32")
s.run(1, betas[:K], mus[:K], cfg.tol)
nat.sync()
torch.cuda.profiler.start()
s.run(K + 1, betas[K:K + Wn], mus[K:K + Wn], cfg.tol)
nat.sync()
torch.cuda.profiler.stop()
s.close()
print("done")
