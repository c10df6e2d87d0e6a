"""Config-3 PGA it/s (200 iterations, tol 1e-300) and the final iterate's relative difference
from a saved reference iterate (pass --save to write it)."""
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
iters = 200
for rep in range(2):
    cfg = L.CompletionConfig(spec=spec, tol=1e-300, max_iters=iters)
    mu0 = cfg.nu * L.fro_norm(np.asarray(m, dtype=np.float64))
    mus, ts, betas = pga_schedule(cfg, mu0)
    s = PGASolver(np.asarray(m, dtype=np.float64), mask, spec, "fp32")
    nat.sync()
    t0 = time.perf_counter()
    k = 1
    while k <= iters:
        n = min(50, iters - k + 1)
        recs, _ = s.run(k, betas[k - 1:k - 1 + n], mus[k - 1:k - 1 + n], cfg.tol)
        k += len(recs)
    nat.sync()
    dt = time.perf_counter() - t0
    x = s.fetch(False)
    s.close()
    print(f"rep {rep}: {iters / dt:7.1f} it/s", flush=True)
out = ROOT / "gpurun_out" / "pga_x_ref.npy"
if "--save" in sys.argv:
    np.save(out, x)
elif out.exists():
    r = np.load(out)
    print("rel diff vs saved iterate:", np.linalg.norm(x - r) / np.linalg.norm(r))
