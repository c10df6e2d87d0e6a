"""Config-3 PGA it/s with the fp32 SVT right-basis carry on / off (late-iteration thresholds)."""
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
for k0, iters in ((1, 200), (150, 20)):
    for qr in (0, 1):
        nat.lib().ltb_debug_set_pga_carry(qr)
        cfg = L.CompletionConfig(spec=spec, tol=1e-300, max_iters=iters + k0 - 1)
        mu0 = cfg.nu * L.fro_norm(np.asarray(m, dtype=np.float64))
        mus, ts, betas = pga_schedule(cfg, mu0)
        s = PGASolver(np.asarray(m, dtype=np.float64), mask, spec, "fp32")
        nat.sync()
        nat.jacobi_stats(reset=True)
        t0 = time.perf_counter()
        k = 1
        while k <= iters:
            n = min(50, iters - k + 1)
            recs, _ = s.run(k, betas[k0 - 2 + k:k0 - 2 + k + n], mus[k0 - 2 + k:k0 - 2 + k + n], cfg.tol)
            k += len(recs)
        nat.sync()
        dt = time.perf_counter() - t0
        sl, sw = nat.jacobi_stats(reset=True)
        x = s.fetch(False)
        s.close()
        print(f"k0={k0} iters={iters} carry={qr}: {iters / dt:7.1f} it/s  sweeps/slice {sw / max(sl, 1):.2f}  |x| {np.linalg.norm(x):.6e}")
nat.lib().ltb_debug_set_pga_carry(1)
