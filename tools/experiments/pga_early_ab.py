"""Config-3 PGA (200 iterations, tol 1e-300): fp32 it/s, Jacobi sweeps and the final iterate's
relative error against the fp64 run, for several early-stop scales (x sqrt(tol)) of the carried SVT."""
import ctypes as C
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

lib = nat.lib()
lib.ltb_debug_set_carry_early.argtypes = [C.c_float]
m, mask = bench._cfg3_data_host()
spec = L.make_spec("dct", bench.CFG3["shape"])
iters = 200
cfg = L.CompletionConfig(spec=spec, tol=1e-300, max_iters=iters)
mu0 = cfg.nu * L.fro_norm(np.asarray(m, dtype=np.float64))
mus, ts, betas = pga_schedule(cfg, mu0)


def run(prec):
    s = PGASolver(np.asarray(m, dtype=np.float64), mask, spec, prec)
    nat.sync()
    nat.jacobi_stats(reset=True)
    t0 = time.perf_counter()
    k = 1
    while k <= iters:
        n = min(50, iters - k + 1)
        recs, _ = s.run(k, betas[k - 1:k - 1 + n], mus[k - 1:k - 1 + n], cfg.tol)
        k += len(recs)
    nat.sync()
    dt = time.perf_counter() - t0
    sl, sw = nat.jacobi_stats(reset=True)
    x = s.fetch(False)
    s.close()
    return x, iters / dt, sw / max(sl, 1)


ref, r64, _ = run("fp64")
print(f"fp64: {r64:.1f} it/s", flush=True)
for es in [float(v) for v in (sys.argv[1:] or ["0", "1", "2"])]:
    lib.ltb_debug_set_carry_early(es)
    run("fp32")
    x, rate, sw = run("fp32")
    print(f"early scale {es:g}: {rate:7.1f} it/s  sweeps/slice {sw:.2f}  rel err vs fp64 "
          f"{np.linalg.norm(x - ref) / np.linalg.norm(ref):.3e}", flush=True)
lib.ltb_debug_set_carry_early(1.0)
