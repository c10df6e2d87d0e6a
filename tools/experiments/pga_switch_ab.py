"""Config-3 PGA (200 iterations, fp32) under a libltb debug switch: it/s, sweeps per slice and
the iterate's distance to the fp64 device path.

    python tools/pga_switch_ab.py ltb_debug_set_qr_ts 16 8"""
import sys
import time
from pathlib import Path
import numpy as np
ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tests"))
import bench  # noqa: E402
import paper_2202_02870_b200 as L  # noqa: E402
from paper_2202_02870_b200 import _native as nat  # noqa: E402
from conftest import rel_err  # noqa: E402

fn = getattr(nat.lib(), sys.argv[1])
vals = [int(v) for v in sys.argv[2:]]
m, mask = bench._cfg3_data_host()
spec = L.make_spec("dct", bench.CFG3["shape"])
cfg = L.CompletionConfig(spec=spec, tol=1e-300, max_iters=200)
ref, _ = L.pga_complete(m.astype(np.float64), mask, cfg, precision="fp64")
for rep in range(2):
    for v in vals:
        fn(v)
        L.pga_complete(m, mask, L.CompletionConfig(spec=spec, tol=1e-300, max_iters=5), precision="fp32")
        nat.jacobi_stats(reset=True)
        t0 = time.perf_counter()
        x, tr = L.pga_complete(m, mask, cfg, precision="fp32")
        dt = time.perf_counter() - t0
        sl, sw = nat.jacobi_stats(reset=True)
        print(f"{sys.argv[1]}={v}: {200 / dt:.1f} it/s (API incl. host setup), sweeps/slice {sw / max(sl, 1):.2f}, "
              f"rel err vs fp64 path {rel_err(x, ref):.2e}", flush=True)
fn(vals[0])
