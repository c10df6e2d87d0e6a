"""Carried-basis SVT rotation threshold: PGA it/s on config 3 (200 iterations) and the fp32
iterate's distance to the fp64 device path (validated against the oracle) at each scale."""
import ctypes as C
import sys
import time
from pathlib import Path
import numpy as np
ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tests")); sys.path.insert(0, str(ROOT / "oracle"))
import bench  # noqa: E402
import paper_2202_02870_b200 as L  # noqa: E402
from paper_2202_02870_b200 import _native as nat  # noqa: E402
from conftest import rel_err  # noqa: E402

lib = nat.lib()
lib.ltb_debug_set_carry_tol_scale.argtypes = [C.c_float]
m, mask = bench._cfg3_data_host()
spec = L.make_spec("dct", bench.CFG3["shape"])
cfg = L.CompletionConfig(spec=spec, tol=1e-300, max_iters=200)
ref, _ = L.pga_complete(m.astype(np.float64), mask, cfg, precision="fp64")
for sc in [float(v) for v in sys.argv[1:]] or [1.0, 10.0, 100.0, 1000.0]:
    lib.ltb_debug_set_carry_tol_scale(sc)
    L.pga_complete(m, mask, L.CompletionConfig(spec=spec, tol=1e-300, max_iters=5), precision="fp32")
    nat.jacobi_stats(reset=True)
    t0 = time.perf_counter()
    x, tr = L.pga_complete(m, mask, cfg, precision="fp32")
    dt = time.perf_counter() - t0
    sl, sw = nat.jacobi_stats(reset=True)
    print(f"tol x{sc:g}: {200 / dt:.1f} it/s (incl. host setup), sweeps/slice {sw / max(sl, 1):.2f}, "
          f"rel err vs fp64 path {rel_err(x, ref):.2e}", flush=True)
lib.ltb_debug_set_carry_tol_scale(1.0)
