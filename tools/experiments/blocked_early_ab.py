"""Blocked-tier svt (config 5, n = 256 / 512, public API) with the fp32 early stop off / on:
wall time, sweeps per slice and the result's relative difference."""
import ctypes as C
import sys
import time
from pathlib import Path
import numpy as np
ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import paper_2202_02870_b200 as L  # noqa: E402
from paper_2202_02870_b200 import _native as nat  # noqa: E402

lib = nat.lib()
lib.ltb_debug_set_qr_early.argtypes = [C.c_float]
for n, tau in ((256, 1.2912667), (512, 1.826952)):
    a = np.random.default_rng(0).standard_normal((n, n, 4, 8, 16), dtype=np.float32)
    spec = L.make_spec("dct", a.shape)
    res = {}
    for early in (0.0, 1.0):
        lib.ltb_debug_set_qr_early(early)
        L.svt(a, tau, spec)
        nat.sync()
        nat.jacobi_stats(reset=True)
        t0 = time.perf_counter()
        res[early] = L.svt(a, tau, spec)
        dt = time.perf_counter() - t0
        sl, sw = nat.jacobi_stats(reset=True)
        print(f"n={n} early {early}: svt API {dt * 1e3:.1f} ms, sweeps/slice {sw / max(sl, 1):.2f}", flush=True)
    print(f"n={n} rel diff", np.linalg.norm(res[1.0] - res[0.0]) / np.linalg.norm(res[0.0]), flush=True)
lib.ltb_debug_set_qr_early(1.0)
