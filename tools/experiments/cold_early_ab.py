"""Config-5 svt (public API, n = 128) and singular values with the cold QR-path early stop
off / on: device time of the K3 launch, sweeps per slice and the result's difference."""
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
a = np.random.default_rng(0).standard_normal((128, 128, 4, 8, 16), dtype=np.float32)
spec = L.make_spec("dct", a.shape)
res = {}
for early in (0.0, 1.0, 0.0, 1.0):
    lib.ltb_debug_set_qr_early(early)
    L.svt(a, 0.9124689, spec)
    nat.sync()
    nat.jacobi_stats(reset=True)
    t0 = time.perf_counter()
    out = L.svt(a, 0.9124689, spec)
    dt = time.perf_counter() - t0
    sl, sw = nat.jacobi_stats(reset=True)
    sv = L.ranks(a, spec)
    res[early] = out
    print(f"early {early}: svt API {dt * 1e3:.2f} ms, sweeps/slice {sw / max(sl, 1):.2f}", flush=True)
print("rel diff", np.linalg.norm(res[1.0] - res[0.0]) / np.linalg.norm(res[0.0]))
lib.ltb_debug_set_qr_early(1.0)
