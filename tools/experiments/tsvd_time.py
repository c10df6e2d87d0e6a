"""Config-5 t_svd / svt through the public API (numpy in, numpy out) at n = 128, 256, 512: best of two calls,
plus the device time of ltb_slice_svd alone on the resident transform-domain stack."""
import sys
import time
from pathlib import Path
import numpy as np
ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import paper_2202_02870_b200 as L  # noqa: E402
from paper_2202_02870_b200 import _native as nat  # noqa: E402

for n in (128, 256, 512):
    rng = np.random.default_rng(0)
    a = rng.standard_normal((n, n, 4, 8, 16), dtype=np.float32)
    spec = L.make_spec("dct", a.shape)
    best = {"svt": 1e9, "t_svd": 1e9}
    for _ in range(2):
        t0 = time.perf_counter(); L.svt(a, 1.0, spec); best["svt"] = min(best["svt"], time.perf_counter() - t0)
        t0 = time.perf_counter(); f = L.t_svd(a, spec); best["t_svd"] = min(best["t_svd"], time.perf_counter() - t0)
    hat = L.linalg._hat_stack(a, spec)
    P, i1, i2 = hat.shape
    u = nat.DeviceArray((P, i1, i1), hat.dtype); v = nat.DeviceArray((P, i2, i2), hat.dtype)
    s = nat.DeviceArray((P, min(i1, i2)), np.float32)
    dev = 1e9
    for _ in range(2):
        nat.sync(); nat.jacobi_stats(reset=True)
        t0 = time.perf_counter()
        nat.check(nat.lib().ltb_slice_svd(nat.context(), hat.code, P, i1, i2, hat.ptr, u.ptr, s.ptr, v.ptr))
        nat.sync(); dev = min(dev, time.perf_counter() - t0)
    sl, sw = nat.jacobi_stats(reset=True)
    rec = L.l_product(L.l_product(f.u, f.s, spec), L.l_transpose(f.v, spec), spec)
    print(f"n={n}: svt {best['svt']*1e3:.1f} ms  t_svd {best['t_svd']*1e3:.1f} ms  slice_svd device {dev*1e3:.1f} ms "
          f"({sw / max(sl, 1):.2f} sweeps/slice)  reconstruction rel err {np.linalg.norm(rec - a) / np.linalg.norm(a):.2e}",
          flush=True)
