"""Per-column accuracy of the fp32 slice SVD factors (ltb_slice_svd) against LAPACK fp64, and
the same SVD run in fp64 on the upcast slices; device time of each."""
import sys
import time

sys.path.insert(0, "/root/repo")
sys.path.insert(0, "/root/repo/tests")
import numpy as np

from paper_2202_02870_b200 import _native as nat
from ltb_testutil import factor_parity

for n in (128, 256, 512):
    rng = np.random.default_rng(0)
    batch = 32
    a = rng.standard_normal((batch, n, n)).astype(np.float32)
    uh, sv, vh = np.linalg.svd(a.astype(np.float64))
    vref = np.swapaxes(vh, 1, 2)
    for dt in (np.float32, np.float64):
        da = nat.DeviceArray.from_numpy(a.astype(dt))
        u = nat.DeviceArray((batch, n, n), dt)
        v = nat.DeviceArray((batch, n, n), dt)
        s = nat.DeviceArray((batch, n), dt)
        nat.check(nat.lib().ltb_slice_svd(nat.context(), nat.dtype_code(dt), batch, n, n, da.ptr, u.ptr, s.ptr, v.ptr))
        nat.sync()
        t0 = time.perf_counter()
        nat.check(nat.lib().ltb_slice_svd(nat.context(), nat.dtype_code(dt), batch, n, n, da.ptr, u.ptr, s.ptr, v.ptr))
        nat.sync()
        dt_s = time.perf_counter() - t0
        U, V, S = u.numpy().astype(np.float64), v.numpy().astype(np.float64), s.numpy().astype(np.float64)
        eu, cu = factor_parity(U, uh, sv)
        ev, cv = factor_parity(V, vref, sv)
        es = np.linalg.norm(S - sv) / np.linalg.norm(sv)
        # per-column error buckets by sigma / sigma_max
        smax = sv.max()
        buckets = {}
        for p in range(batch):
            for j in range(n):
                c = np.vdot(U[p, :, j], uh[p, :, j])
                e = np.linalg.norm(U[p, :, j] * np.sign(c) - uh[p, :, j])
                gap = min(sv[p, j - 1] - sv[p, j] if j else np.inf, sv[p, j] - (sv[p, j + 1] if j + 1 < n else 0))
                key = (int(np.floor(np.log10(sv[p, j] / smax))), int(np.floor(np.log10(max(gap / smax, 1e-9)))))
                buckets.setdefault(key, []).append(e)
        print(f"n={n} {np.dtype(dt).name}: {dt_s * 1e3:.1f} ms for {batch} slices; U err {eu:.2e} ({cu} cols) "
              f"V err {ev:.2e} ({cv}) S err {es:.2e}", flush=True)
        for key in sorted(buckets):
            e = np.array(buckets[key])
            print(f"   log10 sigma/smax {key[0]:3d} log10 gap/smax {key[1]:3d}: {len(e):6d} cols  "
                  f"median {np.median(e):.2e}  max {e.max():.2e}")
