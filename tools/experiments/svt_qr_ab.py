"""A/B of the fp32 SVT: QR-preconditioned Jacobi vs the direct one-sided Jacobi (config-3-like slices)."""
import sys
import time
from pathlib import Path
import numpy as np
ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
from paper_2202_02870_b200 import _native as nat  # noqa: E402

for (batch, m, n) in ((300, 144, 176), (300, 176, 144), (64, 96, 96)):
    rng = np.random.default_rng(0)
    a = (rng.standard_normal((batch, m, n)) * np.linspace(3, 0.01, max(m, n))[:min(m, n)][:, None]
         if m < n else rng.standard_normal((batch, m, n)) * np.linspace(3, 0.01, n)).astype(np.float32)
    da = nat.DeviceArray.from_numpy(a)
    res = {}
    for qr in (0, 1):
        nat.lib().ltb_debug_set_svt_qr(qr)
        out = nat.DeviceArray(a.shape, np.float32)
        for rep in range(3):
            nat.sync()
            nat.jacobi_stats(reset=True)
            t0 = time.perf_counter()
            nat.check(nat.lib().ltb_slice_svt(nat.context(), nat.dtype_code(np.float32), batch, m, n, da.ptr, 0.05,
                                              out.ptr))
            nat.sync()
            dt = time.perf_counter() - t0
        sl, sw = nat.jacobi_stats(reset=True)
        res[qr] = out.numpy()
        print(f"{batch}x{m}x{n} qr={qr}: svt {dt * 1e3:8.3f} ms  sweeps/slice {sw / max(sl, 1):.2f}")
    u, s, vh = np.linalg.svd(a[:8].astype(np.float64), full_matrices=False)
    ref = np.matmul(u * np.maximum(s - 0.05, 0)[:, None, :], vh)
    for qr in (0, 1):
        print(f"   qr={qr} rel err vs numpy (8 slices) {np.linalg.norm(res[qr][:8] - ref) / np.linalg.norm(ref):.2e}")
nat.lib().ltb_debug_set_svt_qr(1)
