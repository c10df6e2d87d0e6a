"""Time of the QR-preconditioned K3 kernel with 0, 1, 2, 4 sweeps on config-3 slices (stage costs)."""
import sys
import time
from pathlib import Path
import numpy as np
ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
from paper_2202_02870_b200 import _native as nat  # noqa: E402

rng = np.random.default_rng(0)
batch, m, n = 300, 144, 176
a = (rng.standard_normal((batch, m, n)) * np.linspace(3, 0.01, n)).astype(np.float32)
da = nat.DeviceArray.from_numpy(a)
out = nat.DeviceArray(a.shape, np.float32)
for ms in (0, 1, 2, 4, 40):
    nat.lib().ltb_debug_set_qr_max_sweeps(ms)
    for rep in range(3):
        nat.sync()
        t0 = time.perf_counter()
        nat.check(nat.lib().ltb_slice_svt(nat.context(), 0, batch, m, n, da.ptr, 0.05, out.ptr))
        nat.sync()
        dt = time.perf_counter() - t0
    print(f"max sweeps {ms:2d}: svt {dt * 1e3:7.3f} ms")
nat.lib().ltb_debug_set_qr_max_sweeps(40)
