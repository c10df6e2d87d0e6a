"""Device-resident SVT timing of the Jacobi tiers at config-4/5 slice sizes (sweeps per slice)."""
import sys
import time
from pathlib import Path
import numpy as np
ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
from paper_2202_02870_b200 import _native as nat  # noqa: E402

cases = [(np.float32, 512, 256, 256), (np.float32, 128, 512, 512), (np.complex64, 24, 1024, 1024),
         (np.float32, 300, 144, 176)]
if len(sys.argv) > 1:
    cases = [c for c in cases if str(c[2]) in sys.argv[1:]]
for dt, batch, m, n in cases:
    rng = np.random.default_rng(0)
    a = rng.standard_normal((batch, m, n)).astype(dt)
    if np.iscomplexobj(a):
        a = a + 1j * rng.standard_normal((batch, m, n)).astype(np.float32)
    da = nat.DeviceArray.from_numpy(a.astype(dt))
    out = nat.DeviceArray(a.shape, dt)
    tau = 0.1 * np.sqrt(max(m, n))
    nat.check(nat.lib().ltb_slice_svt(nat.context(), nat.dtype_code(dt), batch, m, n, da.ptr, tau, out.ptr))
    nat.sync()
    nat.jacobi_stats(reset=True)
    t0 = time.perf_counter()
    nat.check(nat.lib().ltb_slice_svt(nat.context(), nat.dtype_code(dt), batch, m, n, da.ptr, tau, out.ptr))
    nat.sync()
    dt_s = time.perf_counter() - t0
    sl, sw = nat.jacobi_stats(reset=True)
    print(f"{np.dtype(dt).name} batch={batch} {m}x{n}: svt {dt_s * 1e3:9.2f} ms   sweeps/slice {sw / max(sl, 1):.2f}")
