"""One QR-preconditioned K3 launch on config-3 slices with max sweeps from argv (for ncu timing)."""
import sys
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
nat.lib().ltb_debug_set_qr_max_sweeps(int(sys.argv[1]))
nat.check(nat.lib().ltb_slice_svt(nat.context(), 0, batch, m, n, da.ptr, 0.05, out.ptr))
nat.sync()
