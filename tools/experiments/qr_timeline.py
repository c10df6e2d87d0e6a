"""Stage timeline (CTA 0, globaltimer) of the QR-preconditioned K3 kernel on config-3 slices."""
import ctypes as C
import sys
from pathlib import Path
import numpy as np
import torch
ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
from paper_2202_02870_b200 import _native as nat  # noqa: E402

lib = nat.lib()
lib.ltb_debug_set_qr_timeline.argtypes = [C.c_void_p]
rng = np.random.default_rng(0)
for (batch, m, n, mode) in ((300, 144, 176, 0), (2, 144, 176, 0), (2, 144, 176, 1), (2, 144, 176, 2)):
    a = (rng.standard_normal((batch, m, n)) * np.linspace(3, 0.01, n)).astype(np.float32)
    da = nat.DeviceArray.from_numpy(a)
    out = nat.DeviceArray(a.shape, np.float32)
    buf = torch.zeros(16, dtype=torch.int64, device="cuda")
    buf[15] = mode
    nat.check(lib.ltb_slice_svt(nat.context(), 0, batch, m, n, da.ptr, 0.05, out.ptr))
    nat.sync()
    lib.ltb_debug_set_qr_timeline(buf.data_ptr())
    nat.check(lib.ltb_slice_svt(nat.context(), 0, batch, m, n, da.ptr, 0.05, out.ptr))
    nat.sync()
    lib.ltb_debug_set_qr_timeline(None)
    v = buf.cpu().tolist()
    names = ["start", "loaded", "norm check", "QR", "transpose", "sweeps", "emitted"]
    print(f"batch {batch} mode {mode}:", ", ".join(f"{nm} {(v[i] - v[0]) / 1e3:.1f}us" for i, nm in enumerate(names) if v[i]))
