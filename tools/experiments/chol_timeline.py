"""Stage timeline (CTA 0, globaltimer) of the warm Cholesky-preconditioned K3 kernel inside a
late config-3 PGA iteration, plus that iteration's sweep statistics."""
import ctypes as C
import sys
from pathlib import Path
import numpy as np
import torch
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
import paper_2202_02870_b200 as L  # noqa: E402
from paper_2202_02870_b200 import _native as nat  # noqa: E402
from paper_2202_02870_b200.completion import PGASolver, pga_schedule  # noqa: E402

lib = nat.lib()
lib.ltb_debug_set_qr_timeline.argtypes = [C.c_void_p]
m, mask = bench._cfg3_data_host()
spec = L.make_spec("dct", bench.CFG3["shape"])
cfg = L.CompletionConfig(spec=spec, tol=1e-300, max_iters=200)
mu0 = cfg.nu * L.fro_norm(np.asarray(m, dtype=np.float64))
mus, ts, betas = pga_schedule(cfg, mu0)
s = PGASolver(np.asarray(m, dtype=np.float64), mask, spec, "fp32")
buf = torch.zeros(16, dtype=torch.int64, device="cuda")
names = ["start", "loaded", "norm check", "factor", "transpose", "sweeps", "emitted"]
k = 1
for stop in (30, 60, 120, 180):
    s.run(k, betas[k - 1:stop - 1], mus[k - 1:stop - 1], cfg.tol)
    k = stop
    nat.sync()
    nat.jacobi_stats(reset=True)
    buf.zero_()
    lib.ltb_debug_set_qr_timeline(buf.data_ptr())
    s.run(k, betas[k - 1:k], mus[k - 1:k], cfg.tol)
    nat.sync()
    lib.ltb_debug_set_qr_timeline(None)
    k += 1
    sl, sw, mx = nat.jacobi_stats(reset=True, with_max=True)
    v = buf.cpu().tolist()
    print(f"iteration {k - 1}: slices {sl} sweeps/slice {sw / max(sl, 1):.2f} max {mx}; CTA 0:",
          ", ".join(f"{nm} {(v[i] - v[0]) / 1e3:.1f}us" for i, nm in enumerate(names) if v[i]), flush=True)
s.close()
