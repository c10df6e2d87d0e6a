"""Timing of the slice SVT / t_svd at BASELINE config 5 sizes (and config 4 reduced), device-resident."""
import sys, time
from pathlib import Path
import numpy as np
import torch
ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
from paper_2202_02870_b200 import _native as nat  # noqa: E402

def run(P, m, n, dt, tau, full=False):
    x = torch.randn(P, m, n, dtype=dt, device="cuda")
    out = torch.empty_like(x)
    code = {torch.float32: 0, torch.float64: 1, torch.complex64: 2, torch.complex128: 3}[dt]
    nat.jacobi_stats(reset=True)
    torch.cuda.synchronize(); t0 = time.perf_counter()
    if full:
        u = torch.empty(P, m, m, dtype=dt, device="cuda"); v = torch.empty(P, n, n, dtype=dt, device="cuda")
        s = torch.empty(P, min(m, n), dtype=torch.float32 if code in (0, 2) else torch.float64, device="cuda")
        nat.check(nat.lib().ltb_slice_svd(nat.context(), code, P, m, n, x.data_ptr(), u.data_ptr(), s.data_ptr(), v.data_ptr()))
    else:
        nat.check(nat.lib().ltb_slice_svt(nat.context(), code, P, m, n, x.data_ptr(), tau, out.data_ptr()))
    torch.cuda.synchronize(); dt_s = time.perf_counter() - t0
    sl, sw = nat.jacobi_stats(reset=True)
    print(f"{'svd' if full else 'svt'} P={P} {m}x{n} {dt}: {dt_s*1e3:9.1f} ms  sweeps/slice {sw/max(sl,1):.1f}", flush=True)

nat.check(nat.lib().ltb_ctx_set_stream(nat.context(), 1))
for spec in sys.argv[1:]:
    P, m, n, kind, full = spec.split(",")
    dt = {"f32": torch.float32, "c64": torch.complex64, "f64": torch.float64}[kind]
    run(int(P), int(m), int(n), dt, 1.0, full == "1")
