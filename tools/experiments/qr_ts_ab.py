"""fp32 SVT (QR-preconditioned Jacobi, ltb_slice_svt) device time, 16- vs 8-lane pair teams."""
import sys
from pathlib import Path
import numpy as np
import torch
ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
from paper_2202_02870_b200 import _native as nat  # noqa: E402

lib, ctx = nat.lib(), nat.context()
stream = torch.cuda.Stream(); torch.cuda.set_stream(stream)
nat.check(lib.ltb_ctx_set_stream(ctx, stream.cuda_stream))
for (b, m, n) in [(512, 128, 128), (300, 64, 64), (300, 144, 176), (200, 96, 100), (128, 192, 192), (64, 40, 48)]:
    a = torch.randn(b, m, n, device="cuda")
    out = torch.empty_like(a)
    tau = 0.5 * float(np.sqrt(max(m, n)))
    res = {}
    for ts in (16, 8):
        lib.ltb_debug_set_qr_ts(ts)
        for _ in range(2):
            nat.check(lib.ltb_slice_svt(ctx, 0, b, m, n, a.data_ptr(), tau, out.data_ptr()))
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(5):
            nat.check(lib.ltb_slice_svt(ctx, 0, b, m, n, a.data_ptr(), tau, out.data_ptr()))
        e1.record(stream); e1.synchronize()
        res[ts] = (e0.elapsed_time(e1) / 5, out.clone())
    d = float((res[8][1] - res[16][1]).norm() / res[16][1].norm())
    print(f"{b} x {m}x{n}: ts16 {res[16][0]:.3f} ms  ts8 {res[8][0]:.3f} ms  rel diff {d:.1e}", flush=True)
lib.ltb_debug_set_qr_ts(16)
