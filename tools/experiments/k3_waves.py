"""K3 (carried-basis fp32 SVT) device time vs slice count on config-3 late-iteration data:
how much does the 300-slice launch pay for the 4 slices beyond 2 CTAs x 148 SMs?"""
import sys
from pathlib import Path
import numpy as np
import torch
ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
import paper_2202_02870_b200 as L  # noqa: E402
from paper_2202_02870_b200 import _native as nat  # noqa: E402

m, mask = bench._cfg3_data_host()
spec = L.make_spec("dct", bench.CFG3["shape"])
hat = L.linalg._hat_stack(np.where(mask, m, 0).astype(np.float32), spec)  # (300, 144, 176) device
P, i1, i2 = hat.shape
mu0 = 0.9 * float(np.linalg.norm(m.astype(np.float64)))
tau = 1e-4 * mu0
lib, ctx = nat.lib(), nat.context()
stream = torch.cuda.Stream(); torch.cuda.set_stream(stream)
nat.check(lib.ltb_ctx_set_stream(ctx, stream.cuda_stream))
n = min(i1, i2)
for nb in (148, 292, 296, 300):
    out = torch.empty((nb, i1, i2), dtype=torch.float32, device="cuda")
    v = torch.empty((nb, n, n), dtype=torch.float32, device="cuda")
    nat.check(lib.ltb_slice_svt_carry(ctx, nb, i1, i2, hat.ptr, tau, out.data_ptr(), v.data_ptr(), 0))
    ts = []
    for rep in range(6):
        nat.sync()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(torch.cuda.current_stream())
        nat.check(lib.ltb_slice_svt_carry(ctx, nb, i1, i2, hat.ptr, tau, out.data_ptr(), v.data_ptr(), 1))
        e1.record(torch.cuda.current_stream())
        nat.sync(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    print(f"{nb} slices: warm carried SVT {np.median(ts[1:]):.3f} ms", flush=True)
