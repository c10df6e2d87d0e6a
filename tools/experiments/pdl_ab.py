"""A/B of programmatic dependent launch for the config-2 l_product step (one CUDA graph per step)."""
import sys
from pathlib import Path
import numpy as np
import torch
ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import paper_2202_02870_b200 as L  # noqa: E402
from paper_2202_02870_b200 import _native as nat  # noqa: E402
from paper_2202_02870_b200.engine import LProductPlan  # noqa: E402

stream = torch.cuda.Stream(); torch.cuda.set_stream(stream)
nat.check(nat.lib().ltb_ctx_set_stream(nat.context(), stream.cuda_stream))
rng = np.random.default_rng(0)
a_h = rng.standard_normal((256, 128, 3, 32), dtype=np.float32)
b_h = rng.standard_normal((128, 256, 3, 32), dtype=np.float32)
spec = L.make_spec("dct", (256, 256, 3, 32))
plan = LProductPlan(a_h.shape, b_h.shape, spec, np.float32)
a = nat.DeviceArray.from_numpy(a_h); b = nat.DeviceArray.from_numpy(b_h)
c = nat.DeviceArray(plan.c_shape, np.float32)
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
for pdl in (0, 1, 0, 1):
    nat.lib().ltb_tc_debug_set_pdl(pdl)
    for _ in range(2):
        plan.run(a, b, c)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=stream):
        plan.run(a, b, c)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for i in range(25):
        flush.zero_()
        e0.record(stream); g.replay(); e1.record(stream); e1.synchronize()
        if i >= 5:
            ts.append(e0.elapsed_time(e1) * 1e3)
    ref = L.l_product(a_h, b_h, spec)
    out = c.numpy()
    print(f"pdl={pdl}: {np.median(ts):7.2f} us/step (min {min(ts):.2f})  max|diff| vs API {np.abs(out - ref).max():.3g}")
