"""Per-CTA start / end (globaltimer) of each config-2 l_product phase launch, relative to the
earliest CTA start, plus the CUDA-event time of the phase: where does a ~20 us phase go?"""
import ctypes as C
import sys
from pathlib import Path
import numpy as np
import torch
ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
import paper_2202_02870_b200 as L  # noqa: E402
from paper_2202_02870_b200 import _native as nat  # noqa: E402
from paper_2202_02870_b200.engine import LProductPlan  # noqa: E402

lib = nat.lib()
lib.ltb_tc_debug_set_timeline.argtypes = [C.c_void_p]
stream = torch.cuda.Stream(); torch.cuda.set_stream(stream)
nat.check(lib.ltb_ctx_set_stream(nat.context(), stream.cuda_stream))
spec = L.make_spec("dct", (256, 256, 3, 32))
a_h, b_h = bench._cfg2_inputs(0)
plan = LProductPlan(a_h.shape, b_h.shape, spec, np.float32)
a = nat.DeviceArray.from_numpy(a_h); b = nat.DeviceArray.from_numpy(b_h)
c = nat.DeviceArray(plan.c_shape, np.float32)
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
buf = torch.zeros(1024, dtype=torch.int64, device="cuda")
for ph, label in ((0, "forward A+B"), (2, "slice GEMM"), (3, "inverse C")):
    for rep in range(3):
        plan.run(a, b, c)
        flush.zero_()
        torch.cuda.synchronize()
        buf.zero_()
        lib.ltb_tc_debug_set_timeline(buf.data_ptr() if rep == 2 else None)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        plan.run(a, b, c, phases=(ph,))
        e1.record(stream)
        torch.cuda.synchronize()
    lib.ltb_tc_debug_set_timeline(None)
    v = buf.cpu().numpy()
    st = v[256:256 + 2 * 148:2].astype(np.float64); en = v[257:257 + 2 * 148:2].astype(np.float64)
    ok = st > 0
    t0 = st[ok].min()
    s, e = (st[ok] - t0) / 1e3, (en[ok] - t0) / 1e3
    d = e - s
    print(f"{label}: event {e0.elapsed_time(e1) * 1e3:.1f} us; CTAs {ok.sum()}; start spread {s.max():.2f} us; "
          f"end min/med/max {e.min():.2f}/{np.median(e):.2f}/{e.max():.2f} us; CTA duration min/med/max "
          f"{d.min():.2f}/{np.median(d):.2f}/{d.max():.2f} us")
    order = np.argsort(d)
    print("   longest CTAs:", [(int(np.flatnonzero(ok)[i]), round(float(d[i]), 2)) for i in order[-6:]])
