"""CTA-0 device timeline (globaltimer) of the config-2 forward / inverse transform launches."""
import ctypes as C
import sys
from pathlib import Path
import numpy as np
import torch
ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import paper_2202_02870_b200 as L  # noqa: E402
from paper_2202_02870_b200 import _native as nat  # noqa: E402
from paper_2202_02870_b200.engine import LProductPlan  # noqa: E402

lib = nat.lib()
lib.ltb_tc_debug_set_timeline.argtypes = [C.c_void_p]
stream = torch.cuda.Stream(); torch.cuda.set_stream(stream)
nat.check(lib.ltb_ctx_set_stream(nat.context(), stream.cuda_stream))
rng = np.random.default_rng(0)
a_h = rng.standard_normal((256, 128, 3, 32), dtype=np.float32)
b_h = rng.standard_normal((128, 256, 3, 32), dtype=np.float32)
spec = L.make_spec("dct", (256, 256, 3, 32))
plan = LProductPlan(a_h.shape, b_h.shape, spec, np.float32)
a = nat.DeviceArray.from_numpy(a_h); b = nat.DeviceArray.from_numpy(b_h)
c = nat.DeviceArray(plan.c_shape, np.float32)
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
buf = torch.zeros(16, dtype=torch.int64, device="cuda")
names = ["start", "setup done", "first TMA issued", "first split done", "first MMA commit", "epilogue start",
         "tile stored", "before dealloc", "c0 ld start", "c0 ld done", "c1 ld start", "c1 ld done", "c2 ld start",
         "c2 ld done"]
for ph, label in ((0, "forward A (+B when paired)"), (2, "slice GEMM"), (3, "inverse C")):
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
    v = buf.cpu().tolist()
    print(f"{label}: event time {e0.elapsed_time(e1) * 1e3:.1f} us")
    for i, nm in enumerate(names):
        if v[i]:
            print(f"   {nm:18s} {(v[i] - v[0]) / 1e3:8.2f} us")
