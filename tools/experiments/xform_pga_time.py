"""Device time of the PGA-shaped fp32 transforms (config 3, tile engine) through ltb_transform."""
import sys
import time
from pathlib import Path
import numpy as np
ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import paper_2202_02870_b200 as L  # noqa: E402
from paper_2202_02870_b200 import _native as nat, transforms as TR  # noqa: E402

shape = (144, 176, 3, 100)
x = np.random.default_rng(0).standard_normal(shape).astype(np.float32)
spec = L.make_spec("dct", shape)
h = TR.device_spec(spec, shape[2:])
nt, P = 144 * 176, 300
dx = nat.DeviceArray.from_numpy(x.reshape(nt, P))
nat.lib().ltb_debug_set_xform_tc(0)  # force the tile engine (the PGA path)
for inv, li, lo in ((0, nat.TUBE_MAJOR, nat.SLICE_MAJOR), (1, nat.SLICE_MAJOR, nat.TUBE_MAJOR)):
    out, _ = TR.transform_device(dx, h, nt, bool(inv), li, np.float32, lo, (nt, P))
    nat.sync()
    t0 = time.perf_counter()
    for _ in range(20):
        out, _ = TR.transform_device(dx, h, nt, bool(inv), li, np.float32, lo, (nt, P))
    nat.sync()
    print(f"inverse={inv}: {(time.perf_counter() - t0) / 20 * 1e6:8.1f} us")
ref = L.apply_l(x, spec)
nat.lib().ltb_debug_set_xform_tc(0)
got = L.apply_l(x, spec)
print("rel err tile engine vs tc", np.linalg.norm(got - ref) / np.linalg.norm(ref))
nat.lib().ltb_debug_set_xform_tc(1)
