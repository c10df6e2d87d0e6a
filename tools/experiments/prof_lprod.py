"""Profiling driver: BASELINE config 2 l_product (device-resident) a few times."""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402
import paper_2202_02870_b200 as L  # noqa: E402
from paper_2202_02870_b200 import _native as nat  # noqa: E402
from paper_2202_02870_b200.engine import LProductPlan  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
a_h, b_h = bench._cfg2_inputs()
spec = L.make_spec("dct", (256, 256, 3, 32))
plan = LProductPlan(a_h.shape, b_h.shape, spec, np.float32)
a = nat.DeviceArray.from_numpy(a_h)
b = nat.DeviceArray.from_numpy(b_h)
c = nat.DeviceArray(plan.c_shape, np.float32)
for _ in range(reps):
    plan.run(a, b, c)
nat.sync()
print("ok", float(np.abs(c.numpy()).mean()))
