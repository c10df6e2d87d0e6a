"""Config-2 l_product step time (one CUDA graph) under different L2 states before the step:
dirty flush (512 MiB write), clean flush (512 MiB write, then a 512 MiB read so the dirty
lines are written back before the step), and warm L2 (no flush)."""
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

stream = torch.cuda.Stream(); torch.cuda.set_stream(stream)
nat.check(nat.lib().ltb_ctx_set_stream(nat.context(), stream.cuda_stream))
spec = L.make_spec("dct", (256, 256, 3, 32))
a_h, b_h = bench._cfg2_inputs(0)
plan = LProductPlan(a_h.shape, b_h.shape, spec, np.float32)
a = nat.DeviceArray.from_numpy(a_h); b = nat.DeviceArray.from_numpy(b_h)
c = nat.DeviceArray(plan.c_shape, np.float32)
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
fl32 = flush.view(torch.float32)
sink = torch.empty(1, device="cuda")
for _ in range(2):
    plan.run(a, b, c)
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=stream):
    plan.run(a, b, c)
graphs = []
for ph in (0, 2, 3):
    gg = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gg, stream=stream):
        plan.run(a, b, c, phases=(ph,))
    graphs.append(gg)
def dirty():
    flush.zero_()
def clean():
    flush.zero_()
    torch.sum(fl32, dim=(0,), out=sink[0])
def warm():
    pass
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for name, pre in (("dirty flush", dirty), ("clean flush", clean), ("warm L2", warm)):
    for rep in range(2):
        ts = []
        for i in range(25):
            pre()
            e0.record(stream); g.replay(); e1.record(stream); e1.synchronize()
            if i >= 5:
                ts.append(e0.elapsed_time(e1) * 1e3)
        ph = []
        for gg in graphs:
            t = []
            for i in range(15):
                pre()
                e0.record(stream); gg.replay(); e1.record(stream); e1.synchronize()
                if i >= 5:
                    t.append(e0.elapsed_time(e1) * 1e3)
            ph.append(np.median(t))
    print(f"{name:12s}: step median {np.median(ts):6.1f} us min {np.min(ts):6.1f}; phases fwd/gemm/inv "
          + " / ".join(f"{x:5.1f}" for x in ph), flush=True)
