"""Config-2 transforms: tcgen05 Kronecker GEMM vs the CUDA-core tile engine (per-phase graphs, L2 flushed)."""
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
shape_a, shape_b = (256, 128, 3, 32), (128, 256, 3, 32)
if len(sys.argv) > 1:
    shape_a, shape_b = eval(sys.argv[1]), eval(sys.argv[2])
a_h = rng.standard_normal(shape_a, dtype=np.float32)
b_h = rng.standard_normal(shape_b, dtype=np.float32)
spec = L.make_spec("dct", (shape_a[0], shape_b[1]) + shape_a[2:])
plan = LProductPlan(a_h.shape, b_h.shape, spec, np.float32)
a = nat.DeviceArray.from_numpy(a_h); b = nat.DeviceArray.from_numpy(b_h)
c = nat.DeviceArray(plan.c_shape, np.float32)
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
ref = L.l_product(a_h, b_h, spec)
for tc in (1, 0):
    nat.lib().ltb_debug_set_xform_tc(tc)
    for _ in range(2):
        plan.run(a, b, c)
    torch.cuda.synchronize()
    gs = []
    for ph in range(4):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=stream):
            plan.run(a, b, c, phases=(ph,))
        gs.append(g)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
    acc = np.zeros(4)
    for i in range(15):
        flush.zero_()
        for ph in range(4):
            ev[ph].record(stream); gs[ph].replay()
        ev[4].record(stream); ev[4].synchronize()
        if i >= 5:
            acc += [ev[k].elapsed_time(ev[k + 1]) * 1e3 for k in range(4)]
    err = np.linalg.norm(c.numpy() - ref) / np.linalg.norm(ref)
    print(f"xform_tc={tc}: phases us {np.round(acc / 10, 2)}  rel err {err:.2e}")
nat.lib().ltb_debug_set_xform_tc(1)
