"""A/B of libltb debug switches on the config-2 l_product step (CUDA graphs, L2 flushed).

    python tools/lprod_ab.py ltb_tc_debug_set_ct_direct=0,1 [ltb_tc_debug_set_epi_mode=3,1 ...]

Each switch is varied alone (the others at their first value); prints per-phase and
whole-step device times and the error against the single-GPU API."""
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
lib = nat.lib()
nat.check(lib.ltb_ctx_set_stream(nat.context(), stream.cuda_stream))
rng = np.random.default_rng(0)
a_h = rng.standard_normal((256, 128, 3, 32), dtype=np.float32)
b_h = rng.standard_normal((128, 256, 3, 32), dtype=np.float32)
spec = L.make_spec("dct", (256, 256, 3, 32))
plan = LProductPlan(a_h.shape, b_h.shape, spec, np.float32)
a = nat.DeviceArray.from_numpy(a_h); b = nat.DeviceArray.from_numpy(b_h)
c = nat.DeviceArray(plan.c_shape, np.float32)
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
ref = L.l_product(a_h.astype(np.float64), b_h.astype(np.float64), spec)
switches = [(name, [int(v) for v in vals.split(",")]) for name, vals in (arg.split("=") for arg in sys.argv[1:])]


def measure():
    for _ in range(2):
        plan.run(a, b, c)
    torch.cuda.synchronize()
    phases = [0, 2, 3] if plan.paired else [0, 1, 2, 3]
    gs = []
    for ph in phases:
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=stream):
            plan.run(a, b, c, phases=(ph,))
        gs.append(g)
    full = torch.cuda.CUDAGraph()
    with torch.cuda.graph(full, stream=stream):
        plan.run(a, b, c)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(len(gs) + 1)]
    acc = np.zeros(len(gs))
    tot = []
    for i in range(25):
        flush.zero_()
        for k, g in enumerate(gs):
            ev[k].record(stream); g.replay()
        ev[-1].record(stream); ev[-1].synchronize()
        if i >= 5:
            acc += [ev[k].elapsed_time(ev[k + 1]) * 1e3 for k in range(len(gs))]
        flush.zero_()
        ev[0].record(stream); full.replay(); ev[1].record(stream); ev[1].synchronize()
        if i >= 5:
            tot.append(ev[0].elapsed_time(ev[1]) * 1e3)
    err = np.linalg.norm(c.numpy() - ref) / np.linalg.norm(ref)
    return np.round(acc / 20, 2), float(np.median(tot)), err


for name, vals in switches:
    fn = getattr(lib, name)
    for v in vals:
        fn(v)
        ph, tot, err = measure()
        print(f"{name}={v}: phases us {ph}  step {tot:.2f} us  rel err {err:.2e}", flush=True)
    fn(vals[0])
