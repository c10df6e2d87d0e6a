"""Config-2 l_product with the rows of A / C split into H blocks whose phase chains run on
separate streams (one CUDA graph, fork / join events): K1(B) once, then per block
K1(A_h) -> K2_h -> K1'(C_h).  Blocks overlap each other's fill / drain.  Prints the step
time (median of 20, L2 flushed) for H = 1, 2, 4 and the error against the fp64 oracle."""
import sys
from pathlib import Path
import numpy as np
import torch
ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "oracle"))
import paper_2202_02870_b200 as L  # noqa: E402
from paper_2202_02870_b200 import _native as nat  # noqa: E402
from paper_2202_02870_b200.transforms import device_spec  # noqa: E402
import ltensor_oracle as O  # noqa: E402

lib, ctx = nat.lib(), nat.context()
rng = np.random.default_rng(0)
a_h = rng.standard_normal((256, 128, 3, 32), dtype=np.float32)
b_h = rng.standard_normal((128, 256, 3, 32), dtype=np.float32)
spec = L.make_spec("dct", (256, 256, 3, 32))
h = device_spec(spec, (3, 32)).ptr
P, I1, K, I2 = 96, 256, 128, 256
a = nat.DeviceArray.from_numpy(a_h); b = nat.DeviceArray.from_numpy(b_h)
c = nat.DeviceArray((I1, I2, 3, 32), np.float32)
hb = nat.DeviceArray((P, K, I2), np.float32)
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
ref = O.l_product(a_h[:16].astype(np.float64), b_h.astype(np.float64), O.ospec("dct", (16, 256, 3, 32)))
F, TM, SM = nat.F32, nat.TUBE_MAJOR, nat.SLICE_MAJOR
streams = [torch.cuda.Stream() for _ in range(4)]
torch.cuda.set_stream(streams[0])  # flushes and replays on the timed stream


def build(H):
    rows = I1 // H
    has = [nat.DeviceArray((P, rows, K), np.float32) for _ in range(H)]
    hcs = [nat.DeviceArray((P, rows, I2), np.float32) for _ in range(H)]
    g = torch.cuda.CUDAGraph()
    s0 = streams[0]
    with torch.cuda.graph(g, stream=s0):
        start = torch.cuda.Event(); start.record(s0)
        nat.check(lib.ltb_ctx_set_stream(ctx, s0.cuda_stream))
        nat.check(lib.ltb_transform(ctx, h, K * I2, 0, F, TM, b.ptr, F, SM, hb.ptr, None))
        eb = torch.cuda.Event(); eb.record(s0)
        ends = []
        for i in range(H):
            s = streams[i % len(streams)] if i else s0
            if i:
                s.wait_event(start)
            nat.check(lib.ltb_ctx_set_stream(ctx, s.cuda_stream))
            a_i = nat.DeviceArray((rows, K), np.float32, ptr=a.ptr.value + 4 * i * rows * K * P, owner=False)
            c_i = nat.DeviceArray((rows, I2), np.float32, ptr=c.ptr.value + 4 * i * rows * I2 * P, owner=False)
            nat.check(lib.ltb_transform(ctx, h, rows * K, 0, F, TM, a_i.ptr, F, SM, has[i].ptr, None))
            if i:
                s.wait_event(eb)
            nat.check(lib.ltb_slice_gemm(ctx, F, P, rows, I2, K, nat.OP_N, has[i].ptr, K, rows * K, nat.OP_N,
                                         hb.ptr, I2, K * I2, hcs[i].ptr, I2, rows * I2))
            nat.check(lib.ltb_transform(ctx, h, rows * I2, 1, F, SM, hcs[i].ptr, F, TM, c_i.ptr, None))
            if i:
                e = torch.cuda.Event(); e.record(s); ends.append(e)
        for e in ends:
            s0.wait_event(e)
    nat.check(lib.ltb_ctx_set_stream(ctx, s0.cuda_stream))
    return g, (has, hcs)


ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for H in (1, 2, 4, 8):
    g, keep = build(H)
    torch.cuda.synchronize()
    ts = []
    for i in range(25):
        flush.zero_()
        ev0.record(streams[0]); g.replay(); ev1.record(streams[0]); ev1.synchronize()
        if i >= 5:
            ts.append(ev0.elapsed_time(ev1) * 1e3)
    err = np.linalg.norm(c.numpy()[:16] - ref) / np.linalg.norm(ref)
    print(f"H={H}: step {np.median(ts):.2f} us (min {min(ts):.2f})  rel err {err:.2e}", flush=True)
