"""Where does the fixed per-launch cost of the tcgen05 GEMM come from?  (CUDA-graph timed)"""
import sys
from pathlib import Path
import torch
ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
from paper_2202_02870_b200 import _native as nat  # noqa: E402

stream = torch.cuda.Stream(); torch.cuda.set_stream(stream)
nat.check(nat.lib().ltb_ctx_set_stream(nat.context(), stream.cuda_stream))

def timed(fn, reps=50):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=stream):
        for _ in range(reps): fn()
    g.replay(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream); g.replay(); e1.record(stream); e1.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3

x = torch.zeros(1, device="cuda")
print("tiny torch kernel        %.2f us" % timed(lambda: x.add_(1)), flush=True)
def tc(m, n, k, split, a_mn=0, b_mn=0):
    a = torch.randn(k if a_mn else m, m if a_mn else k, device="cuda")
    b = torch.randn(k if b_mn else n, n if b_mn else k, device="cuda")
    c = torch.empty(m, n, device="cuda")
    args = (nat.context(), 1, m, n, k, a_mn, a.data_ptr(), a.shape[1], 0, b_mn, b.data_ptr(), b.shape[1], 0, c.data_ptr(), n, 0, split)
    return lambda: nat.check(nat.lib().ltb_tc_gemm(*args))
for (m, n, k, s) in [(128, 128, 32, 1), (128, 128, 32, 3), (128, 128, 96, 3), (128, 128, 1024, 3), (128, 128, 4096, 3),
                     (128, 128, 4096, 1), (128, 256, 32, 3), (128, 128 * 148, 32, 3)]:
    print(f"tc m={m} n={n} k={k} split={s}: ...", flush=True)
    print("   %.2f us" % timed(tc(m, n, k, s)), flush=True)
