"""Microbenchmark of the tcgen05 fp32 GEMM engine at transform / slice-GEMM shapes (CUDA events)."""
import sys
from pathlib import Path
import numpy as np
import torch
ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
from paper_2202_02870_b200 import _native as nat  # noqa: E402

stream = torch.cuda.Stream(); torch.cuda.set_stream(stream)
nat.check(nat.lib().ltb_ctx_set_stream(nat.context(), stream.cuda_stream))

def bench(batch, m, n, k, a_mn, b_mn, split=3, reps=20):
    a = torch.randn(batch, k if a_mn else m, m if a_mn else k, device="cuda")
    b = torch.randn(batch, k if b_mn else n, n if b_mn else k, device="cuda")
    c = torch.empty(batch, m, n, device="cuda")
    args = (nat.context(), batch, m, n, k, a_mn, a.data_ptr(), a.shape[2], a.shape[1] * a.shape[2], b_mn, b.data_ptr(),
            b.shape[2], b.shape[1] * b.shape[2], c.data_ptr(), n, m * n, split)
    for _ in range(3): nat.check(nat.lib().ltb_tc_gemm(*args))
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=stream):
        for _ in range(reps): nat.check(nat.lib().ltb_tc_gemm(*args))
    g.replay(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    g.replay()
    e1.record(stream); e1.synchronize()
    us = e0.elapsed_time(e1) / reps * 1e3
    byts = 4 * (a.numel() + b.numel() + c.numel())
    print(f"b={batch} m={m} n={n} k={k} amn={a_mn} bmn={b_mn} split={split}: {us:8.2f} us  {byts/us/1e3:8.1f} GB/s  {2*batch*m*n*k/us/1e6:8.1f} TFLOP/s")

for n in (128, 2048, 32768, 327680):
    bench(1, 96, n, 96, 0, 0)
bench(1, 96, 32768, 96, 0, 0, split=1)
bench(96, 256, 256, 128, 0, 1)
bench(96, 256, 256, 128, 0, 1, split=1)
bench(1, 65536, 96, 96, 1, 0)
bench(1, 8192, 8192, 1024, 0, 0)
