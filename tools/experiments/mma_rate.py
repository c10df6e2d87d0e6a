"""Raw kind::tf32 MMA throughput of one SM (M=128, K=8 per instruction) for the operand
patterns of ltb_tc_debug_mma_rate (see ltb_tc_gemm.cu)."""
import ctypes as C
import sys
from pathlib import Path
import torch
ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
from paper_2202_02870_b200 import _native as nat  # noqa: E402

lib = nat.lib()
lib.ltb_tc_debug_mma_rate.argtypes = [C.c_int, C.c_int, C.c_int, C.c_void_p]
out = torch.zeros(2, dtype=torch.int64, device="cuda")
names = ["A smem, fixed operands", "A TMEM, fixed operands", "3xTF32 interleaved (tc3 order)",
         "3xTF32 grouped by operand pair"]
extra = {0: "", 128: " random data", 256 + 128: " random, B cycling 3 K blocks",
         256 + 128 + 64 + 32 + 28: " random, B cycling, x148 + all"}
for bn in (96,):
  for ex, exname in extra.items():
    for pat in (2,) if ex else range(4):
        res = []
        for iters in (16, 256):
            for _ in range(2):
                nat.check(lib.ltb_tc_debug_mma_rate(bn, pat | ex, iters, out.data_ptr()))
                torch.cuda.synchronize()
            res.append(int(out[0].item()))
        per = (res[1] - res[0]) / ((256 - 16) * 12)
        flop_clk = 2 * 128 * bn * 8 / per
        print(f"N={bn:3d} {names[pat] + exname:45s}: {per:6.1f} clk/MMA -> {flop_clk * 148 * 1.965e9 / 1e12:6.0f} TFLOP/s")
