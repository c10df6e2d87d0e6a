"""Does the tensor core truncate fp32 -> tf32?  Compare the 3xTF32 error with an explicit hi vs the raw fp32 tile."""
import ctypes as C, sys
from pathlib import Path
import torch
ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
from paper_2202_02870_b200 import _native as nat  # noqa: E402
lib = nat.lib(); lib.ltb_tc_debug_set_raw_hi.argtypes = [C.c_int]
for k in (128, 1024):
    m = n = 256
    a = torch.randn(m, k, device="cuda"); b = torch.randn(n, k, device="cuda"); c = torch.empty(m, n, device="cuda")
    ref = a.double() @ b.double().T
    for raw in (0, 1):
        lib.ltb_tc_debug_set_raw_hi(raw)
        nat.check(lib.ltb_tc_gemm(nat.context(), 1, m, n, k, 0, a.data_ptr(), k, 0, 0, b.data_ptr(), k, 0, c.data_ptr(), n, 0, 3))
        nat.sync()
        print("k", k, "raw_hi", raw, "err %.3e" % float((c.double() - ref).norm() / ref.norm()), flush=True)
    fp32 = (a @ b.T).double()
    print("k", k, "torch fp32 matmul err %.3e" % float((fp32 - ref).norm() / ref.norm()))
