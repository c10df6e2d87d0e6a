"""Run one tcgen05 GEMM config (m n k split [graph]) and check it against torch fp64."""
import sys
from pathlib import Path
import torch
ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
from paper_2202_02870_b200 import _native as nat  # noqa: E402
m, n, k, split = (int(v) for v in sys.argv[1:5])
stream = torch.cuda.Stream(); torch.cuda.set_stream(stream)
nat.check(nat.lib().ltb_ctx_set_stream(nat.context(), stream.cuda_stream))
a = torch.randn(m, k, device="cuda"); b = torch.randn(n, k, device="cuda"); c = torch.empty(m, n, device="cuda")
nat.check(nat.lib().ltb_tc_gemm(nat.context(), 1, m, n, k, 0, a.data_ptr(), k, 0, 0, b.data_ptr(), k, 0, c.data_ptr(), n, 0, split))
torch.cuda.synchronize()
ref = a.double() @ b.double().T
print(m, n, k, split, "err", float((c.double() - ref).norm() / ref.norm()), flush=True)
