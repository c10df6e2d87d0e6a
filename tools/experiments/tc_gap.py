"""Gap between two back-to-back launches of the tcgen05 GEMM (device globaltimer stamps)."""
import ctypes as C, sys
from pathlib import Path
import torch
ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
from paper_2202_02870_b200 import _native as nat  # noqa: E402
lib = nat.lib(); lib.ltb_tc_debug_set_timeline.argtypes = [C.c_void_p]; lib.ltb_tc_debug_set_epi_mode.argtypes = [C.c_int]
stream = torch.cuda.Stream(); torch.cuda.set_stream(stream)
nat.check(lib.ltb_ctx_set_stream(nat.context(), stream.cuda_stream))
buf = torch.zeros(64, dtype=torch.int64, device="cuda")
m, n, k = 96, 128, 96
a = torch.randn(m, k, device="cuda"); b = torch.randn(n, k, device="cuda"); c = torch.empty(m, n, device="cuda")
def go():
    nat.check(lib.ltb_tc_gemm(nat.context(), 1, m, n, k, 0, a.data_ptr(), k, 0, 0, b.data_ptr(), k, 0, c.data_ptr(), n, 0, 3))
for mode in (0, 2):
    lib.ltb_tc_debug_set_epi_mode(mode)
    go(); go(); torch.cuda.synchronize()
    for i in range(3):
        lib.ltb_tc_debug_set_timeline(buf.data_ptr() + 16 * 8 * i)
        go()
    torch.cuda.synchronize()
    v = buf.cpu()[:48].view(3, 16).tolist()
    t0 = v[0][0]
    for i in range(3):
        print(f"mode {mode} launch {i}: start {(v[i][0]-t0)/1e3:7.2f}  setup {(v[i][1]-t0)/1e3:7.2f}  "
              f"epi {(v[i][5]-t0)/1e3:7.2f}  stored {(v[i][6]-t0)/1e3:7.2f}  dealloc {(v[i][7]-t0)/1e3:7.2f} us")
lib.ltb_tc_debug_set_timeline(None)
