"""Device timeline (globaltimer, CTA 0) of one tcgen05 GEMM launch: where does the fixed cost go?"""
import ctypes as C, sys
from pathlib import Path
import torch
ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
from paper_2202_02870_b200 import _native as nat  # noqa: E402
lib = nat.lib(); lib.ltb_tc_debug_set_timeline.argtypes = [C.c_void_p]
buf = torch.zeros(16, dtype=torch.int64, device="cuda")
names = ["start", "setup done", "first TMA issued", "first split done", "first MMA commit", "epilogue start",
         "tile stored", "before dealloc", "c0 ld start", "c0 ld done", "c1 ld start", "c1 ld done", "c2 ld start", "c2 ld done"]
lib.ltb_tc_debug_set_epi_mode.argtypes = [C.c_int]
for (m, n, k, mode) in [(96, 128, 96, 0), (96, 128, 96, 1), (96, 128, 96, 2), (96, 32768, 96, 0), (96, 32768, 96, 1), (96, 32768, 96, 2)]:
    lib.ltb_tc_debug_set_epi_mode(mode)
    a = torch.randn(m, k, device="cuda"); b = torch.randn(n, k, device="cuda"); c = torch.empty(m, n, device="cuda")
    for rep in range(3):
        buf.zero_(); torch.cuda.synchronize()
        lib.ltb_tc_debug_set_timeline(buf.data_ptr() if rep == 2 else None)
        t0 = torch.cuda.Event(enable_timing=True); t1 = torch.cuda.Event(enable_timing=True)
        t0.record()
        nat.check(lib.ltb_tc_gemm(nat.context(), 1, m, n, k, 0, a.data_ptr(), k, 0, 0, b.data_ptr(), k, 0, c.data_ptr(), n, 0, 3))
        t1.record(); torch.cuda.synchronize()
    v = buf.cpu().tolist()
    print(f"m={m} n={n} k={k} epi_mode={mode}: event time {t0.elapsed_time(t1)*1e3:.1f} us")
    for i, nm in enumerate(names):
        print(f"   {nm:18s} {(v[i]-v[0])/1e3:8.2f} us")
lib.ltb_tc_debug_set_timeline(None)
