"""Per-tile device timeline (globaltimer, CTA 0) of the config-2 l_product tcgen05 phases:
TMA issue of each tile's first k-block, k-block landed (converter saw `full`), split
done, MMA issued, tile's last MMA, epilogue start / done.  Where do ~4 us per tile go?"""
import ctypes as C
import sys
from pathlib import Path
import numpy as np
import torch
ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
import paper_2202_02870_b200 as L  # noqa: E402
from paper_2202_02870_b200 import _native as nat  # noqa: E402
from paper_2202_02870_b200.engine import LProductPlan  # noqa: E402

lib = nat.lib()
lib.ltb_tc_debug_set_timeline.argtypes = [C.c_void_p]
stream = torch.cuda.Stream(); torch.cuda.set_stream(stream)
nat.check(lib.ltb_ctx_set_stream(nat.context(), stream.cuda_stream))
spec = L.make_spec("dct", (256, 256, 3, 32))
a_h, b_h = bench._cfg2_inputs(0)
plan = LProductPlan(a_h.shape, b_h.shape, spec, np.float32)
a = nat.DeviceArray.from_numpy(a_h); b = nat.DeviceArray.from_numpy(b_h)
c = nat.DeviceArray(plan.c_shape, np.float32)
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
buf = torch.zeros(1024, dtype=torch.int64, device="cuda")
for ph, label in ((0, "forward A+B"), (2, "slice GEMM"), (3, "inverse C")):
    for rep in range(3):
        plan.run(a, b, c)
        flush.zero_()
        torch.cuda.synchronize()
        buf.zero_()
        lib.ltb_tc_debug_set_timeline(buf.data_ptr() if rep == 2 else None)
        plan.run(a, b, c, phases=(ph,))
        torch.cuda.synchronize()
    lib.ltb_tc_debug_set_timeline(None)
    v = buf.cpu().numpy().astype(np.float64)
    t0 = v[0]
    us = lambda s: (v[s] - t0) / 1e3 if v[s] else float("nan")  # noqa: E731
    print(f"== {label}: setup {us(1):.2f}  first TMA {us(2):.2f}  first split {us(3):.2f}  "
          f"first MMA {us(4):.2f}  epi start {us(5):.2f}  first tile stored {us(6):.2f}  dealloc {us(7):.2f} us")
    print("   k-block it: landed / split done / MMA start / MMA issued")
    for it in range(16):
        if v[96 + it]:
            print(f"   it {it:2d}: {us(96 + it):7.2f} {us(64 + it):7.2f} {us(80 + it):7.2f} {us(112 + it):7.2f}")
    print("   tile j: TMA issue / last MMA / epi start / chunk0 ld,box,fence,store / tile done")
    for j in range(16):
        if v[16 + j] or v[32 + j]:
            ep = f"{us(160 + 4 * j):7.2f}" if j < 4 else "   -   "
            ch = " ".join(f"{us(176 + 8 * j + k):6.2f}" for k in (3, 0, 1, 2)) if j < 4 else ""
            print(f"   tile {j:2d}: {us(16 + j):7.2f} {us(32 + j):7.2f} {ep} [{ch}] {us(48 + j):7.2f}")
