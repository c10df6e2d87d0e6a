"""Per-tile CTA-0 timeline (globaltimer) of the config-2 tcgen05 launches: when each tile's
first A load is issued, its last MMA committed and its epilogue finished."""
import ctypes as C
import sys
from pathlib import Path
import numpy as np
import torch
ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import paper_2202_02870_b200 as L  # noqa: E402
from paper_2202_02870_b200 import _native as nat  # noqa: E402
from paper_2202_02870_b200.engine import LProductPlan  # noqa: E402

lib = nat.lib()
lib.ltb_tc_debug_set_timeline.argtypes = [C.c_void_p]
stream = torch.cuda.Stream(); torch.cuda.set_stream(stream)
nat.check(lib.ltb_ctx_set_stream(nat.context(), stream.cuda_stream))
rng = np.random.default_rng(0)
a_h = rng.standard_normal((256, 128, 3, 32), dtype=np.float32)
b_h = rng.standard_normal((128, 256, 3, 32), dtype=np.float32)
spec = L.make_spec("dct", (256, 256, 3, 32))
plan = LProductPlan(a_h.shape, b_h.shape, spec, np.float32)
a = nat.DeviceArray.from_numpy(a_h); b = nat.DeviceArray.from_numpy(b_h)
c = nat.DeviceArray(plan.c_shape, np.float32)
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
buf = torch.zeros(256 + 2 * 160, dtype=torch.int64, device="cuda")
lib.ltb_tc_debug_set_epi_mode.argtypes = [C.c_int]
epi = int(sys.argv[1]) if len(sys.argv) > 1 else 3
lib.ltb_tc_debug_set_epi_mode(epi)
print("epilogue mode", epi)
for flushed in (True,):
    for ph, label in ((0, "forward A+B (paired)"), (2, "slice GEMM")):
        for rep in range(3):
            plan.run(a, b, c)
            if flushed:
                flush.zero_()
            torch.cuda.synchronize()
            buf.zero_()
            lib.ltb_tc_debug_set_timeline(buf.data_ptr() if rep == 2 else None)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            plan.run(a, b, c, phases=(ph,))
            e1.record(stream)
            torch.cuda.synchronize()
        lib.ltb_tc_debug_set_timeline(None)
        v = buf.cpu().tolist()
        t0 = v[0]
        f = lambda x: f"{(x - t0) / 1e3:6.2f}" if x else "   -  "
        print(f"{label} ({'L2 flushed' if flushed else 'warm'}): event {e0.elapsed_time(e1) * 1e3:.1f} us; "
              f"setup {f(v[1])} first-split {f(v[3])} end {f(v[7])}")
        for j in range(16):
            if v[16 + j] or v[48 + j]:
                print(f"   tile {j:2d}: load {f(v[16 + j])}  mma-done {f(v[32 + j])}  stored {f(v[48 + j])}")
        st = np.array(v[256::2][:148], dtype=np.float64); en = np.array(v[257::2][:148], dtype=np.float64)
        if st.min() > 0:
            z = st.min()
            print(f"   CTA start: min 0 med {(np.median(st) - z) / 1e3:.2f} max {(st.max() - z) / 1e3:.2f} us; "
                  f"end: min {(en.min() - z) / 1e3:.2f} med {(np.median(en) - z) / 1e3:.2f} max {(en.max() - z) / 1e3:.2f} us; "
                  f"CTA0 starts at {(v[0] - z) / 1e3:.2f}")
        for j in range(4):
            if v[160 + 4 * j]:
                print(f"   epilogue warp 8 tile {j}: acc ready {f(v[160 + 4 * j])}  stores issued {f(v[162 + 4 * j])} "
                      f"{f(v[163 + 4 * j])}")
                for ck in range(2):
                    o = 176 + 8 * j + 4 * ck
                    print(f"      chunk {ck}: ld done {f(v[o + 3])} box free {f(v[o])} written {f(v[o + 1])} "
                          f"fenced {f(v[o + 2])}")
        for it in range(16):
            if v[96 + it]:
                print(f"      k-block {it:2d}: landed {f(v[96 + it])}  in TMEM {f(v[64 + it])} (w5 {f(v[128 + it])})  MMA issue {f(v[80 + it])} .. {f(v[112 + it])} ({v[144 + it]} clk)")
