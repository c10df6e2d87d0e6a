import ctypes as C, sys, numpy as np
sys.path.insert(0, '.')
from paper_2202_02870_b200 import _native as nat
lib = nat.lib()
lib.ltb_tc_debug_set_mn_strides.argtypes = [C.c_uint32, C.c_uint32]
def run(a_mn, b_mn, m=128, n=128, k=32, split=3):
    rng = np.random.default_rng(1)
    a = rng.standard_normal((1, m, k)).astype(np.float32); b = rng.standard_normal((1, k, n)).astype(np.float32)
    a_st = np.ascontiguousarray(np.swapaxes(a, 1, 2) if a_mn else a); b_st = np.ascontiguousarray(b if b_mn else np.swapaxes(b, 1, 2))
    da, db = nat.DeviceArray.from_numpy(a_st), nat.DeviceArray.from_numpy(b_st); dc = nat.DeviceArray((1, m, n), np.float32)
    st = lib.ltb_tc_gemm(nat.context(), 1, m, n, k, a_mn, da.ptr, a_st.shape[2], a_st.size, b_mn, db.ptr, b_st.shape[2], b_st.size, dc.ptr, n, m*n, split)
    ref = a[0].astype(np.float64) @ b[0]
    c = dc.numpy()[0]
    return st, np.linalg.norm(c - ref) / np.linalg.norm(ref), c, ref
for lbo, sbo in [(4096, 512), (512, 4096), (4096, 1024), (1024, 4096), (2048, 512), (512, 2048)]:
    lib.ltb_tc_debug_set_mn_strides(lbo, sbo)
    res = [run(am, bm)[1] for am, bm in [(1, 0), (0, 1), (1, 1)]]
    print(lbo, sbo, ["%.2e" % r for r in res])
lib.ltb_tc_debug_set_mn_strides(4096, 512)
st, err, c, ref = run(1, 0)
np.set_printoptions(precision=3, linewidth=150)
print("st", st, "err", err); print(c[:4, :6]); print(ref[:4, :6])
# find mapping: correlate c rows with ref rows
import itertools
cc = np.corrcoef(c.reshape(128, -1), ref.reshape(128, -1))[:128, 128:]
print("row match:", [int(np.argmax(np.abs(cc[i]))) for i in range(0, 128, 8)])
