import sys; sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import numpy as np
from paper_2202_02870_b200 import _native as nat
import test_gpu_kernels as T
for forced in (0, 1):
    nat.lib().ltb_debug_set_svd_blocked(forced)
    for dt, shape in [(np.float32, (100, 300)), (np.float32, (300, 100)), (np.float32, (40, 70)), (np.complex64, (60, 90)), (np.float32, (140, 150))]:
        rng = np.random.default_rng(1)
        batch = 2
        a = T.rand(rng, (batch,) + shape, dt)
        m, n = shape
        da = nat.DeviceArray.from_numpy(a)
        u = nat.DeviceArray((batch, m, m), dt); v = nat.DeviceArray((batch, n, n), dt)
        s = nat.DeviceArray((batch, min(m, n)), nat.real_of(dt))
        nat.check(nat.lib().ltb_slice_svd(nat.context(), nat.dtype_code(dt), batch, m, n, da.ptr, u.ptr, s.ptr, v.ptr))
        U, S, V = u.numpy(), s.numpy(), v.numpy()
        eu = np.abs(np.conj(np.swapaxes(U, 1, 2)) @ U - np.eye(m)).max()
        ev = np.abs(np.conj(np.swapaxes(V, 1, 2)) @ V - np.eye(n)).max()
        print(forced, dt.__name__, shape, 'U orth', eu, 'V orth', ev)
