import sys; sys.path.insert(0,'/root/repo'); sys.path.insert(0,'/root/repo/tests'); sys.path.insert(0,'/root/repo/oracle')
import numpy as np
import ltensor_oracle as O
import paper_2202_02870_b200 as L
from paper_2202_02870_b200 import _native as nat
from test_gpu_configs import cfg3_data
from conftest import rel_err
m, mask = cfg3_data(shape=(64, 72, 3, 20), rank=4, seed=3)
spec = L.make_spec("dct", m.shape)
ref, recs, _ = O.pga_complete(m, mask, O.ospec("dct", m.shape), tol=1e-300, max_iters=90)
for carry in (0, 1):
    nat.lib().ltb_debug_set_pga_carry(carry)
    for prec in ("fp32", "fp64"):
        x, tr = L.pga_complete(m, mask, L.CompletionConfig(spec=spec, tol=1e-300, max_iters=90), precision=prec)
        print("carry", carry, prec, rel_err(x, ref))
