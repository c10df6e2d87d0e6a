"""A/B of the warm Cholesky-path Jacobi: block pairs (default) vs one pair per team
(LTB_OPT_JACOBI_PAIRS): config-3 PGA it/s over 200 iterations and the K3 kernel's device time
per late iteration (CUPTI)."""
import sys
import time
from collections import defaultdict
from pathlib import Path
import numpy as np
import torch
ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
import paper_2202_02870_b200 as L  # noqa: E402
from paper_2202_02870_b200 import _native as nat  # noqa: E402
from paper_2202_02870_b200.completion import PGASolver, pga_schedule  # noqa: E402

m, mask = bench._cfg3_data_host()
spec = L.make_spec("dct", bench.CFG3["shape"])
cfg = L.CompletionConfig(spec=spec, tol=1e-300, max_iters=200)
mu0 = cfg.nu * L.fro_norm(np.asarray(m, dtype=np.float64))
mus, ts, betas = pga_schedule(cfg, mu0)
for pairs in (2, 0):
    nat.check(nat.lib().ltb_ctx_set_option(nat.context(), nat.OPT_JACOBI_PAIRS, pairs))
    s = PGASolver(np.asarray(m, dtype=np.float64), mask, spec, "fp32")
    nat.sync()
    t0 = time.perf_counter()
    s.run(1, betas[:120], mus[:120], cfg.tol)
    nat.sync()
    with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
        s.run(121, betas[120:125], mus[120:125], cfg.tol)
        nat.sync()
    t1 = time.perf_counter()
    s.run(126, betas[125:], mus[125:], cfg.tol)
    nat.sync()
    t2 = time.perf_counter()
    x = s.result() if hasattr(s, "result") else None
    s.close()
    tot = defaultdict(float)
    for e in prof.events():
        if e.device_type == torch.autograd.DeviceType.CUDA:
            tot[e.name] += e.device_time_total if hasattr(e, "device_time_total") else e.cuda_time_total
    k3 = sum(v for k, v in tot.items() if "jacobi_qr_kernel" in k) / 5
    allk = sum(tot.values()) / 5
    print(f"pairs={pairs}: iterations 126-200 {75 / (t2 - t1):.1f} it/s; late iteration kernels {allk:.1f} us, K3 {k3:.1f} us", flush=True)
nat.check(nat.lib().ltb_ctx_set_option(nat.context(), nat.OPT_JACOBI_PAIRS, 0))
