"""Warm per-kernel device time (CUPTI via torch.profiler) of one config-5 svt / t_svd call
through the public API at n = 128 / 256 / 512 (numpy in / numpy out)."""
import sys
import time
from collections import defaultdict
from pathlib import Path
import numpy as np
import torch
ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import paper_2202_02870_b200 as L  # noqa: E402
from paper_2202_02870_b200 import _native as nat  # noqa: E402

for n in [int(v) for v in (sys.argv[1:] or ["128", "256"])]:
    a = np.random.default_rng(0).standard_normal((n, n, 4, 8, 16), dtype=np.float32)
    spec = L.make_spec("dct", a.shape)
    tau = 0.1 * float(np.median(L.ranks(a, spec).multirank)) if False else 1.0
    for fn, name in ((lambda: L.svt(a, tau, spec), "svt"), (lambda: L.t_svd(a, spec), "t_svd")):
        fn()
        nat.sync()
        t0 = time.perf_counter()
        fn()
        nat.sync()
        wall = time.perf_counter() - t0
        with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
            fn()
            nat.sync()
        tot, cnt = defaultdict(float), defaultdict(int)
        for e in prof.events():
            if e.device_type == torch.autograd.DeviceType.CUDA:
                tot[e.name] += e.device_time_total
                cnt[e.name] += 1
        allt = sum(tot.values())
        print(f"n={n} {name}: wall {wall * 1e3:.1f} ms, device {allt / 1e3:.1f} ms", flush=True)
        for k, t in sorted(tot.items(), key=lambda x: -x[1])[:8]:
            print(f"   {t / 1e3:8.2f} ms x{cnt[k]:<4d} {k[:100]}")
