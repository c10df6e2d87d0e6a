"""Stage timeline (CTA 0, globaltimer) of the warm Cholesky-preconditioned K3 kernel inside a
late config-3 PGA iteration, plus that iteration's sweep statistics."""
import sys
from pathlib import Path
import numpy as np
import torch
ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
import paper_2202_02870_b200 as L  # noqa: E402
from paper_2202_02870_b200 import _native as nat  # noqa: E402
from paper_2202_02870_b200.completion import PGASolver, pga_schedule  # noqa: E402

lib = nat.lib()
m, mask = bench._cfg3_data_host()
spec = L.make_spec("dct", bench.CFG3["shape"])
cfg = L.CompletionConfig(spec=spec, tol=1e-300, max_iters=200)
mu0 = cfg.nu * L.fro_norm(np.asarray(m, dtype=np.float64))
mus, ts, betas = pga_schedule(cfg, mu0)
s = PGASolver(np.asarray(m, dtype=np.float64), mask, spec, "fp32")
buf = torch.zeros(16 + 3 * 300, dtype=torch.int64, device="cuda")
names = ["start", "loaded", "norm check", "factor", "transpose", "sweeps", "emitted", "-", "p0 diag", "p0 trsm", "p0 syrk", "p4 end"]
k = 1
for stop in (30, 60, 120, 180):
    s.run(k, betas[k - 1:stop - 1], mus[k - 1:stop - 1], cfg.tol)
    k = stop
    nat.sync()
    nat.jacobi_stats(reset=True)
    buf.zero_()
    nat.check(lib.ltb_ctx_set_option(nat.context(), nat.OPT_QR_TIMELINE, buf.data_ptr()))
    s.run(k, betas[k - 1:k], mus[k - 1:k], cfg.tol)
    nat.sync()
    nat.check(lib.ltb_ctx_set_option(nat.context(), nat.OPT_QR_TIMELINE, 0))
    k += 1
    sl, sw, mx = nat.jacobi_stats(reset=True, with_max=True)
    v = buf.cpu().tolist()
    print(f"iteration {k - 1}: slices {sl} sweeps/slice {sw / max(sl, 1):.2f} max {mx}; CTA 0:",
          ", ".join(f"{nm} {(v[i] - v[0]) / 1e3:.1f}us" for i, nm in enumerate(names) if v[i]), flush=True)
    c = np.array(v[16:]).reshape(300, 3).astype(np.float64)
    live = c[:, 1] > 0
    if live.any():
        t0 = c[:, 0].min()
        st, en, sw = (c[live, 0] - t0) / 1e3, (c[live, 1] - t0) / 1e3, c[live, 2]
        print(f"   CTAs with sweeps: {live.sum()}; start max {st.max():.1f}us; end min/med/max {en.min():.1f}/{np.median(en):.1f}/{en.max():.1f}us; "
              f"span per sweep count: " + ", ".join(f"{int(k)}: {np.median((en - st)[sw == k]):.1f}us (n={int((sw == k).sum())})" for k in np.unique(sw)), flush=True)
        late = st > 50
        if late.any():
            print(f"   late-starting CTAs: {late.sum()} start {st[late].min():.1f}..{st[late].max():.1f} end {en[late].max():.1f}", flush=True)
s.close()
