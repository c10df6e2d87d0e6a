"""Config-2 l_product step: the fused one-launch kernel vs the four-phase path (CUDA graphs,
L2 flushed before every step), plus per-CTA start / end stamps of the fused kernel."""
import sys
from pathlib import Path
import numpy as np
import torch
ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "oracle"))
import paper_2202_02870_b200 as L  # noqa: E402
from paper_2202_02870_b200 import _native as nat  # noqa: E402
from paper_2202_02870_b200.engine import LProductPlan  # noqa: E402
import ltensor_oracle as O  # noqa: E402

stream = torch.cuda.Stream(); torch.cuda.set_stream(stream)
nat.check(nat.lib().ltb_ctx_set_stream(nat.context(), stream.cuda_stream))
rng = np.random.default_rng(0)
a_h = rng.standard_normal((256, 128, 3, 32), dtype=np.float32)
b_h = rng.standard_normal((128, 256, 3, 32), dtype=np.float32)
spec = L.make_spec("dct", (256, 256, 3, 32))
plan = LProductPlan(a_h.shape, b_h.shape, spec, np.float32)
a = nat.DeviceArray.from_numpy(a_h); b = nat.DeviceArray.from_numpy(b_h)
c = nat.DeviceArray(plan.c_shape, np.float32)
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
ref = O.l_product(a_h[:16].astype(np.float64), b_h.astype(np.float64), O.ospec("dct", (16, 256, 3, 32)))
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
flush_modes = {"write-flush": lambda: flush.zero_(), "read-flush": lambda: flush.view(torch.float32).sum(),
               "no-flush": lambda: None}
for name, fn in (("four-phase", lambda: plan.run(a, b, c)), ("fused", lambda: plan.run_fused(a, b, c))):
  for fname, fl in flush_modes.items():
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=stream):
        fn()
    ts = []
    for i in range(30):
        fl()
        ev0.record(stream); g.replay(); ev1.record(stream); ev1.synchronize()
        if i >= 5:
            ts.append(ev0.elapsed_time(ev1) * 1e3)
    err = np.linalg.norm(c.numpy()[:16] - ref) / np.linalg.norm(ref)
    print(f"{name} {fname}: step median {np.median(ts):.2f} us  min {min(ts):.2f}  rel err {err:.2e}", flush=True)
# per-CTA span of the fused kernel
dbg = torch.zeros(2 * 148, dtype=torch.int64, device="cuda")
nat.check(nat.lib().ltb_ctx_set_option(nat.context(), nat.OPT_TC_TIMELINE, dbg.data_ptr()))
flush.zero_(); plan.run_fused(a, b, c); torch.cuda.synchronize()
nat.check(nat.lib().ltb_ctx_set_option(nat.context(), nat.OPT_TC_TIMELINE, 0))
st = dbg.view(148, 2).cpu().numpy().astype(np.float64)
t0 = st[:, 0].min()
print("CTA start us: min %.2f max %.2f; end us: min %.2f median %.2f max %.2f" % (
    0, (st[:, 0].max() - t0) / 1e3, (st[:, 1].min() - t0) / 1e3, (np.median(st[:, 1]) - t0) / 1e3,
    (st[:, 1].max() - t0) / 1e3))
# per-tile timeline of the fused kernel (slots: see ltb_lprod_fused.cuh)
NT = 32
dbg = torch.zeros(512 + 148 * NT * 8 + 48 * 4, dtype=torch.int64, device="cuda")
nat.check(nat.lib().ltb_ctx_set_option(nat.context(), nat.OPT_TC_TIMELINE, dbg.data_ptr()))
flush.zero_(); plan.run_fused(a, b, c); torch.cuda.synchronize()
nat.check(nat.lib().ltb_ctx_set_option(nat.context(), nat.OPT_TC_TIMELINE, 0))
d = dbg.cpu().numpy()
t0 = d[0:296:2].min()
tl = d[512:512 + 148 * NT * 8].reshape(148, NT, 8).astype(np.float64)
kb = (d[512 + 148 * NT * 8:].reshape(48, 4).astype(np.float64) - t0) / 1e3
nF, nG = 512, 384
kinds = {"F": [], "G": [], "I": []}
for cta in range(148):
    for j in range(NT):
        tid = int(tl[cta, j, 0]) - 1
        if tid < 0:
            continue
        k = "F" if tid < nF else ("G" if tid < nF + nG else "I")
        st = (tl[cta, j, 1:7] - t0) / 1e3
        kinds[k].append(st)
for k, v in kinds.items():
    v = np.array(v)
    if not len(v):
        continue
    print(f"{k}: n={len(v)} claim {np.median(v[:,0]):.1f} [{v[:,0].min():.1f},{v[:,0].max():.1f}]  dep-wait med {np.median(v[:,1]-v[:,0]):.2f} max {np.max(v[:,1]-v[:,0]):.2f}  "
          f"claim->lastTMA {np.median(v[:,2]-v[:,0]):.2f}  lastTMA->lastMMA {np.median(v[:,3]-v[:,2]):.2f}  lastMMA->epi {np.median(v[:,4]-v[:,3]):.2f}  epi {np.median(v[:,5]-v[:,4]):.2f}")
cta = 0
print("CTA 0 tiles:")
for j in range(NT):
    tid = int(tl[cta, j, 0]) - 1
    if tid < 0:
        break
    print(tid, np.round((tl[cta, j, 1:7] - t0) / 1e3, 2))
print("CTA 0 k-blocks: TMA issued, landed (converter), TMEM written, MMA issued")
for i in range(48):
    print(i, np.round(kb[i], 2))
# per dependency group: completion (last epilogue done) and first / last claim
print("groups (F: A0, B0, B1, A1 by 128 tiles; G: (mb,nb) by 96; I: (mb,nb) by 128): done-min / done-max / claim-min / claim-max us")
allt = []
for cta in range(148):
    for j in range(NT):
        tid = int(tl[cta, j, 0]) - 1
        if tid >= 0:
            allt.append((tid, (tl[cta, j, 1] - t0) / 1e3, (tl[cta, j, 6] - t0) / 1e3, (tl[cta, j, 2] - t0) / 1e3, cta))
allt = np.array(allt)
bounds = [(0, 128), (128, 256), (256, 384), (384, 512)] + [(512 + 96 * g, 512 + 96 * (g + 1)) for g in range(4)] + \
    [(896 + 128 * g, 896 + 128 * (g + 1)) for g in range(4)]
for lo, hi in bounds:
    sel = allt[(allt[:, 0] >= lo) & (allt[:, 0] < hi)]
    if len(sel):
        print(f"  tiles {lo}-{hi}: n={len(sel)} done {sel[:, 2].min():.2f} / {sel[:, 2].max():.2f}  claim {sel[:, 1].min():.2f} / {sel[:, 1].max():.2f}  deps met {sel[:, 3].min():.2f} / {np.median(sel[:, 3]):.2f} / {sel[:, 3].max():.2f}")
        k = int(np.argmax(sel[:, 2]))
        print(f"    last done: tile {int(sel[k, 0])} on CTA {int(sel[k, 4])}")
