"""Benchmark of the B200 *_L hot path (contract: see DESIGN.md §Measurement).

Headline (BASELINE.json configs[1], "config 2"): the 4th-order *_L-product
A 256x128x3x32 * B 128x256x3x32, float32 N(0,1), L = DCT along modes 3 and 4,
in GFLOP/s on the algorithmic count of SURVEY.md §8(d) (2,491,416,576 flop per
product).  One step = one product with A, B resident in HBM; L2 is flushed
(512 MiB write) between timed steps.  `e2e` is the same metric through the
public numpy-in / numpy-out API (host copies inside the timed region).

Secondary (BASELINE configs[2], "config 3"): PGA completion iterations/s on the
synthetic 144x176x3x100 colour-video stand-in (tol 1e-300, 200 iterations),
reported in the "pga" object.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
"""

from __future__ import annotations

import argparse
import contextlib
import json
import math
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

CFG2 = dict(a=(256, 128, 3, 32), b=(128, 256, 3, 32), kind="dct")
CFG3 = dict(shape=(144, 176, 3, 100), rank=10, sr=0.2, iters=200)
GFLOP_CFG2 = 2_491_416_576
# the `config` object both arms print (identical, so the driver can pair the lines)
CONFIG2 = {"workload": "config2 l_product A 256x128x3x32 * B 128x256x3x32, DCT modes 3,4",
           "flop_per_step": GFLOP_CFG2}
L2_NOTE = "flushed (512 MiB write) before every timed step"


def _peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), float(d["bf16_tflops"]), "measured"
    return 6650.0, 1590.0, "fallback"


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def _cfg2_inputs(seed=0):
    rng = np.random.default_rng(seed)
    a = rng.standard_normal(CFG2["a"], dtype=np.float32)
    b = rng.standard_normal(CFG2["b"], dtype=np.float32)
    return a, b


def _cpu_info():
    info = {"cores": len(os.sched_getaffinity(0))}
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                info["cpu"] = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    try:
        from threadpoolctl import threadpool_info

        info["blas_threads"] = max((t.get("num_threads", 1) for t in threadpool_info()), default=1)
    except Exception:
        info["blas_threads"] = info["cores"]
    return info


# ----------------------------------------------------------------------------- CPU (oracle) legs
@contextlib.contextmanager
def _host_threads():
    """Every host core this process may run on for the CPU legs: BLAS threads and
    scipy.fft workers (torchrun sets OMP_NUM_THREADS=1 per rank; the CPU legs run on
    rank 0 alone, so they take the whole host)."""
    n = len(os.sched_getaffinity(0))
    with contextlib.ExitStack() as st:
        try:
            from threadpoolctl import threadpool_limits

            st.enter_context(threadpool_limits(limits=n))
        except Exception:
            pass
        import scipy.fft

        st.enter_context(scipy.fft.set_workers(n))
        yield


def cpu_lproduct(steps: int, warmup: int, budget_s: float | None = None):
    """The reference algorithm (oracle port) on the host cores, seconds per product."""
    sys.path.insert(0, str(ROOT / "oracle"))
    import ltensor_oracle as O

    a, b = _cfg2_inputs()
    spec = O.ospec("dct", (256, 256, 3, 32))
    for _ in range(warmup):
        O.l_product(a, b, spec)
    times = []
    t_end = time.perf_counter() + budget_s if budget_s else None
    while True:
        t0 = time.perf_counter()
        O.l_product(a, b, spec)
        times.append(time.perf_counter() - t0)
        if t_end is None and len(times) >= steps:
            break
        if t_end is not None and time.perf_counter() >= t_end and len(times) >= 3:
            break
    return times


def cpu_pga_iters(iters: int):
    sys.path.insert(0, str(ROOT / "oracle"))
    import ltensor_oracle as O

    m, mask = _cfg3_data_host()
    spec = O.ospec("dct", CFG3["shape"])
    t0 = time.perf_counter()
    O.pga_complete(m, mask, spec, tol=1e-300, max_iters=iters)
    return (time.perf_counter() - t0) / iters


def _cfg3_data_host():
    """Config 3 synthetic stand-in: A 144x10x3x100, B 10x176x3x100 N(0,1) f32, X0 = A *_L B
    (DCT, f64), rescaled to [0,1], + N(0, 0.01) noise (std 0.01), f32; Bernoulli(0.2) mask; seed 0."""
    rng = np.random.default_rng(0)
    i1, i2, c, t = CFG3["shape"]
    a = rng.standard_normal((i1, CFG3["rank"], c, t), dtype=np.float32).astype(np.float64)
    b = rng.standard_normal((CFG3["rank"], i2, c, t), dtype=np.float32).astype(np.float64)
    import scipy.fft

    # X0 = A *_L B with the separable DCT, computed with scipy (input synthesis only)
    ah = scipy.fft.dctn(a, type=2, axes=(2, 3), norm="ortho")
    bh = scipy.fft.dctn(b, type=2, axes=(2, 3), norm="ortho")
    xh = np.einsum("ikct,kjct->ijct", ah, bh)
    x0 = scipy.fft.idctn(xh, type=2, axes=(2, 3), norm="ortho")
    x0 = (x0 - x0.min()) / (x0.max() - x0.min())
    m = (x0 + rng.normal(0.0, 0.01, x0.shape)).astype(np.float32)
    mask = rng.random(m.shape) < CFG3["sr"]
    return m, mask


def run_reference(args):
    ws, rank, _ = _dist()
    if rank != 0:
        return
    times = cpu_lproduct(args.steps, args.warmup)
    info = _cpu_info()
    total = sum(times)
    value = GFLOP_CFG2 * len(times) / total / 1e9
    line = {
        "impl": "reference",
        "metric": "*_L-product GFLOP/s",
        "value": value,
        "unit": "GFLOP/s",
        "n_gpus": args.gpus,
        "steps": len(times),
        "warmup": args.warmup,
        "ms_per_step": 1e3 * total / len(times),
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f32",
        "data": "synthetic N(0,1) seed 0 (BASELINE config 2 shapes)",
        "config": dict(CONFIG2),
        "cpu_baseline": {"value": value, "unit": "GFLOP/s", "cores": info["blas_threads"], "kind": "port",
                         "sample": f"{len(times)} full config-2 products (oracle/ltensor_oracle.py, numpy/scipy "
                                   f"OpenBLAS), {info.get('cpu', '?')}"},
        "e2e": {"value": value, "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- clocks sampler
class ClockSampler:
    def __init__(self, index: int):
        self.samples = []
        self.proc = None
        self.index = index

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 7:
                self.samples.append(parts)

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[3 + i] == "Active"})
        loaded = [v for v in sm if v > 0.5 * max(sm)] if sm else []
        return {"sm_mhz": float(np.median(loaded)) if loaded else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


# ----------------------------------------------------------------------------- our arm
def run_ours_dist(args):
    """N > 1: config 2 strong-scaled (the same global product at every N).  Rows of A *_L B depend
    only on the same rows of A and on all of B, so rank g computes the i1-row block R_g of C from
    its rows of A and a full copy of B: K1(A_g), K1(B), the slice GEMM, K1'(C_g).  Transforming B
    on every rank (12.6 MB read + write, ~6 us) replaces the B-hat all-gather of
    distributed.DistLProductPlan (11 MB received per rank over NVLink, plus the collective's
    latency), so the step has no data-path collective.  Time = max over ranks of the device
    (CUDA-event) step time; the job's work is the one config-2 product."""
    import torch
    import torch.distributed as dist

    ws, rank, local = _dist()
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_2202_02870_b200 as L
    from paper_2202_02870_b200 import _native as nat
    from paper_2202_02870_b200.distributed import DeviceEngine, blocks
    from paper_2202_02870_b200.engine import LProductPlan

    nat.set_device(local)
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    nat.check(nat.lib().ltb_ctx_set_stream(nat.context(), stream.cuda_stream))
    spec = L.make_spec("dct", (256, 256, 3, 32))
    a_full, b_h = _cfg2_inputs(seed=0)
    r0, r1 = blocks(256, ws)[rank]
    a_h = np.ascontiguousarray(a_full[r0:r1])
    plan = LProductPlan(a_h.shape, b_h.shape, spec, np.float32)
    a = nat.DeviceArray.from_numpy(a_h)
    b = nat.DeviceArray.from_numpy(b_h)
    c = nat.DeviceArray(plan.c_shape, np.float32)
    flush = torch.empty(512 * 1024 * 1024, dtype=torch.uint8, device="cuda")
    # parity gate: this rank's rows of C against the oracle on a bounded row sample
    plan.run_fused(a, b, c)
    torch.cuda.synchronize()
    gate = _parity_gate(c.numpy(), a_h, b_h)
    for _ in range(2):
        plan.run_fused(a, b, c)
    torch.cuda.synchronize()
    l0 = nat.launch_count()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=stream):
        plan.run_fused(a, b, c)
    launches_per_step = nat.launch_count() - l0
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    times = []
    with ClockSampler(local) as clocks:
        for i in range(args.warmup + args.steps):
            flush.zero_()
            dist.barrier()
            torch.cuda.synchronize()
            e0.record(stream)
            graph.replay()
            e1.record(stream)
            e1.synchronize()
            if i >= args.warmup:
                times.append(e0.elapsed_time(e1) / 1e3)
        launches = launches_per_step * args.steps
        # e2e through the public API per rank: its rows of A and all of B from pinned host
        # memory, its rows of C back to pinned host memory (wall time, max over ranks)
        a_pin = torch.empty(a_h.shape, dtype=torch.float32, pin_memory=True).numpy()
        b_pin = torch.empty(b_h.shape, dtype=torch.float32, pin_memory=True).numpy()
        c_pin = torch.empty(plan.c_shape, dtype=torch.float32, pin_memory=True).numpy()
        a_pin[...] = a_h
        b_pin[...] = b_h
        e2e_times = []
        for i in range(args.warmup + args.steps):
            dist.barrier()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            L.l_product(a_pin, b_pin, spec, out=c_pin)
            if i >= args.warmup:
                e2e_times.append(time.perf_counter() - t0)
    pga = None if (args.skip_extras or args.skip_pga) else bench_pga_dist(L, torch, dist, eng_cls=DeviceEngine,
                                                                          args=args)
    t = torch.tensor([sum(times), sum(e2e_times), gate["rel_err"]], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    t_step, t_e2e, worst = float(t[0].item()), float(t[1].item()), float(t[2].item())
    gate = {"rows_checked_per_rank": gate["rows_checked"], "rel_err_max_over_ranks": worst,
            "tol": 1e-4, "ok": worst < 1e-4}
    hbm_peak, _, peak_src = _peaks()
    E_b = 128 * 256 * 96
    # rank-local fused bytes: its A rows, all of B, its C rows (one read / write each)
    alg_bytes = 4 * ((r1 - r0) * 128 * 96 + E_b + (r1 - r0) * 256 * 96)
    achieved = alg_bytes * args.steps / t_step / 1e9
    line = {
        "metric": "*_L-product GFLOP/s", "value": GFLOP_CFG2 * args.steps / t_step / 1e9, "unit": "GFLOP/s",
        "n_gpus": ws, "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t_step / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic N(0,1) seed 0 (BASELINE config 2 shapes)",
        "config": dict(CONFIG2), "l2": L2_NOTE,
        "parallelism": f"A / C rows sharded x{ws}, B transformed on every rank (no data-path collective)",
        "parity_gate": gate,
        "roofline": {"kernel": "whole rank-local step (fused bytes)", "bound": "hbm", "achieved": achieved,
                     "peak": hbm_peak, "unit": "GB/s", "frac": achieved / hbm_peak,
                     "peak_source": f"{peak_src} HBM copy", "traffic": None},
        "e2e": {"value": GFLOP_CFG2 * len(e2e_times) / t_e2e / 1e9, "unit": "GFLOP/s",
                "h2d_bytes_per_step": int(4 * (256 * 128 * 96 + ws * E_b)),
                "d2h_bytes_per_step": int(4 * 256 * 256 * 96),
                "api": "paper_2202_02870_b200.l_product(numpy, numpy, spec, out=numpy) per rank on pinned host "
                       "arrays (its rows of A, all of B); bytes summed over ranks"},
        "gpu_launches": int(launches), "clocks": clocks.summary(),
    }
    if pga is not None:
        line["pga"] = pga
    if rank == 0:
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()


def _parity_gate(c_rows: np.ndarray, a_rows: np.ndarray, b: np.ndarray, nrows: int = 8) -> dict:
    """Bounded correctness gate of a bench run: the first `nrows` rows of C (rows of A *_L B
    depend only on the same rows of A) against the oracle in float64, relative Frobenius."""
    sys.path.insert(0, str(ROOT / "oracle"))
    import ltensor_oracle as O

    r = min(nrows, a_rows.shape[0])
    ref = O.l_product(a_rows[:r].astype(np.float64), b.astype(np.float64), O.ospec("dct", (r,) + b.shape[1:]))
    err = float(np.linalg.norm((c_rows[:r] - ref).ravel()) / np.linalg.norm(ref.ravel()))
    return {"rows_checked": r, "rel_err": err, "tol": 1e-4, "ok": err < 1e-4}


def bench_pga_dist(L, torch, dist, eng_cls, args):
    """Config-3 PGA over all ranks (SURVEY.md §8(e), strong scaling): rank g owns a block of
    i1 rows for the transforms and gradient step and a block of slices for K3; the layout
    change is an NCCL all-to-all each way per iteration.  Time = max over ranks."""
    from paper_2202_02870_b200.distributed import blocks, dist_pga_complete

    ws, rank = dist.get_world_size(), dist.get_rank()
    m, mask = _cfg3_data_host()
    spec = L.make_spec("dct", CFG3["shape"])
    r0, r1 = blocks(m.shape[0], ws)[rank]
    mu0 = 0.9 * float(np.linalg.norm(m.astype(np.float64)))  # cfg.nu * ||M||_F over the full tensor
    eng = eng_cls(spec, m.shape[2:])
    mt = torch.from_numpy(np.ascontiguousarray(m[r0:r1])).cuda()
    kt = torch.from_numpy(np.ascontiguousarray(mask[r0:r1])).cuda()
    res = None
    for n in (3, args.pga_iters):  # warm-up run, then the timed run
        cfg = L.CompletionConfig(spec=spec, tol=1e-300, max_iters=n)
        torch.cuda.synchronize()
        dist.barrier()
        t0 = time.perf_counter()
        x, trace = dist_pga_complete(mt, kt, cfg, m.shape[0], eng, mu0=mu0)
        torch.cuda.synchronize()
        t = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        res = (trace.iterations, float(t[0]))
    its, secs = res
    return {"metric": "PGA completion iters/sec", "value": its / secs, "unit": "it/s", "iterations": its,
            "seconds": secs, "dtype": "f32", "scaling": "strong", "n_gpus": ws,
            "timing": "device-synchronised wall time of the whole solve, max over ranks",
            "config": {"workload": "config3 144x176x3x100 rank-10 DCT(modes 3,4), Bernoulli(0.2), tol 1e-300",
                       "parallelism": f"i1 rows x{ws} (K1, K1', gradient) / slices x{ws} (K3), NCCL all-to-all",
                       "data": "synthetic stand-in for the paper's colour videos (not in this container)"}}


def run_ours(args):
    import torch

    ws, rank, local = _dist()
    if ws > 1 or args.force_dist:
        return run_ours_dist(args)
    torch.cuda.set_device(local)
    import paper_2202_02870_b200 as L
    from paper_2202_02870_b200 import _native as nat
    from paper_2202_02870_b200.engine import LProductPlan

    nat.set_device(local)
    # one explicit (non-default) stream shared by torch (events, L2 flush) and libltb
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    nat.check(nat.lib().ltb_ctx_set_stream(nat.context(), stream.cuda_stream))

    hbm_peak, tf_peak, peak_src = _peaks()
    spec = L.make_spec("dct", (256, 256, 3, 32))
    a_h, b_h = _cfg2_inputs(seed=rank)
    plan = LProductPlan(a_h.shape, b_h.shape, spec, np.float32)
    a = nat.DeviceArray.from_numpy(a_h)
    b = nat.DeviceArray.from_numpy(b_h)
    c = nat.DeviceArray(plan.c_shape, np.float32)
    flush = torch.empty(512 * 1024 * 1024, dtype=torch.uint8, device="cuda")

    # ---- correctness gate: the first product's leading rows of C against the oracle (float64)
    plan.run(a, b, c)
    torch.cuda.synchronize()
    gate = _parity_gate(c.numpy(), a_h, b_h)

    def barrier():
        if ws > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()

    ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
    step_ms = []
    # the step is the product path: ONE persistent tcgen05 kernel (forward transforms, slice
    # GEMMs, inverse transform; ltb_l_product_device, csrc/ltb_lprod_fused.cuh) captured as a
    # CUDA graph and replayed.  The four-launch path (K1(A,B), K2, K1') is timed beside it, as a
    # whole and per phase (one graph per phase, CUDA events between the replays)
    for _ in range(2):
        plan.run_fused(a, b, c)  # settle kernel attributes / tensor-map caches before capture
        plan.run(a, b, c)
    torch.cuda.synchronize()
    gate_fused = _parity_gate(c.numpy(), a_h, b_h)
    l0 = nat.launch_count()
    full = torch.cuda.CUDAGraph()
    with torch.cuda.graph(full, stream=stream):
        plan.run_fused(a, b, c)
    launches_per_step = nat.launch_count() - l0
    four = torch.cuda.CUDAGraph()
    with torch.cuda.graph(four, stream=stream):
        plan.run(a, b, c)
    four_ms = []
    # per-phase graphs (K1 of A and B is one launch when the plan pairs them)
    E_a, E_b, E_c = 256 * 128 * 96, 128 * 256 * 96, 256 * 256 * 96
    phase_defs = {0: ("transform_fwd_A", 8 * E_a, 70 * E_a, "one f32 read + one write of A"),
                  1: ("transform_fwd_B", 8 * E_b, 70 * E_b, "one f32 read + one write of B"),
                  2: ("slice_gemm", 4 * (E_a + E_b + E_c), 2 * 256 * 128 * 256 * 96,
                      "f32 reads of A-hat, B-hat and the write of C-hat"),
                  3: ("transform_inv_C", 8 * E_c, 70 * E_c, "one f32 read + one write of C")}
    if plan.paired:
        phase_defs[0] = ("transform_fwd_AB", 8 * (E_a + E_b), 70 * (E_a + E_b),
                         "one f32 read + one write of A and of B (one launch)")
        del phase_defs[1]
    phase_ids = sorted(phase_defs)
    graphs = []
    for ph in phase_ids:
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=stream):
            plan.run(a, b, c, phases=(ph,))
        graphs.append(g)
    nph = len(graphs)
    phase_ms = np.zeros(nph)

    def phases(marks):
        for i, g in enumerate(graphs):
            marks(i)
            g.replay()
        marks(nph)

    with ClockSampler(local) as clocks:
        for _ in range(args.warmup):
            flush.zero_()
            full.replay()
        barrier()
        for _ in range(args.steps):
            flush.zero_()  # L2 flush outside the timed events
            ev[0].record(stream)
            full.replay()
            ev[1].record(stream)
            ev[1].synchronize()
            step_ms.append(ev[0].elapsed_time(ev[1]))
        barrier()
        for _ in range(args.steps):
            flush.zero_()
            ev[0].record(stream)
            four.replay()
            ev[1].record(stream)
            ev[1].synchronize()
            four_ms.append(ev[0].elapsed_time(ev[1]))
        for _ in range(args.steps):
            flush.zero_()
            phases(lambda i: ev[i].record(stream))
            ev[nph].synchronize()
            phase_ms += [ev[i].elapsed_time(ev[i + 1]) for i in range(nph)]
        launches = launches_per_step * args.steps
        # e2e: public numpy-in/numpy-out API from / to pinned host buffers, host copies inside the timed region
        a_pin = torch.empty(a_h.shape, dtype=torch.float32, pin_memory=True).numpy()
        b_pin = torch.empty(b_h.shape, dtype=torch.float32, pin_memory=True).numpy()
        c_pin = torch.empty(plan.c_shape, dtype=torch.float32, pin_memory=True).numpy()
        a_pin[...] = a_h
        b_pin[...] = b_h
        e2e_t = []
        for i in range(args.warmup + args.steps):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            out = L.l_product(a_pin, b_pin, spec, out=c_pin)
            dt = time.perf_counter() - t0
            if i >= args.warmup:
                e2e_t.append(dt)
        # the drop-in call exactly as a reference user makes it: plain (pageable) numpy arrays in,
        # a new numpy array out, no `out=` (the library stages pageable buffers through pinned memory)
        e2e_pg = []
        for i in range(args.warmup + args.steps):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            res = L.l_product(a_h, b_h, spec)
            dt = time.perf_counter() - t0
            if i >= args.warmup:
                e2e_pg.append(dt)
        gate_e2e = _parity_gate(res, a_h, b_h)
        pga = None if args.skip_pga else bench_pga(L, nat, torch, args)
        extras = None if args.skip_extras else bench_extras(L, nat, torch, args, cpu=not args.no_cpu_baseline)

    t_step = float(np.sum(step_ms)) / 1e3
    if ws > 1:
        tt = torch.tensor([t_step], device="cuda", dtype=torch.float64)
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        t_step = float(tt.item())
        te = torch.tensor([sum(e2e_t)], device="cuda", dtype=torch.float64)
        torch.distributed.all_reduce(te, op=torch.distributed.ReduceOp.MAX)
        e2e_total = float(te.item())
    else:
        e2e_total = sum(e2e_t)
    value = ws * GFLOP_CFG2 * args.steps / t_step / 1e9
    e2e_value = ws * GFLOP_CFG2 * len(e2e_t) / e2e_total / 1e9

    # roofline of the step's one kernel: the whole product's algorithmic bytes (one read of A
    # and B, one write of C: SURVEY.md section 8(d), 50,331,648 B) over its device time (CUDA
    # events on the launching stream around the graph, which holds only that kernel)
    t_kernel = t_step / args.steps
    fused_bytes = 4 * (E_a + E_b + E_c)
    achieved = fused_bytes / t_kernel / 1e9
    roof = {"kernel": "lprod_fused_kernel (the whole product, one launch)", "bound": "hbm", "achieved": achieved,
            "peak": hbm_peak, "unit": "GB/s", "frac": achieved / hbm_peak,
            "peak_source": f"{peak_src} HBM copy (MEASURED_PEAKS.json)",
            "alg_per_launch": f"{fused_bytes} B (A and B read once, C written once)",
            "traffic": _ncu_traffic("lprod_fused_kernel"),
            # the three-phase algorithm moves every transform-domain stack through memory:
            # A, B, A-hat, B-hat, C-hat, C once each = 151 MB ("unfused")
            "phase_level_bytes": 4 * 3 * (E_a + E_b + E_c),
            "phase_level_frac": 4 * 3 * (E_a + E_b + E_c) / t_kernel / 1e9 / hbm_peak}
    names = [phase_defs[i][0] for i in phase_ids]
    phase_avg = phase_ms / args.steps
    four_phase = {"ms_per_step": float(np.mean(four_ms)),
                  "phase_ms": dict(zip(names, [round(float(x), 5) for x in phase_avg])),
                  "note": "the four-launch path (K1(A,B) paired, K2, K1') on the same buffers, for comparison"}

    line = {
        "metric": "*_L-product GFLOP/s",
        "value": value,
        "unit": "GFLOP/s",
        "n_gpus": ws,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": 1e3 * t_step / args.steps,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f32",
        "data": "synthetic N(0,1) (BASELINE config 2 shapes), seed = rank",
        "config": dict(CONFIG2),
        "l2": L2_NOTE,
        "parallelism": "single GPU",
        "parity_gate": {"device_step": gate_fused, "four_phase": gate, "e2e_pageable": gate_e2e,
                        "ok": gate["ok"] and gate_fused["ok"] and gate_e2e["ok"]},
        "roofline": roof,
        "four_phase": four_phase,
        "e2e": {"value": e2e_value, "unit": "GFLOP/s", "h2d_bytes_per_step": int(a_h.nbytes + b_h.nbytes),
                "d2h_bytes_per_step": int(out.nbytes), "api": "paper_2202_02870_b200.l_product(numpy, numpy, spec, out=numpy) on pinned host arrays"},
        "e2e_pageable": {"value": GFLOP_CFG2 * len(e2e_pg) / sum(e2e_pg) / 1e9, "unit": "GFLOP/s",
                         "h2d_bytes_per_step": int(a_h.nbytes + b_h.nbytes), "d2h_bytes_per_step": int(res.nbytes),
                         "ms_per_step": 1e3 * sum(e2e_pg) / len(e2e_pg),
                         "api": "paper_2202_02870_b200.l_product(a, b, spec) on plain pageable numpy arrays, "
                                "new numpy result (the reference's own signature)"},
        "gpu_launches": int(launches),
        "clocks": clocks.summary(),
    }
    if pga is not None:
        line["pga"] = pga
    if extras is not None:
        line["configs"] = extras
    if rank == 0 and not args.no_cpu_baseline:
        times = cpu_lproduct(1, 1, budget_s=args.cpu_budget)
        info = _cpu_info()
        line["cpu_baseline"] = {"value": GFLOP_CFG2 * len(times) / sum(times) / 1e9, "unit": "GFLOP/s",
                                "cores": info["blas_threads"], "kind": "port",
                                "sample": f"{len(times)} full config-2 products in ~{args.cpu_budget:.0f}s "
                                          f"(oracle port, numpy/scipy OpenBLAS), {info.get('cpu', '?')}"}
        if pga is not None and args.cpu_pga_iters > 0:
            s_it = cpu_pga_iters(args.cpu_pga_iters)
            line["pga"]["cpu_baseline"] = {"value": 1.0 / s_it, "unit": "it/s", "cores": info["blas_threads"],
                                           "kind": "port",
                                           "sample": f"{args.cpu_pga_iters} PGA iterations of config 3 (float64, "
                                                     "as the reference computes)"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if ws > 1:
        torch.distributed.destroy_process_group()


def _ncu_traffic(kernel):
    """dram bytes read + written per launch of `kernel` from the committed ncu captures
    (profiles/r02_traffic.json, then r01_traffic.json; see profiles/rNN_ncu_summary.md), or None."""
    for name in ("r02_traffic.json", "r01_traffic.json"):
        try:
            v = json.load(open(ROOT / "profiles" / name)).get(kernel)
        except (OSError, ValueError):
            v = None
        if v is not None:
            return v
    return None


def bench_pga(L, nat, torch, args):
    m, mask = _cfg3_data_host()
    spec = L.make_spec("dct", CFG3["shape"])
    from paper_2202_02870_b200.completion import PGASolver, pga_schedule

    cfg = L.CompletionConfig(spec=spec, tol=1e-300, max_iters=args.pga_iters)
    mu0 = cfg.nu * L.fro_norm(np.asarray(m, dtype=np.float64))
    mus, ts, betas = pga_schedule(cfg, mu0)
    solver = PGASolver(np.asarray(m, dtype=np.float64), mask, spec, "fp32")
    # warm-up: a separate solver run of a few iterations
    warm = PGASolver(np.asarray(m, dtype=np.float64), mask, spec, "fp32")
    warm.run(1, betas[:3], mus[:3], cfg.tol)
    warm.close()
    torch.cuda.synchronize()
    nat.jacobi_stats(reset=True)
    t0 = time.perf_counter()
    n_done = 0
    k = 1
    while k <= cfg.max_iters:
        n = min(50, cfg.max_iters - k + 1)
        recs, conv = solver.run(k, betas[k - 1:k - 1 + n], mus[k - 1:k - 1 + n], cfg.tol)
        k += len(recs)
        n_done += len(recs)
        if conv:
            break
    dt = time.perf_counter() - t0
    slices, sweeps = nat.jacobi_stats(reset=True)
    x = solver.fetch(False)
    solver.close()
    # K3 alone on a late-iteration-sized problem: the config-3 transform-domain stack of the
    # observed data at tau = mu_150, timed on the device (nominal SVD flops)
    hat = L.linalg._hat_stack(np.where(mask, m, 0).astype(np.float32), spec)
    P3, i1, i2 = hat.shape
    hout = nat.DeviceArray(hat.shape, hat.dtype)
    tau = float(mus[min(149, len(mus) - 1)])
    for _ in range(2):
        nat.check(nat.lib().ltb_slice_svt(nat.context(), hat.code, P3, i1, i2, hat.ptr, tau, hout.ptr))
    nat.sync()
    t0 = time.perf_counter()
    nat.check(nat.lib().ltb_slice_svt(nat.context(), hat.code, P3, i1, i2, hat.ptr, tau, hout.ptr))
    nat.sync()
    t_k3 = time.perf_counter() - t0
    mm, nn = max(i1, i2), min(i1, i2)
    k3_flop = P3 * (6 * mm * nn * nn + 20 * nn ** 3 + 2 * mm * nn * nn)
    fp32_peak = 74.4
    roof = {"kernel": "K3 SVT (QR-preconditioned one-sided Jacobi + recomposition)", "bound": "fp32",
            "achieved": k3_flop / t_k3 / 1e12, "peak": fp32_peak, "unit": "TFLOP/s",
            "frac": k3_flop / t_k3 / 1e12 / fp32_peak,
            "traffic": _ncu_traffic("K3 SVT (QR-preconditioned one-sided Jacobi + recomposition)"),
            "alg_per_launch": f"{k3_flop} flop nominal (300 slices x (6mn^2 + 20n^3 + 2mn^2))",
            "peak_source": "FP32 FFMA nominal 148 SM x 128 x 2 x 1.965 GHz (SURVEY.md §8(d))",
            "k3_ms": t_k3 * 1e3,
            "iteration_ceiling_it_s": 2466, "iteration_frac": (n_done / dt) / 2466,
            "ceiling_source": "SURVEY.md §8(d): max(HBM 305.1 MB, 26.67 GFLOP) per iteration"}
    # the same run at the reference's precision (completion.py:154 computes in float64), the
    # like-for-like pair of the float64 CPU baseline
    _run_pga(L, nat, torch, m, mask, spec, "fp64", 3)
    fp64 = {"value": _run_pga(L, nat, torch, m, mask, spec, "fp64", args.pga_iters), "unit": "it/s",
            "dtype": "f64", "iterations": args.pga_iters,
            "note": "precision='fp64': float64 transforms, Jacobi SVT and recomposition (the reference's precision)"}
    return {"metric": "PGA completion iters/sec", "value": n_done / dt, "unit": "it/s", "iterations": n_done,
            "seconds": dt, "dtype": "f32", "fp64": fp64,
            "jacobi_sweeps_per_slice": sweeps / max(slices, 1), "roofline": roof,
            "config": {"workload": "config3 144x176x3x100 rank-10 DCT(modes 3,4), Bernoulli(0.2), tol 1e-300",
                       "data": "synthetic stand-in for the paper's colour videos (not in this container)"},
            "rse_vs_m": float(np.linalg.norm(x - m) ** 2 / max(np.linalg.norm(x) ** 2, 1e-300))}


def _run_pga(L, nat, torch, m, mask, spec, precision, iters, **cfg_kw):
    """Device-resident PGA run through the solver (setup and fetch outside the timed region)."""
    from paper_2202_02870_b200.completion import PGASolver, pga_schedule

    cfg = L.CompletionConfig(spec=spec, tol=1e-300, max_iters=iters, **cfg_kw)
    m64 = np.asarray(m, dtype=np.float64)
    mu0 = cfg.nu * L.fro_norm(m64) if cfg.mu0 is None else cfg.mu0
    mus, ts, betas = pga_schedule(cfg, mu0)
    solver = PGASolver(m64, mask, spec, precision)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    k = 1
    while k <= iters:
        n = min(50, iters - k + 1)
        recs, _ = solver.run(k, betas[k - 1:k - 1 + n], mus[k - 1:k - 1 + n], cfg.tol)
        k += len(recs)
    dt = time.perf_counter() - t0
    solver.close()
    return iters / dt


def bench_extras(L, nat, torch, args, cpu):
    """The other BASELINE configs (parity is in tests/test_gpu_configs.py): config 1 PGA (fp64),
    config 5 svt / t_svd at n = 128, 256, 512, config 4 PGA at full size (all 50 iterations)."""
    import torch as _t

    sys.path.insert(0, str(ROOT / "oracle"))
    import ltensor_oracle as O

    out = {}
    # ---- config 1: 64x64x16 f64, DCT, mu == 0.01, 100 iterations
    rng = np.random.default_rng(0)
    a1 = rng.standard_normal((64, 5, 16))
    b1 = rng.standard_normal((5, 64, 16))
    spec1 = L.make_spec("dct", (64, 64, 16))
    m1 = L.l_product(a1, b1, spec1)
    mask1 = rng.random(m1.shape) < 0.5
    kw1 = dict(mu0=0.01, mu_bar_ratio=1.0)
    _run_pga(L, nat, torch, m1, mask1, spec1, "fp64", 5, **kw1)  # warm-up
    c1 = {"metric": "PGA completion iters/sec", "value": _run_pga(L, nat, torch, m1, mask1, spec1, "fp64", 100, **kw1),
          "unit": "it/s", "dtype": "f64", "config": "config1 64x64x16 DCT, tubal rank 5, Bernoulli(0.5), mu=0.01, 100 it"}
    if cpu:
        t0 = time.perf_counter()
        O.pga_complete(m1, mask1, O.ospec("dct", m1.shape), mu0=0.01, mu_bar_ratio=1.0, tol=1e-300, max_iters=20)
        c1["cpu_baseline"] = {"value": 20 / (time.perf_counter() - t0), "unit": "it/s", "kind": "port",
                              "cores": _cpu_info()["blas_threads"], "sample": "20 iterations of config 1 (float64)"}
    out["config1_pga"] = c1
    # ---- config 5: n x n x 4 x 8 x 16 f32, DCT^3, svt at tau = 0.1 median sv, t_svd
    c5 = {}
    for n in (128, 256, 512):
        rng = np.random.default_rng(0)
        a5 = rng.standard_normal((n, n, 4, 8, 16), dtype=np.float32)
        spec5 = L.make_spec("dct", a5.shape)
        sv = L.linalg._singular_values(a5, spec5)
        tau = 0.1 * float(np.median(sv))
        _t.cuda.synchronize()
        t_svt = t_tsvd = float("inf")
        for _ in range(2):  # best of two: the first call of a shape grows the workspace pool
            t0 = time.perf_counter()
            L.svt(a5, tau, spec5)
            t_svt = min(t_svt, time.perf_counter() - t0)
        for _ in range(2 if n < 512 else 1):
            t0 = time.perf_counter()
            L.t_svd(a5, spec5)
            t_tsvd = min(t_tsvd, time.perf_counter() - t0)
        # K3 alone on the device-resident transform-domain stack (no host copies, no transforms)
        hat = L.linalg._hat_stack(a5, spec5)
        hout = nat.DeviceArray(hat.shape, hat.dtype)
        P5, i1, i2 = hat.shape
        nat.check(nat.lib().ltb_slice_svt(nat.context(), hat.code, P5, i1, i2, hat.ptr, tau, hout.ptr))
        nat.sync()
        nat.jacobi_stats(reset=True)
        t0 = time.perf_counter()
        nat.check(nat.lib().ltb_slice_svt(nat.context(), hat.code, P5, i1, i2, hat.ptr, tau, hout.ptr))
        nat.sync()
        t_k3 = time.perf_counter() - t0
        sl, sw = nat.jacobi_stats(reset=True)
        gflop_svd = 512 * 26 * n ** 3 / 1e9
        entry = {"svt_s": t_svt, "t_svd_s": t_tsvd, "svt_nominal_gflops": (gflop_svd + 512 * 2 * n ** 3 / 1e9) / t_svt,
                 "t_svd_nominal_gflops": gflop_svd / t_tsvd, "tau": tau,
                 "note": "svt_s / t_svd_s: numpy in / numpy out through the public API (host copies included)",
                 "k3_svt_device_s": t_k3, "k3_sweeps_per_slice": sw / max(sl, 1),
                 "k3_tier": "shared-memory resident" if n * n * 4 <= 225 * 1024 else "blocked (block-cyclic)"}
        if cpu and n == 128:
            t0 = time.perf_counter()
            O.svt(a5, tau, O.ospec("dct", a5.shape))
            entry["cpu_baseline_svt_s"] = time.perf_counter() - t0
        c5[f"n{n}"] = entry
    out["config5"] = c5
    # ---- config 4: 1024x1024x3x64, explicit Q (x) F64 (complex64 transform domain), Bernoulli(0.3)
    if not args.skip_config4:
        rng = np.random.default_rng(0)
        q, _ = np.linalg.qr(rng.standard_normal((3, 3)))
        a4 = rng.standard_normal((1024, 20, 3, 64), dtype=np.float32)
        b4 = rng.standard_normal((20, 1024, 3, 64), dtype=np.float32)
        spec4 = L.make_spec("explicit", (1024, 1024, 3, 64), matrices={3: q, 4: L.build_fourier_matrix(64)})
        m4 = L.l_product(a4.astype(np.float64), b4.astype(np.float64), spec4)
        mask4 = rng.random(m4.shape) < 0.3
        nat.jacobi_stats(reset=True)
        v4 = _run_pga(L, nat, torch, m4.astype(np.float32), mask4, spec4, "fp32", 50)
        sl4, sw4 = nat.jacobi_stats(reset=True)
        out["config4_pga"] = {"metric": "PGA completion iters/sec", "value": v4,
                              "unit": "it/s", "dtype": "c64", "iterations": 50,
                              "config": "config4 1024x1024x3x64 Q(x)DFT64, rank 20, Bernoulli(0.3); all 50 iterations",
                              "jacobi_sweeps_per_slice": sw4 / max(sl4, 1),
                              "note": "99 unique 1024^2 complex slices on the blocked (block-cyclic) Jacobi tier, "
                                      "right bases carried between iterations (ltb_svt_carry_c64_impl), truncated "
                                      "sweeps with the trace-power certificate for the columns below tau; "
                                      "0.72 it/s cold (round-2 start, 2 iterations), 2.39 it/s with full warm sweeps; "
                                      "final iterate 2e-5 from the full-sweep run (tools/experiments/"
                                      "cfg4_truncation_check.py)"}
    return out


def _self_launch(args) -> int:
    """`bench.py --gpus N` outside torchrun: launch N ranks (one per GPU) of this script under
    torch.distributed.run on 127.0.0.1 and return its exit code.  Fails loudly when fewer than
    N GPUs are visible instead of printing a 1-GPU line."""
    import socket

    import torch

    have = torch.cuda.device_count()
    if have < args.gpus:
        print(f"bench.py: --gpus {args.gpus} requested but only {have} CUDA device(s) are visible", file=sys.stderr)
        return 2
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), str(Path(__file__).resolve()), *sys.argv[1:]]
    return subprocess.run(cmd).returncode


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--skip-extras", action="store_true")
    ap.add_argument("--force-dist", action="store_true", help=argparse.SUPPRESS)  # the N>1 path at N=1 (test)
    ap.add_argument("--skip-config4", action="store_true")
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--skip-pga", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=10.0)
    ap.add_argument("--cpu-pga-iters", type=int, default=2)
    ap.add_argument("--pga-iters", type=int, default=CFG3["iters"])
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    in_torchrun = "WORLD_SIZE" in os.environ
    if in_torchrun and int(os.environ["WORLD_SIZE"]) != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={os.environ['WORLD_SIZE']}", file=sys.stderr)
        sys.exit(2)
    if args.impl == "ours" and args.gpus > 1 and not in_torchrun:
        sys.exit(_self_launch(args))
    with _host_threads() if (args.impl == "reference" or int(os.environ.get("WORLD_SIZE", "1")) == 1) \
            else contextlib.nullcontext():
        if args.impl == "reference":
            run_reference(args)
        else:
            run_ours(args)


if __name__ == "__main__":
    main()
