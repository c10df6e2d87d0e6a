"""Low-tubal-rank tensor completion by accelerated proximal gradient on the B200
(drop-in for pkg/src/ltensor/completion.py).

The host keeps the reference's scalar recurrences bit-for-bit (mu_k, t_k and
the momentum weight beta_k are pure functions of k and the config,
completion.py:163-193) and hands them to the device as per-iteration arrays;
the device runs whole chunks of iterations (gradient step fused into the
forward transform, SVT, inverse transform fused with the stopping-rule
norms) and stops itself at the first k with rel <= tol.  The trace is then
rebuilt on the host from the per-iteration sums with the reference formulas.

Precision: the reference always computes in float64 (completion.py:154).  The
drop-in does too for float64 (or any non-float32) input; a float32 `m` runs
the FP32 path (parity bar 1e-4 relative, BASELINE north_star).  Pass
precision="fp64" to force float64.  The result is float64 either way.
"""

from __future__ import annotations

import csv
import ctypes as C
import math
from dataclasses import dataclass, field

import numpy as np

from . import _native as nat
from .core import _float_dtype, _sumsq_max, fro_norm
from .errors import ParameterError, ShapeError, UnsupportedSpecError
from .transforms import IMAG_TOL, TransformSpec, _check_shape, device_spec


def project_omega(x, mask) -> np.ndarray:
    """P_Omega(x) = where(mask, x, 0) (completion.py:23-29), on the GPU."""
    x = np.asarray(x)
    mask = np.asarray(mask, dtype=bool)
    if x.shape != mask.shape:
        raise ShapeError(f"mask shape {mask.shape} does not match data shape {x.shape}")
    dt = np.result_type(x.dtype, 0.0)
    dt = _float_dtype(dt)
    out = nat.DeviceArray(x.shape, dt)
    if out.size:
        dx = nat.DeviceArray.from_numpy(x, dt)
        dm8 = _upload_mask(mask)
        nat.check(nat.lib().ltb_project_omega(nat.context(), out.code, out.size, dx.ptr, dm8.ptr, out.ptr))
    return out.numpy()


class _ByteBuffer:
    """Raw device bytes (the uint8 observation mask)."""

    def __init__(self, data: np.ndarray):
        data = np.ascontiguousarray(data, dtype=np.uint8)
        self.nbytes = int(data.nbytes)
        out = C.c_void_p()
        self.ptr = None
        self._ctx = nat.context()
        nat.check(nat.lib().ltb_malloc(self._ctx, max(self.nbytes, 16), C.byref(out)))
        self.ptr = out
        if self.nbytes:
            nat.check(nat.lib().ltb_memcpy_h2d(self._ctx, self.ptr, data.ctypes.data_as(C.c_void_p), self.nbytes))

    def __del__(self):
        try:
            if self.ptr and nat._lib is not None:
                nat._lib.ltb_free(self._ctx, self.ptr)
        except Exception:
            pass


def _upload_mask(mask: np.ndarray) -> _ByteBuffer:
    return _ByteBuffer(np.ascontiguousarray(mask, dtype=bool).view(np.uint8))


def sample_mask(dims, sr: float, seed: int) -> np.ndarray:
    """Exactly round(sr * prod(dims)) observed entries, uniform without replacement,
    Fortran-order reshape (completion.py:32-42).  Host-side: it must reproduce the
    reference's numpy Generator stream bit for bit."""
    if not 0.0 <= sr <= 1.0:
        raise ParameterError(f"sampling ratio must be in [0, 1], got {sr}")
    dims = tuple(int(d) for d in dims)
    total = int(np.prod(dims, dtype=np.int64))
    picked = np.random.default_rng(seed).choice(total, size=int(round(sr * total)), replace=False)
    flat = np.zeros(total, dtype=bool)
    flat[picked] = True
    return flat.reshape(dims, order="F")


def _pair_sums(obtained, original):
    obtained = np.asarray(obtained)
    original = np.asarray(original)
    if obtained.shape != original.shape:
        raise ShapeError(f"dimension mismatch: {obtained.shape} vs {original.shape}")
    dt = _float_dtype(obtained.dtype, original.dtype)
    do = nat.DeviceArray.from_numpy(obtained, dt)
    dg = nat.DeviceArray.from_numpy(original, dt)
    return do, dg


def rse(obtained, original, denominator: str = "obtained") -> float:
    """||original - obtained||^2 / ||obtained||^2 (or / ||original||^2) (completion.py:45-60)."""
    obtained = np.asarray(obtained)
    original = np.asarray(original)
    if obtained.shape != original.shape:
        raise ShapeError(f"dimension mismatch: {obtained.shape} vs {original.shape}")
    if denominator not in ("obtained", "original"):
        raise ParameterError(f"unknown RSE denominator {denominator!r}")
    den = fro_norm(obtained if denominator == "obtained" else original) ** 2
    if den == 0.0:
        raise ParameterError("RSE undefined: zero denominator tensor")
    if obtained.size == 0:
        return 0.0 / den
    do, dg = _pair_sums(obtained, original)
    return math.sqrt(_sumsq_max(dg, do)[0]) ** 2 / den


def psnr(obtained, original) -> float:
    """10 log10(max(obtained)^2 / ||obtained - original||^2) (completion.py:63-78)."""
    obtained = np.asarray(obtained)
    original = np.asarray(original)
    if obtained.shape != original.shape:
        raise ShapeError(f"dimension mismatch: {obtained.shape} vs {original.shape}")
    if obtained.size == 0:
        return math.inf
    do, dg = _pair_sums(obtained, original)
    s, peak = _sumsq_max(do, dg)
    err = math.sqrt(s) ** 2
    if err == 0.0:
        return math.inf
    if peak == 0.0:
        return -math.inf
    return 10.0 * math.log10(peak ** 2 / err)


@dataclass
class CompletionConfig:
    """Solver parameters; mu0 defaults to nu * ||M||_F at solve time (completion.py:81-102)."""

    spec: TransformSpec
    nu: float = 0.9
    mu0: float | None = None
    mu_bar_ratio: float = 1e-4
    tol: float = 1e-4
    max_iters: int = 100
    reimpose_observed: bool = False
    rse_denominator: str = "obtained"

    def validate(self):
        if not 0.0 < self.nu < 1.0:
            raise ParameterError(f"nu must be in (0, 1), got {self.nu}")
        if self.tol <= 0.0:
            raise ParameterError(f"tol must be > 0, got {self.tol}")
        if self.mu_bar_ratio > 1.0 or self.mu_bar_ratio < 0.0:
            raise ParameterError(f"mu_bar_ratio must be in [0, 1], got {self.mu_bar_ratio}")
        if self.max_iters < 1:
            raise ParameterError(f"max_iters must be >= 1, got {self.max_iters}")


@dataclass
class IterationRecord:
    k: int
    mu: float
    t: float
    rel_change: float
    rse: float | None = None
    psnr: float | None = None


@dataclass
class CompletionTrace:
    records: list = field(default_factory=list)
    status: str = "max-iters"

    @property
    def iterations(self) -> int:
        return len(self.records)

    def write_csv(self, path):
        with open(path, "w", newline="") as fh:
            w = csv.writer(fh)
            w.writerow(["iter", "mu", "t", "rel_change", "rse", "psnr"])
            for r in self.records:
                w.writerow([r.k, repr(r.mu), repr(r.t), repr(r.rel_change),
                            "" if r.rse is None else repr(r.rse), "" if r.psnr is None else repr(r.psnr)])


def pga_schedule(cfg: CompletionConfig, mu0: float):
    """(mu_k, t_k, beta_k) for k = 1..max_iters, computed exactly as completion.py:163-193."""
    mu_bar = cfg.mu_bar_ratio * mu0
    mus, ts, betas = [], [], []
    t_prev, t_cur = 1.0, 1.0
    for k in range(1, cfg.max_iters + 1):
        mus.append(max(cfg.nu**k * mu0, mu_bar))
        ts.append(t_cur)
        betas.append((t_prev - 1.0) / t_cur)
        t_prev, t_cur = t_cur, (1.0 + math.sqrt(4.0 * t_cur**2 + 1.0)) / 2.0
    return mus, ts, betas


def rel_change(s_num: float, s_den: float, pobs_zero: bool) -> float:
    """completion.py:174-181 from the device sums (identical IEEE ops to the device's decision)."""
    num = math.sqrt(s_num)
    den = math.sqrt(s_den)
    if den > 0.0:
        return num / den
    return 0.0 if pobs_zero else math.inf


class PGASolver:
    """Device state of one completion run (ltb_pga): create, run chunks, fetch."""

    def __init__(self, m64: np.ndarray, mask: np.ndarray, spec: TransformSpec, precision: str,
                 ground_truth: np.ndarray | None = None):
        self.shape = m64.shape
        self.dtype = nat.F32 if precision == "fp32" else nat.F64
        handle = device_spec(spec, m64.shape[2:])
        self._spec_handle = handle
        out = C.c_void_p()
        gt = np.ascontiguousarray(ground_truth, dtype=np.float64) if ground_truth is not None else None
        self._m = np.ascontiguousarray(m64, dtype=np.float64)
        mask8 = np.ascontiguousarray(mask, dtype=bool).view(np.uint8)
        nat.check(nat.lib().ltb_pga_create(
            nat.context(), handle.ptr, self.dtype, m64.shape[0], m64.shape[1],
            self._m.ctypes.data_as(C.POINTER(C.c_double)), mask8.ctypes.data_as(C.c_void_p),
            gt.ctypes.data_as(C.POINTER(C.c_double)) if gt is not None else None, C.byref(out)))
        self.ptr = out
        s = C.c_double()
        nat.check(nat.lib().ltb_pga_pobs_sumsq(self.ptr, C.byref(s)))
        self.pobs_sumsq = float(s.value)

    def run(self, k0: int, betas, mus, tol: float):
        n = len(betas)
        b = np.ascontiguousarray(betas, dtype=np.float64)
        mu = np.ascontiguousarray(mus, dtype=np.float64)
        rec = np.zeros((n, 5), dtype=np.float64)
        done, conv = C.c_int(), C.c_int()
        nat.check(nat.lib().ltb_pga_run(self.ptr, k0, n, b.ctypes.data_as(C.POINTER(C.c_double)),
                                        mu.ctypes.data_as(C.POINTER(C.c_double)), float(tol),
                                        rec.ctypes.data_as(C.POINTER(C.c_double)), C.byref(done), C.byref(conv)))
        return rec[: done.value], bool(conv.value)

    def fetch(self, reimpose: bool) -> np.ndarray:
        out = self._m.copy() if reimpose else np.empty(self.shape, dtype=np.float64)
        nat.check(nat.lib().ltb_pga_fetch(self.ptr, int(reimpose), out.ctypes.data_as(C.POINTER(C.c_double))))
        return out

    def close(self):
        if getattr(self, "ptr", None):
            nat.lib().ltb_pga_destroy(self.ptr)
            self.ptr = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _resolve_precision(m_in, precision):
    if precision is None:
        return "fp32" if np.asarray(m_in).dtype == np.float32 else "fp64"
    if precision not in ("fp32", "fp64"):
        raise ParameterError(f"precision must be 'fp32' or 'fp64', got {precision!r}")
    return precision


def pga_complete(m, mask, cfg: CompletionConfig, ground_truth=None, *, precision=None, chunk=None, group=None):
    """Complete P_Omega(m) by accelerated proximal gradient (completion.py:141-202).

    Returns (completed float64 tensor, CompletionTrace).  Keyword-only extras:
    precision ("fp32" / "fp64", default: fp32 for float32 `m`, else fp64),
    chunk (iterations enqueued per device round trip, default adaptive) and
    group (a torch.distributed process group, or "world"): every rank of the group
    makes the same call and the solve is sharded over their GPUs (distributed.py)."""
    cfg.validate()
    if not cfg.spec.unitary_scaled:
        raise UnsupportedSpecError("completion uses SVT, which requires a unitary-scaled transform")
    prec = _resolve_precision(m, precision)
    m64 = np.asarray(m, dtype=float)
    mask = np.asarray(mask, dtype=bool)
    if m64.shape != mask.shape:
        raise ShapeError(f"mask shape {mask.shape} does not match data shape {m64.shape}")
    _check_shape(m64.shape, cfg.spec)
    gt = None
    if ground_truth is not None:
        gt = np.asarray(ground_truth, dtype=float)
        if gt.shape != m64.shape:
            raise ShapeError(f"dimension mismatch: {m64.shape} vs {gt.shape}")

    mu0 = cfg.nu * fro_norm(m64) if cfg.mu0 is None else float(cfg.mu0)
    mus, ts, betas = pga_schedule(cfg, mu0)
    gt_sumsq = fro_norm(gt) ** 2 if (gt is not None and cfg.rse_denominator == "original") else None
    if cfg.rse_denominator not in ("obtained", "original"):
        raise ParameterError(f"unknown RSE denominator {cfg.rse_denominator!r}")

    if group is not None:
        from .distributed import spmd_pga_complete

        return spmd_pga_complete(m64 if prec == "fp64" else np.asarray(m), mask, cfg, gt, precision=prec,
                                 group=group)
    solver = PGASolver(m64, mask, cfg.spec, prec, gt)
    trace = CompletionTrace()
    pobs_zero = solver.pobs_sumsq == 0.0
    k = 1
    step = chunk or 4
    try:
        while k <= cfg.max_iters:
            n = min(step, cfg.max_iters - k + 1)
            recs, converged = solver.run(k, betas[k - 1 : k - 1 + n], mus[k - 1 : k - 1 + n], cfg.tol)
            for i, r in enumerate(recs):
                kk = k + i
                rel = rel_change(r[0], r[1], pobs_zero)
                if prec == "fp64" and r[1] + r[4] > 0:
                    ratio = math.sqrt(r[4]) / math.sqrt(r[1] + r[4])
                    if ratio > IMAG_TOL:
                        from .errors import NumericConsistencyError

                        raise NumericConsistencyError(
                            f"imaginary residual {ratio:.3e} exceeds {IMAG_TOL:.0e} at iteration {kk}")
                rec = IterationRecord(k=kk, mu=mus[kk - 1], t=ts[kk - 1], rel_change=rel)
                if gt is not None:
                    den = math.sqrt(r[1]) ** 2 if cfg.rse_denominator == "obtained" else gt_sumsq
                    err = math.sqrt(r[2]) ** 2
                    rec.rse = math.nan if den == 0.0 else err / den
                    if err == 0.0:
                        rec.psnr = math.inf
                    elif r[3] == 0.0:
                        rec.psnr = -math.inf
                    else:
                        rec.psnr = 10.0 * math.log10(r[3] ** 2 / err)
                trace.records.append(rec)
            k += len(recs)
            if converged:
                trace.status = "converged"
                break
            if chunk is None:
                step = min(step * 2, 32)
        out = solver.fetch(cfg.reimpose_observed)
    finally:
        solver.close()
    return out, trace
