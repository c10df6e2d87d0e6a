"""CPU oracle for the *_L hot path — TEST INFRASTRUCTURE ONLY.

A numpy/scipy restatement of the reference algorithm (arXiv 2202.02870's
`ltensor` package, /root/reference/pkg/src/ltensor).  Only tests/,
__graft_entry__.smoke() and bench.py's CPU-baseline / `--impl reference` leg
may import it, and only as the checker or as the timed CPU baseline; the
product package never imports it.

Pinned: tests/test_oracle_golden.py checks every function below against
golden vectors produced by running the reference itself in the build
container (tests/golden/make_golden.py -> tests/golden/golden.npz) and against
the reference test-suite's known answers (tube examples, pinned completion
RSE values).

The arithmetic of the reference lives in numpy/scipy (numpy >= 1.24,
scipy >= 1.10, unpinned; pkg/pyproject.toml:11-12): LAPACK gesdd via
np.linalg.svd, pocketfft via np.fft, scipy.fft.dct (type II, ortho).  The
oracle calls the same routines in the same order so that it reproduces the
reference's rounding, not just its mathematics.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import scipy.fft


# ------------------------------------------------------------------ operator L
def dct_matrix(n):
    """transforms.py:31-38: orthonormal DCT-II."""
    i = np.arange(n)[:, None]
    j = np.arange(n)[None, :]
    w = np.where(i == 0, math.sqrt(1.0 / n), math.sqrt(2.0 / n))
    return w * np.cos(i * (2 * j + 1) * np.pi / (2 * n))


def dft_matrix(n):
    """transforms.py:41-46: unnormalised DFT."""
    k = np.arange(n)
    return np.exp(-2j * np.pi * np.outer(k, k) / n)


def cprod_matrix(n):
    """transforms.py:49-56: W^{-1} C (I + Z)."""
    c = dct_matrix(n)
    return np.diag(1.0 / c[:, 0]) @ c @ (np.eye(n) + np.eye(n, k=1))


def cprod_inverse(n):
    """transforms.py:59-65: (I + Z)^{-1} C^T W."""
    c = dct_matrix(n)
    return np.linalg.solve(np.eye(n) + np.eye(n, k=1), c.T @ np.diag(c[:, 0]))


@dataclass
class OSpec:
    """kind, 1-based modes, sizes, alpha, unitary flag, explicit matrices (transforms.py:71-158)."""

    kind: str
    modes: tuple
    sizes: tuple
    alpha: float | None
    unitary_scaled: bool
    matrices: dict = field(default_factory=dict)

    def mode_matrix(self, mode):
        if self.kind == "explicit":
            return self.matrices[mode]
        n = self.sizes[self.modes.index(mode)]
        return {"fft": dft_matrix, "dct": dct_matrix, "cprod": cprod_matrix}[self.kind](n)

    def mode_inverse(self, mode):
        if self.kind == "cprod":
            return cprod_inverse(self.sizes[self.modes.index(mode)])
        return np.linalg.inv(self.mode_matrix(mode))


def ospec(kind, shape, modes=None, matrices=None) -> OSpec:
    shape = tuple(int(d) for d in shape)
    modes = tuple(range(3, len(shape) + 1)) if modes is None else tuple(sorted(modes))
    sizes = tuple(shape[m - 1] for m in modes)
    if kind == "fft":
        return OSpec("fft", modes, sizes, float(np.prod(sizes)), True)
    if kind == "dct":
        return OSpec("dct", modes, sizes, 1.0, True)
    if kind == "cprod":
        return OSpec("cprod", modes, sizes, None, False)
    mats = {int(k): np.asarray(v) for k, v in matrices.items()}
    scales, unitary = [], True
    for m in modes:
        g = mats[m] @ mats[m].conj().T
        s = float(np.trace(g).real) / g.shape[0]
        if np.linalg.norm(g - s * np.eye(g.shape[0])) < 1e-10 * max(1.0, s):
            scales.append(s)
        else:
            unitary = False
    return OSpec("explicit", modes, sizes, float(np.prod(scales)) if unitary else None, unitary, mats)


def mode_product(x, u, n):
    """core.py:110-122: multiply every mode-n fibre of x by u, as u @ (mode-n unfolding)
    with the Kolda column order (core.py:90-107), so the GEMM rounding matches."""
    x = np.asarray(x)
    moved = np.moveaxis(x, n - 1, 0)
    unf = moved.reshape(x.shape[n - 1], -1, order="F")
    prod = u @ unf
    return np.moveaxis(prod.reshape((u.shape[0],) + moved.shape[1:], order="F"), 0, n - 1)


def forward(x, spec, explicit=False):
    """transforms.py:176-192."""
    out = np.asarray(x)
    for mode in spec.modes:
        if spec.kind == "fft" and not explicit:
            out = np.fft.fft(out, axis=mode - 1)
        elif spec.kind == "dct" and not explicit:
            out = scipy.fft.dct(out, type=2, axis=mode - 1, norm="ortho")
        else:
            out = mode_product(out, spec.mode_matrix(mode), mode)
    return out


def inverse(xhat, spec, explicit=False, assume_real=False, imag_tol=1e-9):
    """transforms.py:195-226, returning (result, imaginary residual ratio or None)."""
    out = np.asarray(xhat)
    for mode in reversed(spec.modes):
        if spec.kind == "fft" and not explicit:
            out = np.fft.ifft(out, axis=mode - 1)
        elif spec.kind == "dct" and not explicit:
            if np.iscomplexobj(out):
                re = scipy.fft.idct(out.real, type=2, axis=mode - 1, norm="ortho")
                im = scipy.fft.idct(out.imag, type=2, axis=mode - 1, norm="ortho")
                out = re + 1j * im
            else:
                out = scipy.fft.idct(out, type=2, axis=mode - 1, norm="ortho")
        else:
            out = mode_product(out, spec.mode_inverse(mode), mode)
    ratio = None
    if assume_real and np.iscomplexobj(out):
        total = np.linalg.norm(out.ravel())
        ratio = float(np.linalg.norm(out.imag.ravel()) / total) if total > 0 else 0.0
        if ratio > imag_tol:
            raise ValueError(f"imaginary residual {ratio:.3e}")
        out = out.real.copy()
    return out


# ------------------------------------------------------------------ slice stacks (core.py:43-87)
def to_stack(x):
    """(P, I1, I2) in reference p-order (Fortran over trailing dims)."""
    x = np.asarray(x)
    return np.moveaxis(x.reshape(x.shape[0], x.shape[1], -1, order="F"), 2, 0)


def from_stack(stack, trailing):
    return np.moveaxis(np.asarray(stack), 0, 2).reshape(stack.shape[1:] + tuple(trailing), order="F")


def _real(*ts):
    return all(np.isrealobj(t) for t in ts)


# ------------------------------------------------------------------ *_L algebra (linalg.py)
def l_product(a, b, spec):
    """linalg.py:34-43."""
    a, b = np.asarray(a), np.asarray(b)
    c = np.matmul(to_stack(forward(a, spec)), to_stack(forward(b, spec)))
    return inverse(from_stack(c, a.shape[2:]), spec, assume_real=_real(a, b))


def l_transpose(a, spec):
    """linalg.py:54-59."""
    a = np.asarray(a)
    st = np.conj(np.swapaxes(to_stack(forward(a, spec)), 1, 2))
    return inverse(from_stack(st, a.shape[2:]), spec, assume_real=_real(a))


def identity_tensor(n, trailing, spec):
    """linalg.py:46-51."""
    P = int(np.prod(trailing)) if len(trailing) else 1
    return inverse(from_stack(np.broadcast_to(np.eye(n), (P, n, n)).copy(), trailing), spec, assume_real=True)


def t_svd(a, spec):
    """linalg.py:102-118 -> (u, s, v, tube_norms)."""
    a = np.asarray(a)
    i1, i2 = a.shape[:2]
    tr = a.shape[2:]
    uh, sv, vh = np.linalg.svd(to_stack(forward(a, spec)), full_matrices=True)
    real = _real(a)
    k = min(i1, i2)
    sd = np.zeros((sv.shape[0], i1, i2), dtype=sv.dtype)
    sd[:, np.arange(k), np.arange(k)] = sv[:, :k]
    u = inverse(from_stack(uh, tr), spec, assume_real=real)
    s = inverse(from_stack(sd, tr), spec, assume_real=real)
    v = inverse(from_stack(np.conj(np.swapaxes(vh, 1, 2)), tr), spec, assume_real=real)
    norms = np.array([np.linalg.norm(np.ravel(s[i, i])) for i in range(k)])
    return u, s, v, norms


def truncate(u, s, v, k, spec):
    """linalg.py:121-129: u(:,1:k) *_L s(1:k,1:k) *_L v(:,1:k)^T (spec shape-agnostic here)."""
    return l_product(l_product(u[:, :k], s[:k, :k], spec), l_transpose(v[:, :k], spec), spec)


def inner_product(a, b):
    """core.py:26-35: vdot, conjugate-linear in the first argument."""
    out = np.vdot(np.asarray(a), np.asarray(b))
    return float(out.real) if np.isrealobj(a) and np.isrealobj(b) else complex(out)


def is_orthogonal(q, spec, tol=1e-10):
    """linalg.py:62-72."""
    q = np.asarray(q)
    eye = identity_tensor(q.shape[0], q.shape[2:], spec)
    qt = l_transpose(q, spec)
    return fro(l_product(q, qt, spec) - eye) < tol and fro(l_product(qt, q, spec) - eye) < tol


def singular_values(a, spec):
    """compute_uv=False path of linalg.py:137,157,164, (P, min(I1,I2)) in reference p-order."""
    return np.linalg.svd(to_stack(forward(np.asarray(a), spec)), compute_uv=False)


def svt(a, tau, spec):
    """linalg.py:168-181."""
    a = np.asarray(a)
    u, sv, vh = np.linalg.svd(to_stack(forward(a, spec)), full_matrices=False)
    out = np.matmul(u * np.maximum(sv - tau, 0.0)[:, None, :], vh)
    return inverse(from_stack(out, a.shape[2:]), spec, assume_real=_real(a))


# ------------------------------------------------------------------ completion (completion.py)
def project_omega(x, mask):
    """completion.py:23-29."""
    return np.where(np.asarray(mask, dtype=bool), np.asarray(x), 0.0)


def sample_mask(dims, sr, seed):
    """completion.py:32-42."""
    total = int(np.prod(dims))
    flat = np.zeros(total, dtype=bool)
    flat[np.random.default_rng(seed).choice(total, size=int(round(sr * total)), replace=False)] = True
    return flat.reshape(tuple(dims), order="F")


def fro(x):
    return float(np.linalg.norm(np.asarray(x).ravel()))


def rse(obtained, original, denominator="obtained"):
    """completion.py:45-60."""
    den = fro(obtained if denominator == "obtained" else original) ** 2
    return fro(np.asarray(original) - np.asarray(obtained)) ** 2 / den


def psnr(obtained, original):
    """completion.py:63-78."""
    err = fro(np.asarray(obtained) - np.asarray(original)) ** 2
    if err == 0.0:
        return math.inf
    peak = float(np.max(obtained))
    if peak == 0.0:
        return -math.inf
    return 10.0 * math.log10(peak**2 / err)


def pga_complete(m, mask, spec, nu=0.9, mu0=None, mu_bar_ratio=1e-4, tol=1e-4, max_iters=100,
                 reimpose_observed=False, ground_truth=None):
    """completion.py:141-202.  Returns (x, records, status); records are
    (k, mu, t, rel[, rse, psnr]) tuples."""
    m = np.asarray(m, dtype=float)
    mask = np.asarray(mask, dtype=bool)
    p_obs = project_omega(m, mask)
    mu0 = nu * fro(m) if mu0 is None else float(mu0)
    mu_bar = mu_bar_ratio * mu0
    x_prev = np.zeros_like(m)
    x_cur = np.zeros_like(m)
    t_prev = t_cur = 1.0
    records, status = [], "max-iters"
    for k in range(1, max_iters + 1):
        mu_k = max(nu**k * mu0, mu_bar)
        y = x_cur + ((t_prev - 1.0) / t_cur) * (x_cur - x_prev)
        g = y - (project_omega(y, mask) - p_obs)
        x_next = svt(g, mu_k, spec)
        num, den = fro(y - x_next), fro(x_next)
        rel = num / den if den > 0.0 else (0.0 if fro(p_obs) == 0.0 else math.inf)
        rec = (k, mu_k, t_cur, rel)
        if ground_truth is not None:
            try:
                r = rse(x_next, ground_truth)
            except ZeroDivisionError:
                r = math.nan
            rec = rec + (r, psnr(x_next, ground_truth))
        records.append(rec)
        x_prev, x_cur = x_cur, x_next
        t_prev, t_cur = t_cur, (1.0 + math.sqrt(4.0 * t_cur**2 + 1.0)) / 2.0
        if rel <= tol:
            status = "converged"
            break
    out = np.where(mask, m, x_cur) if reimpose_observed else x_cur
    return out, records, status
