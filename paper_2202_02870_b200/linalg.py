"""The *_L algebra on the B200 (drop-in for pkg/src/ltensor/linalg.py).

Every operation is the same sandwich as the reference — forward transform to
the slice stack (K1, slice-major store), a slice-wise kernel (K2 GEMM, K3
Jacobi SVD / SVT), inverse transform (K1') — but the stack never leaves the
device between the three stages.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _native as nat
from .core import fro_norm, num_rep, slice_gemm, slice_order_permutation
from .errors import ParameterError, ShapeError, UnsupportedSpecError
from .transforms import (
    TransformSpec,
    _check_shape,
    _floatify,
    check_real_residual,
    device_spec,
    forward_dtype,
    transform_device,
)

DEFAULT_RANK_THRESHOLD = 1e-10


# ----------------------------------------------------------------- device sandwich helpers
def _hat_stack(x: np.ndarray, spec: TransformSpec, hat_dtype=None) -> nat.DeviceArray:
    """L(x) as a device (P, I1, I2) slice-major stack (linalg.py:22-23 without leaving the GPU)."""
    _check_shape(x.shape, spec)
    hat_dtype = np.dtype(hat_dtype or forward_dtype(x.dtype, spec))
    src_dtype = nat.complex_of(hat_dtype) if np.iscomplexobj(x) else nat.real_of(hat_dtype)
    src = nat.DeviceArray.from_numpy(x, src_dtype)
    trailing = x.shape[2:]
    P = num_rep(x.shape)
    out, _ = transform_device(src, device_spec(spec, trailing), x.shape[0] * x.shape[1], False,
                              nat.TUBE_MAJOR, hat_dtype, nat.SLICE_MAJOR, (P, x.shape[0], x.shape[1]))
    return out


def _from_hat_stack(stack: nat.DeviceArray, lead, trailing, spec: TransformSpec, assume_real: bool,
                    out: np.ndarray | None = None) -> np.ndarray:
    """L^{-1} of a device slice stack back to an (I1, I2, trailing) numpy tensor (linalg.py:26-27)."""
    full = forward_dtype(stack.dtype, spec)
    want_real = assume_real and np.issubdtype(full, np.complexfloating)
    out_dtype = nat.real_of(full) if want_real else full
    # the kernel reads the stack in the output precision (real stays real)
    src_dtype = nat.complex_of(full) if np.issubdtype(stack.dtype, np.complexfloating) else nat.real_of(full)
    src = stack.astype(src_dtype)
    shape = tuple(lead) + tuple(trailing)
    res, sums = transform_device(src, device_spec(spec, trailing), lead[0] * lead[1], True, nat.SLICE_MAJOR,
                                 out_dtype, nat.TUBE_MAJOR, shape, residual=want_real)
    if want_real:
        check_real_residual(sums, out_dtype)
    return res.numpy(out)


def _real_inputs(*tensors) -> bool:
    return all(np.isrealobj(t) for t in tensors)


def _require_unitary(spec, what):
    if not spec.unitary_scaled:
        raise UnsupportedSpecError(f"{what} requires a unitary-scaled transform; the {spec.kind!r} kind is not")


def _singular_values(a: np.ndarray, spec: TransformSpec) -> np.ndarray:
    """Transform-domain singular values, (P, min(I1, I2)) in device slice order, descending per slice."""
    hat = _hat_stack(a, spec)
    P, i1, i2 = hat.shape
    k = min(i1, i2)
    sv = nat.DeviceArray((P, k), nat.real_of(hat.dtype))
    if sv.size:
        nat.check(nat.lib().ltb_slice_singular_values(nat.context(), hat.code, P, i1, i2, hat.ptr, sv.ptr))
    return sv.numpy()


# ----------------------------------------------------------------- public API
def l_product(a, b, spec: TransformSpec, *, out: np.ndarray | None = None, group=None) -> np.ndarray:
    """a *_L b = L^{-1}(L(a) facewise L(b)) (linalg.py:34-43).

    Keyword-only extras (not in the reference signature): `out`, a C-contiguous host
    array of the result's shape and dtype (e.g. pinned memory) that receives the
    product; `group`, a torch.distributed process group (or "world") whose ranks all
    make the same call and split the rows of the product between their GPUs."""
    a = np.asarray(a)
    b = np.asarray(b)
    if group is not None:
        from .distributed import spmd_l_product

        res = spmd_l_product(a, b, spec, group=group)
        if out is not None:
            out[...] = res
            return out
        return res
    if a.shape[2:] != b.shape[2:]:
        raise ShapeError(f"trailing dims differ: {a.shape[2:]} vs {b.shape[2:]}")
    if a.shape[1] != b.shape[0]:
        raise ShapeError(f"inner dims differ: {a.shape[1]} vs {b.shape[0]}")
    _check_shape(a.shape, spec)
    _check_shape(b.shape, spec)
    hat_dtype = np.result_type(forward_dtype(a.dtype, spec), forward_dtype(b.dtype, spec))
    m, k, n = a.shape[0], a.shape[1], b.shape[1]
    trailing = a.shape[2:]
    P = num_rep(a.shape)
    if (a.dtype == b.dtype and a.dtype in (np.float32, np.float64) and not spec.is_complex and spec.modes
            and hat_dtype == a.dtype):
        # real transform domain: one pipelined native call (host copies overlap the compute)
        c_shape = (m, n) + tuple(trailing)
        res = out if out is not None else np.empty(c_shape, a.dtype)
        if res.shape != c_shape or res.dtype != a.dtype or not res.flags.c_contiguous:
            raise ValueError(f"out must be a C-contiguous {a.dtype} array of shape {c_shape}")
        ac, bc = np.ascontiguousarray(a), np.ascontiguousarray(b)
        st = nat.lib().ltb_l_product_host(nat.context(), device_spec(spec, trailing).ptr, m, k, n,
                                          nat.dtype_code(a.dtype), ac.ctypes.data_as(C.c_void_p),
                                          bc.ctypes.data_as(C.c_void_p), res.ctypes.data_as(C.c_void_p))
        if st != 3:  # LTB_EUNSUPPORTED -> the generic path below
            nat.check(st)
            return res
    if a.dtype == b.dtype and np.isrealobj(a) and m * k == k * n and spec.modes:
        # K1 of both operands in one call (one tensor-core launch on the fp32 path)
        src_dtype = nat.real_of(hat_dtype)
        sa = nat.DeviceArray.from_numpy(a, src_dtype)
        sb = nat.DeviceArray.from_numpy(b, src_dtype)
        ha = nat.DeviceArray((P, m, k), hat_dtype)
        hb = nat.DeviceArray((P, k, n), hat_dtype)
        nat.check(nat.lib().ltb_transform_pair(nat.context(), device_spec(spec, trailing).ptr, m * k, 0, sa.code,
                                               nat.TUBE_MAJOR, sa.ptr, sb.ptr, ha.code, nat.SLICE_MAJOR, ha.ptr,
                                               hb.ptr))
    else:
        ha = _hat_stack(a, spec, hat_dtype)
        hb = _hat_stack(b, spec, hat_dtype)
    hc = slice_gemm(ha, hb, P, m, k, n)
    return _from_hat_stack(hc, (m, n), trailing, spec, _real_inputs(a, b), out=out)


def identity_tensor(n: int, trailing_dims, spec: TransformSpec) -> np.ndarray:
    """Tensor whose every transform-domain slice is I_n (linalg.py:46-51)."""
    trailing = tuple(int(d) for d in trailing_dims)
    P = num_rep((n, n) + trailing)
    ones = nat.DeviceArray.from_numpy(np.ones((P, n)))
    stack = nat.DeviceArray((P, n, n), np.float64)
    nat.check(nat.lib().ltb_embed_diag(nat.context(), stack.code, P, n, n, ones.ptr, stack.ptr))
    return _from_hat_stack(stack, (n, n), trailing, spec, True)


def l_transpose(a, spec: TransformSpec) -> np.ndarray:
    """Conjugate-transpose of every transform-domain slice (linalg.py:54-59)."""
    a = np.asarray(a)
    hat = _hat_stack(a, spec)
    P, i1, i2 = hat.shape
    t = nat.DeviceArray((P, i2, i1), hat.dtype)
    nat.check(nat.lib().ltb_slice_transpose(nat.context(), hat.code, P, i1, i2, 1, hat.ptr, t.ptr))
    return _from_hat_stack(t, (i2, i1), a.shape[2:], spec, _real_inputs(a))


def is_orthogonal(q, spec: TransformSpec, tol: float = 1e-10) -> bool:
    """q *_L q^T == I == q^T *_L q within tol (linalg.py:62-72)."""
    q = np.asarray(q)
    if q.shape[0] != q.shape[1]:
        raise ShapeError(f"orthogonality needs square first two dims, got {q.shape[:2]}")
    eye = identity_tensor(q.shape[0], q.shape[2:], spec)
    qt = l_transpose(q, spec)
    return fro_norm(l_product(q, qt, spec) - eye) < tol and fro_norm(l_product(qt, q, spec) - eye) < tol


@dataclass
class LFactors:
    """The *_L-SVD triple plus the tube norms ||S_i||_F (non-increasing) (linalg.py:75-83)."""

    u: np.ndarray
    s: np.ndarray
    v: np.ndarray
    tube_norms: np.ndarray
    spec: TransformSpec


@dataclass
class RankReport:
    tubal: int
    multirank: np.ndarray  # rho_p for p = 1..P (reference p-order)
    average: float


def t_svd(a, spec: TransformSpec) -> LFactors:
    """Full slice-wise SVD in the transform domain, inverse-transformed (linalg.py:102-118).

    K3 runs one-sided Jacobi with V accumulated (in double precision for single-precision
    stacks); U is completed to a full orthonormal basis on the device (full_matrices=True)."""
    a = np.asarray(a)
    i1, i2 = a.shape[:2]
    trailing = a.shape[2:]
    hat = _hat_stack(a, spec)
    P = hat.shape[0]
    k = min(i1, i2)
    rdt = nat.real_of(hat.dtype)
    # single-precision stacks are factored in double precision: the fp32 Jacobi's singular
    # vectors drift ~eps * sigma_max / gap per column (1e-4 relative on config 5, n = 256),
    # outside the 1e-4 factor tolerance; the fp64 kernel's are ~1e-12
    work = hat.astype(nat.complex_of(np.float64) if np.iscomplexobj(np.zeros(0, hat.dtype)) else np.float64)
    u_hat = nat.DeviceArray((P, i1, i1), work.dtype)
    v_hat = nat.DeviceArray((P, i2, i2), work.dtype)
    sv = nat.DeviceArray((P, k), nat.real_of(work.dtype))
    if k > 0:
        nat.check(nat.lib().ltb_slice_svd(nat.context(), work.code, P, i1, i2, work.ptr, u_hat.ptr, sv.ptr,
                                          v_hat.ptr))
    u_hat, v_hat, sv = u_hat.astype(hat.dtype), v_hat.astype(hat.dtype), sv.astype(rdt)
    s_hat = nat.DeviceArray((P, i1, i2), rdt)
    nat.check(nat.lib().ltb_embed_diag(nat.context(), s_hat.code, P, i1, i2, sv.ptr, s_hat.ptr))
    real = _real_inputs(a)
    u = _from_hat_stack(u_hat, (i1, i1), trailing, spec, real)
    s = _from_hat_stack(s_hat, (i1, i2), trailing, spec, real)
    v = _from_hat_stack(v_hat, (i2, i2), trailing, spec, real)
    diag = s[np.arange(k), np.arange(k)].reshape(k, -1)
    tube_norms = np.sqrt(np.sum(np.abs(diag) ** 2, axis=1)) if k else np.zeros(0)
    return LFactors(u=u, s=s, v=v, tube_norms=tube_norms, spec=spec)


def truncate(f: LFactors, k: int) -> np.ndarray:
    """Rank-k truncation u(:,1:k) *_L s(1:k,1:k) *_L v(:,1:k)^T (linalg.py:121-129)."""
    kmax = min(f.s.shape[0], f.s.shape[1])
    if not 1 <= k <= kmax:
        raise ParameterError(f"truncation rank {k} out of range [1, {kmax}]")
    return l_product(l_product(f.u[:, :k], f.s[:k, :k], f.spec), l_transpose(f.v[:, :k], f.spec), f.spec)


def ranks(a, spec: TransformSpec, threshold: float = DEFAULT_RANK_THRESHOLD) -> RankReport:
    """Tubal rank, multirank (reference p-order) and average rank (linalg.py:132-144)."""
    if threshold < 0:
        raise ParameterError(f"threshold must be >= 0, got {threshold}")
    a = np.asarray(a)
    sv = _singular_values(a, spec)
    smax = float(sv.max(initial=0.0))
    if smax == 0.0:
        return RankReport(tubal=0, multirank=np.zeros(sv.shape[0], dtype=int), average=0.0)
    nonzero = sv > threshold * smax
    multirank = nonzero.sum(axis=1)[slice_order_permutation(a.shape[2:])] if a.ndim > 2 else nonzero.sum(axis=1)
    tubal = int(nonzero.any(axis=0).sum())
    return RankReport(tubal=tubal, multirank=multirank, average=float(multirank.mean()))


def spectral_norm(a, spec: TransformSpec) -> float:
    """Largest transform-domain singular value (linalg.py:154-158)."""
    _require_unitary(spec, "spectral_norm")
    return float(_singular_values(np.asarray(a), spec).max(initial=0.0))


def nuclear_norm(a, spec: TransformSpec) -> float:
    """alpha^{-1} * sum of all transform-domain singular values (linalg.py:161-165)."""
    _require_unitary(spec, "nuclear_norm")
    return float(_singular_values(np.asarray(a), spec).sum() / spec.alpha)


def svt(a, tau: float, spec: TransformSpec, *, group=None) -> np.ndarray:
    """Singular value thresholding, the prox of tau * TNN (linalg.py:168-181).

    K3: per-slice one-sided Jacobi in shared memory, then the threshold and the
    rank-limited recomposition as two batched GEMMs, all on the device.  `group`
    (keyword-only, a torch.distributed process group or "world"): every rank makes the
    same call; transforms are row-sharded and the slices split between the GPUs."""
    if tau < 0:
        raise ParameterError(f"tau must be >= 0, got {tau}")
    _require_unitary(spec, "svt")
    a = np.asarray(a)
    if group is not None:
        _check_shape(a.shape, spec)
        from .distributed import spmd_svt

        return spmd_svt(a, tau, spec, group=group)
    hat = _hat_stack(a, spec)
    P, i1, i2 = hat.shape
    out = nat.DeviceArray((P, i1, i2), hat.dtype)
    if np.isrealobj(a):  # conjugate slice pairs of a real tensor's transform are solved once
        nat.check(nat.lib().ltb_spec_slice_svt(nat.context(), device_spec(spec, a.shape[2:]).ptr, hat.code, P, i1,
                                               i2, hat.ptr, float(tau), out.ptr))
    else:
        nat.check(nat.lib().ltb_slice_svt(nat.context(), hat.code, P, i1, i2, hat.ptr, float(tau), out.ptr))
    return _from_hat_stack(out, (i1, i2), a.shape[2:], spec, _real_inputs(a))
