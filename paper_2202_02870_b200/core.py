"""Dense tensor primitives (drop-in for pkg/src/ltensor/core.py).

Index conventions are the reference's: modes and the representative index p
are 1-based, and p runs Fortran-order over the trailing dims,
p = k3 + sum_{i>=4} (k_i - 1) I_3...I_{i-1} (core.py:1-11, 43-60).

Arithmetic (fro_norm, inner_product, mode_n_product, facewise_product) runs on
the B200; the pure index/layout helpers (rep indices, unfold/fold, rep
stacks) are host views with no arithmetic.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _native as nat
from .errors import ModeError, ShapeError


def _as_tensor(x) -> np.ndarray:
    x = np.asarray(x)
    if x.ndim < 2:
        raise ShapeError(f"tensor order must be >= 2, got order {x.ndim}")
    return x


def _float_dtype(*dts) -> np.dtype:
    dt = np.result_type(*dts)
    if dt in (np.float32, np.float64, np.complex64, np.complex128):
        return np.dtype(dt)
    return np.dtype(np.complex128 if np.issubdtype(dt, np.complexfloating) else np.float64)


def _sumsq_max(dev: nat.DeviceArray, other: nat.DeviceArray | None = None):
    out = (C.c_double * 2)()
    nat.check(nat.lib().ltb_reduce_sumsq(nat.context(), dev.code, dev.size, dev.ptr,
                                         other.ptr if other is not None else None, out))
    return float(out[0]), float(out[1])


def fro_norm(a) -> float:
    """Frobenius norm sqrt(sum |a|^2) (core.py:38-40), deterministic float64 device reduction."""
    a = np.asarray(a)
    if a.size == 0:
        return 0.0
    dev = nat.DeviceArray.from_numpy(a, _float_dtype(a.dtype))
    return float(np.sqrt(_sumsq_max(dev)[0]))


def inner_product(a, b):
    """<a, b> = sum conj(a) b (core.py:26-35): float for real operands, complex otherwise."""
    a = _as_tensor(a)
    b = _as_tensor(b)
    if a.shape != b.shape:
        raise ShapeError(f"dimension mismatch: {a.shape} vs {b.shape}")
    dt = _float_dtype(a.dtype, b.dtype)
    out = (C.c_double * 2)()
    if a.size:
        da = nat.DeviceArray.from_numpy(a, dt)
        db = nat.DeviceArray.from_numpy(b, dt)
        nat.check(nat.lib().ltb_reduce_dot(nat.context(), da.code, da.size, da.ptr, db.ptr, out))
    if np.isrealobj(a) and np.isrealobj(b):
        return float(out[0])
    return complex(out[0], out[1])


# ----------------------------------------------------------------- index helpers (host)
def num_rep(dims) -> int:
    """P = I_3 * ... * I_N (1 for order-2 dims)."""
    dims = tuple(dims)
    return int(np.prod(dims[2:], dtype=np.int64)) if len(dims) > 2 else 1


def rep_index_to_multi(p: int, dims) -> tuple:
    """1-based p -> (k_3, ..., k_N), Fortran order over the trailing dims."""
    dims = tuple(int(d) for d in dims)
    P = num_rep(dims)
    if not 1 <= p <= P:
        raise ModeError(f"representative index {p} out of range [1, {P}]")
    rem = int(p) - 1
    multi = []
    for d in dims[2:]:
        multi.append(rem % d + 1)
        rem //= d
    return tuple(multi)


def multi_to_rep_index(multi, dims) -> int:
    """(k_3, ..., k_N) -> 1-based p (inverse of rep_index_to_multi)."""
    dims = tuple(int(d) for d in dims)
    p, stride = 0, 1
    for k, d in zip(multi, dims[2:]):
        p += (int(k) - 1) * stride
        stride *= d
    return p + 1


def rep_matrix(x, p: int) -> np.ndarray:
    """The p-th representative matrix x[:, :, k_3 - 1, ..., k_N - 1] (a view)."""
    x = _as_tensor(x)
    multi = rep_index_to_multi(p, x.shape)
    return x[(slice(None), slice(None)) + tuple(k - 1 for k in multi)]


def as_rep_stack(x) -> np.ndarray:
    """(P, I1, I2) stack of representative matrices in reference p-order (a view when possible)."""
    x = _as_tensor(x)
    flat = x.reshape(x.shape[0], x.shape[1], -1, order="F")
    return np.moveaxis(flat, 2, 0)


def from_rep_stack(stack, trailing_dims) -> np.ndarray:
    """Inverse of as_rep_stack."""
    stack = np.asarray(stack)
    P, i1, i2 = stack.shape
    trailing = tuple(int(d) for d in trailing_dims)
    if P != num_rep((i1, i2) + trailing):
        raise ShapeError(f"stack holds {P} slices, trailing dims {trailing} need "
                         f"{num_rep((i1, i2) + trailing)}")
    return np.moveaxis(stack, 0, 2).reshape((i1, i2) + trailing, order="F")


def slice_order_permutation(trailing) -> np.ndarray:
    """perm[p-1] = device slice index q (C-order over trailing dims) of reference rep index p."""
    trailing = tuple(int(d) for d in trailing)
    if not trailing:
        return np.zeros(1, dtype=np.int64)
    P = int(np.prod(trailing, dtype=np.int64))
    multi = np.unravel_index(np.arange(P), trailing, order="F")
    return np.ravel_multi_index(multi, trailing, order="C")


def mode_n_unfold(x, n: int) -> np.ndarray:
    """Mode-n matricisation, Kolda ordering (core.py:90-95)."""
    x = _as_tensor(x)
    if not 1 <= n <= x.ndim:
        raise ModeError(f"mode {n} out of range [1, {x.ndim}]")
    return np.moveaxis(x, n - 1, 0).reshape(x.shape[n - 1], -1, order="F")


def mode_n_fold(m, n: int, dims) -> np.ndarray:
    """Inverse of mode_n_unfold for target dims (core.py:98-107)."""
    m = np.asarray(m)
    dims = tuple(int(d) for d in dims)
    if not 1 <= n <= len(dims):
        raise ModeError(f"mode {n} out of range [1, {len(dims)}]")
    rest = dims[: n - 1] + dims[n:]
    if m.shape != (dims[n - 1], int(np.prod(rest, dtype=np.int64))):
        raise ShapeError(f"unfolded shape {m.shape} does not match dims {dims}")
    return np.moveaxis(m.reshape((dims[n - 1],) + rest, order="F"), 0, n - 1)


# ----------------------------------------------------------------- device arithmetic
def mode_n_product(x, u, n: int) -> np.ndarray:
    """x x_n u: every mode-n fibre multiplied by u (core.py:110-122), on the GPU."""
    x = _as_tensor(x)
    u = np.atleast_2d(np.asarray(u))
    if not 1 <= n <= x.ndim:
        raise ModeError(f"mode {n} out of range [1, {x.ndim}]")
    if u.shape[1] != x.shape[n - 1]:
        raise ShapeError(f"matrix with {u.shape[1]} columns cannot act on mode of size {x.shape[n - 1]}")
    dt = _float_dtype(u.dtype, x.dtype)
    dims = list(x.shape)
    dims[n - 1] = u.shape[0]
    outer = int(np.prod(x.shape[: n - 1], dtype=np.int64))
    inner = int(np.prod(x.shape[n:], dtype=np.int64))
    out = nat.DeviceArray(dims, dt)
    if out.size:
        dx = nat.DeviceArray.from_numpy(x, dt)
        du = nat.DeviceArray.from_numpy(u, dt)
        nat.check(nat.lib().ltb_mode_product(nat.context(), outer, x.shape[n - 1], inner, u.shape[0],
                                             dx.code, dx.ptr, du.code, du.ptr, out.code, out.ptr))
    return out.numpy()


def tubes_to_slices(dev: nat.DeviceArray, lead, trailing) -> nat.DeviceArray:
    """(I1, I2, trailing...) tube-major -> (P, I1, I2) slice-major, on the device."""
    from .transforms import layout_spec, transform_device

    P = num_rep((1, 1) + tuple(trailing))
    out, _ = transform_device(dev, layout_spec(trailing), lead[0] * lead[1], False, nat.TUBE_MAJOR, dev.dtype,
                              nat.SLICE_MAJOR, (P, lead[0], lead[1]))
    return out


def slices_to_tubes(dev: nat.DeviceArray, lead, trailing, out_dtype=None) -> nat.DeviceArray:
    from .transforms import layout_spec, transform_device

    out, _ = transform_device(dev, layout_spec(trailing), lead[0] * lead[1], False, nat.SLICE_MAJOR,
                              out_dtype or dev.dtype, nat.TUBE_MAJOR, tuple(lead) + tuple(trailing))
    return out


def slice_gemm(a: nat.DeviceArray, b: nat.DeviceArray, P: int, m: int, k: int, n: int) -> nat.DeviceArray:
    """C[q] = A[q] B[q] for slice-major stacks (K2)."""
    out = nat.DeviceArray((P, m, n), a.dtype)
    nat.check(nat.lib().ltb_slice_gemm(nat.context(), a.code, P, m, n, k, nat.OP_N, a.ptr, k, m * k,
                                       nat.OP_N, b.ptr, n, k * n, out.ptr, n, m * n))
    return out


def facewise_product(a, b) -> np.ndarray:
    """Slice-wise matrix product over all P representative matrices (core.py:125-134), on the GPU."""
    a = _as_tensor(a)
    b = _as_tensor(b)
    if a.shape[2:] != b.shape[2:]:
        raise ShapeError(f"trailing dims differ: {a.shape[2:]} vs {b.shape[2:]}")
    if a.shape[1] != b.shape[0]:
        raise ShapeError(f"inner dims differ: {a.shape[1]} vs {b.shape[0]}")
    dt = _float_dtype(a.dtype, b.dtype)
    trailing = a.shape[2:]
    P = num_rep(a.shape)
    m, k, n = a.shape[0], a.shape[1], b.shape[1]
    if m * n * P == 0:
        return np.zeros((m, n) + trailing, dtype=dt)
    sa = tubes_to_slices(nat.DeviceArray.from_numpy(a, dt), (m, k), trailing)
    sb = tubes_to_slices(nat.DeviceArray.from_numpy(b, dt), (k, n), trailing)
    sc = slice_gemm(sa, sb, P, m, k, n)
    return slices_to_tubes(sc, (m, n), trailing).numpy()
