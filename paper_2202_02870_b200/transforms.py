"""The operator L (transform spec) and its device application.

Mirrors pkg/src/ltensor/transforms.py: the matrix builders (:31-65), the
TransformSpec dataclass (:71-100), make_spec (:103-158) and the entry points
apply_l (:176-192) / apply_l_inv (:195-226).  Spec construction stays on the
host (it is O(n^3) in the mode sizes); the mode products run on the B200
through K1/K1' (csrc/ltb_xform_tile.cuh).

Dtype rules follow the reference exactly: the fast fft path returns the
complex type of the input precision, the fast dct path keeps the input
dtype, the matrix path promotes with the float64/complex128 matrices.

Deviation: the real-output contract threshold is 1e-9
relative in double precision, as in the reference; single-precision
computations use 1e-4, because complex64 rounding alone exceeds 1e-9.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _native as nat
from .core import mode_n_product  # noqa: F401  (re-exported as in the reference module)
from .errors import NumericConsistencyError, ParameterError, TransformError

INV_TOL = 1e-10
UNITARY_TOL = 1e-10
IMAG_TOL = 1e-9
IMAG_TOL_SINGLE = 1e-4


# ----------------------------------------------------------------- matrix builders
def build_dct_matrix(n: int) -> np.ndarray:
    """Orthonormal DCT-II: C[i, j] = sqrt((2 - [i == 0]) / n) cos(i (2 j + 1) pi / (2 n)), 0-based
    (transforms.py:31-38)."""
    if n < 1:
        raise ParameterError(f"matrix size must be >= 1, got {n}")
    k = np.arange(n, dtype=np.float64)
    angles = np.pi * np.outer(k, 2.0 * k + 1.0) / (2.0 * n)
    weights = np.full(n, np.sqrt(2.0 / n))
    weights[0] = np.sqrt(1.0 / n)
    return weights[:, None] * np.cos(angles)


def build_fourier_matrix(n: int) -> np.ndarray:
    """Unnormalised DFT matrix F[i, j] = exp(-2 pi i i j / n) (transforms.py:41-46)."""
    if n < 1:
        raise ParameterError(f"matrix size must be >= 1, got {n}")
    k = np.arange(n)
    return np.exp(-2j * np.pi * np.outer(k, k) / n)


def _upper_shift_plus_identity(n: int) -> np.ndarray:
    return np.eye(n) + np.eye(n, k=1)


def build_cproduct_matrix(n: int) -> np.ndarray:
    """Cosine-product matrix W^{-1} C (I + Z), W = diag(first column of C) (transforms.py:49-56)."""
    if n < 1:
        raise ParameterError(f"matrix size must be >= 1, got {n}")
    c = build_dct_matrix(n)
    return (c / c[:, :1]) @ _upper_shift_plus_identity(n)


def build_cproduct_inverse(n: int) -> np.ndarray:
    """Closed-form inverse (I + Z)^{-1} C^T W (transforms.py:59-65)."""
    if n < 1:
        raise ParameterError(f"matrix size must be >= 1, got {n}")
    c = build_dct_matrix(n)
    return np.linalg.solve(_upper_shift_plus_identity(n), c.T * c[:, 0][None, :])


_BUILDERS = {"fft": build_fourier_matrix, "dct": build_dct_matrix, "cprod": build_cproduct_matrix}


# ----------------------------------------------------------------- spec
@dataclass(eq=False)
class TransformSpec:
    """The operator L: transformed modes (1-based, >= 3, ascending), per-mode sizes, the
    unitarity scale alpha and the unitary-scaled flag (transforms.py:71-100)."""

    kind: str
    modes: tuple
    sizes: tuple
    alpha: float | None
    unitary_scaled: bool
    _matrices: dict = field(default_factory=dict, repr=False)
    _device: dict = field(default_factory=dict, repr=False)

    def __eq__(self, other):
        if not isinstance(other, TransformSpec):
            return NotImplemented
        return (self.kind, self.modes, self.sizes) == (other.kind, other.modes, other.sizes)

    __hash__ = None

    def mode_matrix(self, mode: int) -> np.ndarray:
        if mode not in self.modes:
            raise TransformError(f"mode {mode} is not transformed by this spec")
        mats = self._matrices
        if mode not in mats:
            mats[mode] = _BUILDERS[self.kind](self.sizes[self.modes.index(mode)])
        return mats[mode]

    def mode_inverse(self, mode: int) -> np.ndarray:
        m = self.mode_matrix(mode)
        if self.kind == "cprod":
            return build_cproduct_inverse(m.shape[0])
        return np.linalg.inv(m)

    # device-side matrices: exact closed-form inverses where one exists
    def _device_inverse(self, mode: int) -> np.ndarray:
        m = self.mode_matrix(mode)
        if self.kind == "fft":
            return np.conj(m) / m.shape[0]
        if self.kind == "dct":
            return m.T.copy()
        return self.mode_inverse(mode)

    @property
    def is_complex(self) -> bool:
        if self.kind == "fft":
            return True
        if self.kind == "explicit":
            return any(np.iscomplexobj(self._matrices[m]) for m in self.modes)
        return False


def _require_invertible(m, m_inv):
    n = m.shape[0]
    if np.linalg.norm(m @ m_inv - np.eye(n)) >= INV_TOL * max(1.0, float(np.linalg.norm(m))):
        raise TransformError("transform matrix is not invertible to working precision")


def make_spec(kind: str, shape, modes=None, matrices=None) -> TransformSpec:
    """Build a TransformSpec for tensors of `shape` (transforms.py:103-158)."""
    shape = tuple(int(d) for d in shape)
    order = len(shape)
    if order < 3:
        raise TransformError(f"transforms need order >= 3, got shape {shape}")
    modes = tuple(range(3, order + 1)) if modes is None else tuple(sorted(int(m) for m in modes))
    bad = [m for m in modes if m < 3 or m > order]
    if bad:
        raise TransformError(f"mode {bad[0]} out of range [3, {order}] for shape {shape}")
    sizes = tuple(shape[m - 1] for m in modes)

    if kind == "fft":
        return TransformSpec("fft", modes, sizes, float(np.prod(sizes)), True)
    if kind == "dct":
        return TransformSpec("dct", modes, sizes, 1.0, True)
    if kind == "cprod":
        spec = TransformSpec("cprod", modes, sizes, None, False)
        for m in modes:
            _require_invertible(spec.mode_matrix(m), spec.mode_inverse(m))
        return spec
    if kind != "explicit":
        raise TransformError(f"unknown transform kind {kind!r}")
    if matrices is None:
        raise TransformError("explicit kind requires per-mode matrices")
    mats = {int(m): np.asarray(v) for m, v in matrices.items()}
    if set(mats) != set(modes):
        raise TransformError(f"matrices given for modes {sorted(mats)}, expected {modes}")
    unitary = True
    scales = []
    for m in modes:
        mat = mats[m]
        n = shape[m - 1]
        if mat.shape != (n, n):
            raise TransformError(f"matrix for mode {m} has shape {mat.shape}, expected ({n}, {n})")
        try:
            inv = np.linalg.inv(mat)
        except np.linalg.LinAlgError as exc:
            raise TransformError(f"matrix for mode {m} is singular") from exc
        _require_invertible(mat, inv)
        gram = mat @ mat.conj().T
        s = float(np.trace(gram).real) / n
        if np.linalg.norm(gram - s * np.eye(n)) < UNITARY_TOL * max(1.0, s):
            scales.append(s)
        else:
            unitary = False
    spec = TransformSpec("explicit", modes, sizes, float(np.prod(scales)) if unitary else None, unitary)
    spec._matrices = mats
    return spec


def _check_shape(shape, spec):
    for mode, size in zip(spec.modes, spec.sizes):
        if mode > len(shape) or shape[mode - 1] != size:
            raise TransformError(
                f"tensor of shape {tuple(shape)} does not match spec modes {spec.modes} with sizes {spec.sizes}"
            )


# ----------------------------------------------------------------- dtype rules
def _floatify(dt) -> np.dtype:
    dt = np.dtype(dt)
    if dt in (np.float32, np.float64, np.complex64, np.complex128):
        return dt
    if np.issubdtype(dt, np.complexfloating):
        return np.dtype(np.complex128)
    return np.dtype(np.float64)


def _fast(spec, explicit) -> bool:
    return spec.kind in ("fft", "dct") and not explicit


def forward_dtype(x_dtype, spec, explicit=False) -> np.dtype:
    """dtype apply_l returns for an input of x_dtype."""
    dt = _floatify(x_dtype)
    if not spec.modes:
        return np.dtype(x_dtype)
    if _fast(spec, explicit):
        return nat.complex_of(dt) if spec.kind == "fft" else dt
    mat = np.complex128 if spec.is_complex else np.float64
    return np.result_type(dt, mat)


def inverse_dtype(x_dtype, spec, explicit=False, assume_real=False) -> np.dtype:
    """dtype apply_l_inv returns for an input of x_dtype."""
    out = forward_dtype(x_dtype, spec, explicit)
    if assume_real and np.issubdtype(out, np.complexfloating):
        out = nat.real_of(out)
    return out


def imag_tol(dtype) -> float:
    return IMAG_TOL if nat.real_of(dtype) == np.float64 else IMAG_TOL_SINGLE


# ----------------------------------------------------------------- device spec
def hermitian_rows(m: np.ndarray, tol: float = 1e-12) -> np.ndarray:
    """If row (n - i) mod n of `m` is conj(row i) up to rounding (the DFT), make it exactly so.

    With exactly conjugate rows, a real tensor's transform-domain slices q and -q
    are bitwise conjugates, every slice kernel (Jacobi, GEMM) is conjugation-
    equivariant, and the real-output contract (transforms.py:217-225) holds
    structurally instead of up to the conditioning of the slice SVD."""
    n = m.shape[0]
    idx = (-np.arange(n)) % n
    scale = max(1.0, float(np.abs(m).max(initial=0.0)))
    if np.abs(m[idx] - np.conj(m)).max(initial=0.0) > tol * scale:
        return m
    out = m.copy()
    for i in range(n):
        j = idx[i]
        if i < j:
            out[j] = np.conj(out[i])
        elif i == j:
            out[i] = out[i].real
    return out


def device_spec(spec: TransformSpec, trailing: tuple):
    """ltb_spec handle for tensors whose trailing dims are `trailing` (cached on the spec)."""
    trailing = tuple(int(d) for d in trailing)
    key = (trailing, nat.current_device())  # a handle lives on the device (context) that made it
    cache = spec._device
    if key in cache:
        return cache[key]
    axes = [m - 3 for m in spec.modes]
    cplx = spec.is_complex
    fwd, inv = [], []
    for m in spec.modes:
        a = np.asarray(spec.mode_matrix(m), dtype=np.complex128 if cplx else np.float64)
        if cplx:
            a = hermitian_rows(a)
        b = np.asarray(spec._device_inverse(m), dtype=np.complex128 if cplx else np.float64)
        fwd.append(np.ascontiguousarray(a).ravel())
        inv.append(np.ascontiguousarray(b).ravel())
    dt = np.complex128 if cplx else np.float64
    fwd = np.concatenate(fwd) if fwd else np.zeros(1, dt)
    inv = np.concatenate(inv) if inv else np.zeros(1, dt)
    fwd_d = np.ascontiguousarray(fwd.view(np.float64))
    inv_d = np.ascontiguousarray(inv.view(np.float64))
    handle = _create_spec(trailing, axes, cplx, fwd_d, inv_d)
    cache[key] = handle
    return handle


class _SpecHandle:
    __slots__ = ("ptr", "trailing", "P", "_keep")

    def __init__(self, ptr, trailing, keep):
        self.ptr = ptr
        self.trailing = trailing
        self.P = int(np.prod(trailing, dtype=np.int64)) if trailing else 1
        self._keep = keep

    def __del__(self):
        try:
            if self.ptr and nat._lib is not None:
                nat._lib.ltb_spec_destroy(self.ptr)
        except Exception:
            pass


def _create_spec(trailing, axes, cplx, fwd, inv):
    lib = nat.lib()
    ctx = nat.context()
    dims = (C.c_int64 * max(len(trailing), 1))(*trailing)
    ax = (C.c_int * max(len(axes), 1))(*axes)
    out = C.c_void_p()
    nat.check(lib.ltb_spec_create(ctx, len(trailing), dims, len(axes), ax, int(cplx),
                                  fwd.ctypes.data_as(C.POINTER(C.c_double)),
                                  inv.ctypes.data_as(C.POINTER(C.c_double)), C.byref(out)))
    return _SpecHandle(out, trailing, (fwd, inv))


_LAYOUT_SPECS: dict = {}


def layout_spec(trailing: tuple):
    """Identity spec (no modes) used for pure layout changes (tube <-> slice major)."""
    key = (tuple(int(d) for d in trailing), nat.current_device())
    if key not in _LAYOUT_SPECS:
        z = np.zeros(1)
        _LAYOUT_SPECS[key] = _create_spec(key[0], [], False, z, z)
    return _LAYOUT_SPECS[key]


def transform_device(x: nat.DeviceArray, handle, ntubes: int, inverse: bool, layout_in: int, out_dtype,
                     layout_out: int, out_shape, residual: bool = False):
    """Run K1/K1' on a device array already in the compute precision; returns (out, sums|None)."""
    out = nat.DeviceArray(out_shape, out_dtype)
    sums = (C.c_double * 2)() if residual else None
    nat.check(nat.lib().ltb_transform(
        nat.context(), handle.ptr, int(ntubes), int(inverse), x.code, layout_in, x.ptr,
        out.code, layout_out, out.ptr, sums))
    return out, (float(sums[0]), float(sums[1])) if residual else None


def _compute_dtype(in_dtype, out_dtype, spec, explicit) -> np.dtype:
    """Element type the kernel reads: the input converted to the output precision."""
    prec = nat.real_of(out_dtype)
    if np.issubdtype(np.dtype(in_dtype), np.complexfloating):
        return nat.complex_of(prec)
    return prec


def check_real_residual(sums, dtype):
    total, imag = sums
    if total > 0:
        ratio = float(np.sqrt(imag) / np.sqrt(total))
        tol = imag_tol(dtype)
        if ratio > tol:
            raise NumericConsistencyError(
                f"imaginary residual {ratio:.3e} exceeds {tol:.0e}; "
                "transform-domain tensor is not the image of a real tensor"
            )


def _leading(shape):
    """Number of tubes: the product of the (at most two) leading dims."""
    return int(np.prod(shape[:2], dtype=np.int64)) if len(shape) else 1


# ----------------------------------------------------------------- entry points
def apply_l(x, spec: TransformSpec, explicit: bool = False) -> np.ndarray:
    """L(x): mode products with M_k over spec.modes, ascending (transforms.py:176-192), on the GPU."""
    x = np.asarray(x)
    _check_shape(x.shape, spec)
    if not spec.modes:
        return x.copy()
    out_dtype = forward_dtype(x.dtype, spec, explicit)
    src = nat.DeviceArray.from_numpy(x, _compute_dtype(x.dtype, out_dtype, spec, explicit))
    handle = device_spec(spec, x.shape[2:])
    out, _ = transform_device(src, handle, _leading(x.shape), False, nat.TUBE_MAJOR, out_dtype,
                              nat.TUBE_MAJOR, x.shape)
    return out.numpy()


def apply_l_inv(xhat, spec: TransformSpec, explicit: bool = False, assume_real: bool = False) -> np.ndarray:
    """L^{-1}(xhat) in reverse mode order, with the real-output contract (transforms.py:195-226)."""
    xhat = np.asarray(xhat)
    _check_shape(xhat.shape, spec)
    if not spec.modes and not (assume_real and np.iscomplexobj(xhat)):
        return xhat.copy()
    full = forward_dtype(xhat.dtype, spec, explicit)
    want_real = assume_real and np.issubdtype(full, np.complexfloating)
    out_dtype = nat.real_of(full) if want_real else full
    src = nat.DeviceArray.from_numpy(xhat, _compute_dtype(xhat.dtype, full, spec, explicit))
    handle = device_spec(spec, xhat.shape[2:])
    out, sums = transform_device(src, handle, _leading(xhat.shape), True, nat.TUBE_MAJOR, out_dtype,
                                 nat.TUBE_MAJOR, xhat.shape, residual=want_real)
    if want_real:
        check_real_residual(sums, out_dtype)
    return out.numpy()
