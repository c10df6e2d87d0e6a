"""ctypes binding of libltb.so (include/ltb.h) and device-array plumbing.

There is no CPU fallback: if the extension is missing or no CUDA device is
visible, every compute entry point raises DeviceError.
"""

from __future__ import annotations

import ctypes as C
import os
import threading
from pathlib import Path

import numpy as np

from .errors import STATUS_TO_ERROR, DeviceError

LIB_PATH = Path(__file__).resolve().with_name("libltb.so")

F32, F64, C64, C128 = 0, 1, 2, 3
OPT_FORCE_BLOCKED_SVD, OPT_TC_TIMELINE, OPT_QR_TIMELINE, OPT_JACOBI_PAIRS, OPT_FULL_SWEEPS = 1, 2, 3, 4, 5
TUBE_MAJOR, SLICE_MAJOR = 0, 1
OP_N, OP_T, OP_C, OP_H = 0, 1, 2, 3

_NP_TO_CODE = {
    np.dtype(np.float32): F32,
    np.dtype(np.float64): F64,
    np.dtype(np.complex64): C64,
    np.dtype(np.complex128): C128,
}
_CODE_TO_NP = {v: k for k, v in _NP_TO_CODE.items()}

_vp = C.c_void_p
_i64 = C.c_int64
_int = C.c_int
_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)

_SIGNATURES = {
    "ltb_version": ([], _int),
    "ltb_device_count": ([_ip], _int),
    "ltb_ctx_create": ([_int, C.POINTER(_vp)], _int),
    "ltb_ctx_destroy": ([_vp], None),
    "ltb_ctx_last_error": ([_vp], C.c_char_p),
    "ltb_ctx_set_stream": ([_vp, _vp], _int),
    "ltb_ctx_synchronize": ([_vp], _int),
    "ltb_ctx_make_current": ([_vp], _int),
    "ltb_ctx_set_option": ([_vp, _int, _i64], _int),
    "ltb_ctx_launch_count": ([_vp], _i64),
    "ltb_ctx_stats": ([_vp, C.POINTER(_i64), _int], _int),
    "ltb_malloc": ([_vp, _i64, C.POINTER(_vp)], _int),
    "ltb_free": ([_vp, _vp], _int),
    "ltb_memcpy_h2d": ([_vp, _vp, _vp, _i64], _int),
    "ltb_memcpy_d2h": ([_vp, _vp, _vp, _i64], _int),
    "ltb_memcpy_d2d": ([_vp, _vp, _vp, _i64], _int),
    "ltb_memset_zero": ([_vp, _vp, _i64], _int),
    "ltb_convert": ([_vp, _i64, _int, _vp, _int, _vp], _int),
    "ltb_fortran_to_c": ([_vp, _int, _vp, _int, _vp, _vp], _int),
    "ltb_spec_create": ([_vp, _int, C.POINTER(_i64), _int, _ip, _int, _dp, _dp, C.POINTER(_vp)], _int),
    "ltb_spec_destroy": ([_vp], None),
    "ltb_transform": ([_vp, _vp, _i64, _int, _int, _int, _vp, _int, _int, _vp, _dp], _int),
    "ltb_transform_pair": ([_vp, _vp, _i64, _int, _int, _int, _vp, _vp, _int, _int, _vp, _vp], _int),
    "ltb_l_product_host": ([_vp, _vp, _i64, _i64, _i64, _int, _vp, _vp, _vp], _int),
    "ltb_mode_product": ([_vp, _i64, _i64, _i64, _i64, _int, _vp, _int, _vp, _int, _vp], _int),
    "ltb_slice_gemm": ([_vp, _int, _i64, _i64, _i64, _i64, _int, _vp, _i64, _i64, _int, _vp, _i64, _i64,
                        _vp, _i64, _i64], _int),
    "ltb_tc_gemm": ([_vp, _i64, _i64, _i64, _i64, _int, _vp, _i64, _i64, _int, _vp, _i64, _i64, _vp, _i64, _i64, _int],
                    _int),
    "ltb_slice_svt":([_vp, _int, _i64, _i64, _i64, _vp, C.c_double, _vp], _int),
    "ltb_slice_svt_carry": ([_vp, _i64, _i64, _i64, _vp, C.c_double, _vp, _vp, _int], _int),
    "ltb_slice_svt_carry_c64": ([_vp, _i64, _i64, _i64, _vp, C.c_double, _vp, _vp, _int], _int),
    "ltb_reduce_sumsq_device": ([_vp, _int, _i64, _vp, _vp, _vp], _int),
    "ltb_spec_slice_svt": ([_vp, _vp, _int, _i64, _i64, _i64, _vp, C.c_double, _vp], _int),
    "ltb_slice_svd": ([_vp, _int, _i64, _i64, _i64, _vp, _vp, _vp, _vp], _int),
    "ltb_slice_singular_values": ([_vp, _int, _i64, _i64, _i64, _vp, _vp], _int),
    "ltb_reduce_sumsq": ([_vp, _int, _i64, _vp, _vp, _dp], _int),
    "ltb_reduce_dot": ([_vp, _int, _i64, _vp, _vp, _dp], _int),
    "ltb_embed_diag": ([_vp, _int, _i64, _i64, _i64, _vp, _vp], _int),
    "ltb_slice_transpose": ([_vp, _int, _i64, _i64, _i64, _int, _vp, _vp], _int),
    "ltb_project_omega": ([_vp, _int, _i64, _vp, _vp, _vp], _int),
    "ltb_pga_gradient": ([_vp, _int, _i64, _vp, _vp, _vp, _vp, C.c_double, _vp, _vp], _int),
    "ltb_pga_create":([_vp, _vp, _int, _i64, _i64, _dp, _vp, _dp, C.POINTER(_vp)], _int),
    "ltb_pga_pobs_sumsq": ([_vp, _dp], _int),
    "ltb_pga_run": ([_vp, _int, _int, _dp, _dp, C.c_double, _dp, _ip, _ip], _int),
    "ltb_pga_fetch": ([_vp, _int, _dp], _int),
    "ltb_pga_current": ([_vp, C.POINTER(_vp)], _int),
    "ltb_pga_destroy": ([_vp], None),
    "ltb_pack_mask": ([_vp, _i64, _vp, _vp], _int),
    "ltb_l_product_ws_bytes": ([_vp, _i64, _i64, _i64, _int], _i64),
    "ltb_l_product_device": ([_vp, _vp, _i64, _i64, _i64, _int, _vp, _vp, _vp, _vp, _i64, _int], _int),
    "ltb_pga_shard_forward": ([_vp, _vp, _int, _i64, C.c_double, _vp, _vp, _vp, _vp, _vp, _vp], _int),
    "ltb_pga_shard_svt": ([_vp, _int, _i64, _i64, _i64, _vp, C.c_double, _vp, _vp, _int, _vp], _int),
    "ltb_pga_shard_inverse": ([_vp, _vp, _int, _i64, C.c_double, _vp, _vp, _vp, _vp, _vp, _vp, _vp], _int),
    "ltb_pga_shard_decide": ([_vp, _vp, C.c_double, C.c_double, _vp, _vp], _int),
}

# every symbol include/ltb.h declares (checked by the CPU test suite)
EXPORTED_SYMBOLS = tuple(_SIGNATURES)

_lock = threading.RLock()
_lib = None
_device = 0


def load_library(path: Path | str | None = None):
    """Load libltb.so and declare its signatures (no device needed)."""
    global _lib
    with _lock:
        if _lib is not None and path is None:
            return _lib
        p = Path(path) if path is not None else LIB_PATH
        if not p.exists():
            raise DeviceError(
                f"native extension {p} is not built; run `python __graft_entry__.py` (build) first"
            )
        lib = C.CDLL(str(p))
        for name, (argtypes, restype) in _SIGNATURES.items():
            fn = getattr(lib, name)
            fn.argtypes = argtypes
            fn.restype = restype
        if path is None:
            _lib = lib
        return lib


def set_device(device: int) -> None:
    """Select the CUDA device used by subsequent calls (default 0).

    Every device gets its own ltb_ctx, created on first use and kept for the life of
    the process: buffers and spec handles stay bound to the context (and device) that
    made them and are released through it, so switching devices never leaves a live
    object pointing at a destroyed context."""
    global _device
    with _lock:
        _device = int(device)


_ctxs: dict = {}
_tls = threading.local()


def context():
    """The ltb_ctx of the selected device (created on first use)."""
    with _lock:
        ctx = _ctxs.get(_device)
        if ctx is None:
            lib = load_library()
            out = _vp()
            st = lib.ltb_ctx_create(_device, C.byref(out))
            if st != 0:
                raise DeviceError(f"could not create a CUDA context on device {_device} (status {st}); "
                                  "a B200 is required — there is no CPU fallback")
            ctx = _ctxs[_device] = out
        dev = _device
    if getattr(_tls, "device", None) != dev:  # the CUDA current device is per host thread
        load_library().ltb_ctx_make_current(ctx)
        _tls.device = dev
    return ctx


def current_device() -> int:
    return _device


def check(status: int) -> None:
    if status == 0:
        return
    msg = ""
    ctx = _ctxs.get(_device)
    if ctx is not None:
        raw = load_library().ltb_ctx_last_error(ctx)
        msg = raw.decode() if raw else ""
    raise STATUS_TO_ERROR.get(status, DeviceError)(msg or f"libltb status {status}")


def lib():
    return load_library()


def launch_count() -> int:
    return int(lib().ltb_ctx_launch_count(context()))


def jacobi_stats(reset: bool = False, with_max: bool = False) -> tuple:
    """(slices solved, sweeps run[, most sweeps of one slice]) by the Jacobi kernels since the last reset."""
    out = (_i64 * 3)()
    check(lib().ltb_ctx_stats(context(), out, int(reset)))
    return (int(out[0]), int(out[1]), int(out[2])) if with_max else (int(out[0]), int(out[1]))


def dtype_code(dt) -> int:
    dt = np.dtype(dt)
    if dt not in _NP_TO_CODE:
        raise DeviceError(f"unsupported dtype {dt}")
    return _NP_TO_CODE[dt]


def np_dtype(code: int) -> np.dtype:
    return _CODE_TO_NP[code]


def complex_of(dt) -> np.dtype:
    return np.dtype(np.complex64) if np.dtype(dt) in (np.float32, np.complex64) else np.dtype(np.complex128)


def real_of(dt) -> np.dtype:
    return np.dtype(np.float32) if np.dtype(dt) in (np.float32, np.complex64) else np.dtype(np.float64)


class DeviceArray:
    """A device buffer (ltb_malloc) with a numpy-like shape/dtype."""

    __slots__ = ("ptr", "nbytes", "shape", "dtype", "_owner", "_base", "_ctx")

    def __init__(self, shape, dtype, ptr=None, owner=True):
        self._base = None
        self.shape = tuple(int(s) for s in shape)
        self.dtype = np.dtype(dtype)
        self.nbytes = int(np.prod(self.shape, dtype=np.int64)) * self.dtype.itemsize
        self._owner = owner
        self._ctx = None
        if ptr is None:
            out = _vp()
            self._ctx = context()
            check(lib().ltb_malloc(self._ctx, max(self.nbytes, 16), C.byref(out)))
            self.ptr = out
        else:
            self.ptr = _vp(ptr) if not isinstance(ptr, _vp) else ptr
            self._owner = owner

    @property
    def size(self) -> int:
        return int(np.prod(self.shape, dtype=np.int64))

    @property
    def code(self) -> int:
        return dtype_code(self.dtype)

    def __del__(self):
        try:
            if self._owner and self.ptr and _lib is not None and self._ctx is not None:
                _lib.ltb_free(self._ctx, self.ptr)
        except Exception:  # interpreter shutdown
            pass

    @classmethod
    def empty(cls, shape, dtype) -> "DeviceArray":
        return cls(shape, dtype)

    @classmethod
    def zeros(cls, shape, dtype) -> "DeviceArray":
        a = cls(shape, dtype)
        check(lib().ltb_memset_zero(context(), a.ptr, a.nbytes))
        return a

    @classmethod
    def from_numpy(cls, arr, dtype=None) -> "DeviceArray":
        """Upload `arr`; the optional dtype conversion runs on the device."""
        arr = np.asarray(arr)
        if arr.dtype not in _NP_TO_CODE:
            arr = arr.astype(np.complex128 if np.iscomplexobj(arr) else np.float64)
        arr = np.ascontiguousarray(arr)
        src = cls(arr.shape, arr.dtype)
        if src.nbytes:
            check(lib().ltb_memcpy_h2d(context(), src.ptr, arr.ctypes.data_as(_vp), src.nbytes))
        if dtype is None or np.dtype(dtype) == arr.dtype:
            return src
        return src.astype(dtype)

    def astype(self, dtype) -> "DeviceArray":
        dtype = np.dtype(dtype)
        if dtype == self.dtype:
            return self
        out = DeviceArray(self.shape, dtype)
        check(lib().ltb_convert(context(), self.size, self.code, self.ptr, out.code, out.ptr))
        return out

    def numpy(self, out: np.ndarray | None = None) -> np.ndarray:
        """Download; `out` (C-contiguous, same shape and dtype, e.g. pinned host memory) is filled in place."""
        if out is None:
            out = np.empty(self.shape, dtype=self.dtype)
        elif out.shape != self.shape or out.dtype != self.dtype or not out.flags.c_contiguous:
            raise ValueError(f"out must be a C-contiguous {self.dtype} array of shape {self.shape}")
        if self.nbytes:
            check(lib().ltb_memcpy_d2h(context(), out.ctypes.data_as(_vp), self.ptr, self.nbytes))
        return out

    def reshape(self, *shape) -> "DeviceArray":
        if len(shape) == 1 and isinstance(shape[0], (tuple, list)):
            shape = tuple(shape[0])
        view = DeviceArray(shape, self.dtype, ptr=self.ptr, owner=False)
        if view.size != self.size:
            raise ValueError("reshape changes the size")
        view._base = self  # keep the owning buffer alive
        return view


def sync() -> None:
    check(lib().ltb_ctx_synchronize(context()))
