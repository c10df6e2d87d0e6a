"""Device-resident plans for the hot path (no host round trips): used by the
benchmark, the multi-GPU driver and anyone holding inputs on the GPU already.

LProductPlan — l_product (linalg.py:34-43) as K1(A), K1(B), K2, K1' over
preallocated device buffers; `run` optionally records a CUDA event between
phases so per-kernel time shares can be read on the launching stream.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _native as nat
from .core import num_rep
from .transforms import _check_shape, check_real_residual, device_spec, forward_dtype


class LProductPlan:
    def __init__(self, a_shape, b_shape, spec, in_dtype=np.float32):
        a_shape, b_shape = tuple(a_shape), tuple(b_shape)
        _check_shape(a_shape, spec)
        _check_shape(b_shape, spec)
        self.m, self.k, self.n = a_shape[0], a_shape[1], b_shape[1]
        self.trailing = a_shape[2:]
        self.P = num_rep(a_shape)
        self.in_dtype = np.dtype(in_dtype)
        self.hat_dtype = forward_dtype(self.in_dtype, spec)
        self.src_dtype = nat.real_of(self.hat_dtype)
        self.out_real = not np.iscomplexobj(np.zeros(0, self.in_dtype))
        self.out_dtype = nat.real_of(self.hat_dtype) if self.out_real else self.hat_dtype
        self.handle = device_spec(spec, self.trailing)
        self.mode_sizes = list(spec.sizes)
        self.ha = nat.DeviceArray((self.P, self.m, self.k), self.hat_dtype)
        self.hb = nat.DeviceArray((self.P, self.k, self.n), self.hat_dtype)
        self.hc = nat.DeviceArray((self.P, self.m, self.n), self.hat_dtype)
        self.c_shape = (self.m, self.n) + self.trailing
        self._sums = (C.c_double * 2)()
        # K1(A) and K1(B) as one call (one tensor-core launch) when the tube counts match
        self.paired = self.m * self.k == self.k * self.n
        # whole-product entry (ltb_l_product_device): one persistent kernel for fp32 real specs
        self.real_spec = not np.iscomplexobj(np.zeros(0, self.hat_dtype))
        code = nat.dtype_code(self.src_dtype)
        self.ws_bytes = int(nat.lib().ltb_l_product_ws_bytes(self.handle.ptr, self.m, self.k, self.n, code))
        # zero-filled once: the fused kernel leaves its counters zeroed after every launch
        self.ws = nat.DeviceArray.zeros((max(self.ws_bytes, 16),), np.uint8) if self.real_spec else None

    def flops(self) -> int:
        """Algorithmic flop count: slice GEMM + separable real transforms."""
        per = 2 * sum(self.mode_sizes)
        ea, eb, ec = self.m * self.k * self.P, self.k * self.n * self.P, self.m * self.n * self.P
        return 2 * self.m * self.k * self.n * self.P + per * (ea + eb + ec)

    def bytes(self) -> int:
        """Minimal fused HBM traffic: read A, B, write C."""
        s = nat.real_of(self.hat_dtype).itemsize
        return s * (self.m * self.k + self.k * self.n + self.m * self.n) * self.P

    def run_fused(self, a: nat.DeviceArray, b: nat.DeviceArray, c: nat.DeviceArray, fused: bool = True):
        """The whole product through ltb_l_product_device: one persistent tcgen05 kernel (forward
        transforms, slice GEMMs and inverse transform overlapped) when the shape fits, else the
        four phases; real transform domains only."""
        if not self.real_spec:
            return self.run(a, b, c)
        nat.check(nat.lib().ltb_l_product_device(nat.context(), self.handle.ptr, self.m, self.k, self.n, a.code, a.ptr,
                                                 b.ptr, c.ptr, self.ws.ptr, self.ws_bytes, 3 if fused else 0))
        return c

    def run(self, a: nat.DeviceArray, b: nat.DeviceArray, c: nat.DeviceArray, marks=None, check_real=False,
            phases=(0, 1, 2, 3)):
        """Enqueue the phases K1(A)=0, K1(B)=1, K2=2, K1'=3 (all by default); `marks(i)`
        is called before phase i and after the last one (i = 4).  When `paired`, phase 0
        transforms A and B together and phase 1 enqueues nothing."""
        lib, ctx = nat.lib(), nat.context()
        h = self.handle.ptr
        mark = marks or (lambda i: None)
        m, k, n, P = self.m, self.k, self.n, self.P
        sums = None
        mark(0)
        if 0 in phases and self.paired:  # phase 0 transforms both operands, phase 1 is empty
            nat.check(lib.ltb_transform_pair(ctx, h, m * k, 0, a.code, nat.TUBE_MAJOR, a.ptr, b.ptr, self.ha.code,
                                             nat.SLICE_MAJOR, self.ha.ptr, self.hb.ptr))
        elif 0 in phases:
            nat.check(lib.ltb_transform(ctx, h, m * k, 0, a.code, nat.TUBE_MAJOR, a.ptr, self.ha.code,
                                        nat.SLICE_MAJOR, self.ha.ptr, None))
        mark(1)
        if 1 in phases and not self.paired:
            nat.check(lib.ltb_transform(ctx, h, k * n, 0, b.code, nat.TUBE_MAJOR, b.ptr, self.hb.code,
                                        nat.SLICE_MAJOR, self.hb.ptr, None))
        mark(2)
        if 2 in phases:
            nat.check(lib.ltb_slice_gemm(ctx, self.ha.code, P, m, n, k, nat.OP_N, self.ha.ptr, k, m * k, nat.OP_N,
                                         self.hb.ptr, n, k * n, self.hc.ptr, n, m * n))
        mark(3)
        if 3 in phases:
            if check_real and self.out_real and np.iscomplexobj(np.zeros(0, self.hat_dtype)):
                sums = self._sums
            nat.check(lib.ltb_transform(ctx, h, m * n, 1, self.hc.code, nat.SLICE_MAJOR, self.hc.ptr, c.code,
                                        nat.TUBE_MAJOR, c.ptr, sums))
        mark(4)
        if sums is not None:
            check_real_residual((sums[0], sums[1]), c.dtype)
        return c


