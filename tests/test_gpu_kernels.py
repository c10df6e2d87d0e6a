"""Kernel-level checks through the C ABI (device pointers), against numpy on the
same inputs: slice GEMM for every op / dtype, SVT / SVD / singular values for
both slice orientations, the layout-only transform, reductions."""

import ctypes as C

import numpy as np
import paper_2202_02870_b200 as L
import pytest

from paper_2202_02870_b200 import _native as nat
import ltensor_oracle as O
from ltb_testutil import rel_err

pytestmark = pytest.mark.gpu

DTYPES = [np.float32, np.float64, np.complex64, np.complex128]


def rand(rng, shape, dt):
    x = rng.standard_normal(shape)
    if np.issubdtype(dt, np.complexfloating):
        x = x + 1j * rng.standard_normal(shape)
    return x.astype(dt)


def tol(dt):
    return 2e-5 if dt in (np.float32, np.complex64) else 1e-12


def op_apply(x, op):
    return {0: x, 1: np.swapaxes(x, -1, -2), 2: np.conj(x), 3: np.conj(np.swapaxes(x, -1, -2))}[op]


@pytest.mark.parametrize("dt", DTYPES)
@pytest.mark.parametrize("op_a", [0, 1, 2, 3])
@pytest.mark.parametrize("op_b", [0, 1, 2, 3])
@pytest.mark.parametrize("mnk", [(5, 7, 3), (70, 45, 130), (129, 131, 17)])
def test_slice_gemm(dt, op_a, op_b, mnk):
    rng = np.random.default_rng(hash((op_a, op_b, mnk)) % 2**32)
    m, n, k = mnk
    batch = 3
    a_log = rand(rng, (batch, m, k), dt)
    b_log = rand(rng, (batch, k, n), dt)
    a_st = np.ascontiguousarray(op_apply(a_log, op_a) if op_a in (0, 2) else op_apply(a_log, op_a))
    b_st = np.ascontiguousarray(op_apply(b_log, op_b) if op_b in (0, 2) else op_apply(b_log, op_b))
    # stored operands are op^{-1}(logical); op(stored) == logical for all four ops
    a_st = np.ascontiguousarray({0: a_log, 1: np.swapaxes(a_log, 1, 2), 2: np.conj(a_log),
                                 3: np.conj(np.swapaxes(a_log, 1, 2))}[op_a])
    b_st = np.ascontiguousarray({0: b_log, 1: np.swapaxes(b_log, 1, 2), 2: np.conj(b_log),
                                 3: np.conj(np.swapaxes(b_log, 1, 2))}[op_b])
    da = nat.DeviceArray.from_numpy(a_st)
    db = nat.DeviceArray.from_numpy(b_st)
    dc = nat.DeviceArray((batch, m, n), dt)
    lda = a_st.shape[2]
    ldb = b_st.shape[2]
    nat.check(nat.lib().ltb_slice_gemm(nat.context(), nat.dtype_code(dt), batch, m, n, k, op_a, da.ptr, lda,
                                       m * k, op_b, db.ptr, ldb, k * n, dc.ptr, n, m * n))
    ref = np.matmul(a_log.astype(np.complex128), b_log.astype(np.complex128))
    got = dc.numpy()
    assert np.linalg.norm(got - ref) / np.linalg.norm(ref) < tol(dt)


@pytest.mark.parametrize("dt", DTYPES)
@pytest.mark.parametrize("shape", [(6, 4), (4, 6), (1, 5), (5, 1), (33, 70), (70, 33), (64, 64)])
def test_slice_svt_and_values(dt, shape):
    rng = np.random.default_rng(7)
    batch = 4
    a = rand(rng, (batch,) + shape, dt)
    u, s, vh = np.linalg.svd(a.astype(np.complex128 if np.iscomplexobj(a) else np.float64), full_matrices=False)
    tau = float(np.median(s))
    ref = np.matmul(u * np.maximum(s - tau, 0)[:, None, :], vh)
    da = nat.DeviceArray.from_numpy(a)
    out = nat.DeviceArray(a.shape, dt)
    nat.check(nat.lib().ltb_slice_svt(nat.context(), nat.dtype_code(dt), batch, shape[0], shape[1], da.ptr, tau,
                                      out.ptr))
    got = out.numpy()
    assert np.linalg.norm(got - ref) / max(np.linalg.norm(ref), 1e-30) < 50 * tol(dt)
    sv = nat.DeviceArray((batch, min(shape)), nat.real_of(dt))
    nat.check(nat.lib().ltb_slice_singular_values(nat.context(), nat.dtype_code(dt), batch, shape[0], shape[1],
                                                  da.ptr, sv.ptr))
    np.testing.assert_allclose(sv.numpy(), s, rtol=50 * tol(dt), atol=50 * tol(dt) * s.max())


@pytest.mark.parametrize("dt", DTYPES)
@pytest.mark.parametrize("shape", [(6, 4), (4, 6), (5, 5), (3, 1), (120, 40), (40, 120)])
def test_slice_svd_full(dt, shape):
    rng = np.random.default_rng(9)
    batch = 3
    a = rand(rng, (batch,) + shape, dt)
    if shape == (5, 5):
        a[:, :, 3:] = 0  # rank deficient -> completion path
    m, n = shape
    da = nat.DeviceArray.from_numpy(a)
    u = nat.DeviceArray((batch, m, m), dt)
    v = nat.DeviceArray((batch, n, n), dt)
    s = nat.DeviceArray((batch, min(m, n)), nat.real_of(dt))
    nat.check(nat.lib().ltb_slice_svd(nat.context(), nat.dtype_code(dt), batch, m, n, da.ptr, u.ptr, s.ptr, v.ptr))
    U, S, V = u.numpy(), s.numpy(), v.numpy()
    k = min(m, n)
    sig = np.zeros((batch, m, n))
    sig[:, np.arange(k), np.arange(k)] = S
    recon = U @ sig @ np.conj(np.swapaxes(V, 1, 2))
    t = 50 * tol(dt)
    assert np.linalg.norm(recon - a) / np.linalg.norm(a) < t
    eye_m = np.broadcast_to(np.eye(m), (batch, m, m))
    eye_n = np.broadcast_to(np.eye(n), (batch, n, n))
    assert np.abs(np.conj(np.swapaxes(U, 1, 2)) @ U - eye_m).max() < t
    assert np.abs(np.conj(np.swapaxes(V, 1, 2)) @ V - eye_n).max() < t
    assert np.all(np.diff(S, axis=1) <= 0)


@pytest.mark.parametrize("dt", DTYPES)
def test_reductions(dt):
    rng = np.random.default_rng(3)
    x = rand(rng, (1000, 37), dt)
    y = rand(rng, (1000, 37), dt)
    dx, dy = nat.DeviceArray.from_numpy(x), nat.DeviceArray.from_numpy(y)
    out = (C.c_double * 2)()
    nat.check(nat.lib().ltb_reduce_sumsq(nat.context(), dx.code, dx.size, dx.ptr, dy.ptr, out))
    ref = np.sum(np.abs(x.astype(np.complex128) - y) ** 2)
    assert abs(out[0] - ref) / ref < 1e-6
    assert out[1] == pytest.approx(float(np.max(x.real)))
    nat.check(nat.lib().ltb_reduce_dot(nat.context(), dx.code, dx.size, dx.ptr, dy.ptr, out))
    ref = np.vdot(x.astype(np.complex128), y.astype(np.complex128))
    assert abs(complex(out[0], out[1]) - ref) / abs(ref) < 1e-5


@pytest.mark.parametrize("split", [3, 1])
@pytest.mark.parametrize("a_mn", [0, 1])
@pytest.mark.parametrize("b_mn", [0, 1])
@pytest.mark.parametrize("mnk", [(128, 128, 32), (256, 256, 128), (96, 200, 96), (300, 72, 36)])
def test_tc_gemm_tf32(split, a_mn, b_mn, mnk):
    """tcgen05 kind::tf32 engine (3xTF32 split) vs float64 numpy."""
    rng = np.random.default_rng(11)
    m, n, k = mnk
    batch = 2
    a = rng.standard_normal((batch, m, k)).astype(np.float32)
    b = rng.standard_normal((batch, k, n)).astype(np.float32)
    a_st = np.ascontiguousarray(np.swapaxes(a, 1, 2) if a_mn else a)  # a_mn: stored k x m
    b_st = np.ascontiguousarray(b if b_mn else np.swapaxes(b, 1, 2))  # b_mn: stored k x n, else n x k
    da, db = nat.DeviceArray.from_numpy(a_st), nat.DeviceArray.from_numpy(b_st)
    dc = nat.DeviceArray((batch, m, n), np.float32)
    lda, ldb = a_st.shape[2], b_st.shape[2]
    st = nat.lib().ltb_tc_gemm(nat.context(), batch, m, n, k, a_mn, da.ptr, lda, a_st.shape[1] * lda, b_mn, db.ptr,
                               ldb, b_st.shape[1] * ldb, dc.ptr, n, m * n, split)
    if st == 3:
        pytest.skip("tensor-core path unsupported for this alignment")
    nat.check(st)
    ref = np.matmul(a.astype(np.float64), b.astype(np.float64))
    err = np.linalg.norm(dc.numpy() - ref) / np.linalg.norm(ref)
    assert err < (2e-6 if split == 3 else 2e-3), err


# ---- blocked (block-cyclic, shared-memory column pairs) tier: slices beyond the resident tier,
# and small slices forced through it (odd column counts, a single block pair, n = 1)
BLOCKED_CASES = [(np.float32, (300, 280)), (np.float64, (240, 260)), (np.complex64, (250, 270)),
                 (np.complex128, (210, 200))]


@pytest.fixture
def force_blocked():
    nat.check(nat.lib().ltb_ctx_set_option(nat.context(), nat.OPT_FORCE_BLOCKED_SVD, 1))
    yield
    nat.check(nat.lib().ltb_ctx_set_option(nat.context(), nat.OPT_FORCE_BLOCKED_SVD, 0))


def _svt_check(dt, shape, batch=2, seed=11):
    rng = np.random.default_rng(seed)
    a = rand(rng, (batch,) + shape, dt)
    u, s, vh = np.linalg.svd(a.astype(np.complex128 if np.iscomplexobj(a) else np.float64), full_matrices=False)
    tau = float(np.median(s))
    ref = np.matmul(u * np.maximum(s - tau, 0)[:, None, :], vh)
    da = nat.DeviceArray.from_numpy(a)
    out = nat.DeviceArray(a.shape, dt)
    nat.check(nat.lib().ltb_slice_svt(nat.context(), nat.dtype_code(dt), batch, shape[0], shape[1], da.ptr, tau,
                                      out.ptr))
    assert np.linalg.norm(out.numpy() - ref) / max(np.linalg.norm(ref), 1e-30) < 50 * tol(dt)
    sv = nat.DeviceArray((batch, min(shape)), nat.real_of(dt))
    nat.check(nat.lib().ltb_slice_singular_values(nat.context(), nat.dtype_code(dt), batch, shape[0], shape[1],
                                                  da.ptr, sv.ptr))
    np.testing.assert_allclose(sv.numpy(), s, rtol=50 * tol(dt), atol=50 * tol(dt) * s.max())


def _svd_check(dt, shape, batch=2, seed=12):
    rng = np.random.default_rng(seed)
    a = rand(rng, (batch,) + shape, dt)
    m, n = shape
    da = nat.DeviceArray.from_numpy(a)
    u = nat.DeviceArray((batch, m, m), dt)
    v = nat.DeviceArray((batch, n, n), dt)
    s = nat.DeviceArray((batch, min(m, n)), nat.real_of(dt))
    nat.check(nat.lib().ltb_slice_svd(nat.context(), nat.dtype_code(dt), batch, m, n, da.ptr, u.ptr, s.ptr, v.ptr))
    U, S, V = u.numpy(), s.numpy(), v.numpy()
    k = min(m, n)
    sig = np.zeros((batch, m, n))
    sig[:, np.arange(k), np.arange(k)] = S
    t = 50 * tol(dt)
    assert np.linalg.norm(U @ sig @ np.conj(np.swapaxes(V, 1, 2)) - a) / np.linalg.norm(a) < t
    assert np.abs(np.conj(np.swapaxes(V, 1, 2)) @ V - np.eye(n)).max() < t
    assert np.all(np.diff(S, axis=1) <= 0)


@pytest.mark.parametrize("dt,shape", BLOCKED_CASES)
def test_blocked_tier_svt_and_values(dt, shape):
    _svt_check(dt, shape)


@pytest.mark.parametrize("dt,shape", [(np.float32, (260, 250)), (np.complex64, (240, 260))])
def test_blocked_tier_svd_full(dt, shape):
    _svd_check(dt, shape)


@pytest.mark.parametrize("dt", DTYPES)
@pytest.mark.parametrize("shape", [(6, 4), (4, 7), (5, 1), (33, 70), (71, 33), (64, 64), (3, 130)])
def test_blocked_tier_forced_small(dt, shape, force_blocked):
    _svt_check(dt, shape, batch=3)
    _svd_check(dt, shape, batch=3)


# ---- the tensor-core transform (dense Kronecker GEMM, resident pre-split K when P <= 96) in every
# layout orientation, against the CPU oracle's mode products (fp32 tolerance 1e-4 rel. Frobenius)
@pytest.mark.parametrize("trail", [(3, 2), (5, 8), (3, 32), (4, 25)])
@pytest.mark.parametrize("nt", [1, 130, 1000])
def test_tc_transform_layouts(trail, nt):
    import ltensor_oracle as O
    from paper_2202_02870_b200 import transforms as TR
    import paper_2202_02870_b200 as L

    rng = np.random.default_rng(len(trail) * 1000 + nt)
    shape = (nt, 1) + trail
    x = rng.standard_normal(shape).astype(np.float32)
    spec = L.make_spec("dct", shape)
    ref = O.forward(x.astype(np.float64), O.ospec("dct", shape)).reshape(nt, -1)  # tube-major (t, q)
    P = ref.shape[1]
    handle = TR.device_spec(spec, trail)
    dx = nat.DeviceArray.from_numpy(x.reshape(nt, P))
    for lo, shp, want in ((nat.TUBE_MAJOR, (nt, P), ref), (nat.SLICE_MAJOR, (P, nt), ref.T)):
        out, _ = TR.transform_device(dx, handle, nt, False, nat.TUBE_MAJOR, np.float32, lo, shp)
        got = out.numpy()
        assert np.linalg.norm(got - want) / np.linalg.norm(want) < 1e-5
    # inverse from slice-major input back to tube-major
    hat = nat.DeviceArray.from_numpy(np.ascontiguousarray(ref.T.astype(np.float32)))
    back, _ = TR.transform_device(hat, handle, nt, True, nat.SLICE_MAJOR, np.float32, nat.TUBE_MAJOR, (nt, P))
    assert np.linalg.norm(back.numpy() - x.reshape(nt, P)) / np.linalg.norm(x) < 1e-5


# ---- conjugate-pair SVT: for a real tensor under a DFT-type spec, solving one slice of every
# conjugate pair and mirroring must equal solving every slice (the Jacobi kernel is conjugation-
# equivariant), bit for bit
@pytest.mark.parametrize("kind,shape", [("fft", (20, 16, 6)), ("fft", (12, 30, 4, 5)), ("dct", (10, 9, 4))])
def test_spec_svt_mirror_matches_full(kind, shape):
    import paper_2202_02870_b200 as L
    from paper_2202_02870_b200 import linalg, transforms as TR

    rng = np.random.default_rng(21)
    x = rng.standard_normal(shape)
    spec = L.make_spec(kind, shape)
    hat = linalg._hat_stack(x, spec)
    P, i1, i2 = hat.shape
    tau = 0.7
    full = nat.DeviceArray(hat.shape, hat.dtype)
    mirr = nat.DeviceArray(hat.shape, hat.dtype)
    nat.check(nat.lib().ltb_slice_svt(nat.context(), hat.code, P, i1, i2, hat.ptr, tau, full.ptr))
    nat.check(nat.lib().ltb_spec_slice_svt(nat.context(), TR.device_spec(spec, shape[2:]).ptr, hat.code, P, i1, i2,
                                           hat.ptr, tau, mirr.ptr))
    np.testing.assert_array_equal(mirr.numpy(), full.numpy())


# ---- fp32 SVT through the QR-preconditioned kernel: rank-deficient, zero and duplicated-column
# slices (Householder steps with vanishing columns), both orientations
@pytest.mark.parametrize("shape", [(40, 50), (50, 40), (64, 64), (150, 170)])
def test_svt_qr_rank_deficient(shape):
    rng = np.random.default_rng(31)
    m, n = shape
    batch = 4
    a = np.zeros((batch, m, n), np.float32)
    a[0] = (rng.standard_normal((m, 5)) @ rng.standard_normal((5, n))).astype(np.float32)  # rank 5
    a[1] = 0.0                                                                              # zero slice
    col = rng.standard_normal((m, 1))
    a[2] = np.repeat(col, n, axis=1).astype(np.float32)                                     # rank 1, equal columns
    a[3] = rng.standard_normal((m, n)).astype(np.float32)                                   # full rank
    u, s, vh = np.linalg.svd(a.astype(np.float64), full_matrices=False)
    tau = 0.5
    ref = np.matmul(u * np.maximum(s - tau, 0)[:, None, :], vh)
    da = nat.DeviceArray.from_numpy(a)
    out = nat.DeviceArray(a.shape, np.float32)
    nat.check(nat.lib().ltb_slice_svt(nat.context(), nat.dtype_code(np.float32), batch, m, n, da.ptr, tau, out.ptr))
    got = out.numpy()
    for i in range(batch):
        den = max(np.linalg.norm(ref[i]), 1e-30)
        assert np.linalg.norm(got[i] - ref[i]) / den < 1e-4 or np.linalg.norm(got[i]) < 1e-6


@pytest.mark.parametrize("nbytes", [4, (1 << 20) + 4, (16 << 20) - 4, (16 << 20) + 4, (40 << 20) + 12])
def test_host_device_copies_pageable_and_pinned(nbytes):
    """Uploads / downloads of pageable numpy buffers go through the pinned staging pipeline
    (chunks of 16 MiB, threaded host copies): bit-exact round trips at chunk boundaries, and
    the same through pinned host memory (direct DMA)."""
    import torch

    rng = np.random.default_rng(nbytes)
    x = rng.integers(0, 2**32, size=nbytes // 4, dtype=np.uint32).view(np.float32)
    d = nat.DeviceArray.from_numpy(x)
    np.testing.assert_array_equal(d.numpy().view(np.uint32), x.view(np.uint32))
    pin = torch.empty(x.shape, dtype=torch.float32, pin_memory=True).numpy()
    d.numpy(out=pin)
    np.testing.assert_array_equal(pin.view(np.uint32), x.view(np.uint32))
    d2 = nat.DeviceArray.from_numpy(pin)
    np.testing.assert_array_equal(d2.numpy().view(np.uint32), x.view(np.uint32))


@pytest.mark.parametrize("i1,l,i2,trail", [
    (256, 128, 256, (3, 32)),   # BASELINE config 2
    (128, 40, 384, (3, 32)),    # L not a multiple of 32 (partial GEMM k-block), three column blocks
    (384, 64, 128, (4, 8)),     # P = 32: one k-block, three row blocks
    (128, 16, 128, (3, 8)),     # P = 24: partial transform k-block (zero-filled)
    (128, 40, 200, (3, 32)),    # I2 % 128 != 0: the four-launch path
])
def test_lprod_fused_kernel(i1, l, i2, trail):
    """The one-launch persistent *_L product (ltb_lprod_fused.cuh) against the fp64 oracle
    and against the four-launch path on the same buffers."""
    import ltensor_oracle as O
    from paper_2202_02870_b200.engine import LProductPlan

    rng = np.random.default_rng(i1 + l + i2)
    a_h = rng.standard_normal((i1, l) + trail, dtype=np.float32)
    b_h = rng.standard_normal((l, i2) + trail, dtype=np.float32)
    spec = L.make_spec("dct", (i1, i2) + trail)
    plan = LProductPlan(a_h.shape, b_h.shape, spec, np.float32)
    a = nat.DeviceArray.from_numpy(a_h)
    b = nat.DeviceArray.from_numpy(b_h)
    c = nat.DeviceArray(plan.c_shape, np.float32)
    c4 = nat.DeviceArray(plan.c_shape, np.float32)
    for _ in range(2):  # counters are reset per launch
        plan.run_fused(a, b, c)
    plan.run_fused(a, b, c4, fused=False)
    ref = O.l_product(a_h.astype(np.float64), b_h.astype(np.float64), O.ospec("dct", (i1, i2) + trail))
    got = c.numpy()
    assert np.isfinite(got).all()
    assert np.linalg.norm(got - ref) / np.linalg.norm(ref) < 1e-4
    assert np.linalg.norm(got - c4.numpy()) / np.linalg.norm(ref) < 1e-5


@pytest.mark.parametrize("dt,a_shape,n", [(np.float32, (256, 128, 3, 32), 256), (np.float64, (96, 40, 2, 16), 128),
                                           (np.float32, (200, 24, 4, 8), 130), (np.float32, (64, 16, 100), 66)])
def test_l_product_pinned_host_pipeline(dt, a_shape, n):
    """Pinned A, B and C go straight to the DMA engines in the chunked host pipeline (no staging):
    the product matches the oracle and the pageable (staged) path bit for bit, including a ragged
    last row chunk."""
    import torch

    rng = np.random.default_rng(7)
    b_shape = (a_shape[1], n) + a_shape[2:]
    a = rng.standard_normal(a_shape).astype(dt)
    b = rng.standard_normal(b_shape).astype(dt)
    spec = L.make_spec("dct", (a_shape[0], n) + a_shape[2:])
    tdt = torch.float32 if dt == np.float32 else torch.float64
    pa = torch.empty(a_shape, dtype=tdt, pin_memory=True).numpy()
    pb = torch.empty(b_shape, dtype=tdt, pin_memory=True).numpy()
    pc = torch.empty((a_shape[0], n) + a_shape[2:], dtype=tdt, pin_memory=True).numpy()
    pa[...] = a
    pb[...] = b
    L.l_product(pa, pb, spec, out=pc)
    plain = L.l_product(a, b, spec)
    ref = O.l_product(a.astype(np.float64), b.astype(np.float64), O.ospec("dct", pc.shape))
    assert rel_err(pc, ref) < (1e-4 if dt == np.float32 else 1e-10)
    np.testing.assert_array_equal(pc, plain)


@pytest.mark.parametrize("trail,kind", [((5, 120), "dct"), ((3, 100, 2), "dct"), ((7, 90), "explicit_dct"),
                                        ((6, 98), "explicit_rand")])
def test_tile_engine_even_odd_modes(trail, kind):
    """fp32 transforms through the shared-memory tile engine (P > 512, so not the tensor-core
    Kronecker path): DCT modes (and an explicit DCT matrix) take the even/odd half-matrix mode
    steps, a random explicit matrix the full ones; forward and inverse against the oracle."""
    rng = np.random.default_rng(11)
    shape = (9, 7) + trail
    x = rng.standard_normal(shape).astype(np.float32)
    if kind == "dct":
        spec, ospec = L.make_spec("dct", shape), O.ospec("dct", shape)
    else:
        n = trail[-1]
        m = L.build_dct_matrix(n) if kind == "explicit_dct" else np.linalg.qr(rng.standard_normal((n, n)))[0]
        mats = {len(shape): m}
        md = [len(shape)]
        spec = L.make_spec("explicit", shape, modes=md, matrices=mats)
        ospec = O.ospec("explicit", shape, modes=md, matrices=mats)
    y = L.apply_l(x, spec)
    ref = O.forward(x.astype(np.float64), ospec)
    assert rel_err(y, ref) < 1e-5
    back = L.apply_l_inv(y, spec)
    assert rel_err(back, x) < 1e-5
