"""Complex64 work on the tensor cores and the carried (warm-started) complex SVT of the blocked
Jacobi tier (config 4's path: 1024 x 1024 complex slices), against numpy / the fp64 oracle on the
same seeded inputs.  The blocked tier is forced on small slices (OPT_FORCE_BLOCKED_SVD) so that
the tests finish in seconds; the full-size run is timed by bench.py.

Reference: svt linalg.py:168-181, pga_complete completion.py:141-202, mode products core.py:110-134."""

import numpy as np
import paper_2202_02870_b200 as L
import pytest

from paper_2202_02870_b200 import _native as nat
import ltensor_oracle as O
from ltb_testutil import rel_err

pytestmark = pytest.mark.gpu


def crand(rng, shape):
    return (rng.standard_normal(shape) + 1j * rng.standard_normal(shape)).astype(np.complex64)


@pytest.fixture
def force_blocked():
    nat.check(nat.lib().ltb_ctx_set_option(nat.context(), nat.OPT_FORCE_BLOCKED_SVD, 1))
    yield
    nat.check(nat.lib().ltb_ctx_set_option(nat.context(), nat.OPT_FORCE_BLOCKED_SVD, 0))


# ---- complex64 GEMM through the real 2 x 2 representation on tcgen05 (op_a N / C, every op_b),
# shapes whose strides TMA accepts (even k, n), shared B (stride 0), row scaling
@pytest.mark.parametrize("op_a", [0, 2])
@pytest.mark.parametrize("op_b", [0, 1, 2, 3])
@pytest.mark.parametrize("mnk", [(128, 64, 32), (200, 96, 130), (1024, 256, 64), (64, 32, 16)])
def test_complex_gemm_tensor_core(op_a, op_b, mnk):
    rng = np.random.default_rng(hash((op_a, op_b, mnk)) % 2**32)
    m, n, k = mnk
    batch = 3
    a_log = crand(rng, (batch, m, k))
    b_log = crand(rng, (batch, k, n))
    a_st = np.ascontiguousarray({0: a_log, 2: np.conj(a_log)}[op_a])
    b_st = np.ascontiguousarray({0: b_log, 1: np.swapaxes(b_log, 1, 2), 2: np.conj(b_log),
                                 3: np.conj(np.swapaxes(b_log, 1, 2))}[op_b])
    da, db = nat.DeviceArray.from_numpy(a_st), nat.DeviceArray.from_numpy(b_st)
    dc = nat.DeviceArray((batch, m, n), np.complex64)
    nat.check(nat.lib().ltb_slice_gemm(nat.context(), nat.dtype_code(np.complex64), batch, m, n, k, op_a, da.ptr,
                                       a_st.shape[2], m * k, op_b, db.ptr, b_st.shape[2], k * n, dc.ptr, n, m * n))
    ref = np.matmul(a_log.astype(np.complex128), b_log.astype(np.complex128))
    assert rel_err(dc.numpy(), ref) < 5e-6


def test_complex_gemm_shared_b():
    rng = np.random.default_rng(5)
    batch, m, n, k = 4, 128, 64, 48
    a = crand(rng, (batch, m, k))
    b = crand(rng, (k, n))
    da, db = nat.DeviceArray.from_numpy(a), nat.DeviceArray.from_numpy(b)
    dc = nat.DeviceArray((batch, m, n), np.complex64)
    nat.check(nat.lib().ltb_slice_gemm(nat.context(), nat.dtype_code(np.complex64), batch, m, n, k, 0, da.ptr, k,
                                       m * k, 0, db.ptr, n, 0, dc.ptr, n, m * n))
    assert rel_err(dc.numpy(), a.astype(np.complex128) @ b.astype(np.complex128)) < 5e-6


def _svt_ref(g, tau):
    u, s, vh = np.linalg.svd(g.astype(np.complex128), full_matrices=False)
    return np.matmul(u * np.maximum(s - tau, 0)[:, None, :], vh), s


def _carry_call(g, tau, vt, warm):
    batch, i1, i2 = g.shape
    dg = nat.DeviceArray.from_numpy(g)
    out = nat.DeviceArray(g.shape, np.complex64)
    nat.check(nat.lib().ltb_slice_svt_carry_c64(nat.context(), batch, i1, i2, dg.ptr, float(tau), out.ptr, vt.ptr,
                                                int(warm)))
    return out.numpy()


@pytest.mark.parametrize("shape", [(96, 64), (130, 48), (64, 64)])
def test_carried_complex_svt_blocked(shape, force_blocked):
    """Cold call, then warm calls on slowly moving slices: every call matches numpy's SVT, the
    carried V^T is unitary and a warm call takes fewer Jacobi sweeps than the cold one."""
    rng = np.random.default_rng(3)
    batch, (i1, i2) = 5, shape
    low = crand(rng, (batch, i1, 6)) @ crand(rng, (batch, 6, i2))
    g = (low + 0.3 * crand(rng, (batch, i1, i2))).astype(np.complex64)
    g[3] *= 1e-3  # ||G||_F <= tau: exact zero output, not solved
    ref, s = _svt_ref(g, 0.0)
    tau = float(np.median(s[0])) * 1.5
    vt = nat.DeviceArray((batch, i2, i2), np.complex64)
    sweeps = []
    for it in range(4):
        nat.jacobi_stats(reset=True)
        got = _carry_call(g, tau, vt, warm=it > 0)
        sl, sw = nat.jacobi_stats(reset=True)
        sweeps.append(sw / max(sl, 1))
        ref, s = _svt_ref(g, tau)
        assert rel_err(got, ref) < 1e-4, (it, rel_err(got, ref))
        assert not np.any(got[3])
        v = vt.numpy()
        for b in (0, 1, 2, 4):
            assert np.abs(v[b].conj() @ v[b].T - np.eye(i2)).max() < 1e-4
        # rows of VT are right singular vectors of G: |VT conj(V_ref)| ~ identity on separated sigma
        g = (g + 0.01 * crand(rng, g.shape) * np.abs(g).mean()).astype(np.complex64)
    assert min(sweeps[1:]) < sweeps[0], sweeps  # (truncated warm sweeps are cheaper, not always fewer)


@pytest.mark.parametrize("tau_scale", [2.0, 0.6])
def test_carried_complex_svt_truncated_sweeps(tau_scale, force_blocked):
    """Warm calls rotate only the block pairs that involve a leading block (sigma-sorted carried
    bases) and certify the rest by the trace bound tr(S^64): tau at twice the top of the noise
    bulk (the certificate holds: far fewer block rounds than full sweeps) and inside the bulk
    (it fails or every block leads: full sweeps); every call matches numpy's SVT."""
    rng = np.random.default_rng(21)
    batch, i1, i2 = 3, 200, 144
    low = crand(rng, (batch, i1, 6)) @ crand(rng, (batch, 6, i2))
    noise = 0.3
    g = (low + noise * crand(rng, (batch, i1, i2))).astype(np.complex64)
    bulk_top = noise * np.sqrt(2.0) * (np.sqrt(i1) + np.sqrt(i2))
    tau = tau_scale * bulk_top
    vt = nat.DeviceArray((batch, i2, i2), np.complex64)
    sweeps = []
    for it in range(5):
        nat.jacobi_stats(reset=True)
        got = _carry_call(g, tau, vt, warm=it > 0)
        sl, sw = nat.jacobi_stats(reset=True)
        sweeps.append(sw / max(sl, 1))
        ref, s = _svt_ref(g, tau)
        assert rel_err(got, ref) < 1e-4, (it, rel_err(got, ref))
        v = vt.numpy()
        for b in range(batch):
            assert np.abs(v[b].conj() @ v[b].T - np.eye(i2)).max() < 1e-4
        g = (g + 0.02 * noise * crand(rng, g.shape)).astype(np.complex64)


def test_carried_complex_svt_rank_deficient(force_blocked):
    """Vanishing singular values: the tiny columns' inner products are so small that their squares
    underflow (the packed rotation computes the phase scaled by the larger component); every
    call stays correct, the carried basis finite and unitary."""
    rng = np.random.default_rng(8)
    batch, i1, i2 = 2, 80, 40
    g = (crand(rng, (batch, i1, 5)) @ crand(rng, (batch, 5, i2))).astype(np.complex64)  # rank 5 of 40
    vt = nat.DeviceArray((batch, i2, i2), np.complex64)
    for it in range(3):
        ref, s = _svt_ref(g, 1.0)
        got = _carry_call(g, 1.0, vt, warm=it > 0)
        assert rel_err(got, ref) < 1e-4
        v = vt.numpy()
        assert np.all(np.isfinite(v))
        for b in range(batch):
            assert np.abs(v[b].conj() @ v[b].T - np.eye(i2)).max() < 1e-4


def test_carried_complex_svt_unsupported_shapes():
    rng = np.random.default_rng(1)
    g = crand(rng, (2, 48, 64))  # I1 < I2
    vt = nat.DeviceArray((2, 48, 48), np.complex64)
    dg = nat.DeviceArray.from_numpy(g)
    out = nat.DeviceArray(g.shape, np.complex64)
    st = nat.lib().ltb_slice_svt_carry_c64(nat.context(), 2, 48, 64, dg.ptr, 1.0, out.ptr, vt.ptr, 0)
    with pytest.raises(L.errors.UnsupportedSpecError):
        nat.check(st)


def test_config4_recipe_pga_blocked_carry(force_blocked):
    """Config 4's recipe (explicit Q (x) DFT, complex64 transform domain, conjugate-mirrored slices,
    Bernoulli(0.3)) at 64 x 48 x 3 x 8 with the blocked tier forced, so the PGA loop takes the
    carried complex SVT that the 1024 x 1024 slices take: 50 iterations against the fp64 oracle."""
    rng = np.random.default_rng(0)
    shape = (64, 48, 3, 8)
    q, _ = np.linalg.qr(rng.standard_normal((3, 3)))
    f = L.build_fourier_matrix(8)
    a = rng.standard_normal((64, 5, 3, 8), dtype=np.float32)
    b = rng.standard_normal((5, 48, 3, 8), dtype=np.float32)
    spec = L.make_spec("explicit", shape, matrices={3: q, 4: f})
    ospec = O.ospec("explicit", shape, matrices={3: q, 4: f})
    m = O.l_product(a.astype(np.float64), b.astype(np.float64), ospec).astype(np.float32)
    mask = rng.random(m.shape) < 0.3
    nat.jacobi_stats(reset=True)
    x, trace = L.pga_complete(m, mask, L.CompletionConfig(spec=spec, tol=1e-300, max_iters=50))
    ref, recs, _ = O.pga_complete(m.astype(np.float64), mask, ospec, tol=1e-300, max_iters=50)
    assert trace.iterations == 50
    assert rel_err(x, ref) < 1e-4
    rc = np.array([r.rel_change for r in trace.records])
    rr = np.array([r[3] for r in recs])
    fin = np.isfinite(rr)
    np.testing.assert_array_equal(np.isfinite(rc), fin)
    assert np.max(np.abs(rc[fin] - rr[fin]) / np.maximum(rr[fin], 1e-12)) < 1e-2


def test_config4_recipe_256_truncated_vs_oracle_and_full_sweeps():
    """Config 4's recipe at 256 x 256 x 3 x 8 (complex64 slices beyond shared memory: the carried blocked
    path with truncated sweeps is what runs by default), 45 iterations: against the fp64 oracle (1e-4) and
    against the same run with full sweeps (LTB_OPT_FULL_SWEEPS)."""
    rng = np.random.default_rng(0)
    shape = (256, 256, 3, 8)
    q, _ = np.linalg.qr(rng.standard_normal((3, 3)))
    f = L.build_fourier_matrix(8)
    a = rng.standard_normal((256, 8, 3, 8), dtype=np.float32)
    b = rng.standard_normal((8, 256, 3, 8), dtype=np.float32)
    spec = L.make_spec("explicit", shape, matrices={3: q, 4: f})
    ospec = O.ospec("explicit", shape, matrices={3: q, 4: f})
    m = O.l_product(a.astype(np.float64), b.astype(np.float64), ospec).astype(np.float32)
    mask = rng.random(m.shape) < 0.3
    cfg = L.CompletionConfig(spec=spec, tol=1e-300, max_iters=45)
    nat.jacobi_stats(reset=True)
    x, trace = L.pga_complete(m, mask, cfg)
    sl_t, sw_t = nat.jacobi_stats(reset=True)
    nat.check(nat.lib().ltb_ctx_set_option(nat.context(), nat.OPT_FULL_SWEEPS, 1))
    try:
        xf, _ = L.pga_complete(m, mask, cfg)
    finally:
        nat.check(nat.lib().ltb_ctx_set_option(nat.context(), nat.OPT_FULL_SWEEPS, 0))
    ref, recs, _ = O.pga_complete(m.astype(np.float64), mask, ospec, tol=1e-300, max_iters=45)
    assert trace.iterations == 45
    assert rel_err(x, ref) < 1e-4
    assert rel_err(xf, ref) < 1e-4
    assert rel_err(x, xf) < 1e-4
    assert np.count_nonzero(x) > 0  # the run got past the all-zero iterations
