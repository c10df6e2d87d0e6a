"""Edge cases of the reference's own test suite (pkg/tests/test_linalg.py, test_completion.py)
on the CUDA path: zero tensors, 1x1 slices, thresholds that keep nothing or everything,
empty / full observation masks, an all-zero observation, order-2 input.  Expected values are
what the reference returns on the same inputs (checked in this container)."""

import numpy as np
import pytest

import paper_2202_02870_b200 as L
from paper_2202_02870_b200.errors import TransformError

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("kind", ["dct", "fft"])
def test_zero_tensor_family(kind):
    z = np.zeros((3, 4, 5))
    spec = L.make_spec(kind, z.shape)
    np.testing.assert_array_equal(L.svt(z, 0.5, spec), z)
    f = L.t_svd(z, spec)
    assert np.all(f.s == 0) and f.s.shape == (3, 4, 5)
    # the factors stay orthogonal (completion of a rank-0 slice)
    eye_u = L.l_product(L.l_transpose(f.u, spec), f.u, spec)
    np.testing.assert_allclose(eye_u, L.identity_tensor(3, (5,), spec), atol=1e-10)
    r = L.ranks(z, spec)
    assert r.tubal == 0 and np.all(r.multirank == 0) and r.average == 0.0
    assert L.spectral_norm(z, spec) == 0.0
    assert L.nuclear_norm(z, spec) == 0.0


def test_one_by_one_slices():
    x = np.ones((1, 1, 5))
    spec = L.make_spec("dct", x.shape)
    f = L.t_svd(x, spec)
    np.testing.assert_allclose(L.l_product(L.l_product(f.u, f.s, spec), L.l_transpose(f.v, spec), spec), x,
                               atol=1e-12)


def test_threshold_extremes():
    rng = np.random.default_rng(0)
    m = rng.standard_normal((4, 4, 3))
    spec = L.make_spec("dct", m.shape)
    np.testing.assert_array_equal(L.svt(m, 1e9, spec), np.zeros_like(m))
    np.testing.assert_allclose(L.svt(m, 0.0, spec), m, atol=1e-12)
    m32 = m.astype(np.float32)
    np.testing.assert_array_equal(L.svt(m32, 1e9, spec), np.zeros_like(m32))


def test_pga_mask_extremes():
    m = np.random.default_rng(0).standard_normal((4, 4, 3))
    spec = L.make_spec("dct", m.shape)
    x, tr = L.pga_complete(m, np.zeros(m.shape, bool), L.CompletionConfig(spec=spec, max_iters=5))
    np.testing.assert_array_equal(x, np.zeros_like(m))
    assert tr.status == "converged" and tr.iterations == 1 and tr.records[0].rel_change == 0.0
    assert tr.records[0].mu == pytest.approx(4.951257123176576, rel=1e-14)
    x, tr = L.pga_complete(m, np.ones(m.shape, bool), L.CompletionConfig(spec=spec, max_iters=5))
    assert tr.status == "max-iters" and tr.iterations == 5
    x, tr = L.pga_complete(np.zeros((4, 4, 3)), np.ones((4, 4, 3), bool), L.CompletionConfig(spec=spec, max_iters=5))
    rec = tr.records[-1]
    assert tr.iterations == 1 and rec.mu == 0.0 and rec.rel_change == 0.0 and tr.status == "converged"
    np.testing.assert_array_equal(x, np.zeros((4, 4, 3)))


def test_order_two_refused():
    with pytest.raises(TransformError):
        L.make_spec("dct", (2, 2))
