"""CUDA path vs the reference's own outputs (golden fixtures) on the same seeded
inputs.  Tolerances (BASELINE north_star): relative Frobenius error <= 1e-10 for
float64 work, <= 1e-4 for float32; masks / indices bit-exact; SVD factors
compared through the factor-independent quantities (singular values, S, the
reconstruction, orthogonality)."""

import numpy as np
import pytest

import paper_2202_02870_b200 as L
from paper_2202_02870_b200 import core
from ltb_testutil import build_spec, case_names, meta, rel_err

pytestmark = pytest.mark.gpu


def tol_for(*arrays):
    return 1e-4 if any(np.asarray(a).dtype in (np.float32, np.complex64) for a in arrays) else 1e-10


@pytest.mark.parametrize("name", case_names("t_"))
def test_transform_parity(golden, name):
    spec = build_spec(L, golden, name)
    x = golden[f"{name}/x"]
    ref_fwd = golden[f"{name}/fwd"]
    fwd = L.apply_l(x, spec)
    assert fwd.dtype == ref_fwd.dtype
    assert rel_err(fwd, ref_fwd) < tol_for(x)
    inv = L.apply_l_inv(ref_fwd, spec, assume_real=True)
    assert inv.dtype == golden[f"{name}/inv"].dtype
    assert rel_err(inv, golden[f"{name}/inv"]) < tol_for(x)
    if f"{name}/fwd_explicit" in golden.files:
        fe = L.apply_l(x, spec, explicit=True)
        assert fe.dtype == golden[f"{name}/fwd_explicit"].dtype
        assert rel_err(fe, golden[f"{name}/fwd_explicit"]) < 1e-10


@pytest.mark.parametrize("name", case_names("p_"))
def test_product_parity(golden, name):
    spec = build_spec(L, golden, name)
    a, b = golden[f"{name}/a"], golden[f"{name}/b"]
    c = L.l_product(a, b, spec)
    assert c.dtype == golden[f"{name}/c"].dtype
    assert rel_err(c, golden[f"{name}/c"]) < tol_for(a, b)


def test_product_known_answers():
    tube = lambda *v: np.asarray(v, dtype=float).reshape(1, 1, len(v))  # noqa: E731
    np.testing.assert_allclose(L.l_product(tube(1, 2), tube(3, 4), L.make_spec("fft", (1, 1, 2))).ravel(),
                               [11.0, 10.0], atol=1e-12)
    np.testing.assert_allclose(L.l_product(tube(1, 2), tube(3, 4), L.make_spec("cprod", (1, 1, 2))).ravel(),
                               [3.0, 26.0], atol=1e-12)
    np.testing.assert_allclose(L.apply_l(tube(1, 2), L.make_spec("cprod", (1, 1, 2))).ravel(), [5.0, 1.0],
                               atol=1e-12)
    np.testing.assert_allclose(L.facewise_product(np.array([5.0, 1.0]).reshape(1, 1, 2),
                                                  np.array([11.0, 3.0]).reshape(1, 1, 2)).ravel(), [55.0, 3.0])
    np.testing.assert_allclose(L.mode_n_product(tube(1, 2), np.array([[1.0, 2.0], [1.0, 0.0]]), 3).ravel(), [5, 1])


@pytest.mark.parametrize("name", case_names("s_"))
def test_svd_family_parity(golden, name):
    spec = build_spec(L, golden, name)
    x = golden[f"{name}/x"]
    tol = tol_for(x)
    f = L.t_svd(x, spec)
    assert rel_err(f.s, golden[f"{name}/s"]) < tol
    np.testing.assert_allclose(f.tube_norms, golden[f"{name}/tube_norms"], rtol=tol, atol=tol)
    # reconstruction u * s * v^T == x and orthogonality of the factors
    recon = L.l_product(L.l_product(f.u, f.s, L.make_spec(spec.kind, (x.shape[0], x.shape[1]) + x.shape[2:])),
                        L.l_transpose(f.v, L.make_spec(spec.kind, f.v.shape)), spec) if spec.kind != "cprod" else None
    if recon is not None:
        assert rel_err(recon, x) < 10 * tol
    # singular values: device slice order -> reference p-order
    sv = L.linalg._singular_values(x, spec)
    perm = core.slice_order_permutation(x.shape[2:])
    np.testing.assert_allclose(sv[perm], golden[f"{name}/sv"], rtol=tol, atol=tol * max(1.0, golden[f"{name}/sv"].max()))
    rr = L.ranks(x, spec)
    np.testing.assert_array_equal(rr.multirank, golden[f"{name}/multirank"])
    assert rr.tubal == int(golden[f"{name}/tubal"])
    if f"{name}/svt" in golden.files:
        tau = meta(golden, name)["tau"]
        out = L.svt(x, tau, spec)
        assert out.dtype == golden[f"{name}/svt"].dtype
        assert rel_err(out, golden[f"{name}/svt"]) < tol
        assert np.isclose(L.nuclear_norm(x, spec), float(golden[f"{name}/nuclear"]), rtol=tol)
        assert np.isclose(L.spectral_norm(x, spec), float(golden[f"{name}/spectral"]), rtol=tol)


@pytest.mark.parametrize("name", case_names("c_"))
def test_completion_parity(golden, name):
    md = meta(golden, name)
    m = golden[f"{name}/m"]
    spec = build_spec(L, golden, name, shape=m.shape)
    gt = golden[f"{name}/gt"] if f"{name}/gt" in golden.files else None
    cfg = L.CompletionConfig(spec=spec, **md["cfg"])
    x, trace = L.pga_complete(m, golden[f"{name}/mask"], cfg, ground_truth=gt, precision="fp64")
    assert x.dtype == np.float64
    assert trace.status == md["status"]
    assert trace.iterations == len(golden[f"{name}/mu"])
    assert [r.t for r in trace.records] == list(golden[f"{name}/t"])
    np.testing.assert_allclose([r.mu for r in trace.records], golden[f"{name}/mu"], rtol=1e-14)
    np.testing.assert_allclose([r.rel_change for r in trace.records], golden[f"{name}/rel"], rtol=1e-7)
    assert rel_err(x, golden[f"{name}/x_out"]) < 1e-10
    if gt is not None:
        np.testing.assert_allclose([r.rse for r in trace.records], golden[f"{name}/rse"], rtol=1e-8)
        np.testing.assert_allclose([r.psnr for r in trace.records], golden[f"{name}/psnr"], rtol=1e-8)


def test_completion_fp32_path(golden):
    name = "c_config3s"
    md = meta(golden, name)
    m = golden[f"{name}/m"]
    assert m.dtype == np.float32
    spec = build_spec(L, golden, name, shape=m.shape)
    x, trace = L.pga_complete(m, golden[f"{name}/mask"], L.CompletionConfig(spec=spec, **md["cfg"]))
    assert x.dtype == np.float64 and trace.iterations == 20
    assert rel_err(x, golden[f"{name}/x_out"]) < 1e-4


def test_pinned_rse_regression(golden):
    pinned = {"fft": 0.0003459755997733272, "dct": 0.00020922751673777}
    for kind, val in pinned.items():
        m = golden[f"c_pinned_{kind}/m"]
        spec = L.make_spec(kind, m.shape)
        mask = L.sample_mask(m.shape, 0.5, 7)
        out, trace = L.pga_complete(m, mask, L.CompletionConfig(spec=spec, max_iters=300))
        final = L.rse(out, m)
        assert final < 1e-2 and np.isclose(final, val, rtol=1e-6), (kind, final, val, trace.iterations)


def test_project_omega_bit_exact(golden):
    m = golden["c_fft/m"]
    mask = golden["c_fft/mask"]
    out = L.project_omega(m, mask)
    np.testing.assert_array_equal(out, np.where(mask, m, 0.0))
    np.testing.assert_array_equal(L.project_omega(out, mask), out)


def test_deterministic_bitwise(golden):
    m = golden["c_fft/m"]
    mask = golden["c_fft/mask"]
    cfg = L.CompletionConfig(spec=L.make_spec("fft", m.shape), max_iters=40)
    a, _ = L.pga_complete(m, mask, cfg)
    b, _ = L.pga_complete(m, mask, cfg)
    np.testing.assert_array_equal(a, b)


@pytest.mark.parametrize("name", case_names("b_"))
def test_cprod_product_matches_btph(golden, name):
    """The CUDA l_product under the non-unitary cprod transform equals the reference's
    block-Toeplitz-plus-Hankel matrix product (btph.py:140-149) on the same inputs."""
    spec = build_spec(L, golden, name)
    c = L.l_product(golden[f"{name}/a"], golden[f"{name}/b"], spec)
    assert rel_err(c, golden[f"{name}/c"]) < 1e-10
