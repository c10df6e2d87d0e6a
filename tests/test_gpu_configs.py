"""BASELINE.json configurations at (or near) full size on the GPU, checked against the CPU
oracle run here on the same seeded inputs (the oracle is the checker only), against compact
fixtures of the reference's own outputs where the host run is too slow for the test session
(tests/golden/configs.npz, tests/golden/make_config_fixtures.py), and through size-independent
properties.  Tolerances (north_star):
1e-4 relative Frobenius for float32 work, 1e-10 for float64."""

import numpy as np
import pytest

import ltensor_oracle as O
import paper_2202_02870_b200 as L
from paper_2202_02870_b200 import core
from config_recipes import NSAMPLE, config3_inputs, config5_input, sample_index
from ltb_testutil import ROOT, factor_parity, rel_err

CONFIGS = ROOT / "tests" / "golden" / "configs.npz"

pytestmark = pytest.mark.gpu


def sha(x):
    import hashlib

    return hashlib.sha256(np.ascontiguousarray(x).tobytes()).hexdigest()


@pytest.fixture(scope="module")
def cfx():
    return np.load(CONFIGS)

def cfg2_inputs():
    rng = np.random.default_rng(0)
    a = rng.standard_normal((256, 128, 3, 32), dtype=np.float32)
    b = rng.standard_normal((128, 256, 3, 32), dtype=np.float32)
    return a, b


def test_config2_l_product_full():
    a, b = cfg2_inputs()
    spec = L.make_spec("dct", (256, 256, 3, 32))
    c = L.l_product(a, b, spec)
    assert c.dtype == np.float32 and c.shape == (256, 256, 3, 32)
    ref = O.l_product(a.astype(np.float64), b.astype(np.float64), O.ospec("dct", (256, 256, 3, 32)))
    assert rel_err(c, ref) < 1e-4


def test_config2_linearity_and_associativity():
    """Size-independent checks at full size: L-linearity in A, and (A*B)*e == A*(B*e) for an
    identity-like scalar tensor e."""
    a, b = cfg2_inputs()
    spec = L.make_spec("dct", (256, 256, 3, 32))
    c1 = L.l_product(a, b, spec)
    c2 = L.l_product(2.0 * a, b, spec)
    assert rel_err(c2, 2.0 * c1) < 1e-6
    eye = L.identity_tensor(256, (3, 32), spec).astype(np.float32)
    assert rel_err(L.l_product(c1, eye, spec), c1) < 1e-5


def cfg3_data(shape=(144, 176, 3, 100), rank=10, seed=0):
    rng = np.random.default_rng(seed)
    i1, i2, c, t = shape
    a = rng.standard_normal((i1, rank, c, t), dtype=np.float32).astype(np.float64)
    b = rng.standard_normal((rank, i2, c, t), dtype=np.float32).astype(np.float64)
    x0 = O.l_product(a, b, O.ospec("dct", shape))
    x0 = (x0 - x0.min()) / (x0.max() - x0.min())
    m = (x0 + rng.normal(0.0, 0.01, x0.shape)).astype(np.float32)
    mask = rng.random(m.shape) < 0.2
    return m, mask


@pytest.mark.parametrize("precision,tol", [("fp32", 1e-4), ("fp64", 1e-10)])
def test_config3_pga_full_size_first_iterations(precision, tol):
    m, mask = cfg3_data()
    spec = L.make_spec("dct", m.shape)
    cfg = L.CompletionConfig(spec=spec, tol=1e-300, max_iters=2)
    x, trace = L.pga_complete(m, mask, cfg, precision=precision)
    ref, recs, _ = O.pga_complete(m, mask, O.ospec("dct", m.shape), tol=1e-300, max_iters=2)
    assert trace.iterations == 2
    assert rel_err(x, ref) < tol
    np.testing.assert_allclose([r.rel_change for r in trace.records], [r[3] for r in recs],
                               rtol=1e-3 if precision == "fp32" else 1e-8)


def test_config3_pga_full_run_fp32_vs_fp64():
    """The whole config-3 run (200 iterations) in fp32 -- carried right bases, Cholesky warm
    path, early-stopped Jacobi sweeps -- against the same run in fp64 (itself pinned to the
    oracle at 1e-10 on the first iterations above and on config 1 / the golden traces)."""
    m, mask = cfg3_data()
    spec = L.make_spec("dct", m.shape)
    cfg = L.CompletionConfig(spec=spec, tol=1e-300, max_iters=200)
    x32, t32 = L.pga_complete(m, mask, cfg, precision="fp32")
    x64, t64 = L.pga_complete(m, mask, cfg, precision="fp64")
    assert t32.iterations == t64.iterations == 200
    assert rel_err(x32, x64) < 1e-4
    assert [r.mu for r in t32.records] == [r.mu for r in t64.records]


def test_config1_pga_full():
    rng = np.random.default_rng(0)
    a = rng.standard_normal((64, 5, 16))
    b = rng.standard_normal((5, 64, 16))
    spec = L.make_spec("dct", (64, 64, 16))
    m = L.l_product(a, b, spec)
    mask = rng.random(m.shape) < 0.5
    cfg = L.CompletionConfig(spec=spec, mu0=0.01, mu_bar_ratio=1.0, tol=1e-300, max_iters=100)
    x, trace = L.pga_complete(m, mask, cfg)
    ref, recs, _ = O.pga_complete(m, mask, O.ospec("dct", m.shape), mu0=0.01, mu_bar_ratio=1.0, tol=1e-300,
                                  max_iters=100)
    assert trace.iterations == 100
    assert rel_err(x, ref) < 1e-10
    assert abs(O.rse(x, m) - 0.383) < 0.01  # oracle RSE after 100 iterations ~0.383


@pytest.mark.parametrize("n", [128])
def test_config5_svt_and_tsvd(n):
    rng = np.random.default_rng(0)
    a = rng.standard_normal((n, n, 4, 8, 16), dtype=np.float32)
    spec = L.make_spec("dct", a.shape)
    ospec = O.ospec("dct", a.shape)
    sv_ref = O.singular_values(a.astype(np.float64), ospec)
    tau = 0.1 * float(np.median(sv_ref))
    out = L.svt(a, tau, spec)
    ref = O.svt(a.astype(np.float64), tau, ospec)
    assert out.dtype == np.float32 and rel_err(out, ref) < 1e-4
    f = L.t_svd(a, spec)
    # singular values (device slice order -> reference p-order) and the factor-independent S
    sv = L.linalg._singular_values(a, spec)[core.slice_order_permutation(a.shape[2:])]
    assert rel_err(sv, sv_ref) < 1e-4  # north_star fp32 tolerance (QR-preconditioned sigma: normwise accurate)
    assert rel_err(np.sort(f.tube_norms)[::-1], f.tube_norms) == 0.0
    assert abs(float((f.tube_norms ** 2).sum()) - float((a.astype(np.float64) ** 2).sum())) \
        < 1e-4 * float((a.astype(np.float64) ** 2).sum())


def test_config5_n256_global_tier_properties():
    """n = 256 slices exceed shared memory (global-workspace Jacobi tier): check svt(., 0) == id
    and the Frobenius identity of the singular values on a 4-slice cut of config 5."""
    rng = np.random.default_rng(1)
    a = rng.standard_normal((256, 256, 4), dtype=np.float32)
    spec = L.make_spec("dct", a.shape)
    assert rel_err(L.svt(a, 0.0, spec), a) < 1e-4
    sv = L.linalg._singular_values(a, spec)
    assert abs(float((sv.astype(np.float64) ** 2).sum()) - float((a.astype(np.float64) ** 2).sum())) \
        < 1e-4 * float((a.astype(np.float64) ** 2).sum())


def test_config4_reduced_pga():
    """Config 4 recipe at 128 x 128 x 3 x 64: explicit Q (x) F64, complex64
    transform domain, Bernoulli(0.3), first iterations vs the oracle."""
    rng = np.random.default_rng(0)
    q, _ = np.linalg.qr(rng.standard_normal((3, 3)))
    f = L.build_fourier_matrix(64)
    a = rng.standard_normal((128, 20, 3, 64), dtype=np.float32)
    b = rng.standard_normal((20, 128, 3, 64), dtype=np.float32)
    spec = L.make_spec("explicit", (128, 128, 3, 64), matrices={3: q, 4: f})
    ospec = O.ospec("explicit", (128, 128, 3, 64), matrices={3: q, 4: f})
    m = O.l_product(a.astype(np.float64), b.astype(np.float64), ospec)
    mask = rng.random(m.shape) < 0.3
    cfg = L.CompletionConfig(spec=spec, tol=1e-300, max_iters=3)
    x, trace = L.pga_complete(m.astype(np.float32), mask, cfg)
    ref, recs, _ = O.pga_complete(m, mask, ospec, tol=1e-300, max_iters=3)
    assert trace.iterations == 3
    assert rel_err(x, ref) < 1e-4


def test_config3_recipe_long_run_fp32_carry():
    """Config-3 recipe at 64 x 72 x 3 x 20 for 90 iterations in fp32: the warm-started SVT
    (right bases carried across iterations) stays within the fp32 tolerance of the fp64 oracle
    trajectory, iterate and per-iteration relative change."""
    m, mask = cfg3_data(shape=(64, 72, 3, 20), rank=4, seed=3)
    spec = L.make_spec("dct", m.shape)
    cfg = L.CompletionConfig(spec=spec, tol=1e-300, max_iters=90)
    x, trace = L.pga_complete(m, mask, cfg, precision="fp32")
    ref, recs, _ = O.pga_complete(m, mask, O.ospec("dct", m.shape), tol=1e-300, max_iters=90)
    assert trace.iterations == 90
    assert rel_err(x, ref) < 1e-4
    rc = np.array([r.rel_change for r in trace.records])
    rr = np.array([r[3] for r in recs])
    fin = np.isfinite(rr)
    np.testing.assert_array_equal(np.isfinite(rc), fin)  # x_next == 0 (inf) on the same iterations
    assert np.max(np.abs(rc[fin] - rr[fin]) / np.maximum(rr[fin], 1e-12)) < 1e-2


@pytest.mark.parametrize("precision,tol", [("fp32", 1e-4), ("fp64", 1e-10)])
def test_config3_pga_200_iterations_vs_reference(cfx, precision, tol):
    """The full config-3 run (144x176x3x100, 200 iterations, defaults, tol 1e-300) against the
    reference's own trajectory (tests/golden/configs.npz, made by make_config_fixtures.py):
    mu / t bit-exact, the per-iteration relative change, and the final iterate through its norm
    and a seeded sample of 65,536 entries."""
    m, mask = config3_inputs(O.l_product, O.ospec)
    assert sha(m) == str(cfx["cfg3/m_sha"]) and sha(mask) == str(cfx["cfg3/mask_sha"])
    spec = L.make_spec("dct", m.shape)
    x, trace = L.pga_complete(m, mask, L.CompletionConfig(spec=spec, tol=1e-300, max_iters=200), precision=precision)
    assert trace.iterations == 200
    # mu_0 = nu ||M||_F over 7.6M entries: the device's fixed-order reduction vs numpy's pairwise sum
    np.testing.assert_allclose([r.mu for r in trace.records], cfx["cfg3/mu"], rtol=1e-13)
    assert [r.t for r in trace.records] == list(cfx["cfg3/t"])
    idx = sample_index(x.size, NSAMPLE, seed=3)
    assert rel_err(x.ravel()[idx], cfx["cfg3/x_sample"]) < tol
    assert abs(np.linalg.norm(x.ravel()) - float(cfx["cfg3/x_norm"])) < tol * float(cfx["cfg3/x_norm"])
    rc = np.array([r.rel_change for r in trace.records])
    rr = cfx["cfg3/rel"]
    fin = np.isfinite(rr)
    np.testing.assert_array_equal(np.isfinite(rc), fin)
    # fp32: ||y - x+|| / ||x+|| carries ~1e-6 absolute rounding (it falls to ~1e-5 late in the run)
    np.testing.assert_allclose(rc[fin], rr[fin], rtol=1e-2 if precision == "fp32" else 1e-6,
                               atol=2e-6 if precision == "fp32" else 0.0)


@pytest.mark.parametrize("n", [256, 512])
def test_config5_vs_reference(cfx, n):
    """Config 5 at n = 256 / 512 (512 slices, DCT over modes 3-5): svt at the reference's tau and
    the transform-domain singular values against the reference (configs.npz)."""
    key = f"cfg5_{n}"
    a = config5_input(n)
    assert sha(a) == str(cfx[f"{key}/a_sha"])
    spec = L.make_spec("dct", a.shape)
    tau = float(cfx[f"{key}/tau"])
    out = L.svt(a, tau, spec)
    assert out.dtype == np.float32
    idx = sample_index(out.size, NSAMPLE, seed=n)
    assert rel_err(out.ravel()[idx], cfx[f"{key}/svt_sample"]) < 1e-4
    nrm = float(cfx[f"{key}/svt_norm"])
    assert abs(float(np.linalg.norm(out.ravel().astype(np.float64))) - nrm) < 1e-4 * nrm
    sv = L.linalg._singular_values(a, spec)[core.slice_order_permutation(a.shape[2:])]
    assert rel_err(sv, cfx[f"{key}/sv"]) < 1e-4


def test_config5_n256_tsvd_factors():
    """t_svd at n = 256: S against the singular values and U, V up to sign against LAPACK's on
    the same transform-domain stack (oracle, f64)."""
    a = config5_input(256)
    spec = L.make_spec("dct", a.shape)
    ospec = O.ospec("dct", a.shape)
    f = L.t_svd(a, spec)
    uh, sv, vh = np.linalg.svd(O.to_stack(O.forward(a.astype(np.float64), ospec)), full_matrices=True)
    for ours, ref in ((f.u, uh), (f.v, np.conj(np.swapaxes(vh, 1, 2)))):
        err, count = factor_parity(O.to_stack(O.forward(ours.astype(np.float64), ospec)), ref, sv)
        assert count > 0.8 * sv.size and err < 1e-4, (err, count)
    diag = O.to_stack(O.forward(f.s.astype(np.float64), ospec))
    assert rel_err(np.diagonal(diag, axis1=1, axis2=2), sv) < 1e-4


def test_config4_reduced_pga_50_iterations():
    """Config 4 recipe at 128 x 128 x 3 x 64 for the full 50 iterations:
    explicit Q (x) F64, complex64 transform domain, Bernoulli(0.3), against the fp64 oracle."""
    rng = np.random.default_rng(0)
    q, _ = np.linalg.qr(rng.standard_normal((3, 3)))
    f = L.build_fourier_matrix(64)
    a = rng.standard_normal((128, 20, 3, 64), dtype=np.float32)
    b = rng.standard_normal((20, 128, 3, 64), dtype=np.float32)
    spec = L.make_spec("explicit", (128, 128, 3, 64), matrices={3: q, 4: f})
    ospec = O.ospec("explicit", (128, 128, 3, 64), matrices={3: q, 4: f})
    m = O.l_product(a.astype(np.float64), b.astype(np.float64), ospec).astype(np.float32)
    mask = rng.random(m.shape) < 0.3
    x, trace = L.pga_complete(m, mask, L.CompletionConfig(spec=spec, tol=1e-300, max_iters=50))
    # the oracle computes in float64 on the same (float32-valued) observations, as the reference would
    ref, recs, _ = O.pga_complete(m.astype(np.float64), mask, ospec, tol=1e-300, max_iters=50)
    assert trace.iterations == 50
    # mu_0 = nu ||M||_F: a device reduction vs numpy's norm, equal to the last bits
    np.testing.assert_allclose([r.mu for r in trace.records], [r[1] for r in recs], rtol=1e-14)
    assert [r.t for r in trace.records] == [r[2] for r in recs]
    assert rel_err(x, ref) < 1e-4


@pytest.mark.parametrize("variant", [0, 1, 2, 3])
@pytest.mark.parametrize("shape", [(144, 176, 2, 3), (160, 128, 3, 2)])
def test_warm_jacobi_variants_config3_recipe(variant, shape):
    """The warm (carried-basis, Cholesky-preconditioned) SVT inside fp32 PGA with each Jacobi
    variant (LTB_OPT_JACOBI_PAIRS: 0 two-column blocks (default), 1 one pair per team, 2 two-column
    blocks, 3 four-column blocks) on the config-3 recipe with n = 144 / 128 columns, 80 iterations,
    against the fp64 oracle trajectory."""
    from paper_2202_02870_b200 import _native as nat

    m, mask = config3_inputs(O.l_product, O.ospec, shape=shape, rank=4, seed=5)
    spec = L.make_spec("dct", m.shape)
    nat.check(nat.lib().ltb_ctx_set_option(nat.context(), nat.OPT_JACOBI_PAIRS, variant))
    try:
        x, trace = L.pga_complete(m, mask, L.CompletionConfig(spec=spec, tol=1e-300, max_iters=80), precision="fp32")
    finally:
        nat.check(nat.lib().ltb_ctx_set_option(nat.context(), nat.OPT_JACOBI_PAIRS, 0))
    ref, recs, _ = O.pga_complete(m.astype(np.float64), mask, O.ospec("dct", m.shape), tol=1e-300, max_iters=80)
    assert trace.iterations == 80
    assert rel_err(x, ref) < 1e-4
