"""Pin the CPU oracle (oracle/ltensor_oracle.py) against the reference's own outputs
(tests/golden/golden.npz, produced by tests/golden/make_golden.py) and the reference
test-suite's known answers.  CPU only."""

import numpy as np
import pytest

import ltensor_oracle as O
from ltb_testutil import build_spec, case_names, meta, rel_err


@pytest.mark.parametrize("name", case_names("t_"))
def test_transforms(golden, name):
    spec = build_spec(O, golden, name)
    x = golden[f"{name}/x"]
    fwd = O.forward(x, spec)
    assert fwd.dtype == golden[f"{name}/fwd"].dtype
    assert rel_err(fwd, golden[f"{name}/fwd"]) < 1e-14
    back = O.inverse(golden[f"{name}/fwd"], spec, assume_real=True, imag_tol=1e-4 if x.dtype == np.float32 else 1e-9)
    assert rel_err(back, golden[f"{name}/inv"]) < 1e-14
    if f"{name}/fwd_explicit" in golden.files:
        assert rel_err(O.forward(x, spec, explicit=True), golden[f"{name}/fwd_explicit"]) < 1e-12


@pytest.mark.parametrize("name", case_names("p_"))
def test_products(golden, name):
    spec = build_spec(O, golden, name)
    c = O.l_product(golden[f"{name}/a"], golden[f"{name}/b"], spec)
    assert c.dtype == golden[f"{name}/c"].dtype
    assert rel_err(c, golden[f"{name}/c"]) < 1e-12


def test_known_answer_tubes(golden):
    np.testing.assert_allclose(golden["p_fft_tubes/c"].ravel(), [11.0, 10.0], atol=1e-12)
    np.testing.assert_allclose(golden["p_cprod_tubes/c"].ravel(), [3.0, 26.0], atol=1e-12)
    np.testing.assert_allclose(golden["t_tube_cprod/fwd"].ravel(), [5.0, 1.0], atol=1e-12)


@pytest.mark.parametrize("name", case_names("s_"))
def test_svd_family(golden, name):
    spec = build_spec(O, golden, name)
    x = golden[f"{name}/x"]
    u, s, v, norms = O.t_svd(x, spec)
    assert rel_err(s, golden[f"{name}/s"]) < (1e-6 if x.dtype == np.float32 else 1e-12)
    np.testing.assert_allclose(norms, golden[f"{name}/tube_norms"], rtol=1e-6 if x.dtype == np.float32 else 1e-12)
    np.testing.assert_allclose(O.singular_values(x, spec), golden[f"{name}/sv"],
                               rtol=1e-5 if x.dtype == np.float32 else 1e-12, atol=1e-12)
    if f"{name}/svt" in golden.files:
        tau = meta(golden, name)["tau"]
        assert rel_err(O.svt(x, tau, spec), golden[f"{name}/svt"]) < (1e-5 if x.dtype == np.float32 else 1e-12)


@pytest.mark.parametrize("name", case_names("c_"))
def test_completion(golden, name):
    md = meta(golden, name)
    m = golden[f"{name}/m"]
    spec = build_spec(O, golden, name, shape=m.shape)
    gt = golden[f"{name}/gt"] if f"{name}/gt" in golden.files else None
    x, recs, status = O.pga_complete(m, golden[f"{name}/mask"], spec, ground_truth=gt, **md["cfg"])
    assert status == md["status"]
    assert len(recs) == len(golden[f"{name}/mu"])
    assert [r[1] for r in recs] == list(golden[f"{name}/mu"])  # exact
    assert [r[2] for r in recs] == list(golden[f"{name}/t"])  # exact
    np.testing.assert_allclose([r[3] for r in recs], golden[f"{name}/rel"], rtol=1e-9)
    assert rel_err(x, golden[f"{name}/x_out"]) < 1e-11


def test_pinned_completion_rse(golden):
    # the reference suite's pinned values (test_acceptance.py:225), rtol 1e-6
    pinned = {"fft": 0.0003459755997733272, "dct": 0.00020922751673777}
    for kind, val in pinned.items():
        name = f"c_pinned_{kind}"
        assert np.isclose(O.rse(golden[f"{name}/x_out"], golden[f"{name}/m"]), val, rtol=1e-6)
        assert np.isclose(meta(golden, name)["final_rse"], val, rtol=1e-6)


@pytest.mark.parametrize("name", case_names("m_"))
def test_sample_mask(golden, name):
    md = meta(golden, name)
    np.testing.assert_array_equal(O.sample_mask(md["dims"], md["sr"], md["seed"]), golden[f"{name}/mask"])


@pytest.mark.parametrize("name", case_names("b_"))
def test_oracle_cprod_equals_btph(golden, name):
    """the oracle's cprod l_product equals the reference's btph construction."""
    spec = build_spec(O, golden, name)
    c = O.l_product(golden[f"{name}/a"], golden[f"{name}/b"], spec)
    assert rel_err(c, golden[f"{name}/c"]) < 1e-12


@pytest.mark.parametrize("name", case_names("s_"))
def test_svd_factors(golden, name):
    """The oracle's t_svd factors are the reference's (same LAPACK call on the same stack)."""
    spec = build_spec(O, golden, name)
    x = golden[f"{name}/x"]
    u, s, v, _ = O.t_svd(x, spec)
    tol = 1e-6 if x.dtype == np.float32 else 1e-12
    assert rel_err(u, golden[f"{name}/u"]) < tol and rel_err(v, golden[f"{name}/v"]) < tol


@pytest.mark.parametrize("name", case_names("a_"))
def test_algebra(golden, name):
    spec = build_spec(O, golden, name)
    if name.startswith("a_truncate"):
        u, s, v, _ = O.t_svd(golden[f"{name}/x"], spec)
        out = O.truncate(u, s, v, meta(golden, name)["k"], spec)
        assert rel_err(out, golden[f"{name}/out"]) < 1e-12
    elif name.startswith("a_inner"):
        assert O.inner_product(golden[f"{name}/a"], golden[f"{name}/b"]) == golden[f"{name}/value"][()]
    else:
        assert O.is_orthogonal(golden[f"{name}/q"], spec) == bool(golden[f"{name}/orth"])
        assert bool(golden[f"{name}/orth"]) and not bool(golden[f"{name}/nonorth"])


@pytest.mark.parametrize("name", case_names("n_"))
def test_mode_products(golden, name):
    out = O.mode_product(golden[f"{name}/x"], golden[f"{name}/u"], int(golden[f"{name}/n"]))
    assert out.dtype == golden[f"{name}/out"].dtype
    np.testing.assert_array_equal(out, golden[f"{name}/out"])
