"""t_svd factors "up to sign", the rest of the *_L algebra (truncate, inner_product,
is_orthogonal, mode_n_product on real shapes) and the real-output error path, against
the reference's outputs (golden fixtures) and the oracle.

Tolerances (north_star): 1e-4 relative Frobenius for float32 work, 1e-10 for float64;
SVD factors are compared in the transform domain column by column after sign / phase
alignment, on columns with a singular-value gap > 1e-3 sigma_max."""

import numpy as np
import pytest

import ltensor_oracle as O
import paper_2202_02870_b200 as L
from paper_2202_02870_b200.errors import NumericConsistencyError
from ltb_testutil import build_spec, case_names, factor_parity, meta, rel_err

pytestmark = pytest.mark.gpu


def tol_for(*arrays):
    return 1e-4 if any(np.asarray(a).dtype in (np.float32, np.complex64) for a in arrays) else 1e-10


def hat(ospec_factory, f):
    """Transform-domain (P, n, n) stack of a spatial factor, reference p-order (oracle = checker)."""
    return O.to_stack(O.forward(f, ospec_factory(f.shape)))


@pytest.mark.parametrize("name", case_names("s_"))
def test_tsvd_factors_up_to_sign(golden, name):
    md = meta(golden, name)
    x = golden[f"{name}/x"]
    spec = build_spec(L, golden, name)
    f = L.t_svd(x, spec)
    assert f.u.dtype == golden[f"{name}/u"].dtype and f.v.dtype == golden[f"{name}/v"].dtype
    assert f.u.shape == golden[f"{name}/u"].shape and f.v.shape == golden[f"{name}/v"].shape

    def ospec(shape):
        return build_spec(O, golden, name, shape=shape)

    sv = golden[f"{name}/sv"]
    tol = tol_for(x)
    for ours, key in ((f.u, "u"), (f.v, "v")):
        err, count = factor_parity(hat(ospec, ours), hat(ospec, golden[f"{name}/{key}"]), sv)
        assert count > 0, f"{name}/{key}: no well-separated column to compare"
        assert err < tol, f"{name}/{key}: {err:.3e} over {count} columns ({md['kind']})"


def test_tsvd_factors_config5_n128():
    """Config 5 at n = 128 (512 slices of 128 x 128, DCT over modes 3-5): U and V against
    LAPACK's on the same transform-domain stack, up to sign."""
    rng = np.random.default_rng(0)
    a = rng.standard_normal((128, 128, 4, 8, 16), dtype=np.float32)
    spec = L.make_spec("dct", a.shape)
    ospec = O.ospec("dct", a.shape)
    f = L.t_svd(a, spec)
    uh, sv, vh = np.linalg.svd(O.to_stack(O.forward(a.astype(np.float64), ospec)), full_matrices=True)
    vref = np.conj(np.swapaxes(vh, 1, 2))
    for ours, ref in ((f.u, uh), (f.v, vref)):
        err, count = factor_parity(O.to_stack(O.forward(ours.astype(np.float64), ospec)), ref, sv)
        assert count > 0.9 * sv.size  # Gaussian slices: nearly every column is separated
        assert err < 1e-4, f"{err:.3e} over {count} columns"


@pytest.mark.parametrize("name", case_names("a_truncate"))
def test_truncate_parity(golden, name):
    x = golden[f"{name}/x"]
    spec = build_spec(L, golden, name)
    out = L.truncate(L.t_svd(x, spec), meta(golden, name)["k"])
    assert out.dtype == golden[f"{name}/out"].dtype
    assert rel_err(out, golden[f"{name}/out"]) < 1e-10


def test_truncate_eckart_young_fp32():
    """fp32 truncation at a realistic size: the residual equals the discarded singular
    values' energy (Eckart-Young in the transform domain, unitary DCT)."""
    rng = np.random.default_rng(5)
    x = rng.standard_normal((48, 40, 3, 8), dtype=np.float32)
    spec = L.make_spec("dct", x.shape)
    k = 7
    out = L.truncate(L.t_svd(x, spec), k)
    sv = O.singular_values(x.astype(np.float64), O.ospec("dct", x.shape))
    resid = float(np.linalg.norm((x.astype(np.float64) - out).ravel()))
    assert abs(resid - float(np.sqrt((sv[:, k:] ** 2).sum()))) < 1e-4 * resid
    ref = O.truncate(*O.t_svd(x.astype(np.float64), O.ospec("dct", x.shape))[:3], k, O.ospec("dct", x.shape))
    assert rel_err(out, ref) < 1e-4


@pytest.mark.parametrize("name", case_names("a_inner"))
def test_inner_product_parity(golden, name):
    a, b = golden[f"{name}/a"], golden[f"{name}/b"]
    val = L.inner_product(a, b)
    ref = golden[f"{name}/value"][()]
    assert isinstance(val, complex if np.iscomplexobj(ref) else float)
    assert abs(val - ref) <= 1e-12 * max(1.0, abs(ref))
    # conjugate-linear in the first argument
    assert abs(L.inner_product(b, a) - np.conj(ref)) <= 1e-12 * max(1.0, abs(ref))


def test_inner_product_fp32_large():
    rng = np.random.default_rng(9)
    a = rng.standard_normal((256, 128, 3, 32), dtype=np.float32)
    b = rng.standard_normal((256, 128, 3, 32), dtype=np.float32)
    ref = O.inner_product(a.astype(np.float64), b.astype(np.float64))
    val = L.inner_product(a, b)
    assert abs(val - ref) <= 1e-4 * float(np.linalg.norm(a) * np.linalg.norm(b))


@pytest.mark.parametrize("name", case_names("a_orth"))
def test_is_orthogonal_parity(golden, name):
    spec = build_spec(L, golden, name)
    q = golden[f"{name}/q"]
    assert L.is_orthogonal(q, spec) is bool(golden[f"{name}/orth"]) is True
    assert L.is_orthogonal(golden[f"{name}/q"] * 1.001, spec) is False
    # factors built on the device are *_L-orthogonal too (the true case on our own t_svd output)
    f = L.t_svd(q, spec)
    assert L.is_orthogonal(f.u, spec) and L.is_orthogonal(f.v, spec)


@pytest.mark.parametrize("name", case_names("n_"))
def test_mode_n_product_parity(golden, name):
    x, u, n = golden[f"{name}/x"], golden[f"{name}/u"], int(golden[f"{name}/n"])
    out = L.mode_n_product(x, u, n)
    ref = golden[f"{name}/out"]
    assert out.dtype == ref.dtype and out.shape == ref.shape
    assert rel_err(out, ref) < 1e-12


def test_mode_n_product_large_real():
    """A config-shaped mode product (mode 3 of a 64 x 48 x 100 x 3 tensor by a 100 x 100 matrix)."""
    rng = np.random.default_rng(4)
    x = rng.standard_normal((64, 48, 100, 3))
    u = rng.standard_normal((100, 100))
    for n in (1, 2, 3, 4):
        uu = u[: x.shape[n - 1], : x.shape[n - 1]] if n != 3 else u
        assert rel_err(L.mode_n_product(x, uu, n), O.mode_product(x, uu, n)) < 1e-12


@pytest.mark.parametrize(
    "shape,n,dtype",
    [
        ((40, 30, 20), 3, np.float64),       # inner == 1: one GEMM X M^T
        ((40, 30, 20), 3, np.float32),       # (tcgen05 3xTF32 engine)
        ((7, 33, 48), 2, np.float32),        # batched GEMMs with the matrix shared (inner >= 16)
        ((7, 33, 48), 2, np.complex64),
        ((5, 6, 40, 17), 3, np.complex128),
        ((9, 20, 5), 2, np.float64),         # inner 2..15: the per-output kernel
        ((70000, 2, 16), 2, np.float64),     # more than 65535 GEMM batches
        ((0, 4, 3), 2, np.float64),
    ],
)
def test_mode_n_product_gemm_paths(shape, n, dtype):
    rng = np.random.default_rng(11)
    x = rng.standard_normal(shape)
    u = rng.standard_normal((shape[n - 1] + 3, shape[n - 1]))
    if np.iscomplexobj(np.zeros(1, dtype)):
        x = x + 1j * rng.standard_normal(shape)
        u = u - 0.5j * rng.standard_normal(u.shape)
    x, u = x.astype(dtype), u.astype(dtype)
    out = L.mode_n_product(x, u, n)
    ref = O.mode_product(x.astype(np.complex128 if np.iscomplexobj(x) else np.float64), u, n)
    assert out.shape == ref.shape and out.dtype == np.result_type(x.dtype, u.dtype)
    tol = 1e-5 if dtype in (np.float32, np.complex64) else 1e-12
    assert rel_err(out, ref) < tol if ref.size else out.size == 0


@pytest.mark.parametrize("kind,dtype", [("fft", np.complex128), ("fft", np.complex64), ("dct", np.complex128)])
def test_numeric_consistency_error_on_corrupted_spectrum(kind, dtype):
    """apply_l_inv(assume_real=True) raises when the transform-domain tensor is not the image
    of a real tensor (transforms.py:217-225; the reference's test_transforms.py:102-106)."""
    rng = np.random.default_rng(2)
    x = rng.standard_normal((6, 5, 8, 3))
    spec = L.make_spec(kind, x.shape)
    xh = O.forward(x, O.ospec(kind, x.shape)).astype(dtype)
    # a clean spectrum passes and returns the real tensor
    back = L.apply_l_inv(xh, spec, assume_real=True)
    assert np.isrealobj(back) and rel_err(back, x) < tol_for(xh)
    bad = xh.copy()
    bad[2, 3, 1, 0] += 0.5j * (1 + abs(bad[2, 3, 1, 0]))  # breaks the conjugate symmetry / realness
    with pytest.raises(NumericConsistencyError):
        L.apply_l_inv(bad, spec, assume_real=True)
    # without the contract the complex result comes back
    assert np.iscomplexobj(L.apply_l_inv(bad, spec))


def test_numeric_consistency_error_tube():
    """The reference's exact case (test_transforms.py:102-106)."""
    spec = L.make_spec("fft", (1, 1, 3))
    with pytest.raises(NumericConsistencyError):
        L.apply_l_inv(np.array([1.0 + 2j, 0.5, 0.25]).reshape(1, 1, 3), spec, assume_real=True)
