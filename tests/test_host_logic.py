"""Host-side logic of the drop-in that needs no GPU: spec construction, matrix
builders, index helpers, the exact scalar recurrences of PGA, typed errors
raised before any device work, and the C-ABI library surface."""

import math
import re
from pathlib import Path

import numpy as np
import pytest

import paper_2202_02870_b200 as L
from paper_2202_02870_b200 import _native, completion, core, transforms
from paper_2202_02870_b200.errors import (
    ModeError,
    ParameterError,
    ShapeError,
    TransformError,
    UnsupportedSpecError,
)
from ltb_testutil import ROOT, case_names, meta, random_shape


# ----------------------------------------------------------------- C ABI surface
def header_symbols():
    text = (ROOT / "include" / "ltb.h").read_text()
    return sorted(set(re.findall(r"\b(ltb_[a-z0-9_]+)\s*\(", text)))


def test_header_and_binding_agree():
    assert header_symbols() == sorted(_native.EXPORTED_SYMBOLS)


def test_library_loads_and_exports_every_symbol():
    lib = _native.load_library()
    for name in header_symbols():
        assert hasattr(lib, name), name
    assert lib.ltb_version() == 1


def test_library_is_sm100a():
    import subprocess

    out = subprocess.run(["cuobjdump", "--list-elf", str(_native.LIB_PATH)], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


# ----------------------------------------------------------------- builders & spec
def test_dct_matrix_values():
    r = 1 / np.sqrt(2)
    np.testing.assert_allclose(L.build_dct_matrix(1), [[1.0]])
    np.testing.assert_allclose(L.build_dct_matrix(2), [[r, r], [r, -r]], atol=1e-12)
    for n in (2, 3, 4, 7):
        c = L.build_dct_matrix(n)
        assert np.linalg.norm(c @ c.T - np.eye(n)) < 1e-12
    with pytest.raises(ParameterError):
        L.build_dct_matrix(0)


def test_fourier_and_cprod_matrices():
    np.testing.assert_allclose(L.build_fourier_matrix(2), [[1, 1], [1, -1]], atol=1e-12)
    np.testing.assert_allclose(L.build_fourier_matrix(4)[:, 1], [1, -1j, -1, 1j], atol=1e-12)
    np.testing.assert_allclose(L.build_cproduct_matrix(2), [[1, 2], [1, 0]], atol=1e-12)
    for n in (2, 3, 5):
        f = L.build_fourier_matrix(n)
        assert np.linalg.norm(f @ f.conj().T - n * np.eye(n)) < 1e-10
        assert np.linalg.norm(L.build_cproduct_matrix(n) @ transforms.build_cproduct_inverse(n) - np.eye(n)) < 1e-12


def test_builders_match_oracle():
    import ltensor_oracle as O

    for n in (1, 2, 3, 16, 100):
        np.testing.assert_allclose(L.build_dct_matrix(n), O.dct_matrix(n), atol=1e-14)
        np.testing.assert_allclose(L.build_fourier_matrix(n), O.dft_matrix(n), atol=1e-12)
        np.testing.assert_allclose(L.build_cproduct_matrix(n), O.cprod_matrix(n), rtol=1e-12, atol=1e-12)


def test_spec_construction():
    assert L.make_spec("fft", (2, 2, 3, 4)).unitary_scaled
    assert L.make_spec("fft", (2, 2, 3, 4)).alpha == 12.0
    assert L.make_spec("dct", (2, 2, 3, 4)).alpha == 1.0
    assert not L.make_spec("cprod", (2, 2, 3)).unitary_scaled
    rng = np.random.default_rng(0)
    q, _ = np.linalg.qr(rng.standard_normal((3, 3)))
    s = L.make_spec("explicit", (2, 2, 3), matrices={3: 2.0 * q})
    assert s.unitary_scaled and np.isclose(s.alpha, 4.0)
    assert not L.make_spec("explicit", (2, 2, 3), matrices={3: np.eye(3) + np.diag([0.5, 0.5], 1)}).unitary_scaled
    with pytest.raises(TransformError):
        L.make_spec("explicit", (2, 2, 2), matrices={3: np.ones((2, 2))})
    with pytest.raises(TransformError):
        L.make_spec("wavelet", (2, 2, 2))
    with pytest.raises(TransformError):
        L.make_spec("fft", (2, 2))
    with pytest.raises(TransformError):
        L.make_spec("fft", (2, 2, 3), modes=(4,))
    # config 4's mixed transform is an explicit spec
    s4 = L.make_spec("explicit", (8, 8, 3, 64), matrices={3: q, 4: L.build_fourier_matrix(64)})
    assert s4.unitary_scaled and np.isclose(s4.alpha, 64.0)
    assert s4.is_complex


def test_spec_equality_and_modes():
    assert L.make_spec("dct", (2, 2, 3)) == L.make_spec("dct", (5, 7, 3))
    assert L.make_spec("fft", (2, 3, 4, 2), modes=(3,)).modes == (3,)
    assert L.make_spec("fft", (2, 3, 4, 2), modes=(3,)).alpha == 4.0


def test_dtype_rules():
    dct = L.make_spec("dct", (2, 2, 3))
    fft = L.make_spec("fft", (2, 2, 3))
    cpr = L.make_spec("cprod", (2, 2, 3))
    assert transforms.forward_dtype(np.float32, dct) == np.float32
    assert transforms.forward_dtype(np.float32, fft) == np.complex64
    assert transforms.forward_dtype(np.float64, fft) == np.complex128
    assert transforms.forward_dtype(np.float32, cpr) == np.float64
    assert transforms.forward_dtype(np.int64, dct) == np.float64
    assert transforms.inverse_dtype(np.complex64, fft, assume_real=True) == np.float32
    assert transforms.imag_tol(np.float64) == 1e-9


# ----------------------------------------------------------------- index helpers
def seq_tensor(shape):
    return np.arange(1.0, np.prod(shape) + 1.0).reshape(shape, order="F")


def test_rep_index_bijection():
    dims = (2, 2, 3, 2, 2)
    seen = set()
    for p in range(1, core.num_rep(dims) + 1):
        multi = core.rep_index_to_multi(p, dims)
        assert core.multi_to_rep_index(multi, dims) == p
        seen.add(multi)
    assert len(seen) == core.num_rep(dims)
    assert core.rep_index_to_multi(3, (2, 2, 2, 2)) == (1, 2)
    np.testing.assert_array_equal(L.rep_matrix(seq_tensor((2, 2, 2, 2)), 3), seq_tensor((2, 2, 2, 2))[:, :, 0, 1])
    with pytest.raises(ModeError):
        L.rep_matrix(np.ones((2, 2, 2)), 3)


def test_slice_order_permutation():
    trailing = (3, 4, 2)
    x = np.random.default_rng(1).standard_normal((2, 2) + trailing)
    ref_stack = core.as_rep_stack(x)  # reference p-order
    dev_stack = np.moveaxis(x.reshape(2, 2, -1), 2, 0)  # C-order q (device order)
    perm = core.slice_order_permutation(trailing)
    np.testing.assert_array_equal(ref_stack, dev_stack[perm])


def test_unfold_fold():
    x = seq_tensor((2, 2, 2))
    np.testing.assert_array_equal(L.mode_n_unfold(x, 1), [[1, 3, 5, 7], [2, 4, 6, 8]])
    rng = np.random.default_rng(3)
    for _ in range(20):
        shape = random_shape(rng)
        n = int(rng.integers(1, len(shape) + 1))
        y = rng.standard_normal(shape)
        np.testing.assert_array_equal(L.mode_n_fold(L.mode_n_unfold(y, n), n, shape), y)
    with pytest.raises(ModeError):
        L.mode_n_unfold(np.ones((2, 2, 2)), 4)
    stack = core.as_rep_stack(y)
    np.testing.assert_array_equal(core.from_rep_stack(stack, y.shape[2:]), y)


# ----------------------------------------------------------------- errors raised before device work
def test_shape_errors_before_device():
    spec = L.make_spec("fft", (2, 2, 3))
    with pytest.raises(ShapeError):
        L.l_product(np.ones((2, 3, 3)), np.ones((2, 2, 3)), spec)
    with pytest.raises(ShapeError):
        L.l_product(np.ones((2, 2, 3)), np.ones((2, 2, 4)), spec)
    with pytest.raises(TransformError):
        L.apply_l(np.ones((2, 2, 4)), spec)
    with pytest.raises(ShapeError):
        L.facewise_product(np.ones((2, 3, 2)), np.ones((2, 2, 2)))
    with pytest.raises(ShapeError):
        L.mode_n_product(np.ones((2, 2, 3)), np.ones((2, 2)), 3)
    with pytest.raises(ShapeError):
        L.project_omega(np.ones((2, 2, 2)), np.ones((2, 2, 3), dtype=bool))
    with pytest.raises(ShapeError):
        L.is_orthogonal(np.ones((2, 3, 2)), L.make_spec("fft", (2, 3, 2)))
    with pytest.raises(ShapeError):
        L.inner_product(np.ones((2, 2, 2)), np.ones((2, 2, 3)))


def test_parameter_errors_before_device():
    with pytest.raises(ParameterError):
        L.svt(np.ones((2, 2, 2)), -0.1, L.make_spec("dct", (2, 2, 2)))
    with pytest.raises(UnsupportedSpecError):
        L.svt(np.ones((2, 2, 3)), 0.5, L.make_spec("cprod", (2, 2, 3)))
    for fn in (L.spectral_norm, L.nuclear_norm):
        with pytest.raises(UnsupportedSpecError):
            fn(np.ones((2, 2, 3)), L.make_spec("cprod", (2, 2, 3)))
    with pytest.raises(ParameterError):
        L.ranks(np.ones((2, 2, 2)), L.make_spec("dct", (2, 2, 2)), threshold=-1.0)
    spec = L.make_spec("fft", (2, 2, 2))
    for kwargs in ({"nu": 1.0}, {"nu": 0.0}, {"tol": 0.0}, {"mu_bar_ratio": 2.0}, {"max_iters": 0}):
        with pytest.raises(ParameterError):
            L.CompletionConfig(spec=spec, **kwargs).validate()
    L.CompletionConfig(spec=L.make_spec("dct", (2, 2, 2))).validate()
    with pytest.raises(UnsupportedSpecError):
        L.pga_complete(np.ones((2, 2, 2)), np.ones((2, 2, 2), dtype=bool),
                       L.CompletionConfig(spec=L.make_spec("cprod", (2, 2, 2))))
    with pytest.raises(ShapeError):
        L.pga_complete(np.ones((2, 2, 2)), np.ones((2, 2, 3), dtype=bool), L.CompletionConfig(spec=spec))
    with pytest.raises(ParameterError):
        L.sample_mask((2, 2, 2), 1.5, 0)
    with pytest.raises(ParameterError):
        L.rse(np.ones((2, 2, 2)), np.ones((2, 2, 2)), denominator="mean")


# ----------------------------------------------------------------- PGA host recurrences
def test_pga_schedule_is_exact():
    spec = L.make_spec("fft", (8, 8, 2))
    cfg = L.CompletionConfig(spec=spec, nu=0.8, mu0=5.0, mu_bar_ratio=1e-2, tol=1e-12, max_iters=40)
    mus, ts, betas = completion.pga_schedule(cfg, 5.0)
    t = 1.0
    t_prev = 1.0
    for k in range(1, 41):
        assert mus[k - 1] == max(0.8**k * 5.0, 1e-2 * 5.0)
        assert ts[k - 1] == t
        assert betas[k - 1] == (t_prev - 1.0) / t
        t_prev, t = t, (1.0 + math.sqrt(4.0 * t * t + 1.0)) / 2.0


@pytest.mark.parametrize("name", case_names("c_"))
def test_pga_schedule_matches_reference_trace(golden, name):
    md = meta(golden, name)
    cfg_kw = {k: v for k, v in md["cfg"].items() if k in ("nu", "mu0", "mu_bar_ratio", "tol", "max_iters")}
    spec = L.make_spec(md["kind"], golden[f"{name}/m"].shape)
    cfg = L.CompletionConfig(spec=spec, **cfg_kw)
    mu_ref = golden[f"{name}/mu"]
    t_ref = golden[f"{name}/t"]
    mu0 = cfg.mu0 if cfg.mu0 is not None else mu_ref[0] / cfg.nu
    mus, ts, _ = completion.pga_schedule(cfg, mu0)
    assert ts[: len(t_ref)] == list(t_ref)
    if cfg.mu0 is not None:
        assert mus[: len(mu_ref)] == list(mu_ref)
    else:
        np.testing.assert_allclose(mus[: len(mu_ref)], mu_ref, rtol=1e-15)


def test_rel_change_rules():
    assert completion.rel_change(4.0, 16.0, False) == 0.5
    assert completion.rel_change(1.0, 0.0, True) == 0.0
    assert completion.rel_change(1.0, 0.0, False) == math.inf


@pytest.mark.parametrize("name", case_names("m_"))
def test_sample_mask_matches_reference(golden, name):
    md = meta(golden, name)
    np.testing.assert_array_equal(L.sample_mask(md["dims"], md["sr"], md["seed"]), golden[f"{name}/mask"])


def test_sample_mask_properties():
    assert L.sample_mask((4, 5, 3), 0.5, 0).sum() == 30
    assert not np.array_equal(L.sample_mask((6, 6, 4), 0.5, 1), L.sample_mask((6, 6, 4), 0.5, 2))
    assert not L.sample_mask((3, 3, 2), 0.0, 0).any()
    assert L.sample_mask((3, 3, 2), 1.0, 0).all()


def test_trace_csv(tmp_path):
    trace = L.CompletionTrace(records=[completion.IterationRecord(1, 0.5, 1.0, 0.25, 0.1, 12.5),
                                       completion.IterationRecord(2, 0.25, 1.618, 0.125)])
    p = tmp_path / "t.csv"
    trace.write_csv(p)
    lines = p.read_text().strip().splitlines()
    assert lines[0] == "iter,mu,t,rel_change,rse,psnr"
    assert float(lines[1].split(",")[1]) == 0.5
    assert lines[2].endswith(",,")
    assert trace.iterations == 2


def test_public_names_match_reference_surface():
    expected = {
        "facewise_product", "fro_norm", "inner_product", "mode_n_fold", "mode_n_product", "mode_n_unfold",
        "num_rep", "rep_matrix", "TransformSpec", "apply_l", "apply_l_inv", "build_cproduct_matrix",
        "build_dct_matrix", "build_fourier_matrix", "make_spec", "LFactors", "RankReport", "identity_tensor",
        "is_orthogonal", "l_product", "l_transpose", "nuclear_norm", "ranks", "spectral_norm", "svt", "t_svd",
        "truncate", "CompletionConfig", "CompletionTrace", "pga_complete", "project_omega", "psnr", "rse",
        "sample_mask", "export_ppm_dir", "import_ppm_dir", "read_container", "write_container",
    }
    assert expected <= set(L.__all__)


REF_SRC = Path("/root/reference/pkg/src/ltensor")
SUBMODULES = ("core", "transforms", "linalg", "completion", "errors", "io", "cli")


def _public_defs(path: Path, imports: bool = False) -> set:
    """Top-level public functions / classes (and relative imports) of a module, by AST (no import)."""
    import ast

    names = set()
    for node in ast.parse(path.read_text()).body:
        if isinstance(node, (ast.FunctionDef, ast.ClassDef)):
            names.add(node.name)
        elif imports and isinstance(node, ast.ImportFrom) and node.level == 1:
            names.update(a.asname or a.name for a in node.names)
    return {n for n in names if not n.startswith("_")}


@pytest.mark.skipif(not REF_SRC.is_dir(), reason="reference tree not present (GPU box)")
def test_public_names_cover_reference_modules():
    """Every public name of the reference package and of each of its modules the
    drop-in replaces exists under the same module here (pkg/src/ltensor/__init__.py:3-45)."""
    import importlib

    assert _public_defs(REF_SRC / "__init__.py", imports=True) <= set(dir(L))
    for mod in SUBMODULES:
        ours = importlib.import_module(f"paper_2202_02870_b200.{mod}")
        missing = _public_defs(REF_SRC / f"{mod}.py") - set(dir(ours))
        assert not missing, f"{mod}: {sorted(missing)}"


def test_no_oracle_in_product_package():
    pkg = ROOT / "paper_2202_02870_b200"
    for f in pkg.rglob("*.py"):
        text = f.read_text()
        assert "ltensor_oracle" not in text and "oracle" not in re.findall(r"^\s*(?:from|import)\s+(\S+)", text, re.M)
