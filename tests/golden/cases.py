"""Seeded case recipes for the golden fixtures (inputs are stored in golden.npz
alongside the reference's outputs, so the tests never need to regenerate them).

`lp(a, b, kind, shape)` is the l_product used to build low-rank inputs; the
generator passes the reference's own l_product.
"""

from __future__ import annotations

import numpy as np


def _q3(seed):
    q, _ = np.linalg.qr(np.random.default_rng(seed).standard_normal((3, 3)))
    return q


def _f(n):
    k = np.arange(n)
    return np.exp(-2j * np.pi * np.outer(k, k) / n)


def transform_cases():
    r = np.random.default_rng(11)
    c = {}
    for kind in ("fft", "dct", "cprod"):
        x = r.standard_normal((3, 2, 4, 3))
        c[f"t_{kind}4"] = dict(kind=kind, x=x, spec_shape=x.shape)
    x = r.standard_normal((2, 3, 4, 2))
    c["t_fft_mode3"] = dict(kind="fft", x=x, spec_shape=x.shape, modes=(3,))
    x = r.standard_normal((2, 3, 2, 3, 4))
    c["t_dct5"] = dict(kind="dct", x=x, spec_shape=x.shape)
    x = r.standard_normal((4, 3, 3, 8))
    c["t_explicit"] = dict(kind="explicit", x=x, spec_shape=x.shape, matrices={3: _q3(5), 4: _f(8)})
    c["t_tube_cprod"] = dict(kind="cprod", x=np.array([1.0, 2.0]).reshape(1, 1, 2), spec_shape=(1, 1, 2))
    x = r.standard_normal((5, 4, 6, 4)).astype(np.float32)
    c["t_dct_f32"] = dict(kind="dct", x=x, spec_shape=x.shape)
    x = r.standard_normal((3, 3, 7))
    c["t_fft_odd"] = dict(kind="fft", x=x, spec_shape=x.shape)
    return c


def product_cases():
    r = np.random.default_rng(22)
    c = {}
    tube = lambda *v: np.asarray(v, dtype=float).reshape(1, 1, len(v))  # noqa: E731
    c["p_fft_tubes"] = dict(kind="fft", a=tube(1, 2), b=tube(3, 4), spec_shape=(1, 1, 2))
    c["p_cprod_tubes"] = dict(kind="cprod", a=tube(1, 2), b=tube(3, 4), spec_shape=(1, 1, 2))
    for kind in ("fft", "dct", "cprod"):
        a = r.standard_normal((4, 3, 2, 3))
        b = r.standard_normal((3, 5, 2, 3))
        c[f"p_{kind}"] = dict(kind=kind, a=a, b=b, spec_shape=(4, 5, 2, 3))
    a = r.standard_normal((6, 2, 3, 8))
    b = r.standard_normal((2, 5, 3, 8))
    c["p_explicit"] = dict(kind="explicit", a=a, b=b, spec_shape=(6, 5, 3, 8), matrices={3: _q3(6), 4: _f(8)})
    a = r.standard_normal((32, 16, 3, 8)).astype(np.float32)
    b = r.standard_normal((16, 32, 3, 8)).astype(np.float32)
    c["p_dct_f32"] = dict(kind="dct", a=a, b=b, spec_shape=(32, 32, 3, 8))
    a = r.standard_normal((5, 4, 3, 5)) + 1j * r.standard_normal((5, 4, 3, 5))
    b = r.standard_normal((4, 3, 3, 5))
    c["p_fft_complex"] = dict(kind="fft", a=a, b=b, spec_shape=(5, 3, 3, 5))
    return c


def svd_cases():
    r = np.random.default_rng(33)
    c = {}
    c["s_fft"] = dict(kind="fft", x=r.standard_normal((4, 3, 2, 2)), tau=0.5)
    c["s_dct"] = dict(kind="dct", x=r.standard_normal((3, 5, 2, 3)), tau=0.3)
    c["s_dct_sq"] = dict(kind="dct", x=r.standard_normal((6, 6, 4)), tau=1.0)
    c["s_cprod"] = dict(kind="cprod", x=r.standard_normal((3, 3, 2, 2)), tau=0.0)
    x = r.standard_normal((5, 4, 3))
    x[:, 2:] = 0.0
    c["s_rankdef"] = dict(kind="fft", x=x, tau=0.2)
    c["s_dct_f32"] = dict(kind="dct", x=r.standard_normal((8, 6, 2, 2, 3)).astype(np.float32), tau=0.5)
    c["s_fft_wide"] = dict(kind="fft", x=r.standard_normal((3, 7, 5)), tau=0.4)
    # round 2: complex input, a wide 5th-order DCT, a tall fp32 slice stack
    c["s_fft_cplx"] = dict(kind="fft", x=r.standard_normal((5, 4, 3)) + 1j * r.standard_normal((5, 4, 3)), tau=0.6)
    c["s_dct5_wide"] = dict(kind="dct", x=r.standard_normal((4, 9, 2, 3, 2)), tau=0.5)
    c["s_dct_f32_tall"] = dict(kind="dct", x=r.standard_normal((40, 24, 3, 4)).astype(np.float32), tau=0.8)
    for v in c.values():
        v["spec_shape"] = v["x"].shape
    return c


def completion_cases(lp):
    c = {}
    r = np.random.default_rng(44)
    m = lp(r.standard_normal((10, 2, 3)), r.standard_normal((2, 10, 3)), "fft", (10, 10, 3))
    mask = np.asarray(r.random(m.shape) < 0.5)
    c["c_fft"] = dict(kind="fft", m=m, mask=mask, cfg=dict(max_iters=40))
    m = lp(r.standard_normal((12, 2, 3, 2)), r.standard_normal((2, 10, 3, 2)), "dct", (12, 10, 3, 2))
    mask = np.asarray(r.random(m.shape) < 0.6)
    c["c_dct"] = dict(kind="dct", m=m, mask=mask, cfg=dict(max_iters=60))
    m = lp(r.standard_normal((8, 2, 2)), r.standard_normal((2, 8, 2)), "fft", (8, 8, 2))
    mask = np.asarray(r.random(m.shape) < 0.5)
    c["c_gt"] = dict(kind="fft", m=m, mask=mask, gt=m, cfg=dict(max_iters=15, tol=1e-12, reimpose_observed=True))
    # the reference suite's pinned regression problem (test_acceptance.py:213-240 recipe)
    r7 = np.random.default_rng(7)
    probs = {}
    for kind in ("fft", "dct"):
        probs[kind] = lp(r7.standard_normal((20, 2, 3, 5)), r7.standard_normal((2, 20, 3, 5)), kind, (20, 20, 3, 5))
    for kind in ("fft", "dct"):
        c[f"c_pinned_{kind}"] = dict(kind=kind, m=probs[kind], mask=None, mask_seed=(0.5, 7),
                                     cfg=dict(max_iters=300))
    # BASELINE config 1: seed 0, A 64x5x16, B 5x64x16, Bernoulli(0.5)
    r0 = np.random.default_rng(0)
    a = r0.standard_normal((64, 5, 16))
    b = r0.standard_normal((5, 64, 16))
    m = lp(a, b, "dct", (64, 64, 16))
    mask = np.asarray(r0.random(m.shape) < 0.5)
    c["c_config1"] = dict(kind="dct", m=m, mask=mask,
                          cfg=dict(mu0=0.01, mu_bar_ratio=1.0, tol=1e-300, max_iters=100))
    # BASELINE config 3 at reduced size: A 36x4x3x10, B 4x44x3x10, [0,1] rescale, N(0, 0.01) noise, f32
    r3 = np.random.default_rng(0)
    a = r3.standard_normal((36, 4, 3, 10)).astype(np.float32)
    b = r3.standard_normal((4, 44, 3, 10)).astype(np.float32)
    x0 = lp(a.astype(np.float64), b.astype(np.float64), "dct", (36, 44, 3, 10))
    x0 = (x0 - x0.min()) / (x0.max() - x0.min())
    m = (x0 + r3.normal(0.0, 0.01, x0.shape)).astype(np.float32)
    mask = np.asarray(r3.random(m.shape) < 0.2)
    c["c_config3s"] = dict(kind="dct", m=m, mask=mask, cfg=dict(tol=1e-300, max_iters=20))
    return c


def mask_cases():
    return {"m_a": ((4, 5, 3), 0.5, 0), "m_b": ((6, 6, 4), 0.3, 42), "m_c": ((8, 8, 3), 0.3, 3),
            "m_d": ((3, 3, 2), 1.0, 0), "m_e": ((3, 3, 2), 0.0, 0)}


def btph_cases():
    """Small cprod products checked against the reference's btph construction (btph.py:140-149)."""
    r = np.random.default_rng(314)
    c = {}
    for name, (sa, sb) in {"b_cprod3": ((3, 4, 5), (4, 2, 5)), "b_cprod4": ((2, 3, 3, 4), (3, 2, 3, 4)),
                           "b_cprod_tube": ((1, 1, 6), (1, 1, 6))}.items():
        c[name] = dict(kind="cprod", a=r.standard_normal(sa), b=r.standard_normal(sb),
                       spec_shape=(sa[0], sb[1]) + tuple(sa[2:]))
    return c


def algebra_cases():
    """*_L algebra beyond the product (linalg.py:46-72,121-129; core.py:26-36,110-122)."""
    r = np.random.default_rng(55)
    c = {}
    for kind, shape, k in (("dct", (6, 5, 3, 2), 2), ("fft", (5, 7, 4), 3), ("fft", (4, 4, 2, 3), 1)):
        c[f"a_truncate_{kind}{len(shape)}_{k}"] = dict(kind=kind, x=r.standard_normal(shape), k=k, spec_shape=shape)
    c["a_inner_real"] = dict(kind="dct", a=r.standard_normal((4, 3, 5)), b=r.standard_normal((4, 3, 5)),
                             spec_shape=(4, 3, 5))
    c["a_inner_cplx"] = dict(kind="dct", a=r.standard_normal((3, 2, 4)) + 1j * r.standard_normal((3, 2, 4)),
                             b=r.standard_normal((3, 2, 4)) - 2j * r.standard_normal((3, 2, 4)),
                             spec_shape=(3, 2, 4))
    # orthogonal tensors: the u factor of a t-SVD under dct / fft
    c["a_orth_dct"] = dict(kind="dct", x=r.standard_normal((5, 5, 3, 2)), spec_shape=(5, 5, 3, 2))
    c["a_orth_fft"] = dict(kind="fft", x=r.standard_normal((4, 4, 6)), spec_shape=(4, 4, 6))
    return c


def mode_product_cases():
    """mode_n_product on real shapes (core.py:110-122; the reference's test_core.py:103-119 recipes)."""
    r = np.random.default_rng(66)
    c = {}
    x = r.standard_normal((4, 3, 5, 2))
    for n in (1, 2, 3, 4):
        c[f"n_mode{n}"] = dict(x=x, u=r.standard_normal((6, x.shape[n - 1])), n=n)
    x = r.standard_normal((3, 4, 6))
    c["n_cplx_u"] = dict(x=x, u=r.standard_normal((5, 6)) + 1j * r.standard_normal((5, 6)), n=3)
    c["n_f32"] = dict(x=r.standard_normal((8, 7, 5)).astype(np.float32), u=r.standard_normal((3, 7)), n=2)
    return c
