"""Seeded input recipes of the BASELINE configs, shared by the
fixture generator (tests/golden/make_config_fixtures.py, run against the reference) and
the GPU tests, so both see the same bytes (pinned by SHA-256 in the fixture)."""

from __future__ import annotations

import numpy as np

NSAMPLE = 65536


def sample_index(size: int, count: int, seed: int) -> np.ndarray:
    """Seeded sorted sample of flat indices (with replacement)."""
    return np.sort(np.random.default_rng(seed).integers(0, size, size=min(count, size)))


def config5_input(n: int) -> np.ndarray:
    return np.random.default_rng(0).standard_normal((n, n, 4, 8, 16), dtype=np.float32)


def config3_inputs(l_product, make_spec, shape=(144, 176, 3, 100), rank=10, seed=0):
    """A 144x10x3x100, B 10x176x3x100 N(0,1) f32 -> X0 = A *_L B (f64), min-max to [0,1],
    + N(0, 0.01) noise (std 0.01), cast to f32; Bernoulli(0.2) mask (C-order draws)."""
    rng = np.random.default_rng(seed)
    i1, i2, c, t = shape
    a = rng.standard_normal((i1, rank, c, t), dtype=np.float32).astype(np.float64)
    b = rng.standard_normal((rank, i2, c, t), dtype=np.float32).astype(np.float64)
    x0 = l_product(a, b, make_spec("dct", shape))
    x0 = (x0 - x0.min()) / (x0.max() - x0.min())
    m = (x0 + rng.normal(0.0, 0.01, x0.shape)).astype(np.float32)
    mask = rng.random(m.shape) < 0.2
    return m, mask
