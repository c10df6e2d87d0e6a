import json
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
for p in (ROOT, ROOT / "oracle", ROOT / "tests"):
    if str(p) not in sys.path:
        sys.path.insert(0, str(p))

GOLDEN = ROOT / "tests" / "golden" / "golden.npz"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built libltb.so")


@pytest.fixture(scope="session")
def golden():
    return np.load(GOLDEN)


@pytest.fixture
def rng():
    return np.random.default_rng(1234)


def random_shape(rng, min_order=3, max_order=5, max_dim=4):
    order = int(rng.integers(min_order, max_order + 1))
    return tuple(int(d) for d in rng.integers(1, max_dim + 1, size=order))


def case_names(prefix):
    g = np.load(GOLDEN)
    return sorted({k.split("/")[0] for k in g.files if k.startswith(prefix)})


def meta(g, name):
    return json.loads(str(g[f"{name}/meta"]))


def build_spec(module, g, name, shape=None):
    """Spec for case `name` from `module` (the package's make_spec or the oracle's ospec)."""
    md = meta(g, name)
    shape = tuple(shape or md["spec_shape"])
    mats = None
    if md["kind"] == "explicit":
        mats = {int(k.split("/mat")[1]): g[k] for k in g.files if k.startswith(f"{name}/mat")}
    if hasattr(module, "make_spec"):
        return module.make_spec(md["kind"], shape, modes=md["modes"], matrices=mats)
    return module.ospec(md["kind"], shape, modes=md["modes"], matrices=mats)


def rel_err(a, b):
    a = np.asarray(a)
    b = np.asarray(b)
    den = max(float(np.linalg.norm(b.ravel())), 1e-300)
    return float(np.linalg.norm((a - b).ravel())) / den
