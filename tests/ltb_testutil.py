"""Shared test helpers (imported by the test modules; tests/conftest.py holds the fixtures)."""

import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
for p in (ROOT, ROOT / "oracle", ROOT / "tests"):
    if str(p) not in sys.path:
        sys.path.insert(0, str(p))

GOLDEN = ROOT / "tests" / "golden" / "golden.npz"


def random_shape(rng, min_order=3, max_order=5, max_dim=4):
    """Same draw as the reference's pkg/tests/conftest.py:10-12."""
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


def factor_parity(ours_hat, ref_hat, sv_ref, gap_rel=1e-3):
    """Compare SVD factors "up to sign".

    ours_hat / ref_hat: (P, n, n) transform-domain factors in the same slice order
    (columns are the singular vectors); sv_ref: (P, k) reference singular values,
    descending.  Column j of slice p is compared only if j < rank (sigma_j >
    gap_rel * sigma_max) and sigma_j is separated from its neighbours (and from the
    null space) by more than gap_rel * sigma_max; the null-space columns of a
    full_matrices factor are ignored.  Each compared column is aligned by the unit
    phase of <ours, ref> (a sign for real slices).  Returns (relative Frobenius error
    over the compared columns, number of columns compared)."""
    ours_hat = np.asarray(ours_hat)
    ref_hat = np.asarray(ref_hat)
    sv_ref = np.asarray(sv_ref, dtype=np.float64)
    smax = float(sv_ref.max(initial=0.0))
    num = den = 0.0
    count = 0
    for p in range(ref_hat.shape[0]):
        s = sv_ref[p]
        for j in range(len(s)):
            if s[j] <= gap_rel * smax:
                continue
            left = s[j - 1] - s[j] if j > 0 else np.inf
            right = s[j] - (s[j + 1] if j + 1 < len(s) else 0.0)
            if min(left, right) <= gap_rel * smax:
                continue
            a = ours_hat[p, :, j].astype(np.complex128)
            b = ref_hat[p, :, j].astype(np.complex128)
            c = np.vdot(a, b)
            phase = c / abs(c) if abs(c) > 0 else 1.0
            num += float(np.sum(np.abs(a * phase - b) ** 2))
            den += float(np.sum(np.abs(b) ** 2))
            count += 1
    return (np.sqrt(num / den) if den > 0 else 0.0), count
