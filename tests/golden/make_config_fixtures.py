"""Compact reference fixtures for the BASELINE configs too large to re-run on the host
inside the GPU test session (tests/test_gpu_configs.py reads tests/golden/configs.npz).

Run in the build container only (the reference is not on the GPU box):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_config_fixtures.py

Inputs are regenerated in the tests from the same seeded recipes;
a SHA-256 of each input pins that the test feeds the bytes the reference saw.  Outputs
too large to commit are stored as size-independent summaries: the Frobenius norm, the
singular values (float32), and the values at a seeded sample of flat indices.
"""

from __future__ import annotations

import hashlib
import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent))

import ltensor as ref  # noqa: E402  (the reference, via PYTHONPATH)
from ltensor.completion import CompletionConfig  # noqa: E402

from config_recipes import NSAMPLE, config3_inputs, config5_input, sample_index  # noqa: E402


def sha(x: np.ndarray) -> np.ndarray:
    return np.array(hashlib.sha256(np.ascontiguousarray(x).tobytes()).hexdigest())


def main(which=("cfg5_256", "cfg5_512", "cfg3")):
    path = HERE / "configs.npz"
    out = dict(np.load(path)) if path.exists() else {}
    for n in (256, 512):
        key = f"cfg5_{n}"
        if key not in which:
            continue
        t0 = time.time()
        a = config5_input(n)
        spec = ref.make_spec("dct", a.shape)
        a64 = a.astype(np.float64)
        sv = np.linalg.svd(ref.core.as_rep_stack(ref.apply_l(a64, spec)), compute_uv=False)
        tau = 0.1 * float(np.median(sv))
        s = ref.svt(a64, tau, spec)
        idx = sample_index(s.size, NSAMPLE, seed=n)
        out.update({f"{key}/a_sha": sha(a), f"{key}/tau": np.array(tau), f"{key}/sv": sv.astype(np.float32),
                    f"{key}/svt_norm": np.array(np.linalg.norm(s.ravel())),
                    f"{key}/svt_sample": s.ravel()[idx]})
        print(f"{key}: tau {tau:.6f} in {time.time() - t0:.1f} s", flush=True)
    if "cfg3" in which:
        t0 = time.time()
        m, mask = config3_inputs(ref.l_product, ref.make_spec)
        spec = ref.make_spec("dct", m.shape)
        cfg = CompletionConfig(spec=spec, tol=1e-300, max_iters=200)
        x, trace = ref.pga_complete(m, mask, cfg)
        idx = sample_index(x.size, NSAMPLE, seed=3)
        out.update({"cfg3/m_sha": sha(m), "cfg3/mask_sha": sha(mask),
                    "cfg3/mu": np.array([r.mu for r in trace.records]),
                    "cfg3/t": np.array([r.t for r in trace.records]),
                    "cfg3/rel": np.array([r.rel_change for r in trace.records]),
                    "cfg3/x_norm": np.array(np.linalg.norm(x.ravel())), "cfg3/x_sample": x.ravel()[idx]})
        print(f"cfg3: {trace.iterations} iterations in {time.time() - t0:.1f} s", flush=True)
    np.savez_compressed(path, **out)
    print(f"wrote {len(out)} arrays -> {path}")


if __name__ == "__main__":
    main(tuple(sys.argv[1:]) or ("cfg5_256", "cfg5_512", "cfg3"))
