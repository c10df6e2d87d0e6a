"""Generate tests/golden/golden.npz by running the REFERENCE implementation.

Run in the build container only (the reference is not on the GPU box):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

The fixture holds, per case, the seeded inputs, the spec metadata (JSON) and
the outputs of `ltensor` (the reference) on those inputs.  It pins the CPU
oracle (tests/test_oracle_golden.py) and the CUDA path (tests/test_gpu_*.py).
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE))

import cases  # noqa: E402
import ltensor as ref  # noqa: E402  (the reference, via PYTHONPATH)
from ltensor.completion import CompletionConfig  # noqa: E402


def spec_of(case):
    if case["kind"] == "explicit":
        return ref.make_spec("explicit", case["spec_shape"], modes=case.get("modes"), matrices=case["matrices"])
    return ref.make_spec(case["kind"], case["spec_shape"], modes=case.get("modes"))


def put_meta(out, name, case, **extra):
    meta = {"kind": case["kind"], "spec_shape": list(case["spec_shape"]),
            "modes": list(case["modes"]) if case.get("modes") else None}
    meta.update(extra)
    out[f"{name}/meta"] = np.array(json.dumps(meta))
    for mode, mat in (case.get("matrices") or {}).items():
        out[f"{name}/mat{mode}"] = np.asarray(mat)


def lp(a, b, kind, shape):
    return ref.l_product(a, b, ref.make_spec(kind, shape))


def main():
    out = {}
    for name, case in cases.transform_cases().items():
        spec = spec_of(case)
        put_meta(out, name, case)
        out[f"{name}/x"] = case["x"]
        fwd = ref.apply_l(case["x"], spec)
        out[f"{name}/fwd"] = fwd
        out[f"{name}/inv"] = ref.apply_l_inv(fwd, spec, assume_real=True)
        if spec.kind in ("fft", "dct"):
            out[f"{name}/fwd_explicit"] = ref.apply_l(case["x"], spec, explicit=True)
    for name, case in cases.product_cases().items():
        put_meta(out, name, case)
        out[f"{name}/a"] = case["a"]
        out[f"{name}/b"] = case["b"]
        out[f"{name}/c"] = ref.l_product(case["a"], case["b"], spec_of(case))
    # the generalized c-product through the reference's block-Toeplitz-plus-Hankel
    # construction (btph.py:140-149), the paper's independent characterisation of cprod
    from ltensor.btph import cproduct_via_btph

    for name, case in cases.btph_cases().items():
        put_meta(out, name, case)
        out[f"{name}/a"] = case["a"]
        out[f"{name}/b"] = case["b"]
        out[f"{name}/c"] = cproduct_via_btph(case["a"], case["b"])
    for name, case in cases.svd_cases().items():
        spec = spec_of(case)
        put_meta(out, name, case, tau=case["tau"])
        out[f"{name}/x"] = case["x"]
        f = ref.t_svd(case["x"], spec)
        out[f"{name}/s"] = f.s
        out[f"{name}/u"] = f.u
        out[f"{name}/v"] = f.v
        out[f"{name}/tube_norms"] = f.tube_norms
        out[f"{name}/sv"] = np.linalg.svd(ref.core.as_rep_stack(ref.apply_l(case["x"], spec)), compute_uv=False)
        if spec.unitary_scaled:
            out[f"{name}/svt"] = ref.svt(case["x"], case["tau"], spec)
            out[f"{name}/nuclear"] = np.array(ref.nuclear_norm(case["x"], spec))
            out[f"{name}/spectral"] = np.array(ref.spectral_norm(case["x"], spec))
        rr = ref.ranks(case["x"], spec)
        out[f"{name}/multirank"] = np.asarray(rr.multirank)
        out[f"{name}/tubal"] = np.array(rr.tubal)
    for name, case in cases.completion_cases(lp).items():
        spec = spec_of(dict(case, spec_shape=case["m"].shape))
        mask = case["mask"]
        if mask is None:
            mask = ref.sample_mask(case["m"].shape, *case["mask_seed"])
        cfg = CompletionConfig(spec=spec, **case["cfg"])
        x, trace = ref.pga_complete(case["m"], mask, cfg, ground_truth=case.get("gt"))
        put_meta(out, name, dict(case, spec_shape=case["m"].shape), cfg=case["cfg"],
                 status=trace.status, final_rse=ref.rse(x, case["m"]))
        out[f"{name}/m"] = case["m"]
        out[f"{name}/mask"] = mask
        if case.get("gt") is not None:
            out[f"{name}/gt"] = case["gt"]
        out[f"{name}/x_out"] = x
        out[f"{name}/mu"] = np.array([r.mu for r in trace.records])
        out[f"{name}/t"] = np.array([r.t for r in trace.records])
        out[f"{name}/rel"] = np.array([r.rel_change for r in trace.records])
        if case.get("gt") is not None:
            out[f"{name}/rse"] = np.array([r.rse for r in trace.records])
            out[f"{name}/psnr"] = np.array([r.psnr for r in trace.records])
    for name, case in cases.algebra_cases().items():
        spec = spec_of(case)
        put_meta(out, name, case, **({"k": case["k"]} if "k" in case else {}))
        if name.startswith("a_truncate"):
            out[f"{name}/x"] = case["x"]
            out[f"{name}/out"] = ref.truncate(ref.t_svd(case["x"], spec), case["k"])
        elif name.startswith("a_inner"):
            out[f"{name}/a"] = case["a"]
            out[f"{name}/b"] = case["b"]
            out[f"{name}/value"] = np.array(ref.inner_product(case["a"], case["b"]))
        else:
            q = ref.t_svd(case["x"], spec).u
            out[f"{name}/q"] = q
            out[f"{name}/orth"] = np.array(ref.is_orthogonal(q, spec))
            out[f"{name}/nonorth"] = np.array(ref.is_orthogonal(case["x"], spec))
    for name, case in cases.mode_product_cases().items():
        out[f"{name}/x"] = case["x"]
        out[f"{name}/u"] = case["u"]
        out[f"{name}/n"] = np.array(case["n"])
        out[f"{name}/out"] = ref.mode_n_product(case["x"], case["u"], case["n"])
    for name, (dims, sr, seed) in cases.mask_cases().items():
        out[f"{name}/meta"] = np.array(json.dumps({"dims": list(dims), "sr": sr, "seed": seed}))
        out[f"{name}/mask"] = ref.sample_mask(dims, sr, seed)
    # TLT1 container bytes written by the reference (io.py:39-51) for a few dtypes / orders
    import tempfile

    from ltensor.io import write_container

    r = np.random.default_rng(2718)
    io_cases = {"io_f64": r.standard_normal((3, 4, 2, 5)), "io_f32": r.standard_normal((2, 3, 4)).astype(np.float32),
                "io_c128": r.standard_normal((2, 2, 3)) + 1j * r.standard_normal((2, 2, 3)),
                "io_mask": r.random((5, 4, 3, 2)) < 0.37}
    with tempfile.TemporaryDirectory() as td:
        for name, x in io_cases.items():
            path = Path(td) / f"{name}.tlt"
            write_container(path, x)
            out[f"{name}/x"] = x
            out[f"{name}/bytes"] = np.frombuffer(path.read_bytes(), dtype=np.uint8)
    np.savez_compressed(HERE / "golden.npz", **out)
    total = sum(np.asarray(v).nbytes for v in out.values())
    print(f"wrote {len(out)} arrays, {total / 1e6:.2f} MB raw -> {HERE / 'golden.npz'}")


if __name__ == "__main__":
    main()
