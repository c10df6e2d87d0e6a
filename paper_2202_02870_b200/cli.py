"""Command line interface over the B200 path (drop-in for pkg/src/ltensor/cli.py).

The command surface (sub-commands, flags, printed lines, exit codes 0 success /
1 usage / 2 numeric, format or device error) is the reference's; every numeric
command runs on the GPU through this package's API (no CPU fallback) and moves
tensors in TLT1 containers (io.py).

    python -m paper_2202_02870_b200 product --a A.tlt --b B.tlt --transform dct --out C.tlt
"""

from __future__ import annotations

import argparse
import math
import sys

from . import completion, io, linalg
from .errors import LTensorError
from .transforms import make_spec


def _int_list(text):
    try:
        dims = tuple(int(d) for d in text.split(","))
    except ValueError:
        raise argparse.ArgumentTypeError(f"bad dims {text!r}, expected e.g. 10,10,3")
    if min(dims) < 1:
        raise argparse.ArgumentTypeError("dims must be positive")
    return dims


def _mode_list(text):
    if text == "3..N":
        return None  # every trailing mode (make_spec's default)
    try:
        return tuple(int(m) for m in text.split(","))
    except ValueError:
        raise argparse.ArgumentTypeError(f"bad modes {text!r}, expected '3..N' or e.g. '3'")


# (flag, argparse keyword arguments); "T" marks the shared --transform/--modes pair
_TRANSFORM = [("--transform", dict(choices=("fft", "dct", "cprod"), required=True)),
              ("--modes", dict(default="3..N", help="'3..N' (default) or comma list like '3'"))]
_REQ = dict(required=True)
_COMMAND_FLAGS = {
    "complete": ("run tensor completion",
                 [("--input", _REQ), ("--mask", _REQ), "T", ("--nu", dict(type=float, default=0.9)),
                  ("--mu0", dict(type=float, default=None)), ("--mu-bar-ratio", dict(type=float, default=1e-4)),
                  ("--tol", dict(type=float, default=1e-4)), ("--max-iters", dict(type=int, default=100)),
                  ("--ground-truth", dict(default=None)), ("--trace-csv", dict(default=None)), ("--out", _REQ),
                  ("--reimpose-observed", dict(action="store_true")),
                  ("--rse-denominator", dict(choices=("obtained", "original"), default="obtained"))]),
    "tsvd": ("compute the *_L-SVD factors",
             [("--input", _REQ), "T", ("--out-u", _REQ), ("--out-s", _REQ), ("--out-v", _REQ),
              ("--truncate", dict(type=int, default=None, metavar="K"))]),
    "product": ("compute a *_L product", [("--a", _REQ), ("--b", _REQ), "T", ("--out", _REQ)]),
    "svt": ("singular value thresholding",
            [("--input", _REQ), ("--tau", dict(type=float, required=True)), "T", ("--out", _REQ)]),
    "metrics": ("print RSE and PSNR between two tensors",
                [("--a", dict(required=True, help="obtained tensor")),
                 ("--b", dict(required=True, help="original tensor"))]),
}


def build_parser() -> argparse.ArgumentParser:
    parser = argparse.ArgumentParser(prog="ltensor", description=__doc__)
    sub = parser.add_subparsers(dest="command", required=True)
    mask = sub.add_parser("mask", help="observation mask utilities")
    gen = mask.add_subparsers(dest="mask_command", required=True).add_parser(
        "gen", help="sample a uniform observation mask")
    for flag, kw in (("--dims", dict(type=_int_list, required=True)), ("--sr", dict(type=float, required=True)),
                     ("--seed", dict(type=int, required=True)), ("--out", _REQ)):
        gen.add_argument(flag, **kw)
    for name, (help_text, flags) in _COMMAND_FLAGS.items():
        p = sub.add_parser(name, help=help_text)
        for item in flags:
            for flag, kw in (_TRANSFORM if item == "T" else [item]):
                p.add_argument(flag, **kw)
    return parser


def _spec_for(ns, shape):
    return make_spec(ns.transform, shape, modes=_mode_list(ns.modes))


def run_mask(ns):
    io.write_container(ns.out, completion.sample_mask(ns.dims, ns.sr, ns.seed))


def run_complete(ns):
    m = io.read_container(ns.input)
    cfg = completion.CompletionConfig(
        spec=_spec_for(ns, m.shape), nu=ns.nu, mu0=ns.mu0, mu_bar_ratio=ns.mu_bar_ratio, tol=ns.tol,
        max_iters=ns.max_iters, reimpose_observed=ns.reimpose_observed, rse_denominator=ns.rse_denominator)
    truth = None if ns.ground_truth is None else io.read_container(ns.ground_truth)
    x, trace = completion.pga_complete(m, io.read_container(ns.mask), cfg, ground_truth=truth)
    io.write_container(ns.out, x)
    if ns.trace_csv:
        trace.write_csv(ns.trace_csv)
    final = trace.records[-1]
    lines = [f"status {trace.status} after {trace.iterations} iterations, rel_change {final.rel_change:.3e}"]
    if final.rse is not None:
        lines += [f"RSE {final.rse:.6g}", f"PSNR {final.psnr:.6g}"]
    print("\n".join(lines))


def run_tsvd(ns):
    a = io.read_container(ns.input)
    f = linalg.t_svd(a, _spec_for(ns, a.shape))
    factors = [f.u, f.s, f.v]
    if ns.truncate is not None:
        k, top = ns.truncate, min(f.s.shape[:2])
        if k < 1 or k > top:
            raise LTensorError(f"truncation rank {k} out of range [1, {top}]")
        factors = [f.u[:, :k], f.s[:k, :k], f.v[:, :k]]
    for path, t in zip((ns.out_u, ns.out_s, ns.out_v), factors):
        io.write_container(path, t)


def run_product(ns):
    a, b = io.read_container(ns.a), io.read_container(ns.b)
    io.write_container(ns.out, linalg.l_product(a, b, _spec_for(ns, a.shape)))


def run_svt(ns):
    a = io.read_container(ns.input)
    io.write_container(ns.out, linalg.svt(a, ns.tau, _spec_for(ns, a.shape)))


def run_metrics(ns):
    got, ref = io.read_container(ns.a), io.read_container(ns.b)
    peak = completion.psnr(got, ref)
    print(f"RSE {completion.rse(got, ref):.12g}")
    print("PSNR inf" if math.isinf(peak) else f"PSNR {peak:.12g}")


def main(argv=None) -> int:
    try:
        ns = build_parser().parse_args(argv)
    except SystemExit as exc:  # argparse: --help exits 0, usage errors 2 -> our 1
        return 0 if exc.code == 0 else 1
    runner = {"mask": run_mask, "complete": run_complete, "tsvd": run_tsvd, "product": run_product,
              "svt": run_svt, "metrics": run_metrics}[ns.command]
    try:
        runner(ns)
    except (LTensorError, OSError) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 2
    return 0


if __name__ == "__main__":
    sys.exit(main())
