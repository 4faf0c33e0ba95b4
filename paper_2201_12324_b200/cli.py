"""``lin`` command line: the reference's file-driven
entropic OT entry (otkit/cli.py:58-73, 123-172, 350-419) on the GPU path.

    python -m paper_2201_12324_b200 lin --x X.csv --y Y.csv [--a A.csv] [--b B.csv]
        [--eps E | --eps-rel R] [--threshold T] [--max-iters N]
        [--coupling-out P.csv] [--out summary.json]
    python -m paper_2201_12324_b200 lin --cost-matrix C.csv ...

Same CSV conventions (comma-separated, no header, '#' comments; fileio.py),
same weight checks and rescaling (_as_cli_weights), same JSON summary keys,
same exit codes (0 converged, 1 input error, 2 not converged / diverged) and
atomic writes.  Differences, all on the side of doing more: the regularised
cost is computed online (no 4e6-entry cap), and the n x m coupling is only
materialised when --coupling-out asks for it (the reference always builds
it, cli.py:157, so it refuses every problem above the cap).  The low-rank
solver, the LP ``--verify`` oracle and the other subcommands (quad,
softsort, gmm) are outside this build's hot path and exit
with an input error.

    python -m paper_2201_12324_b200 barycenter --support S.csv --hist H1.csv
        --hist H2.csv [--weights 0.3,0.7 | --weights W.csv] [--cost sqeucl|eucl|cosine]
        [--eps E | --eps-rel R] [--threshold T] [--max-iters N]
        [--barycenter-out P.csv] [--out summary.json]

mirrors the reference's barycenter subcommand (cli.py:233-273) on the
one-launch GPU solve (csrc/bary.cu); ``--grid`` (separable GridGeometry)
is not part of this build.
"""

from __future__ import annotations

import argparse
import json
import logging
import os
import sys
import tempfile

import numpy as np

from .errors import DivergedError

logger = logging.getLogger(__name__)

__all__ = ["main"]


class _InputError(Exception):
    pass


class _Parser(argparse.ArgumentParser):
    def error(self, message):  # usage errors -> exit code 1 (cli.py:48-51)
        raise _InputError(message)


# ---- file I/O (reference fileio.py conventions) ----
def read_matrix(path: str) -> np.ndarray:
    try:
        data = np.loadtxt(path, delimiter=",", comments="#", ndmin=2)
    except Exception as exc:
        raise ValueError(f"could not parse {path} as CSV: {exc}") from exc
    if data.size == 0:
        raise ValueError(f"{path} contains no data rows")
    return data


def read_vector(path: str) -> np.ndarray:
    data = read_matrix(path)
    if 1 not in data.shape:
        raise ValueError(f"{path} must contain a single row or column, got shape {data.shape}")
    return data.reshape(-1)


def _write_atomic(path: str, text: str) -> None:
    directory = os.path.dirname(os.path.abspath(path))
    fd, tmp = tempfile.mkstemp(dir=directory, prefix=".tmp-", text=True)
    try:
        with os.fdopen(fd, "w") as fh:
            fh.write(text)
        os.replace(tmp, path)
    except BaseException:
        os.unlink(tmp)
        raise


def write_json_atomic(path: str, payload: dict) -> None:
    _write_atomic(path, json.dumps(payload, indent=2) + "\n")


def write_matrix_atomic(path: str, matrix) -> None:
    matrix = np.atleast_2d(np.asarray(matrix))
    _write_atomic(path, "\n".join(",".join(repr(float(v)) for v in row) for row in matrix) + "\n")


# ---- helpers (cli.py:79-117) ----
def _as_cli_weights(w: np.ndarray, size: int, name: str) -> np.ndarray:
    if w.size != size:
        raise _InputError(f"{name} must have {size} entries, got {w.size}")
    if np.any(w < 0) or not np.all(np.isfinite(w)):
        raise _InputError(f"{name} must be entrywise finite and nonnegative")
    total = w.sum()
    if abs(total - 1.0) > 1e-6:
        raise _InputError(f"{name} sums to {total!r}; expected 1 (within 1e-6)")
    if total != 1.0:
        if abs(total - 1.0) > 1e-9:
            logger.warning("%s sums to %.12g; rescaling to 1", name, total)
        w = w / total
    return w


def _resolve_eps(args, geom):
    if args.eps is not None and args.eps_rel is not None:
        raise _InputError("--eps and --eps-rel are mutually exclusive")
    if args.eps is not None:
        return args.eps
    if args.eps_rel is not None:
        return args.eps_rel * geom.mean_cost()
    return None


def _emit(args, payload: dict) -> None:
    if args.out:
        write_json_atomic(args.out, payload)
    else:
        print(json.dumps(payload, indent=2))


def _cmd_lin(args) -> int:
    from .geometry import DenseGeometry, PointCloudGeometry
    from .sinkhorn import LinearProblem, reg_ot_cost, solve_sinkhorn, transport_matrix
    if (args.cost_matrix is None) == (args.x is None or args.y is None):
        raise _InputError("provide either --cost-matrix or both --x and --y")
    if args.solver != "sinkhorn":
        raise _InputError("--solver lr (low-rank Sinkhorn) is outside this build's hot path")
    if args.verify:
        raise _InputError("--verify (exact LP oracle) is outside this build's hot path")
    if args.cost_matrix is not None:
        geom = DenseGeometry(read_matrix(args.cost_matrix))
    else:
        geom = PointCloudGeometry(read_matrix(args.x), read_matrix(args.y), args.cost)
    n, m = geom.shape
    a = _as_cli_weights(read_vector(args.a), n, "a") if args.a else None
    b = _as_cli_weights(read_vector(args.b), m, "b") if args.b else None
    prob = LinearProblem(geom, a, b)
    eps = _resolve_eps(args, geom)
    opts = {}
    if args.threshold is not None:
        opts["threshold"] = args.threshold
    if args.max_iters is not None:
        opts["max_iters"] = args.max_iters
    out = solve_sinkhorn(prob, eps, **opts)
    costs = reg_ot_cost(out, prob)
    payload = {
        "command": "lin",
        "solver": "sinkhorn",
        "transport_cost": costs.transport_cost,
        "dual_objective": costs.dual_objective,
        "iterations": out.iterations,
        "converged": out.converged,
        "eps": out.eps,
    }
    if args.coupling_out:
        write_matrix_atomic(args.coupling_out, transport_matrix(out, prob).matrix)
    _emit(args, payload)
    return 0 if payload["converged"] else 2


def _parse_weights_arg(raw: str | None, size: int):
    """cli.py:262-272: a CSV path or comma-separated floats, checked like weights."""
    if raw is None:
        return None
    if os.path.exists(raw):
        w = read_vector(raw)
    else:
        try:
            w = np.array([float(tok) for tok in raw.split(",")])
        except ValueError:
            raise _InputError(f"--weights must be a CSV path or comma-separated floats, "
                              f"got {raw!r}") from None
    return _as_cli_weights(w, size, "weights")


def _cmd_barycenter(args) -> int:
    from .barycenter import BarycenterProblem, solve_barycenter
    from .geometry import PointCloudGeometry
    if (args.support is None) == (args.grid is None):
        raise _InputError("provide either --support or --grid")
    if args.grid is not None:
        raise _InputError("--grid (separable GridGeometry) is outside this build's hot path")
    support = read_matrix(args.support)
    geom = PointCloudGeometry(support, support, args.cost)
    hists = np.stack([read_vector(p) for p in args.hist])
    hists = np.stack([_as_cli_weights(h, geom.shape[0], f"histogram {i}")
                      for i, h in enumerate(hists)])
    weights = _parse_weights_arg(args.weights, hists.shape[0])
    bp = BarycenterProblem(geom, hists, weights)
    eps = _resolve_eps(args, geom)
    opts = {}
    if args.threshold is not None:
        opts["threshold"] = args.threshold
    if args.max_iters is not None:
        opts["max_iters"] = args.max_iters
    out = solve_barycenter(bp, eps, **opts)
    payload = {
        "command": "barycenter",
        "converged": out.converged,
        "iterations": out.iterations,
        "eps": out.eps,
        "num_histograms": int(hists.shape[0]),
        "support_size": int(geom.shape[0]),
        "barycenter": out.barycenter.tolist(),
    }
    if args.barycenter_out:
        write_matrix_atomic(args.barycenter_out, out.barycenter.reshape(-1, 1))
    _emit(args, payload)
    return 0 if out.converged else 2


def _unsupported(args) -> int:
    raise _InputError(f"subcommand {args.command!r} is outside this build's hot path "
                      "(only 'lin' with the Sinkhorn solver and 'barycenter' are provided)")


def _build_parser() -> argparse.ArgumentParser:
    parser = _Parser(prog="paper_2201_12324_b200",
                     description="entropic OT between two discrete measures on a B200")
    commands = parser.add_subparsers(dest="command", required=True)
    lin = commands.add_parser("lin", help="entropic OT between two discrete measures")
    lin.add_argument("--x", help="source points CSV (one point per row)")
    lin.add_argument("--y", help="target points CSV")
    lin.add_argument("--cost-matrix", help="explicit cost matrix CSV (alternative to --x/--y)")
    lin.add_argument("--cost", choices=("sqeucl", "eucl", "cosine"), default="sqeucl")
    lin.add_argument("--a", help="source weights CSV (default uniform)")
    lin.add_argument("--b", help="target weights CSV (default uniform)")
    lin.add_argument("--solver", choices=("sinkhorn", "lr"), default="sinkhorn")
    lin.add_argument("--rank", type=int)
    lin.add_argument("--seed", type=int, default=0)
    lin.add_argument("--coupling-out", help="write the coupling matrix CSV here")
    lin.add_argument("--verify", action="store_true")
    lin.add_argument("--eps", type=float, help="absolute regularization strength")
    lin.add_argument("--eps-rel", type=float, help="regularization as a fraction of the mean cost")
    lin.add_argument("--threshold", type=float, help="solver convergence threshold")
    lin.add_argument("--max-iters", type=int, help="solver iteration cap")
    lin.add_argument("--out", help="write the JSON summary here instead of stdout")
    lin.set_defaults(handler=_cmd_lin)
    bary = commands.add_parser("barycenter", help="fixed-support barycenter of histograms")
    bary.add_argument("--support", help="support points CSV (dense mode)")
    bary.add_argument("--grid", nargs="+", help="per-axis coordinate CSVs (not in this build)")
    bary.add_argument("--cost", choices=("sqeucl", "eucl", "cosine"), default="sqeucl")
    bary.add_argument("--hist", action="append", required=True,
                      help="histogram CSV; repeat per input")
    bary.add_argument("--weights", help="barycentric weights: comma-separated floats or a CSV path")
    bary.add_argument("--barycenter-out", help="write the barycenter CSV here")
    bary.add_argument("--eps", type=float, help="absolute regularization strength")
    bary.add_argument("--eps-rel", type=float, help="regularization as a fraction of the mean cost")
    bary.add_argument("--threshold", type=float, help="solver convergence threshold")
    bary.add_argument("--max-iters", type=int, help="solver iteration cap")
    bary.add_argument("--out", help="write the JSON summary here instead of stdout")
    bary.set_defaults(handler=_cmd_barycenter)
    for name in ("quad", "softsort", "gmm"):
        sub = commands.add_parser(name, help="(not in this build)")
        sub.set_defaults(handler=_unsupported)
    return parser


def main(argv: list[str] | None = None) -> int:
    level = os.environ.get("OTKIT_LOG", "WARNING").upper()
    logging.basicConfig(level=getattr(logging, level, logging.WARNING),
                        format="%(levelname)s %(name)s: %(message)s")
    parser = _build_parser()
    try:
        args, extra = parser.parse_known_args(argv)
        if extra and args.command in ("lin", "barycenter"):
            raise _InputError(f"unrecognized arguments: {' '.join(extra)}")
        return args.handler(args)
    except _InputError as err:
        print(f"error: {err}", file=sys.stderr)
        return 1
    except DivergedError as err:
        print(f"error: {err}", file=sys.stderr)
        return 2
    except (ValueError, OSError) as err:
        print(f"error: {err}", file=sys.stderr)
        return 1
