"""Command line of the B200 engine: the reference CLI's experiment drivers (cli.py:136-240).

    python -m paper_2110_01470_b200 run   [--function f5 --schedule parallel --nsol ... --runs N --out r.csv]
    python -m paper_2110_01470_b200 sweep [--function f1 --triples builtin|FILE --runs N --out r.csv]

Same flags, JSON ``--config`` layering (hard defaults < file < explicit
flags; unknown keys rejected) and exit codes (0 ok, 1 usage error, 2 runtime
failure) as the reference ``sso`` CLI (cli.py:44-69, 355-386); extra flags
``--dtype`` and ``--rng``.  Every cell runs on the device (harness.py here);
the records CSV has the reference schema, so the reference's ``sso compare``,
``sso stats`` and ``sso plot-data`` (statistics and plotting, outside the hot
path) read it unchanged.
"""

from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

import numpy as np

from . import harness
from .parallel import LayoutMode
from .records import ScheduleKind

EXIT_OK = 0
EXIT_USAGE = 1
EXIT_RUNTIME = 2

FUNCTIONS = [f"f{i}" for i in range(1, 10)]


class UsageError(Exception):
    pass


class _Parser(argparse.ArgumentParser):
    def error(self, message):  # argparse would exit 2; the CLI contract says 1
        raise UsageError(message)


def _merged(args: argparse.Namespace, defaults: dict) -> dict:
    """hard defaults < config file < explicit flags (reference cli.py:51-69)."""
    merged = dict(defaults)
    if args.config is not None:
        try:
            loaded = json.loads(Path(args.config).read_text(encoding="utf-8"))
        except FileNotFoundError:
            raise UsageError(f"config file not found: {args.config}")
        except json.JSONDecodeError as exc:
            raise UsageError(f"config file is not valid JSON: {exc}")
        for key, value in loaded.items():
            if key not in defaults:
                raise UsageError(f"unknown config key {key!r}")
            merged[key] = value
    for key in defaults:
        value = getattr(args, key, None)
        if value is not None:
            merged[key] = value
    return merged


def _build_parser() -> _Parser:
    parser = _Parser(prog="psso-b200", description=__doc__.split("\n\n")[0])
    sub = parser.add_subparsers(dest="command", required=True)

    run = sub.add_parser("run", help="repeated optimization runs on the device, results to CSV")
    run.add_argument("--function", choices=FUNCTIONS)
    run.add_argument("--schedule", choices=["sequential", "parallel"])
    run.add_argument("--workers", type=int)
    run.add_argument("--nsol", type=int)
    run.add_argument("--nvar", type=int)
    run.add_argument("--iters", type=int)
    run.add_argument("--cw", type=float)
    run.add_argument("--cp", type=float)
    run.add_argument("--cg", type=float)
    run.add_argument("--seed", type=int, help="base seed; run r uses seed + r")
    run.add_argument("--runs", type=int)
    run.add_argument("--layout", choices=[str(m) for m in LayoutMode])
    run.add_argument("--out", type=Path)
    run.add_argument("--trajectory", action="store_true", default=None,
                     help="also write <out>.trajectories.dat")
    run.add_argument("--dtype", choices=["float64", "float32"])
    run.add_argument("--rng", choices=["reference", "philox"])
    run.add_argument("--config", type=Path, default=None)

    sweep = sub.add_parser("sweep", help="threshold triples, one device cell each")
    sweep.add_argument("--function", choices=FUNCTIONS)
    sweep.add_argument("--triples", help="'builtin' or a file with one 'cw,cp,cg' line each")
    sweep.add_argument("--runs", type=int)
    sweep.add_argument("--nsol", type=int)
    sweep.add_argument("--nvar", type=int)
    sweep.add_argument("--iters", type=int)
    sweep.add_argument("--workers", type=int)
    sweep.add_argument("--seed", type=int)
    sweep.add_argument("--out", type=Path)
    sweep.add_argument("--schedule", choices=["sequential", "parallel"])
    sweep.add_argument("--config", type=Path, default=None)
    return parser


def _print_summaries(summaries) -> None:  # reference cli.py:172-177
    print(f"{'function':<10}{'schedule':<12}{'n':>4}{'mean':>16}{'std':>16}{'min':>16}")
    for row in summaries:
        std = f"{row.std:.6g}" if row.std is not None else "-"
        print(f"{row.function:<10}{str(row.schedule):<12}{row.n:>4}"
              f"{row.mean:>16.6g}{std:>16}{row.min:>16.6g}")


def _cmd_run(args) -> int:
    cfg = _merged(args, {
        "function": "f1", "schedule": "parallel", "workers": 1,
        "nsol": harness.DEFAULT_NSOL, "nvar": harness.DEFAULT_NVAR, "iters": harness.DEFAULT_NITER,
        "cw": harness.DEFAULT_THRESHOLDS[0], "cp": harness.DEFAULT_THRESHOLDS[1],
        "cg": harness.DEFAULT_THRESHOLDS[2], "seed": 0, "runs": harness.DEFAULT_REPLICATIONS,
        "layout": str(LayoutMode.PARTICLE_MAJOR), "out": None, "trajectory": False,
        "dtype": "float64", "rng": "reference",
    })
    try:
        config = harness.ExperimentConfig(
            functions=[cfg["function"]], schedules=[ScheduleKind(cfg["schedule"])],
            replications=int(cfg["runs"]), base_seed=int(cfg["seed"]),
            nsol=int(cfg["nsol"]), nvar=int(cfg["nvar"]), niter=int(cfg["iters"]),
            cw=float(cfg["cw"]), cp=float(cfg["cp"]), cg=float(cfg["cg"]),
            workers=int(cfg["workers"]), layout=LayoutMode(cfg["layout"]),
            record_trajectory=bool(cfg["trajectory"]), dtype=cfg["dtype"], rng=cfg["rng"])
    except ValueError as exc:
        raise UsageError(str(exc))
    report = harness.run_experiment(config, out=cfg["out"])
    if cfg["out"] is not None and cfg["trajectory"]:
        side = Path(cfg["out"]).with_suffix(Path(cfg["out"]).suffix + ".trajectories.dat")
        harness.write_trajectories(report.records, side)
        print(f"trajectories -> {side}")
    _print_summaries(report.summaries)
    if cfg["out"] is not None:
        print(f"records -> {cfg['out']}")
    return EXIT_OK


def _parse_triples(token) -> tuple:  # reference cli.py:180-199
    if token in (None, "builtin"):
        return harness.DEFAULT_TRIPLES
    path = Path(token)
    if not path.exists():
        raise UsageError(f"--triples expects 'builtin' or an existing file, got {token!r}")
    triples = []
    for line in path.read_text(encoding="utf-8").splitlines():
        line = line.strip()
        if not line or line.startswith("#"):
            continue
        parts = [float(v) for v in line.replace(",", " ").split()]
        if len(parts) != 3:
            raise UsageError(f"triple line must have 3 values, got {line!r}")
        triples.append(tuple(parts))
    if not triples:
        raise UsageError(f"no triples found in {path}")
    return tuple(triples)


def _cmd_sweep(args) -> int:
    cfg = _merged(args, {
        "function": "f1", "triples": "builtin", "runs": harness.DEFAULT_REPLICATIONS,
        "nsol": harness.DEFAULT_NSOL, "nvar": harness.DEFAULT_NVAR, "iters": harness.DEFAULT_NITER,
        "workers": 1, "seed": 0, "out": None, "schedule": "parallel",
    })
    try:
        config = harness.SweepConfig(
            function=cfg["function"], triples=_parse_triples(cfg["triples"]),
            replications=int(cfg["runs"]), base_seed=int(cfg["seed"]), nsol=int(cfg["nsol"]),
            nvar=int(cfg["nvar"]), niter=int(cfg["iters"]), workers=int(cfg["workers"]),
            schedule=ScheduleKind(cfg["schedule"]))
        report = harness.parameter_sweep(config)
    except ValueError as exc:
        raise UsageError(str(exc))
    if cfg["out"] is not None:
        harness.write_records(report.records, cfg["out"])
        print(f"records -> {cfg['out']}")
    print(f"{'cw':>6}{'cp':>6}{'cg':>6}{'n':>4}{'mean':>16}{'std':>16}{'min':>16}")
    for triple, values in report.groups.items():
        arr = np.asarray(values)
        std = f"{arr.std(ddof=1):.6g}" if arr.size > 1 else "-"
        print(f"{triple[0]:>6}{triple[1]:>6}{triple[2]:>6}{arr.size:>4}"
              f"{arr.mean():>16.6g}{std:>16}{arr.min():>16.6g}")
    print(report.note)
    return EXIT_OK


_COMMANDS = {"run": _cmd_run, "sweep": _cmd_sweep}


def main(argv=None) -> int:
    parser = _build_parser()
    try:
        args = parser.parse_args(argv)
        return _COMMANDS[args.command](args)
    except UsageError as exc:
        print(f"usage error: {exc}", file=sys.stderr)
        return EXIT_USAGE
    except (ValueError, OSError, RuntimeError) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return EXIT_RUNTIME


if __name__ == "__main__":
    sys.exit(main())
