"""Experiment cells on the B200 engine: the reference harness's run loop, batched.

SURVEY §8(f) "next" #2: the reference harness (``harness.py``) runs every
(function, schedule) cell as ``replications`` independent ``run_parallel``
calls with seeds ``base_seed + run_id`` (``_run_one``, harness.py:148-163;
``run_experiment``, :217-263) and streams a results CSV (schema :46, writer
:187-214).  Here a parallel-schedule cell is ONE device job: all its seeds run
side by side in the whole-run kernel (``run_parallel_batch``), and the records
-- bit-identical per seed to ``run_parallel`` -- are written in the
reference's CSV schema and formatting, so the reference's readers, summaries,
statistics and plotting tools consume them unchanged.

Both schedules run on the device: a sequential cell is likewise ONE job
(``run_sequential_batch``: one k_seq launch, one CTA per seed), bit-identical
per seed to the reference's ``run_sequential``.  Shapes the batched kernels
do not take (nvar > 128, or nsol*nvar > 2^22) fall back to one device run per
seed (the parallel schedule; the sequential one needs nvar <= 128).
"""

from __future__ import annotations

from dataclasses import dataclass, field, replace
from pathlib import Path
from typing import Optional, Sequence, Union

import numpy as np

from .benchmarks import BenchmarkFn, make_function
from .core import NonFiniteFitnessError, SsoParams
from .core import run_sequential
from .parallel import LayoutMode, run_parallel, run_parallel_batch, run_sequential_batch
from .records import RunRecord, ScheduleKind

__all__ = [
    "CSV_HEADER",
    "DEFAULT_TRIPLES",
    "SweepConfig",
    "SweepReport",
    "parameter_sweep",
    "write_trajectories",
    "write_trajectory_rows",
    "read_trajectory_rows",
    "ExperimentConfig",
    "ExperimentReport",
    "SpeedupReport",
    "SummaryRow",
    "compute_speedup",
    "read_records",
    "run_cell",
    "run_experiment",
    "summarize",
    "write_records",
    "write_summary",
]

#: reference defaults (harness.py:49-68): the paper's setup
DEFAULT_TRIPLES = ((0.1, 0.3, 0.7), (0.1, 0.4, 0.8), (0.2, 0.4, 0.6), (0.2, 0.5, 0.9),
                   (0.3, 0.4, 0.5), (0.3, 0.6, 0.8))
DEFAULT_NSOL = 100
DEFAULT_NVAR = 50
DEFAULT_NITER = 1000
DEFAULT_THRESHOLDS = (0.3, 0.6, 0.8)
DEFAULT_REPLICATIONS = 20
DEFAULT_POWER_A = 84.0
DEFAULT_POWER_B = 180.0
#: trajectory sidecar header (harness.py:318)
TRAJECTORY_HEADER = "# columns: run_id schedule function iteration gbest_fitness"

#: results CSV columns, identical to the reference (harness.py:46)
CSV_HEADER = "run_id,schedule,function,nsol,nvar,niter,cw,cp,cg,seed,best_fitness,wall_time_s"
_BATCH_MAX_ELEMS = 1 << 22


def _cell(value) -> str:
    # floats in repr form, like the reference's writer, so rows round-trip exactly
    return repr(value) if isinstance(value, float) else str(value)


@dataclass(frozen=True)
class SummaryRow:
    """Per-cell best-fitness statistics (reference harness.py:71-79)."""

    function: str
    schedule: ScheduleKind
    n: int
    mean: float
    std: Optional[float]  # None for a single replication, like the reference
    min: float


@dataclass(frozen=True)
class SpeedupReport:
    """Mean-time ratio and power-rectified efficiency (reference harness.py:82-93)."""

    mean_time_a: float
    mean_time_b: float
    speedup: float
    power_a: float
    power_b: float
    power_ratio: float
    rectified_efficiency: float
    nsol: Optional[int] = None


@dataclass
class ExperimentConfig:
    """The reference's experiment configuration (harness.py:96-128), same fields and defaults.

    Extra keyword fields: ``dtype`` and ``rng`` as in ``run_parallel``, and
    ``per_run_timing``: False (default) runs each cell's replications as one
    batched device job and gives every record the batch's loop time divided by
    the number of runs; True runs and times every replication on its own, the
    reference's protocol (harness.py:148-163), for speedup / RE comparisons
    (harness.py:354-384).  ``workers``, ``layout`` and ``block_size`` are
    accepted and have no effect on results, as in the reference;
    ``parallel_cells`` runs the cells concurrently on the device (see
    ``run_experiment``).
    """

    functions: Sequence[Union[str, BenchmarkFn]] = ("f1",)
    schedules: Sequence[ScheduleKind] = (ScheduleKind.SEQUENTIAL, ScheduleKind.PARALLEL)
    replications: int = 20
    base_seed: int = 0
    nsol: int = 100
    nvar: int = 50
    niter: int = 1000
    cw: float = 0.3
    cp: float = 0.6
    cg: float = 0.8
    workers: int = 1
    layout: LayoutMode = LayoutMode.PARTICLE_MAJOR
    record_trajectory: bool = False
    parallel_cells: bool = False
    block_size: int = 1024
    dtype: str = "float64"
    rng: str = "reference"
    per_run_timing: bool = False

    def __post_init__(self):
        if not self.functions:
            raise ValueError("config key 'functions' must list at least one function")
        if not self.schedules:
            raise ValueError("config key 'schedules' must list at least one schedule")
        self.schedules = [ScheduleKind(s) for s in self.schedules]
        self.layout = LayoutMode(self.layout)
        if not 0.0 <= self.cw <= self.cp <= self.cg <= 1.0:
            raise ValueError(
                f"thresholds must satisfy 0 <= cw <= cp <= cg <= 1, "
                f"got ({self.cw}, {self.cp}, {self.cg})"
            )
        for key in ("replications", "nsol", "nvar", "niter", "workers"):
            if int(getattr(self, key)) < 1:
                raise ValueError(f"config key {key!r} must be >= 1")


@dataclass
class ExperimentReport:
    config: ExperimentConfig
    records: list
    summaries: list
    metadata: dict = field(default_factory=dict)


def _function(entry, nvar: int) -> BenchmarkFn:
    return entry if isinstance(entry, BenchmarkFn) else make_function(entry, nvar)


def run_cell(fn: BenchmarkFn, config: ExperimentConfig, run_ids: Sequence[int],
             schedule: ScheduleKind = ScheduleKind.PARALLEL) -> list:
    """Replications ``run_ids`` of one cell (reference _run_one, harness.py:148-163).

    Seeds are ``base_seed + run_id``.  One batched launch when the shape allows
    it; ``wall_time_s`` is then the batch's loop time divided evenly over its
    runs (per-run device time; the reference times each run separately).
    """
    params = SsoParams(cw=config.cw, cp=config.cp, cg=config.cg, var_min=fn.var_min,
                       var_max=fn.var_max, nsol=config.nsol, nvar=config.nvar,
                       niter=config.niter)
    seeds = [config.base_seed + rid for rid in run_ids]
    sequential = ScheduleKind(schedule) is ScheduleKind.SEQUENTIAL
    batched = (not config.per_run_timing and config.nvar <= 128
               and config.nsol * config.nvar <= _BATCH_MAX_ELEMS)
    if batched:
        batch = run_sequential_batch if sequential else run_parallel_batch
        recs = batch(params, fn, seeds, dtype=config.dtype, rng=config.rng)
        per_run = recs[0].wall_time_s / len(recs)
        recs = [replace(r, run_id=rid, wall_time_s=per_run) for r, rid in zip(recs, run_ids)]
    elif sequential:
        recs = [replace(run_sequential(params, fn, s, dtype=config.dtype, rng=config.rng), run_id=rid)
                for s, rid in zip(seeds, run_ids)]
    else:
        recs = [replace(run_parallel(params, fn, s, workers=config.workers, layout=config.layout,
                                     dtype=config.dtype, rng=config.rng), run_id=rid)
                for s, rid in zip(seeds, run_ids)]
    out = []
    for r in recs:
        r = replace(r, function=fn.id)
        if not config.record_trajectory:
            r = replace(r, trajectory=None)
        out.append(r)
    return out


def summarize(records: Sequence[RunRecord]) -> list:
    """Per (function, schedule) mean / sample std / min, in first-seen order (harness.py:166-184)."""
    cells: dict = {}
    for rec in records:
        cells.setdefault((rec.function, rec.schedule), []).append(rec.best_fitness)
    out = []
    for (function, schedule), vals in cells.items():
        a = np.asarray(vals, dtype=np.float64)
        out.append(SummaryRow(function=function, schedule=schedule, n=int(a.size),
                              mean=float(a.mean()),
                              std=float(a.std(ddof=1)) if a.size > 1 else None,
                              min=float(a.min())))
    return out


class _Rows:
    """Streaming results CSV in the reference format (harness.py:187-214)."""

    def __init__(self, path):
        self.fh = None if path is None else open(path, "w", encoding="utf-8")
        if self.fh:
            self.fh.write(CSV_HEADER + "\n")
            self.fh.flush()

    def add(self, rec: RunRecord):
        if self.fh:
            row = rec.scalar_row()
            self.fh.write(",".join(_cell(row[c]) for c in CSV_HEADER.split(",")) + "\n")
            self.fh.flush()

    def failed(self, exc: BaseException):
        if self.fh:
            self.fh.write(f"# FAILED: {type(exc).__name__}: {exc}\n")
            self.fh.flush()

    def close(self):
        if self.fh:
            self.fh.close()
            self.fh = None


def run_experiment(config: ExperimentConfig, out=None, summary_out=None) -> ExperimentReport:
    """Every cell, all replications, records streamed to ``out`` (reference harness.py:217-263).

    A failure mid-experiment (e.g. ``NonFiniteFitnessError``) leaves the
    completed cells' rows plus a ``# FAILED`` marker, like the reference.
    ``parallel_cells=True`` runs the cells concurrently, as the reference does
    with a thread pool: each host thread drives its cell's batched launch on
    its own CUDA stream, so the cells share the GPU's SMs (rows are still
    written in cell order; wall times then include the contention, as the
    reference warns).
    """
    functions = [_function(e, config.nvar) for e in config.functions]
    cells = [(fn, schedule) for fn in functions for schedule in config.schedules]
    sink = _Rows(None if out is None else Path(out))
    records = []

    def emit(recs):
        for rec in recs:
            sink.add(rec)
            records.append(rec)

    def one_cell(cell):
        fn, schedule = cell
        return run_cell(fn, config, range(config.replications), schedule)

    try:
        if config.parallel_cells and len(cells) > 1:
            from concurrent.futures import ThreadPoolExecutor

            with ThreadPoolExecutor(max_workers=len(cells)) as pool:
                for recs in pool.map(one_cell, cells):  # a failed cell raises here, in order
                    emit(recs)
        else:
            for fn, schedule in cells:
                try:
                    cell = one_cell((fn, schedule))
                except NonFiniteFitnessError:
                    # a batched cell fails as a whole: replay it run by run so the
                    # rows of the replications before the failing one are written
                    # first, as the reference's sequential loop leaves them
                    cell = []
                    for rid in range(config.replications):
                        try:
                            one = run_cell(fn, replace(config, per_run_timing=True), [rid],
                                           schedule)
                        except NonFiniteFitnessError:
                            emit(cell)
                            raise
                        cell.extend(one)
                emit(cell)
    except BaseException as exc:
        sink.failed(exc)
        raise
    finally:
        sink.close()
    report = ExperimentReport(config=config, records=records, summaries=summarize(records),
                              metadata={"block_size": config.block_size, "engine": "b200",
                                        "wall_time_s": "per run (the reference protocol)"
                                        if config.per_run_timing else
                                        "batched cell: loop time of the batch / runs"})
    if summary_out is not None:
        write_summary(report.summaries, summary_out)
    return report


def write_records(records: Sequence[RunRecord], path) -> None:
    sink = _Rows(Path(path))
    try:
        for rec in records:
            sink.add(rec)
    finally:
        sink.close()


def read_records(path) -> list:
    """Results CSV (this module's or the reference's) back into records (harness.py:275-305)."""
    recs = []
    with open(path, encoding="utf-8") as fh:
        header = fh.readline().strip()
        if header != CSV_HEADER:
            raise ValueError(f"unexpected CSV header {header!r}")
        for line in fh:
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            p = line.split(",")
            if len(p) != 12:
                raise ValueError(f"malformed row: {line!r}")
            recs.append(RunRecord(run_id=int(p[0]), schedule=ScheduleKind(p[1]), function=p[2],
                                  nsol=int(p[3]), nvar=int(p[4]), niter=int(p[5]),
                                  cw=float(p[6]), cp=float(p[7]), cg=float(p[8]), seed=int(p[9]),
                                  best_fitness=float(p[10]), wall_time_s=float(p[11])))
    return recs


def write_summary(summaries: Sequence[SummaryRow], path) -> None:
    """Summary CSV in the reference format (harness.py:308-315)."""
    with open(path, "w", encoding="utf-8") as fh:
        fh.write("function,schedule,n,mean,std,min\n")
        for s in summaries:
            std = "" if s.std is None else repr(s.std)
            fh.write(f"{s.function},{s.schedule},{s.n},{s.mean!r},{std},{s.min!r}\n")


def compute_speedup(times_a, times_b, power_a: float, power_b: float,
                    nsol: Optional[int] = None) -> SpeedupReport:
    """Speedup = mean(a)/mean(b); RE = speedup / (power_b/power_a) (harness.py:354-384, Eq. 3.1-3.3)."""
    a = np.asarray(times_a, dtype=np.float64)
    b = np.asarray(times_b, dtype=np.float64)
    if a.size == 0 or b.size == 0:
        raise ValueError("time samples must be nonempty")
    if (a <= 0).any() or (b <= 0).any():
        raise ValueError("wall times must be positive")
    if power_a <= 0 or power_b <= 0:
        raise ValueError("power ratings must be positive")
    ma, mb = float(a.mean()), float(b.mean())
    s = ma / mb
    ratio = power_b / power_a
    return SpeedupReport(mean_time_a=ma, mean_time_b=mb, speedup=s, power_a=power_a,
                         power_b=power_b, power_ratio=ratio, rectified_efficiency=s / ratio,
                         nsol=nsol)


def write_trajectories(records: Sequence[RunRecord], path) -> None:
    """Sidecar with the per-iteration gBest curve of each run (reference harness.py:321-336)."""
    write_trajectory_rows(((rec.run_id, str(rec.schedule), rec.function, t, float(value))
                           for rec in records if rec.trajectory is not None
                           for t, value in enumerate(rec.trajectory)), path)


def write_trajectory_rows(rows, path) -> None:
    """(run_id, schedule, function, t, value) rows in the sidecar format (reference harness.py:332-336)."""
    with open(path, "w", encoding="utf-8") as fh:
        fh.write(TRAJECTORY_HEADER + "\n")
        for run_id, schedule, function, t, value in rows:
            fh.write(f"{run_id} {schedule} {function} {t} {float(value)!r}\n")


def read_trajectory_rows(path) -> list:
    """The sidecar's rows back as (run_id, schedule, function, t, value) (reference harness.py:339-351)."""
    rows = []
    with open(path, encoding="utf-8") as fh:
        for line in fh:
            line = line.strip()
            if line and not line.startswith("#"):
                rid, sched, fn, t, value = line.split()
                rows.append((int(rid), sched, fn, int(t), float(value)))
    if not rows:
        raise ValueError(f"no trajectory rows in {path}")
    return rows


@dataclass
class SweepConfig:
    """Threshold sweep (reference harness.py:388-398)."""

    function: Union[str, BenchmarkFn] = "f1"
    triples: Sequence[tuple] = DEFAULT_TRIPLES
    replications: int = DEFAULT_REPLICATIONS
    base_seed: int = 0
    nsol: int = DEFAULT_NSOL
    nvar: int = DEFAULT_NVAR
    niter: int = DEFAULT_NITER
    workers: int = 1
    schedule: ScheduleKind = ScheduleKind.PARALLEL
    dtype: str = "float64"
    rng: str = "reference"


@dataclass
class SweepReport:
    config: SweepConfig
    records: list
    groups: dict
    summaries: list
    note: Optional[str] = None


def parameter_sweep(config: SweepConfig) -> SweepReport:
    """Every threshold triple as one device cell (reference harness.py:410-444).

    The between-group Kruskal-Wallis test of the reference is statistics on
    the records, outside the hot path: the records CSV written from
    ``SweepReport.records`` has the reference schema, so the reference's
    ``sso stats --test kruskal --group-by cw,cp,cg`` runs on it unchanged.
    """
    fn = _function(config.function, config.nvar)
    for triple in config.triples:  # reject malformed triples before any compute
        SsoParams(cw=triple[0], cp=triple[1], cg=triple[2], var_min=fn.var_min,
                  var_max=fn.var_max, nsol=config.nsol, nvar=config.nvar, niter=config.niter)
    records, groups = [], {}
    for triple in config.triples:
        cell = ExperimentConfig(functions=[fn], schedules=[config.schedule],
                                replications=config.replications, base_seed=config.base_seed,
                                nsol=config.nsol, nvar=config.nvar, niter=config.niter,
                                cw=triple[0], cp=triple[1], cg=triple[2], workers=config.workers,
                                dtype=config.dtype, rng=config.rng)
        cell_records = run_experiment(cell).records
        records.extend(cell_records)
        groups[tuple(triple)] = [r.best_fitness for r in cell_records]
    note = ("only one combination swept; no between-group comparison" if len(groups) < 2 else
            "between-group test: reference `sso stats --test kruskal --group-by cw,cp,cg` on the records")
    return SweepReport(config, records, groups, summarize(records), note=note)
