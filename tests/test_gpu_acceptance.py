"""The reference's acceptance experiment (tests/test_acceptance.py:127-196 of
/root/reference/pkg: criterion 5 and the sequential-f1 regression band) run
through the device harness, with every run pinned to the oracle.

The reference's precision report is nine functions x two schedules x twenty
replications at population 100, dimension 50, 1000 iterations (run_experiment
with base_seed 0).  The device runs it as 18 batched launches; the oracle (the
reference's algorithm in C) recomputes all 360 runs on the host.  Every run's
best fitness must agree with the oracle's -- f1-f4 (no transcendentals) to
the bit, f5-f9 within the 1e-12 relative fitness tolerance -- so the cell means
the criteria read are the reference's, and each criterion must come out the
way it does for the reference itself (the reference README lists an f9
known failure: its band sits below the as-printed function's floor).
"""

import warnings
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2110_01470_b200 as psso  # noqa: E402
from oracle import oracle as O  # noqa: E402  (the checker)
from paper_2110_01470_b200.harness import ExperimentConfig, run_experiment  # noqa: E402
from paper_2110_01470_b200.records import ScheduleKind  # noqa: E402

FIDS = ("f1", "f2", "f3", "f4", "f5", "f6", "f7", "f8", "f9")
RUNS, NSOL, NVAR, NITER = 20, 100, 50, 1000
# reference study's accelerated-schedule column (test_acceptance.py:150-162)
BANDS = {
    "f1": (41.0156 * 0.5, 41.0156 * 1.5),
    "f5": (220.6183 * 0.5, 220.6183 * 1.5),
    "f6": (15.2896 * 0.5, 15.2896 * 1.5),
    "f9": (20708.0471 - 60.0, 20708.0471 + 60.0),
}


def _fn(fid):
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")  # f8 at dimension 50 truncates to 48
        return psso.make_function(fid, NVAR)


def _oracle_run(args):
    fid, schedule, seed = args
    fn = _fn(fid)
    o = O.Oracle(fid, NSOL, NVAR, 0.3, 0.6, 0.8, fn.var_min, fn.var_max, seed)
    sw = o.initialize()
    traj = (o.run if schedule == "parallel" else o.run_sequential)(sw, 0, NITER)
    return float(traj[-1])


@pytest.fixture(scope="module")
def precision_report():
    config = ExperimentConfig(functions=[_fn(f) for f in FIDS],
                              schedules=[ScheduleKind.SEQUENTIAL, ScheduleKind.PARALLEL],
                              replications=RUNS, base_seed=0, nsol=NSOL, nvar=NVAR, niter=NITER)
    return run_experiment(config)


@pytest.fixture(scope="module")
def oracle_finals():
    jobs = [(fid, sch, s) for fid in FIDS for sch in ("sequential", "parallel") for s in range(RUNS)]
    with ThreadPoolExecutor(max_workers=O.max_threads()) as ex:  # ctypes releases the GIL; no fork of a CUDA process
        out = list(ex.map(_oracle_run, jobs, chunksize=4))
    return {(j[0], j[1], j[2]): v for j, v in zip(jobs, out)}


def _means(finals):
    return {(fid, sch): float(np.mean([finals[(fid, sch, s)] for s in range(RUNS)]))
            for fid in FIDS for sch in ("sequential", "parallel")}


def test_every_run_equals_the_reference_algorithm(precision_report, oracle_finals):
    assert len(precision_report.records) == len(FIDS) * 2 * RUNS
    for r in precision_report.records:
        want = oracle_finals[(r.function, ScheduleKind(r.schedule).value, r.seed)]
        if r.function in ("f1", "f2", "f3", "f4"):
            assert r.best_fitness == want, (r.function, r.schedule, r.seed)
        else:
            assert abs(r.best_fitness - want) <= 1e-12 * abs(want), (r.function, r.schedule, r.seed)


def test_criterion_5_same_outcome_as_the_reference(precision_report, oracle_finals):
    dev = {(row.function, ScheduleKind(row.schedule).value): row.mean
           for row in precision_report.summaries}
    ref = _means(oracle_finals)
    for key, m in ref.items():
        assert abs(dev[key] - m) <= 1e-12 * abs(m), key
    for fid, (lo, hi) in BANDS.items():  # criterion 5: precision bands
        assert (lo <= dev[(fid, "parallel")] <= hi) == (lo <= ref[(fid, "parallel")] <= hi), fid
    # criterion 5: parallel mean <= sequential mean on >= 6 of 9 functions
    wins = lambda m: sum(m[(f, "parallel")] <= m[(f, "sequential")] for f in FIDS)  # noqa: E731
    assert wins(dev) == wins(ref)
    # sequential f1 regression band: reference 54.9497 +- 2 * 7.4781
    assert (abs(dev[("f1", "sequential")] - 54.9497) <= 2 * 7.4781) == \
        (abs(ref[("f1", "sequential")] - 54.9497) <= 2 * 7.4781)
