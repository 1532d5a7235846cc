"""The reference's property tests, run on the device path.

Each test restates one of the reference suite's properties
(tests/test_parallel.py, tests/test_core.py, tests/test_benchmarks.py of
/root/reference/pkg) against the CUDA engine and device objectives, and pins
the device result to the oracle where the property alone would not.
"""

import warnings

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2110_01470_b200 as psso  # noqa: E402
from oracle import oracle as O  # noqa: E402  (the checker)
from paper_2110_01470_b200 import _lib  # noqa: E402
from paper_2110_01470_b200.engine import DeviceEngine  # noqa: E402


def _fn(fid, d):
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        return psso.make_function(fid, d)


def _params(fn, nsol, niter, **kw):
    return psso.SsoParams(cw=kw.get("cw", 0.3), cp=kw.get("cp", 0.6), cg=kw.get("cg", 0.8),
                          var_min=fn.var_min, var_max=fn.var_max, nsol=nsol,
                          nvar=fn.dimension, niter=niter)


# ------------------------------------------------------------ schedules ----

@pytest.mark.parametrize("fid", ["f1", "f4"])
def test_single_particle_parallel_coincides_with_sequential(fid):
    """test_parallel.py:213-220 / acceptance criterion 2: with one particle the
    two schedules are the same algorithm -- bitwise, and equal to the oracle."""
    fn = _fn(fid, 12)
    p = _params(fn, 1, 40)
    par = psso.run_parallel(p, fn, 17)
    seq = psso.run_sequential(p, fn, 17)
    assert np.array_equal(par.trajectory, seq.trajectory)
    assert np.array_equal(par.best_position, seq.best_position)
    o = O.Oracle.from_params(p, fid, 17)
    assert np.array_equal(o.run(o.initialize(), 0, 40), par.trajectory)


def test_schedules_can_differ_with_many_particles():
    """test_parallel.py:222-227: with 30 particles the live gBest of the
    sequential schedule changes the trajectory."""
    fn = _fn("f1", 10)
    p = _params(fn, 30, 30)
    seq = psso.run_sequential(p, fn, 1)
    par = psso.run_parallel(p, fn, 1)
    assert not np.array_equal(seq.trajectory, par.trajectory)
    o = O.Oracle.from_params(p, "f1", 1)
    assert np.array_equal(o.run_sequential(o.initialize(), 0, 30), seq.trajectory)


@pytest.mark.parametrize("schedule", ["parallel", "sequential"])
def test_trajectory_monotone_inside_box_and_consistent(schedule):
    """test_parallel.py:204-211, test_core.py:160-174: g_f never rises, the best
    position lies in the box and its fitness is the record's."""
    fn = _fn("f5", 8)
    p = _params(fn, 16, 50)
    run = psso.run_parallel if schedule == "parallel" else psso.run_sequential
    rec = run(p, fn, 11)
    assert (np.diff(rec.trajectory) <= 0).all()
    assert rec.trajectory.size == p.niter
    assert rec.best_fitness == rec.trajectory[-1]
    assert rec.best_position.min() >= p.var_min and rec.best_position.max() <= p.var_max
    assert float(fn(rec.best_position)) == rec.best_fitness


def test_sequential_is_bitwise_deterministic_and_a_prefix():
    """test_core.py:176-191: same seed, same bits; a shorter budget is a prefix."""
    fn = _fn("f7", 12)
    a = psso.run_sequential(_params(fn, 15, 30), fn, 123)
    b = psso.run_sequential(_params(fn, 15, 30), fn, 123)
    assert a.best_fitness == b.best_fitness
    assert np.array_equal(a.best_position, b.best_position)
    assert np.array_equal(a.trajectory, b.trajectory)
    assert a.wall_time_s > 0
    short = psso.run_sequential(_params(fn, 15, 18), fn, 123)
    assert np.array_equal(a.trajectory[:18], short.trajectory)


# ---------------------------------------------------- phase invariants ----

def test_invariants_hold_along_phased_run():
    """test_parallel.py:229-246 on the device phase API, state read back after
    every phase quartet, and each iteration's state equal to the oracle's."""
    fn = _fn("f2", 7)
    p = _params(fn, 12, 15)
    eng = DeviceEngine(p, fn, 13)
    o = O.Oracle.from_params(p, "f2", 13)
    osw = o.initialize()
    try:
        eng.initialize()
        g_prev = eng.to_host().g_f
        for t in range(p.niter):
            eng.search(t)
            eng.evaluate(t)
            eng.update_pbests()
            eng.update_gbest()
            eng.check()
            sw = eng.to_host()
            o.step(osw, t)
            assert np.all(sw.p_f <= sw.sol_f)
            assert np.all(sw.g_f <= sw.p_f)
            assert sw.g_f <= g_prev
            for arr in (sw.sol, sw.pbests, sw.gbest):
                assert arr.min() >= p.var_min and arr.max() <= p.var_max
            assert sw.g_f == float(fn(sw.gbest))
            assert np.array_equal(sw.sol, osw.sol) and np.array_equal(sw.pbests, osw.pbests)
            assert sw.g_f == osw.g_f and np.array_equal(sw.gbest, osw.gbest)
            g_prev = sw.g_f
    finally:
        eng.close()


def test_initial_population_inside_box_and_bests_consistent():
    """test_core.py:108-118 on the device initialization."""
    fn = _fn("f1", 8)
    p = _params(fn, 40, 1)
    eng = DeviceEngine(p, fn, 11)
    try:
        eng.initialize()
        sw = eng.to_host()
        gf, gi = eng.result()
    finally:
        eng.close()
    assert sw.sol.shape == (40, 8)
    assert sw.sol.min() >= p.var_min and sw.sol.max() <= p.var_max
    assert np.array_equal(sw.pbests, sw.sol) and np.array_equal(sw.p_f, sw.sol_f)
    best = int(np.argmin(sw.p_f))
    assert gi == best and sw.g_f == gf == sw.p_f[best]
    assert np.array_equal(sw.gbest, sw.pbests[best])
    assert np.array_equal(sw.sol, O.init_positions(11, 40, 8, p.var_min, p.var_max))


@pytest.mark.parametrize("dtype", ["float64", "float32"])
def test_tiny_interval_stays_inside(dtype):
    """test_core.py:120-128: a 1e-9-wide box -- positions in [0, 1e-9) at
    initialization (== the oracle's in fp64) and inside the box after 20
    iterations of fresh draws."""
    fn = psso.probe_function(1, float("inf"), bounds=(0.0, 1e-9))
    p = psso.SsoParams(cw=0.3, cp=0.6, cg=0.8, var_min=0.0, var_max=1e-9, nsol=64, nvar=1,
                       niter=20)
    eng = DeviceEngine(p, fn, 0, dtype=dtype)
    try:
        eng.initialize()
        sw0 = eng.to_host()
        eng.run(0, p.niter)
        eng.check()
        sw = eng.to_host()
    finally:
        eng.close()
    assert (sw0.sol >= 0.0).all() and (sw0.sol < 1e-9).all()
    if dtype == "float64":
        assert np.array_equal(sw0.sol, O.init_positions(0, 64, 1, 0.0, 1e-9))
    assert np.array_equal(sw0.gbest, sw0.sol[int(np.argmin(sw0.p_f))])
    for arr in (sw.sol, sw.pbests, sw.gbest):
        assert arr.min() >= 0.0 and arr.max() <= 1e-9


@pytest.mark.parametrize("cw,cp,cg", [(0.3, 0.3, 0.8), (0.3, 0.8, 0.8), (0.5, 0.5, 0.5)])
def test_equal_thresholds_are_legal_and_match_the_oracle(cw, cp, cg):
    """test_core.py:46-52: cw == cp or cp == cg empty a branch; the device run
    equals the reference's (oracle) bit for bit."""
    fn = _fn("f4", 10)
    p = _params(fn, 23, 25, cw=cw, cp=cp, cg=cg)
    rec = psso.run_parallel(p, fn, 42)
    o = O.Oracle(fid="f4", nsol=23, nvar=10, cw=cw, cp=cp, cg=cg, var_min=fn.var_min,
                 var_max=fn.var_max, seed=42)
    osw = o.initialize()
    assert np.array_equal(o.run(osw, 0, 25), rec.trajectory)
    assert np.array_equal(osw.gbest, rec.best_position)


# ------------------------------------------------- device objectives ----

@pytest.mark.parametrize("fid", ["f1", "f2", "f5", "f6", "f7"])
def test_even_in_every_coordinate(fid):
    """test_benchmarks.py:86-94 on the device objectives."""
    fn = _fn(fid, 12)
    x = np.random.default_rng(3).uniform(fn.var_min, fn.var_max, size=12)
    rows = np.repeat(x[None, :], 13, axis=0)
    for j in range(12):
        rows[j + 1, j] = -rows[j + 1, j]
    f = fn(rows)
    assert f[1:] == pytest.approx(np.full(12, f[0]), rel=1e-12, abs=1e-12)


@pytest.mark.parametrize("fid", ["f1", "f2", "f5", "f9"])
def test_separable_functions_decompose_coordinatewise(fid):
    """test_benchmarks.py:97-108 on the device objectives."""
    fn = _fn(fid, 16)
    x = np.random.default_rng(4).uniform(fn.var_min, fn.var_max, size=16)
    rows = np.zeros((17, 16))
    for j in range(16):
        rows[j + 1, j] = x[j]
    f = fn(rows)
    acc = f[0] + sum(f[j + 1] - f[0] for j in range(16))
    assert acc == pytest.approx(float(fn(x)), rel=1e-9, abs=1e-9)


@pytest.mark.parametrize("fid", ["f1", "f2", "f3", "f4", "f5", "f7", "f8"])
@pytest.mark.parametrize("dtype", ["float64", "float32"])
def test_nonnegative_and_finite_on_box_samples(fid, dtype):
    """test_benchmarks.py:111-122: 100,000 box samples at 48 dimensions are
    finite and >= 0, in both device precisions; fp64 values equal the oracle's."""
    fn = _fn(fid, 48)
    block = np.random.default_rng(5).uniform(fn.var_min, fn.var_max, size=(100_000, 48))
    f = psso.benchmarks.evaluate_rows(fn, block, dtype=dtype)
    assert np.isfinite(f).all() and f.min() >= 0.0
    if dtype == "float64":
        ref = O.evaluate(fid, block[:2000], threads=O.max_threads())
        assert f[:2000] == pytest.approx(ref, rel=1e-12, abs=1e-12)


def test_f6_f9_finite_on_box_samples():
    """test_benchmarks.py:118-122 for the two objectives not covered above."""
    for fid in ("f6", "f9"):
        fn = _fn(fid, 48)
        block = np.random.default_rng(6).uniform(fn.var_min, fn.var_max, size=(10_000, 48))
        assert np.isfinite(fn(block)).all(), fid


def test_truncated_powell_ignores_trailing_coordinates():
    """test_benchmarks.py:131-146: f8 at 50 dimensions uses the first 48 only,
    and agrees with the 48-variable instance on that prefix -- on the device."""
    fn = _fn("f8", 50)
    assert fn.truncated_to == 48
    x = np.zeros(50)
    x[-2:] = 3.0
    assert fn(x) == 0.0
    full = _fn("f8", 48)
    y = np.random.default_rng(7).uniform(-4, 5, size=50)
    assert fn(y) == full(y[:48])


def test_out_of_bounds_is_flagged_not_clamped():
    """test_benchmarks.py:156-164: the device objective evaluates outside the box."""
    fn = _fn("f1", 3)
    with pytest.warns(psso.benchmarks.OutOfBoundsWarning):
        value, in_bounds = fn.evaluate_flagged(np.array([6.0, 0.0, 0.0]))
    assert value == 36.0 and not in_bounds
    value, in_bounds = fn.evaluate_flagged(np.array([1.0, 0.0, 0.0]))
    assert value == 1.0 and in_bounds


@pytest.mark.parametrize("fid,nsol,nvar,dtype,box,kernel", [
    ("f5", 4096, 128, "float64", None, "k_chain"),
    ("f5", 4096, 128, "float32", None, "k_chain"),
    ("f6", 64, 1024, "float64", None, "k_rows"),
    ("f7", 1000, 100, "float64", None, "k_swarm"),
    ("f9", 1000, 100, "float64", None, "k_swarm"),
    ("f6", 300, 300, "float64", None, "k_fused"),
    ("f5", 200, 301, "float64", None, "k_tile"),
    ("f5", 200, 301, "float32", None, "k_tile"),
    ("f5", 4096, 128, "float64", 1e13, "k_fused"),
])
def test_reevaluated_pbests_equal_in_run_fitness(fid, nsol, nvar, dtype, box, kernel):
    """test_core.py:168-174 (`fn(best_position) == best_fitness`) for every
    kernel family: each pBest row re-evaluated by psso_eval_rows equals the
    p_f the iteration kernel computed for it, bit for bit -- one set of
    objective instructions on every device path (psso_device.cuh obj_cos)."""
    fn = _fn(fid, nvar)
    p = psso.SsoParams(cw=0.3, cp=0.6, cg=0.8, var_min=-box if box else fn.var_min,
                       var_max=box if box else fn.var_max, nsol=nsol, nvar=nvar, niter=6)
    eng = DeviceEngine(p, fn, 3, dtype=dtype)
    try:
        name = _lib.load().psso_kernel_name(eng.ctx).decode()
        assert name.startswith(kernel), name
        eng.initialize()
        eng.run(0, p.niter)
        eng.check()
        sw = eng.to_host()
        gf, gi = eng.result()
    finally:
        eng.close()
    again = psso.benchmarks.evaluate_rows(fn, sw.pbests, dtype=dtype)
    assert np.array_equal(again, sw.p_f)
    assert psso.benchmarks.evaluate_rows(fn, sw.gbest[None, :], dtype=dtype)[0] == gf
